# default bench line with the solve block + GPU tests (end of round 2)
mkdir -p gpurun_out/final_r2c
O=gpurun_out/final_r2c
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4.json; echo
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-batch > $O/bench_c2_128.json 2> $O/bench_c2_128.err; tail -c 200 $O/bench_c2_128.json; echo
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 500 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
