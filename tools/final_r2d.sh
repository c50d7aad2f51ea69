# last check of the round: full GPU suite, smoke, default bench line
mkdir -p gpurun_out/final_r2d
O=gpurun_out/final_r2d
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 500 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 400 $O/bench_c4.json; echo
