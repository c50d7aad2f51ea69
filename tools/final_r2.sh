# End-of-round-2 measurement set (one GPU)
mkdir -p gpurun_out/final_r2
O=gpurun_out/final_r2
NCU=/usr/local/cuda/bin/ncu
timeout 1300 python -m pytest tests -q -m gpu -x --timeout 400 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 600 $O/bench_c4.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 700 $O/bench_ref.json; echo
timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 --no-batch > $O/bench_c3.json 2> $O/bench_c3.err; tail -c 300 $O/bench_c3.json; echo
timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 --no-batch > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json; echo
timeout 900 python bench.py --workload c1 --steps 20 --warmup 3 --no-batch > $O/bench_c1.json 2> $O/bench_c1.err; tail -c 300 $O/bench_c1.json; echo
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity --ordering identity > $O/launches.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o $O/k_persist_c4_128 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants default > $O/ncu_c4.log 2>&1
$NCU -i $O/k_persist_c4_128.ncu-rep --page raw --csv > $O/k_persist_c4_128_raw.csv 2>/dev/null
$NCU -i $O/k_persist_c4_128.ncu-rep --page details > $O/k_persist_c4_128_details.txt 2>/dev/null
rm -f $O/*.ncu-rep
ls $O
