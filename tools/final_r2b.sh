# End-of-round-2 measurement set after the chain split (one GPU): tests, smoke,
# bench lines (C4 default + C5 sub, reference arm, C3/C2/C1, C3@240, C5),
# launch list of the default bench command, ncu --set full of k_persist C4@128.
mkdir -p gpurun_out/final_r2b
O=gpurun_out/final_r2b
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 500 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json; echo
for w in "c3 128" "c2 128" "c1 128" "c3 240" "c2 240"; do set -- $w
timeout 900 python bench.py --workload $1 --tile $2 --steps 5 --warmup 3 --no-batch > $O/bench_$1_$2.json 2> $O/bench_$1_$2.err; tail -c 200 $O/bench_$1_$2.json; echo
done
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 300 $O/bench_c5.json; echo
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity --ordering identity > $O/launches.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o $O/k_persist_c4_128 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants default > $O/ncu_c4.log 2>&1
$NCU -i $O/k_persist_c4_128.ncu-rep --page raw --csv > $O/k_persist_c4_128_raw.csv 2>/dev/null
$NCU -i $O/k_persist_c4_128.ncu-rep --page details > $O/k_persist_c4_128_details.txt 2>/dev/null
rm -f $O/*.ncu-rep
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128.txt 2>&1
ls $O
