export TC_UPD_SHAPE=128x64
for R in 0 8 16; do
export TC_RESERVE=$R
echo "== reserve $R"
timeout 600 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > gpurun_out/r2n_trace_c4_$R.txt 2>&1; tail -11 gpurun_out/r2n_trace_c4_$R.txt
done
