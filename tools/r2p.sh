export TC_UPD_SHAPE=128x64 TC_DEBUG_ORDER=1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2p_pytest.log 2>&1; tail -3 gpurun_out/r2p_pytest.log
for R in 0 12; do
export TC_RESERVE=$R
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default,la8,la12 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default,la8 2>&1 | grep -v Warn
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 12 > gpurun_out/r2p_trace_c4_$R.txt 2>&1; tail -14 gpurun_out/r2p_trace_c4_$R.txt
done
