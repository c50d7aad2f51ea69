timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2w_pytest.log 2>&1; tail -3 gpurun_out/r2w_pytest.log
export TC_UPD_SHAPE=128x64
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default,la4 2>&1 | grep -v Warn
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants la3,la4,la6 2>&1 | grep -v Warn
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 4 > gpurun_out/r2w_trace_c4.txt 2>&1; tail -68 gpurun_out/r2w_trace_c4.txt
