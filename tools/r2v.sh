timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2v_pytest.log 2>&1; tail -3 gpurun_out/r2v_pytest.log
timeout 600 python tools/ab_sched.py --workload c2 --tile 120 --reps 2 --variants default,la4 2>&1 | grep -v Warn
export TC_UPD_SHAPE=128x64
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default,la4,la8 2>&1 | grep -v Warn
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default,la4,la8,la16,la32 2>&1 | grep -v Warn
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 8 > gpurun_out/r2v_trace_c4.txt 2>&1; tail -68 gpurun_out/r2v_trace_c4.txt
