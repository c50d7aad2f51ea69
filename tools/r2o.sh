export TC_UPD_SHAPE=128x64 TC_DEBUG_ORDER=1
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default,la4,la8,la12,la16 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default,la4,la8,la12 2>&1 | grep -v Warn
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 12 > gpurun_out/r2o_trace_c4.txt 2>&1; tail -22 gpurun_out/r2o_trace_c4.txt
