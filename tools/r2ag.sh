export TC_DEBUG_ORDER=1
export TC_ORDER=1
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants la2,default,la4 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 1 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c3 --tile 128 --reps 1 --variants default 2>&1 | grep -v Warn
TC_UPD_SHAPE=128x64 timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants default,la4 2>&1 | grep -v Warn
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 3 > gpurun_out/r2ag_trace.txt 2>&1; head -16 gpurun_out/r2ag_trace.txt
