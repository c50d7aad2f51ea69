timeout 1200 python -m pytest tests -q -m gpu -x --timeout 400 > gpurun_out/r2at_pytest.log 2>&1; tail -2 gpurun_out/r2at_pytest.log
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default,la2,la4 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c3 --tile 128 --reps 2 --variants default,la2,la4 2>&1 | grep -v Warn
TC_UPD_SHAPE=128x64 timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants la3,la4,la6 2>&1 | grep -v Warn
TC_UPD_SHAPE=128x64 timeout 900 python tools/ab_sched.py --workload c3 --tile 128 --reps 2 --variants default,la4 2>&1 | grep -v Warn
timeout 900 python tools/ab_sched.py --workload c4 --tile 120 --reps 1 --variants default 2>&1 | grep -v Warn
timeout 900 python tools/ab_sched.py --workload c4 --tile 160 --reps 1 --variants default 2>&1 | grep -v Warn
