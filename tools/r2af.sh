export TILECHOL_EXPERIMENTAL=1
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 4 --variants default,occ2,occ2la4 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 4 --variants default,occ2 2>&1 | grep -v Warn
timeout 900 python tools/ab_sched.py --workload c3 --tile 128 --reps 4 --variants default,occ2 2>&1 | grep -v Warn
timeout 900 python tools/ab_sched.py --workload c3 --tile 120 --reps 2 --variants default,occ2 2>&1 | grep -v Warn
timeout 900 python tools/ab_sched.py --workload c4 --tile 120 --reps 2 --variants default,occ2 2>&1 | grep -v Warn
