echo "== rhead (committed TMA)"
cd rhead
timeout 600 python tools/ab_sched.py --workload c4 --tile 160 --reps 1 --variants default 2>&1 | grep -v Warn
TC_UPD_TMA=0 timeout 600 python tools/ab_sched.py --workload c4 --tile 160 --reps 1 --variants default 2>&1 | grep -v Warn
TC_UPD_SHAPE=128x64 timeout 600 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants default 2>&1 | grep -v Warn
cd ..
echo "== current, graph executor"
timeout 900 python tools/ab_sched.py --workload c4 --tile 160 --reps 1 --variants graph 2>&1 | grep -v Warn
