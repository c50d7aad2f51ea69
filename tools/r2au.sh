for nt in 120 128 160 192 240 256; do timeout 600 python tools/ab_sched.py --workload c4 --tile $nt --reps 1 --variants default 2>&1 | grep -v Warn; done
TC_UPD_SHAPE=128x64 timeout 600 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants default,la4 2>&1 | grep -v Warn
for nt in 120 128 160 240; do timeout 600 python tools/ab_sched.py --workload c3 --tile $nt --reps 1 --variants default,la4 2>&1 | grep -v Warn; done
for nt in 120 128 160 240 320; do timeout 600 python tools/ab_sched.py --workload c2 --tile $nt --reps 1 --variants default 2>&1 | grep -v Warn; done
TC_UPD_TMA_SB=1 TC_UPD_SHAPE=128x64 timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 1 --variants default 2>&1 | grep -v Warn
TC_UPD_TMA=0 timeout 600 python tools/ab_sched.py --workload c2 --tile 160 --reps 1 --variants default 2>&1 | grep -v Warn
