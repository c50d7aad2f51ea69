timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "tile_kernels or tile_size_sweep or solve_persistent" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 400 -k "c3_full_inla or arrowhead_logdet" 2>&1 | tail -3
for nt in 192 200 240 256; do timeout 600 python tools/ab_sched.py --workload c3 --tile $nt --reps 1 --variants default 2>&1 | grep -v Warn; done
for nt in 192 240 256; do timeout 600 python tools/ab_sched.py --workload c2 --tile $nt --reps 1 --variants default 2>&1 | grep -v Warn; done
for nt in 240 256; do timeout 900 python tools/ab_sched.py --workload c4 --tile $nt --reps 1 --variants default 2>&1 | grep -v Warn; done
