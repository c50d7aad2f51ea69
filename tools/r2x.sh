timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2x_pytest.log 2>&1; tail -3 gpurun_out/r2x_pytest.log
export TC_UPD_SHAPE=128x64
for U in 0 24 48; do for SP in 2 4; do
export TC_URGENT=$U TC_URGENT_SPAN=$SP
echo "urgent $U span $SP"
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants la4,la6 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 1 --variants la4 2>&1 | grep -v Warn
done; done
