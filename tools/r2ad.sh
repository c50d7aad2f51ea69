timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2ad_pytest.log 2>&1; tail -3 gpurun_out/r2ad_pytest.log
for sh in 64x64 128x64; do
export TC_UPD_SHAPE=$sh
echo "== $sh"
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants default,la3 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 1 --variants default,la3 2>&1 | grep -v Warn
done
unset TC_UPD_SHAPE
timeout 600 python tools/ab_sched.py --workload c2 --tile 120 --reps 1 --variants default 2>&1 | grep -v Warn
