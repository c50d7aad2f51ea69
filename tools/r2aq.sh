timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r2aq_pytest.log 2>&1; tail -3 gpurun_out/r2aq_pytest.log
for f in 0 1; do
export TC_SYRK_FUSE=$f
echo "== fuse $f"
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default,la4 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c3 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 120 --reps 2 --variants default 2>&1 | grep -v Warn
done
export TC_SYRK_FUSE=1
timeout 600 python tools/trace_legacy.py --workload c4 --tile 128 --ordering identity > gpurun_out/r2aq_trace.txt 2>&1; tail -14 gpurun_out/r2aq_trace.txt
