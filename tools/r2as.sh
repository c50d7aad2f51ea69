timeout 1200 python -m pytest tests -q -m gpu -x --timeout 400 > gpurun_out/r2as_pytest.log 2>&1; tail -3 gpurun_out/r2as_pytest.log
for t in 0 1; do
export TC_UPD_TMA=$t
echo "== tma $t"
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c3 --tile 128 --reps 2 --variants default 2>&1 | grep -v Warn
TC_UPD_SHAPE=128x64 timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default,la4 2>&1 | grep -v Warn
done
export TC_UPD_TMA=1
timeout 600 python tools/trace_legacy.py --workload c4 --tile 128 --ordering identity > gpurun_out/r2as_trace.txt 2>&1; tail -14 gpurun_out/r2as_trace.txt
