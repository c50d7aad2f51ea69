for sh in none 128x64 128x128; do
  if [ $sh != none ]; then export TC_UPD_SHAPE=$sh; fi
  echo "== shape $sh"
  timeout 600 python tools/ab_sched.py --workload c4 --tile 128 --reps 2 --variants default,neither 2>&1 | grep -v Warn
  timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 2 --variants default,neither 2>&1 | grep -v Warn
done
export TC_UPD_SHAPE=128x64
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > gpurun_out/r2m_trace_c4.txt 2>&1; tail -16 gpurun_out/r2m_trace_c4.txt
