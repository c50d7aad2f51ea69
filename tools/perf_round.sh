#!/bin/bash
# usage: tools/perf_round.sh TAG "tiles" [ncu]   (runs on the GPU box under gpurun)
TAG=$1; TILES=${2:-"120 240"}; NCU=${3:-0}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.log
for t in $TILES; do
  timeout 900 python bench.py --workload c2 --tile $t --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_c2_$t.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_c2_$t.log | cut -c1-200
done
if [ "$NCU" != "0" ]; then
  for k in k_potrf k_trsm k_update; do
    ncu --set full --import-source on --clock-control none -k regex:$k -s 40 -c 2 -o gpurun_out/prof_${TAG}_$k python tools/prof_driver.py --workload c2 --tile $NCU > gpurun_out/ncu_${TAG}_$k.log 2>&1
  done
fi
true
