#!/bin/bash
# C3 / C4 measurements (runs on the GPU box)
mkdir -p gpurun_out
for t in ${C3TILES:-120 240}; do
  timeout 900 python bench.py --workload c3 --tile $t --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${1}_c3_$t.log 2>&1
  tail -1 gpurun_out/bench_${1}_c3_$t.log | cut -c1-150
done
for t in ${C4TILES:-240}; do
  timeout 1800 python bench.py --workload c4 --tile $t --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --ordering identity --no-profile > gpurun_out/bench_${1}_c4_$t.log 2>&1
  tail -3 gpurun_out/bench_${1}_c4_$t.log | cut -c1-300
done
true
