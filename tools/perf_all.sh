#!/bin/bash
mkdir -p gpurun_out
for t in ${C2TILES:-120 160}; do
  timeout 900 python bench.py --workload c2 --tile $t --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${1}_c2_$t.log 2>&1
done
for t in ${C3TILES:-120 160 240}; do
  timeout 900 python bench.py --workload c3 --tile $t --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${1}_c3_$t.log 2>&1
done
for t in ${C4TILES:-120 160}; do
  timeout 1800 python bench.py --workload c4 --tile $t --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --ordering identity --no-profile > gpurun_out/bench_${1}_c4_$t.log 2>&1
done
for f in gpurun_out/bench_${1}_*.log; do echo $f; tail -1 $f | cut -c1-160; done
true
