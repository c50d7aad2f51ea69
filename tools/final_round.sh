#!/bin/bash
# Round-end measurement set (GPU box): default bench + reference arm, C1/C3/C4/C5 lines,
# ncu launch list of the default bench, ncu --set full of k_persist (C2 and C4), traffic.
TAG=${1:-r1f}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -1 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -1 gpurun_out/bench_ref_$TAG.json | cut -c1-200
for w in c1:120 c3:120 c5:120; do IFS=: read wl t <<< "$w"
  timeout 1200 python bench.py --workload $wl --tile $t --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_${TAG}_$wl.json 2> gpurun_out/bench_${TAG}_$wl.err; tail -1 gpurun_out/bench_${TAG}_$wl.json | cut -c1-160; done
timeout 1200 python bench.py --workload c5 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline --share 4 > gpurun_out/bench_${TAG}_c5share4.json 2> gpurun_out/bench_${TAG}_c5share4.err; tail -1 gpurun_out/bench_${TAG}_c5share4.json | cut -c1-160
timeout 1800 python bench.py --workload c4 --tile 120 --ordering identity --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-profile > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err; tail -1 gpurun_out/bench_${TAG}_c4.json | cut -c1-160
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o gpurun_out/prof_${TAG}_c2 python tools/prof_driver.py --workload c2 --tile 120 --reps 2 > gpurun_out/ncu_full_${TAG}_c2.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o gpurun_out/prof_${TAG}_c3 python tools/prof_driver.py --workload c3 --tile 120 --reps 2 > gpurun_out/ncu_full_${TAG}_c3.log 2>&1
ls gpurun_out | grep $TAG
true
