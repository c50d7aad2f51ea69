#!/bin/bash
# usage: tools/sweep.sh TAG "workload:tile[:extra]" ...   (GPU box) — one bench line per case
TAG=$1; shift
mkdir -p gpurun_out
for w in "$@"; do
  IFS=: read wl t extra <<< "$w"
  timeout 1500 python bench.py --workload $wl --tile $t --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-profile $extra > gpurun_out/sw_${TAG}_${wl}_$t.log 2>&1
  tail -1 gpurun_out/sw_${TAG}_${wl}_$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl $t', round(d['ms_per_step'],2), 'ms frac', round(d['fp64_roofline']['frac'],3), 'TF', round(d['roofline']['achieved'],2), 'e2e', round(d['e2e']['ms_per_step'],1), 'setup', round(d['setup_s'],1))" 2>&1 | tail -1
done
true
