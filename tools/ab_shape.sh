#!/bin/bash
# A/B of persistent-kernel update shapes / tile sizes; args are "workload tile occ shape [lookahead]" tuples
mkdir -p gpurun_out
if [ -n "$AB_TESTS" ]; then python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3; fi
for w in "$@"; do
  set -- $w
  extra=""; [ "$1" = "c4" ] && extra="--ordering identity"
  la=${5:-1}; tag=${1}_${2}_o${3}_s${4}_la$la
  TC_PERSIST_SHAPE=$4 timeout 1200 python bench.py --workload $1 --tile $2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --no-profile --occupancy $3 --lookahead $la $extra > gpurun_out/ab_$tag.log 2>&1
  tail -1 gpurun_out/ab_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['ms_per_step'],2), 'ms', round(d['fp64_roofline']['frac'],3), 'kern', round(d['roofline']['achieved'],2))" 2>&1 | tail -1
done
