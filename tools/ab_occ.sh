#!/bin/bash
mkdir -p gpurun_out
./tools/potrf_trace | grep -E "nt=|last"
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for w in "c2 120" "c3 120" "c4 120"; do
  set -- $w
  for occ in 1 2; do
    extra=""; [ "$1" = "c4" ] && extra="--ordering identity"
    timeout 1200 python bench.py --workload $1 --tile $2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --no-profile --occupancy $occ $extra > gpurun_out/ab_${1}_${2}_occ$occ.log 2>&1
    tail -1 gpurun_out/ab_${1}_${2}_occ$occ.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 occ$occ', round(d['ms_per_step'],2), 'ms', round(d['fp64_roofline']['frac'],3))" 2>&1 | tail -1
  done
done
