#!/bin/bash
# A/B of tuning environment settings (GPU box):
#   tools/ab_env.sh "ENV=a ENV=b ..." "workload:tile ..."
# each setting runs bench.py in its own process (the library reads the
# variables once); prints ms per step and the FP64 roofline fraction
for w in $2; do
  IFS=: read wl t <<< "$w"
  for E in $1; do
    r=$(env $E timeout 900 python bench.py --workload $wl --tile $t --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-profile --no-batch --no-parity $3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'ms frac', round(d['roofline']['frac'],3), 'logdet', d.get('logdet'))" 2>&1 | tail -1)
    echo "$wl@$t $E: $r"
  done
done
