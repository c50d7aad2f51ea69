#!/bin/bash
# A/B of library builds: tools/ab.sh "lib1 lib2 ..." "workload:tile ..."   (GPU box)
for w in $2; do
  IFS=: read wl t <<< "$w"
  for L in $1; do
    r=$(TILECHOL_B200_LIB=$PWD/tools/ab/$L.so timeout 900 python bench.py --workload $wl --tile $t --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-profile $3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'ms frac', round(d['fp64_roofline']['frac'],3))" 2>&1 | tail -1)
    echo "$wl@$t $L: $r"
  done
done
