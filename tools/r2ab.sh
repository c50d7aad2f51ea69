for sh in 64x64 128x64; do
export TC_UPD_SHAPE=$sh
echo "== $sh"
timeout 900 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants la2,la4,nosplit2,nosplit4,neither2 2>&1 | grep -v Warn
timeout 600 python tools/ab_sched.py --workload c2 --tile 128 --reps 1 --variants la2,la4,nosplit2,nosplit4,neither2 2>&1 | grep -v Warn
done
