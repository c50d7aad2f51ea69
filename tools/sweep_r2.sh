# Tile-size sweep (round 2): bench lines per workload x tile into gpurun_out/sweep_r2/
mkdir -p gpurun_out/sweep_r2
for nt in 120 128 160 192 240 256 320 384 480; do
  timeout 600 python bench.py --workload c2 --tile $nt --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity --no-profile --ordering identity > gpurun_out/sweep_r2/c2_$nt.json 2> gpurun_out/sweep_r2/c2_$nt.err
  tail -c 300 gpurun_out/sweep_r2/c2_$nt.err | tail -2
done
for nt in 120 128 240; do
  timeout 600 python bench.py --workload c3 --tile $nt --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity --no-profile --ordering identity > gpurun_out/sweep_r2/c3_$nt.json 2> gpurun_out/sweep_r2/c3_$nt.err
done
for nt in 120 128 160 192 240 256 320; do
  timeout 900 python bench.py --workload c4 --tile $nt --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity --no-profile --ordering identity > gpurun_out/sweep_r2/c4_$nt.json 2> gpurun_out/sweep_r2/c4_$nt.err
  tail -c 300 gpurun_out/sweep_r2/c4_$nt.err | tail -2
done
python - <<'PY'
import json, glob, os
rows = []
for f in sorted(glob.glob("gpurun_out/sweep_r2/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    rows.append((os.path.basename(f)[:-5], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel_ms"], d.get("e2e", {}).get("ms_per_step")))
for r in rows: print("%-10s step %9.2f ms  kernel %9.2f ms  frac %.3f  e2e %s" % (r[0], r[1], r[3], r[2], r[4]))
PY
