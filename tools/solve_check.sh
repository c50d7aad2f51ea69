# solve GEMVs with independent loads in flight: timing + solve parity tests
mkdir -p gpurun_out/r3
O=gpurun_out/r3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "solve" > $O/pytest_solve.log 2>&1; tail -2 $O/pytest_solve.log
for w in c2 c4; do
timeout 900 python bench.py --workload $w --steps 2 --warmup 3 --no-batch --no-cpu-baseline --e2e-steps 1 > $O/solve_$w.json 2> $O/solve_$w.err
python -c "import json; d=json.loads(open('$O/solve_$w.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], json.dumps(d.get('solve')))"
done
