# Round-2 re-entry check on one GPU: gpu tests, smoke, default bench, C3/C2 at tile 240.
mkdir -p gpurun_out/r3
O=gpurun_out/r3
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 500 > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 400 $O/bench_c4.json; echo
for t in 128 240; do
timeout 600 python bench.py --workload c3 --tile $t --steps 5 --warmup 3 --no-batch --no-cpu-baseline --e2e-steps 1 > $O/bench_c3_$t.json 2> $O/bench_c3_$t.err; python -c "import json,sys; d=json.loads(open('$O/bench_c3_$t.json').read().strip().splitlines()[-1]); print('c3',$t,d['ms_per_step'],d['roofline']['frac'])"
done
