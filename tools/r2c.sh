export TILECHOL_EXPERIMENTAL=1
timeout 900 python -m pytest tests/test_gpu_stress.py -q -x > gpurun_out/r2c_stress.log 2>&1; tail -5 gpurun_out/r2c_stress.log
for occ in 2 1; do
timeout 900 python tools/trace.py --workload c4 --tile 120 --ordering identity --occupancy $occ > gpurun_out/r2c_trace_c4_occ$occ.txt 2>&1; cat gpurun_out/r2c_trace_c4_occ$occ.txt
done
for i in 1 2 3; do
timeout 900 python bench.py --workload c4 --ordering identity --occupancy 2 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity > gpurun_out/r2c_c4_occ2_$i.json 2> gpurun_out/r2c_c4_occ2_$i.err
python -c "import json;d=json.loads(open('gpurun_out/r2c_c4_occ2_$i.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['bitwise_reproducible'],d['logdet'])"
done
