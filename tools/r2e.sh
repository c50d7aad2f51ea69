export TILECHOL_EXPERIMENTAL=1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/potrf_bench tools/potrf_bench.cu 2>&1 | grep -i error | head
timeout 120 /tmp/potrf_bench > gpurun_out/r2e_potrf.txt 2>&1; cat gpurun_out/r2e_potrf.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2e_pytest.log 2>&1; tail -15 gpurun_out/r2e_pytest.log
for occ in 1 2; do
timeout 900 python tools/trace.py --workload c4 --tile 120 --ordering identity --occupancy $occ > gpurun_out/r2e_trace_c4_occ$occ.txt 2>&1; cat gpurun_out/r2e_trace_c4_occ$occ.txt | tail -14
done
for occ in 1 2 2; do
timeout 900 python bench.py --workload c4 --ordering identity --occupancy $occ --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity > gpurun_out/r2e_c4.json 2> gpurun_out/r2e_c4.err
python -c "import json;d=json.loads(open('gpurun_out/r2e_c4.json').read().strip().splitlines()[-1]);print('c4 occ',$occ,d['ms_per_step'],d['roofline']['frac'],d['bitwise_reproducible'],repr(d['logdet']))"; tail -2 gpurun_out/r2e_c4.err
done
for w in c2 c3; do
timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-parity --no-profile > gpurun_out/r2e_$w.json 2> gpurun_out/r2e_$w.err
python -c "import json;d=json.loads(open('gpurun_out/r2e_$w.json').read().strip().splitlines()[-1]);print('$w',d['ms_per_step'],d['roofline']['frac'],d['bitwise_reproducible'],repr(d['logdet']))"; tail -2 gpurun_out/r2e_$w.err
done
