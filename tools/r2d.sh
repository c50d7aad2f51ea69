export TILECHOL_EXPERIMENTAL=1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/gemm_bench tools/gemm_bench.cu 2>&1 | grep -v Warn | head -5
/tmp/gemm_bench > gpurun_out/r2d_gemm_bench.txt 2>&1; cat gpurun_out/r2d_gemm_bench.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "solve" > gpurun_out/r2d_solve.log 2>&1; tail -15 gpurun_out/r2d_solve.log
for occ in 2 2 1; do
timeout 900 python bench.py --workload c4 --ordering identity --occupancy $occ --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity > gpurun_out/r2d_c4.json 2> gpurun_out/r2d_c4.err
python -c "import json;d=json.loads(open('gpurun_out/r2d_c4.json').read().strip().splitlines()[-1]);print('occ',$occ,d['ms_per_step'],d['roofline']['frac'],d['bitwise_reproducible'],repr(d['logdet']))"
done
