set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2g_pytest.log 2>&1; tail -15 gpurun_out/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; tail -3 gpurun_out/r2g_smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; tail -c 3000 gpurun_out/r2g_bench.json; tail -5 gpurun_out/r2g_bench.err
