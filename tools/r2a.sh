set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -m pytest tests -q -m gpu -x > gpurun_out/r2a_pytest.log 2>&1; tail -3 gpurun_out/r2a_pytest.log
timeout 900 python bench.py --workload c4 --tile 120 --ordering identity --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline --no-profile > gpurun_out/r2a_c4_120.json 2> gpurun_out/r2a_c4_120.err; tail -c 600 gpurun_out/r2a_c4_120.json
timeout 900 python bench.py --workload c4 --tile 240 --ordering identity --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-profile > gpurun_out/r2a_c4_240.json 2> gpurun_out/r2a_c4_240.err; tail -c 600 gpurun_out/r2a_c4_240.json; tail -5 gpurun_out/r2a_c4_240.err
