timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2ak_bench.json 2> gpurun_out/r2ak_bench.err; tail -c 4000 gpurun_out/r2ak_bench.json; tail -5 gpurun_out/r2ak_bench.err
timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 --no-batch > gpurun_out/r2ak_c2.json 2> gpurun_out/r2ak_c2.err; tail -c 1500 gpurun_out/r2ak_c2.json
