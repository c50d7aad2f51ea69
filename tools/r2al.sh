timeout 600 python tools/trace_legacy.py --workload c4 --tile 128 --ordering identity > gpurun_out/r2al_c4.txt 2>&1; tail -14 gpurun_out/r2al_c4.txt
timeout 600 python tools/trace_legacy.py --workload c2 --tile 128 > gpurun_out/r2al_c2.txt 2>&1; tail -14 gpurun_out/r2al_c2.txt
