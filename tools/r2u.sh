export TC_UPD_SHAPE=128x64
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 4 > gpurun_out/r2u_trace_c4.txt 2>&1; tail -60 gpurun_out/r2u_trace_c4.txt
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 32 > gpurun_out/r2u_trace_c4_32.txt 2>&1; tail -90 gpurun_out/r2u_trace_c4_32.txt
