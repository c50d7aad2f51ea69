export TC_UPD_SHAPE=128x64
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity --lookahead 2 > gpurun_out/r2r_trace_c4.txt 2>&1; tail -30 gpurun_out/r2r_trace_c4.txt
