timeout 900 python tools/ab_sched.py --workload c4 --variants default,nochain,nosplit,neither,la3 > gpurun_out/r2h_ab_c4.txt 2>&1; cat gpurun_out/r2h_ab_c4.txt
timeout 600 python tools/ab_sched.py --workload c2 --variants default,nochain,nosplit,neither > gpurun_out/r2h_ab_c2.txt 2>&1; cat gpurun_out/r2h_ab_c2.txt
timeout 600 python tools/trace.py --workload c4 --tile 120 --ordering identity > gpurun_out/r2h_trace_c4.txt 2>&1; cat gpurun_out/r2h_trace_c4.txt | tail -16
timeout 600 python tools/trace.py --workload c2 --tile 120 > gpurun_out/r2h_trace_c2.txt 2>&1; cat gpurun_out/r2h_trace_c2.txt | tail -16
