timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2l_pytest.log 2>&1; tail -3 gpurun_out/r2l_pytest.log
timeout 900 python tools/ab_sched.py --workload c2 --variants default,nochain,neither > gpurun_out/r2l_ab_c2.txt 2>&1; cat gpurun_out/r2l_ab_c2.txt
timeout 900 python tools/ab_sched.py --workload c4 --variants default,nochain,neither > gpurun_out/r2l_ab_c4.txt 2>&1; cat gpurun_out/r2l_ab_c4.txt
timeout 600 python tools/trace.py --workload c2 --tile 120 > gpurun_out/r2l_trace_c2.txt 2>&1; tail -16 gpurun_out/r2l_trace_c2.txt
timeout 600 python tools/trace.py --workload c4 --tile 120 --ordering identity > gpurun_out/r2l_trace_c4.txt 2>&1; tail -16 gpurun_out/r2l_trace_c4.txt
