# TRSMr late (with per-column guard) + plan-order test
mkdir -p gpurun_out/r3
O=gpurun_out/r3
bash tools/ab_env.sh "TC_TRSMR_LATE=0 TC_TRSMR_LATE=1" "c4:128"
TC_DEBUG_ORDER=1 TC_TRSMR_LATE=1 timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_b10.txt 2>&1; grep -i topolog $O/trace_c4_128_b10.txt; head -40 $O/trace_c4_128_b10.txt | tail -30
timeout 600 python -m pytest tests/test_gpu_plan_order.py -m gpu -x -q > $O/pytest_b10.log 2>&1; tail -2 $O/pytest_b10.log
TC_TRSMR_LATE=1 timeout 600 python -m pytest tests/test_gpu_plan_order.py tests/test_gpu_stress.py -m gpu -x -q > $O/pytest_b10l.log 2>&1; tail -2 $O/pytest_b10l.log
