# Md/M split of the near update (TC_MSPLIT): A/B, trace, parity subset; standalone POTRF latency
mkdir -p gpurun_out/r3
O=gpurun_out/r3
./tools/potrf_ab > $O/potrf_ab.txt 2>&1; cat $O/potrf_ab.txt
bash tools/ab_env.sh "TC_MSPLIT=0 TC_MSPLIT=1" "c4:128 c3:128 c2:128"
TC_DEBUG_ORDER=1 timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_ms.txt 2>&1; head -12 $O/trace_c4_128_ms.txt; grep -A40 "launch timeline" $O/trace_c4_128_ms.txt | head -40; grep -i topolog $O/trace_c4_128_ms.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -x -q --timeout 300 > $O/pytest_ms.log 2>&1; tail -2 $O/pytest_ms.log
