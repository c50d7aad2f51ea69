# critical split (L_crit / TRSMc, TC_CRIT): A/B, trace, parity subset
mkdir -p gpurun_out/r3
O=gpurun_out/r3
bash tools/ab_env.sh "TC_CRIT=0 TC_CRIT=1" "c4:128 c3:128 c2:128 c3:240"
TC_DEBUG_ORDER=1 timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_crit.txt 2>&1; head -40 $O/trace_c4_128_crit.txt; grep -A30 "launch timeline" $O/trace_c4_128_crit.txt | tail -22; grep -i topolog $O/trace_c4_128_crit.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -x -q --timeout 300 > $O/pytest_crit.log 2>&1; tail -2 $O/pytest_crit.log
