# non-critical TRSM(k) ticketed behind B(k+D) (TC_TRSMR_LATE); lookahead 2
mkdir -p gpurun_out/r3
O=gpurun_out/r3
bash tools/ab_env.sh "TC_TRSMR_LATE=0 TC_TRSMR_LATE=1" "c4:128"
bash tools/ab.sh "base" "c4:128" "--no-batch --no-parity --lookahead 2"
TC_DEBUG_ORDER=1 TC_TRSMR_LATE=1 timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_b9.txt 2>&1; grep -i topolog $O/trace_c4_128_b9.txt; head -40 $O/trace_c4_128_b9.txt | tail -34
