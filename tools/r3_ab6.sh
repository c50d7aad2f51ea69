# builds: base (KC 32 x ST 4, B split) / st3 (KC 32 x ST 3) / kc16 (KC 16 x ST 4); B split on/off
mkdir -p gpurun_out/r3
O=gpurun_out/r3
bash tools/ab.sh "base st3 kc16" "c4:128 c3:128 c2:128" "--no-batch --no-parity"
bash tools/ab_env.sh "TC_BSPLIT=0" "c4:128 c3:128"
TC_DEBUG_ORDER=1 timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_b6.txt 2>&1; head -40 $O/trace_c4_128_b6.txt | tail -32; grep -A40 "launch timeline" $O/trace_c4_128_b6.txt | sed -n 10,40p; grep -i topolog $O/trace_c4_128_b6.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -x -q --timeout 300 > $O/pytest_b6.log 2>&1; tail -2 $O/pytest_b6.log
