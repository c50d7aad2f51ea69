# builds: base (metadata prefetch) / nopf; lookahead 4 on C4; chain-first order on C3
mkdir -p gpurun_out/r3
O=gpurun_out/r3
bash tools/ab.sh "base nopf" "c4:128 c3:128 c2:128" "--no-batch --no-parity"
bash tools/ab.sh "base" "c4:128" "--no-batch --no-parity --lookahead 4"
bash tools/ab_env.sh "TC_ORDER=1" "c3:128 c2:128"
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_b7.txt 2>&1; head -40 $O/trace_c4_128_b7.txt | tail -32
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -x -q --timeout 300 > $O/pytest_b7.log 2>&1; tail -2 $O/pytest_b7.log
