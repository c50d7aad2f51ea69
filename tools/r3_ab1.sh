# two-level POTRF at nt=128 (TC_POTRF2_MIN): parity under the switch, then A/B
mkdir -p gpurun_out/r3
O=gpurun_out/r3
TC_POTRF2_MIN=16 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 > $O/pytest_p2.log 2>&1; tail -2 $O/pytest_p2.log
TC_POTRF2_MIN=128 timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q --timeout 400 -k "c2_whole or c3_full or c4_full" > $O/pytest_p2f.log 2>&1; tail -2 $O/pytest_p2f.log
bash tools/ab_env.sh "TC_POTRF2_MIN=185 TC_POTRF2_MIN=120" "c2:128 c4:128 c3:128 c2:120"
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128.txt 2>&1; head -30 $O/trace_c4_128.txt
TC_POTRF2_MIN=120 timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_p2.txt 2>&1; head -30 $O/trace_c4_128_p2.txt
