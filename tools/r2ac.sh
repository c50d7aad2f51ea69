cd r806
timeout 600 python tools/trace.py --workload c2 --tile 128 > ../gpurun_out/r2ac_c2.txt 2>&1; tail -12 ../gpurun_out/r2ac_c2.txt
timeout 600 python tools/trace.py --workload c2 --tile 120 > ../gpurun_out/r2ac_c2_120.txt 2>&1; grep span ../gpurun_out/r2ac_c2_120.txt
timeout 900 python tools/trace.py --workload c4 --tile 128 --ordering identity > ../gpurun_out/r2ac_c4_128.txt 2>&1; tail -12 ../gpurun_out/r2ac_c4_128.txt
