cd r1ref
timeout 600 python tools/trace.py --workload c2 --tile 120 > ../gpurun_out/r2aa_r1_c2.txt 2>&1; tail -16 ../gpurun_out/r2aa_r1_c2.txt
timeout 900 python tools/trace.py --workload c4 --tile 120 --ordering identity > ../gpurun_out/r2aa_r1_c4.txt 2>&1; tail -16 ../gpurun_out/r2aa_r1_c4.txt
timeout 900 python tools/trace.py --workload c4 --tile 128 --ordering identity > ../gpurun_out/r2aa_r1_c4_128.txt 2>&1; tail -16 ../gpurun_out/r2aa_r1_c4_128.txt
