export TILECHOL_EXPERIMENTAL=1
timeout 600 python tools/occ_diff.py --workload c4 > gpurun_out/r2f_occdiff.txt 2>&1; cat gpurun_out/r2f_occdiff.txt | tail -26
timeout 600 python tools/occ_diff.py --workload c4 --tree off > gpurun_out/r2f_occdiff_notree.txt 2>&1; cat gpurun_out/r2f_occdiff_notree.txt | tail -26
bash tools/r2e.sh
