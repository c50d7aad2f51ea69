# Round-2 profiling set: launch list of the default bench, ncu --set full of
# k_persist (C4@128, C2@128) and of the per-class kernels (direct executor, C2@128)
mkdir -p gpurun_out/prof_r2
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof_r2/launches_c4.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-batch --no-parity --ordering identity > gpurun_out/prof_r2/launches_bench.log 2>&1
echo launches $?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o gpurun_out/prof_r2/k_persist_c4_128 python tools/ab_sched.py --workload c4 --tile 128 --reps 1 --variants default > gpurun_out/prof_r2/ncu_c4.log 2>&1
echo c4 $?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_persist -s 1 -c 1 -o gpurun_out/prof_r2/k_persist_c2_128 python tools/ab_sched.py --workload c2 --tile 128 --reps 1 --variants default > gpurun_out/prof_r2/ncu_c2.log 2>&1
echo c2 $?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_update|k_potrf|k_trsm" -s 600 -c 12 -o gpurun_out/prof_r2/classes_c2_128 python tools/ab_sched.py --workload c2 --tile 128 --reps 1 --variants direct > gpurun_out/prof_r2/ncu_cls.log 2>&1
echo cls $?
for f in k_persist_c4_128 k_persist_c2_128 classes_c2_128; do
  $NCU -i gpurun_out/prof_r2/$f.ncu-rep --page raw --csv > gpurun_out/prof_r2/${f}_raw.csv 2>/dev/null
  $NCU -i gpurun_out/prof_r2/$f.ncu-rep --page details > gpurun_out/prof_r2/${f}_details.txt 2>/dev/null
done
ls -la gpurun_out/prof_r2
