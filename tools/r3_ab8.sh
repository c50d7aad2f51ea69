# Bd(k+D+1) one column earlier (TC_BD_EARLY); C5 batch grid share 1/2/4
mkdir -p gpurun_out/r3
O=gpurun_out/r3
bash tools/ab_env.sh "TC_BD_EARLY=0 TC_BD_EARLY=1" "c4:128 c3:128"
for sh in 1 2 4; do
timeout 600 python bench.py --workload c5 --share $sh --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-profile > $O/c5_share$sh.json 2> $O/c5_share$sh.err
python -c "import json; d=json.loads(open('$O/c5_share$sh.json').read().strip().splitlines()[-1]); print('c5 share $sh', round(d['value'],2), 'fact/s e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3), 'repro', d.get('bitwise_reproducible'))"
done
timeout 600 python tools/trace.py --workload c4 --tile 128 --ordering identity > $O/trace_c4_128_b8.txt 2>&1; head -40 $O/trace_c4_128_b8.txt | tail -22
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -x -q --timeout 300 > $O/pytest_b8.log 2>&1; tail -2 $O/pytest_b8.log
