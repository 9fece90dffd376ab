timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu6.log 2>&1
tail -2 gpurun_out/pytest_gpu6.log
for q in 0 4; do
DD_AUX_K1MAXQ=$q timeout 300 python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b1_q$q.json 2> gpurun_out/b1_q$q.err
python -c "import json;d=json.loads(open('gpurun_out/b1_q$q.json').read().splitlines()[-1]);print('cfg1 maxq=$q factor_ms',d['factor_ms'],'k1',d['phases']['k1_diag_bk']['ms_per_step'],'solve/batch',d['solve_ms_per_batch'])"
done
tools/ab_env.sh cfg2 gpurun_out/ab6 "-" "DD_AUX_K3CFG=13" > gpurun_out/ab6.txt 2>&1
tools/ab_env.sh cfg3 gpurun_out/ab7 "-" "DD_AUX_K3CFG=13" >> gpurun_out/ab6.txt 2>&1
cat gpurun_out/ab6.txt
