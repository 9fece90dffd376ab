timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_assemble.py -x -q > gpurun_out/pytest_fw.log 2>&1; tail -2 gpurun_out/pytest_fw.log
for fw in 0 1 0 1; do
  DD_AUX_K1FULLW=$fw timeout 300 python bench.py --config cfg1 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b1_fw.json 2> gpurun_out/b1_fw.err
  python -c "import json;d=json.loads(open('gpurun_out/b1_fw.json').read().splitlines()[-1]);print('fullw=$fw cfg1 factor_ms',round(d['factor_ms'],2),'k1',round(d['phases']['k1_diag_bk']['ms_per_step'],2),'berr',d['accuracy']['berr_max'],'graphs',round(d['graphs']['factor_ms'],2))"
done
tools/ab_env.sh cfg2 gpurun_out/ab13 "DD_AUX_K1FULLW=0" "-" > gpurun_out/ab13.txt 2>&1; cat gpurun_out/ab13.txt
