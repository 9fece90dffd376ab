timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu9.log 2>&1
tail -3 gpurun_out/pytest_gpu9.log
timeout 300 python bench.py --config cfg1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b1_z.json 2> gpurun_out/b1_z.err
python -c "import json;d=json.loads(open('gpurun_out/b1_z.json').read().splitlines()[-1]);print('cfg1 factor_ms',d['factor_ms'],'k1',d['phases']['k1_diag_bk']['ms_per_step'],'solve/batch',d['solve_ms_per_batch'])"
timeout 900 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b3_z.json 2> gpurun_out/b3_z.err
python -c "import json;d=json.loads(open('gpurun_out/b3_z.json').read().splitlines()[-1]);print('cfg3 factor_ms',d['factor_ms'],'solve/batch',d['solve_ms_per_batch'],{k:(round(v['ms_per_step'],1),v['tflops']) for k,v in d['phases'].items() if k in ['fupd','bupd','spmv','fdiag','bdiag']}, d['accuracy']['berr_max'])"
