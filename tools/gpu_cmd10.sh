timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu7.log 2>&1
tail -2 gpurun_out/pytest_gpu7.log
timeout 300 python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b1_x.json 2> gpurun_out/b1_x.err
python -c "import json;d=json.loads(open('gpurun_out/b1_x.json').read().splitlines()[-1]);print('cfg1 factor_ms',d['factor_ms'],'k1',d['phases']['k1_diag_bk']['ms_per_step'],'solve/batch',d['solve_ms_per_batch'])"
timeout 300 python bench.py --config cfg0 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b0.json 2> gpurun_out/b0.err
python -c "import json;d=json.loads(open('gpurun_out/b0.json').read().splitlines()[-1]);print('cfg0 factor_ms',d['factor_ms'],'solve/batch',d['solve_ms_per_batch'])"
