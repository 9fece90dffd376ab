timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu12.log 2>&1; tail -2 gpurun_out/pytest_gpu12.log
timeout 300 python bench.py --config cfg1 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b1_k2.json 2> gpurun_out/b1_k2.err
python -c "import json;d=json.loads(open('gpurun_out/b1_k2.json').read().splitlines()[-1]);print('cfg1 factor_ms',round(d['factor_ms'],2),{k:round(v['ms_per_step'],2) for k,v in d['phases'].items() if k in ['k1_diag_bk','k2_panel','k3_update','linv','rowperm']})"
timeout 900 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b2_k2.json 2> gpurun_out/b2_k2.err
python -c "import json;d=json.loads(open('gpurun_out/b2_k2.json').read().splitlines()[-1]);print('cfg2 factor_ms',round(d['factor_ms'],1),{k:(round(v['ms_per_step'],1),v['tflops']) for k,v in d['phases'].items() if k in ['k2_panel','k3_update']})"
