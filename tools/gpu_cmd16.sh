timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu10.log 2>&1; tail -2 gpurun_out/pytest_gpu10.log
run1() { timeout 300 python bench.py --config cfg1 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b1_v.json 2> gpurun_out/b1_v.err; python -c "import json;d=json.loads(open('gpurun_out/b1_v.json').read().splitlines()[-1]);print('$1 cfg1 factor_ms',round(d['factor_ms'],2),'k1',round(d['phases']['k1_diag_bk']['ms_per_step'],2),'solve/batch',round(d['solve_ms_per_batch'],2),'graphs',d['graphs']['factor_ms'])"; }
run1 "chains2 split1"
DD_AUX_K3A_SPLIT=0 run1 "chains2 split0"
DD_AUX_DEFS="DDK_K1_CHAINS=1" python dd_build.py --force > /dev/null 2>&1
run1 "chains1 split1"
DD_AUX_K3A_SPLIT=0 run1 "chains1 split0"
python dd_build.py --force > /dev/null 2>&1
