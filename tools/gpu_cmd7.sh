timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu4.log 2>&1
tail -2 gpurun_out/pytest_gpu4.log
timeout 300 python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b1_pf.json 2> gpurun_out/b1_pf.err
python -c "import json;d=json.loads(open('gpurun_out/b1_pf.json').read().splitlines()[-1]);print('cfg1 factor_ms',d['factor_ms'],'k1',d['phases']['k1_diag_bk']['ms_per_step'])"
tools/ab_env.sh cfg2 gpurun_out/ab4 "-" "DD_AUX_K3CFG=11" "DD_AUX_K3CFG=12" > gpurun_out/ab4.txt 2>&1
tools/ab_env.sh cfg3 gpurun_out/ab5 "-" "DD_AUX_K3CFG=11" >> gpurun_out/ab4.txt 2>&1
cat gpurun_out/ab4.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k3_update --launch-skip 6 --launch-count 1 -o gpurun_out/k3_cfg2_r1b python bench.py --config cfg2 --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k3.log 2>&1
tail -2 gpurun_out/ncu_k3.log
