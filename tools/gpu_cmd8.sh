timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu5.log 2>&1
tail -2 gpurun_out/pytest_gpu5.log
./tools/engine_bench.bin > gpurun_out/engine2.txt 2>&1; tail -8 gpurun_out/engine2.txt
timeout 900 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --trace-out gpurun_out/trace_cfg2c.json > gpurun_out/b2c.json 2> gpurun_out/b2c.err
python -c "import json;d=json.loads(open('gpurun_out/b2c.json').read().splitlines()[-1]);print('cfg2 factor',d['factor_ms'],d['value'],'solve/batch',d['solve_ms_per_batch'],{k:(round(v['ms_per_step'],1),v['tflops']) for k,v in d['phases'].items() if k in ['fupd','bupd','spmv','assemble']}, d.get('assemble'))"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_diag_bk --launch-skip 12 --launch-count 1 -o gpurun_out/k1_cfg1 python bench.py --config cfg1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1.log 2>&1
tail -1 gpurun_out/ncu_k1.log
