timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1
tail -2 gpurun_out/pytest_gpu8.log
timeout 300 python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b1_y.json 2> gpurun_out/b1_y.err
python -c "import json;d=json.loads(open('gpurun_out/b1_y.json').read().splitlines()[-1]);print('cfg1 factor_ms',d['factor_ms'],'k1',d['phases']['k1_diag_bk']['ms_per_step'],'linv',d['phases']['linv']['ms_per_step'],'solve/batch',d['solve_ms_per_batch'], d['graphs'])"
tools/ab_env.sh cfg3 gpurun_out/ab8 "-" > gpurun_out/ab8.txt 2>&1; cat gpurun_out/ab8.txt
