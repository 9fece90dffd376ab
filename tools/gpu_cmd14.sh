for nb in 16 32 48 64; do
DD_AUX_K1NB=$nb timeout 300 python bench.py --config cfg1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b1_nb$nb.json 2> gpurun_out/b1_nb$nb.err
python -c "import json;d=json.loads(open('gpurun_out/b1_nb$nb.json').read().splitlines()[-1]);print('nb=$nb factor_ms',d['factor_ms'],'k1',d['phases']['k1_diag_bk']['ms_per_step'])"
done
