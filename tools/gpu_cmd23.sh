for defs in "-" "DDK_NT1=128" "DDK_NT1=512"; do
  d=$defs; [ "$d" = "-" ] && d=""
  DD_AUX_DEFS="$d" python dd_build.py --force > /dev/null 2>&1 || { echo "build $defs failed"; continue; }
  timeout 300 python bench.py --config cfg1 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b1_nt.json 2> gpurun_out/b1_nt.err
  python -c "import json;d=json.loads(open('gpurun_out/b1_nt.json').read().splitlines()[-1]);print('$defs cfg1 factor_ms',round(d['factor_ms'],2),'k1',round(d['phases']['k1_diag_bk']['ms_per_step'],2),'berr',d['accuracy']['berr_max'])" || tail -3 gpurun_out/b1_nt.err
done
DD_AUX_DEFS="DDK_NT1=128" python dd_build.py --force > /dev/null 2>&1
DD_AUX_DEFS="DDK_NT1=128" timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "isolated or cfg1_full or spec" > gpurun_out/pytest_nt128.log 2>&1; tail -2 gpurun_out/pytest_nt128.log
python dd_build.py --force > /dev/null 2>&1
