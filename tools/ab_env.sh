#!/bin/bash
# A/B of runtime env switches (e.g. DD_AUX_K3CFG) on one GPU box, same build:
#   tools/ab_env.sh CFG OUTDIR "VAR=val VAR2=val" ...   ("-" = defaults)
cfg=$1; out=$2; shift 2
mkdir -p "$out"
i=0
for envs in "$@"; do
  [ "$envs" = "-" ] && envs=""
  env $envs timeout 900 python bench.py --config "$cfg" --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e \
      --trace-out "$out/trace_${cfg}_$i.json" > "$out/bench_${cfg}_$i.json" 2> "$out/bench_${cfg}_$i.err"
  python - "$out/trace_${cfg}_$i.json" "$envs" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1])); t = d["trace"]
    print(f"env [{sys.argv[2]}] factor_ms={d['line']['factor_ms']:.1f} k3_ms={t['k3_update']['ms']:.1f} "
          f"k3_tf={t['k3_update']['flops']/t['k3_update']['ms']/1e9:.2f} berr={d['line']['accuracy']['berr_max']:.2e}")
except Exception as e:
    print(f"env [{sys.argv[2]}] failed: {e}")
PY
  i=$((i+1))
done
