#!/bin/bash
# A/B of runtime env switches on the solve of a config (same build):  tools/ab_solve.sh CFG OUT "ENV" ...
cfg=$1; out=$2; shift 2; mkdir -p "$out"; i=0
for envs in "$@"; do
  [ "$envs" = "-" ] && envs=""
  env $envs timeout 900 python bench.py --config "$cfg" --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > "$out/b_$i.json" 2> "$out/b_$i.err"
  python - "$out/b_$i.json" "$envs" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); p = d["phases"]
    print(f"env [{sys.argv[2]}] solve_ms/1000={d['solve_ms_per_1000_rhs']:.1f} bupd={p['bupd']['ms_per_step']:.1f} "
          f"fupd={p['fupd']['ms_per_step']:.1f} berr={d['accuracy']['berr_max']:.2e}")
except Exception as e:
    print(f"env [{sys.argv[2]}] failed: {e}")
PY
  i=$((i+1))
done
