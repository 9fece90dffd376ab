#!/bin/bash
# A/B of compile-time kernel variants on one GPU box:
#   tools/ab_variants.sh CFG OUTDIR "DEFS1" "DEFS2" ...   (each DEFS: space-separated -D switches, "-" = none)
# Rebuilds libdd_aux.so per variant (DD_AUX_DEFS) and runs a short traced bench of CFG.
cfg=$1; out=$2; shift 2
mkdir -p "$out"
i=0
for defs in "$@"; do
  [ "$defs" = "-" ] && defs=""
  DD_AUX_DEFS="$defs" python dd_build.py --force > "$out/build_$i.log" 2>&1 || { echo "build $i failed"; continue; }
  timeout 900 python bench.py --config "$cfg" --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e \
      --trace-out "$out/trace_${cfg}_$i.json" > "$out/bench_${cfg}_$i.json" 2> "$out/bench_${cfg}_$i.err"
  python - "$out/trace_${cfg}_$i.json" "$defs" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); t = d["trace"]
print(f"variant [{sys.argv[2]}] factor_ms={d['line']['factor_ms']:.1f} k3_ms={t['k3_update']['ms']:.1f} "
      f"k3_tf={t['k3_update']['flops']/t['k3_update']['ms']/1e9:.2f}")
PY
  i=$((i+1))
done
python dd_build.py --force > /dev/null 2>&1
