#!/bin/bash
# round 2 call 16: solve-kernel copy spread (KN layouts) 1 / 2 (default) / 4 on cfg3 (complex) and cfg2 (real) with the final epilogues
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for sp in 1 4; do
  DD_AUX_DEFS="DDK_FASTLD_SPREAD_KN=$sp" python dd_build.py > /dev/null
  timeout 900 python bench.py --config cfg3 $A > gpurun_out/c16_cfg3_kn$sp.log 2>&1
  timeout 900 python bench.py --config cfg2 $A > gpurun_out/c16_cfg2_kn$sp.log 2>&1
done
python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c16_cfg3_kn2.log 2>&1
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c16_cfg2_kn2.log 2>&1
