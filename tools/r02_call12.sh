#!/bin/bash
# round 2 call 12: complex K3 at 3 CTAs/SM (A/B cfg 19) with the fast loader, copies spread over 1 / 2 / 4 k-steps
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for sp in 1 2 4; do
  DD_AUX_DEFS="DD_AUX_AB DDK_FASTLD_SPREAD=$sp" python dd_build.py > /dev/null
  DD_AUX_K3CFG=19 timeout 900 python bench.py --config cfg3 $A > gpurun_out/c12_cfg3_k19_spread$sp.log 2>&1
done
python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c12_cfg3_default.log 2>&1
