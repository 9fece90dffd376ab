#!/bin/bash
# round 2 call 5: full GPU suite on HEAD, then A/B 3 (K3 search) and the K3 tile-shape A/B on cfg2
mkdir -p gpurun_out
python dd_build.py > /dev/null
( time timeout 1800 python -m pytest tests -m gpu -x -q ) > gpurun_out/c5_tests.log 2>&1; echo rc=$? >> gpurun_out/c5_tests.log
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c5_cfg2_s32.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c5_cfg3_s32.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c5_cfg1.log 2>&1
DD_AUX_DEFS="DDK_K3_SEARCH32=0" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c5_cfg2_bin.log 2>&1
DD_AUX_DEFS="DD_AUX_AB" python dd_build.py > /dev/null
for c in 16 17 18; do DD_AUX_K3CFG=$c timeout 900 python bench.py --config cfg2 $A > gpurun_out/c5_cfg2_k$c.log 2>&1; done
DD_AUX_K3CFG=19 timeout 900 python bench.py --config cfg3 $A > gpurun_out/c5_cfg3_k19.log 2>&1
python dd_build.py > /dev/null
