#!/bin/bash
# round 2 call 14: complex 3M K3 default = fast loader at 3 CTAs/SM (copies up front); backward update without the fold;
# real K3 copy spread 3 vs 6 (BK = 24); then the affected bench lines
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
( time timeout 2400 python -m pytest tests -m gpu -q ) > gpurun_out/c14_pytest.log 2>&1; echo rc=$? >> gpurun_out/c14_pytest.log
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c14_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c14_cfg3.log 2>&1
DD_AUX_DEFS="DDK_FASTLD_SPREAD=3" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c14_cfg2_spread3.log 2>&1
DD_AUX_DEFS="DDK_FASTLD_SPREAD=4" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c14_cfg2_spread4.log 2>&1
python dd_build.py > /dev/null
