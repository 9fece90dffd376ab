#!/bin/bash
# round 2 A/B 3: 32-ary target search in K3 (default) vs binary search; complex 3M tile at 3 CTAs/SM
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schur.py -q -x > gpurun_out/ab3_tests.log 2>&1; echo rc=$? >> gpurun_out/ab3_tests.log
timeout 900 python bench.py --config cfg2 $A > gpurun_out/ab3_cfg2_s32.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab3_cfg3_s32.log 2>&1
DD_AUX_DEFS="DDK_K3_SEARCH32=0" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/ab3_cfg2_bin.log 2>&1
DD_AUX_DEFS="DD_AUX_AB" python dd_build.py > /dev/null
DD_AUX_K3CFG=19 timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab3_cfg3_k19.log 2>&1
DD_AUX_K3CFG=9 timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab3_cfg3_k9.log 2>&1
python dd_build.py > /dev/null
