#!/bin/bash
# round 2 call 13: backward-update split-K reduction: in-kernel fold only for G <= 8 (batched partial loads), separate reduce kernel above
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
( time timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -x -q ) > gpurun_out/c13_tests.log 2>&1; echo rc=$? >> gpurun_out/c13_tests.log
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c13_cfg1.log 2>&1
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c13_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c13_cfg3.log 2>&1
for g in 0 4 32; do
  DD_AUX_DEFS="DDK_BUPD_FOLD_MAXG=$g" python dd_build.py > /dev/null
  timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c13_cfg1_g$g.log 2>&1
  timeout 900 python bench.py --config cfg2 $A > gpurun_out/c13_cfg2_g$g.log 2>&1
  timeout 900 python bench.py --config cfg3 $A > gpurun_out/c13_cfg3_g$g.log 2>&1
done
python dd_build.py > /dev/null
