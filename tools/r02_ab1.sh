#!/bin/bash
# round 2 A/B: K1 redux argmax (cfg1), persistent K3 (cfg2, cfg3)
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_cfg1_base.log 2>&1
timeout 900 python bench.py --config cfg2 $A > gpurun_out/ab_cfg2_base.log 2>&1
DD_AUX_K3PERSIST=1 timeout 900 python bench.py --config cfg2 $A > gpurun_out/ab_cfg2_persist.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab_cfg3_base.log 2>&1
DD_AUX_K3PERSIST=1 timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab_cfg3_persist.log 2>&1
DD_AUX_DEFS="DDK_REDUX=1" python dd_build.py > /dev/null
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_cfg1_redux.log 2>&1
DD_AUX_DEFS="DDK_REDUX=1 DDK_K1_CHAINS=2" python dd_build.py > /dev/null
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_cfg1_redux_ch2.log 2>&1
python dd_build.py > /dev/null
