#!/bin/bash
# round 2 call 8: ncu of K3 with the fast loader; engine microbench (8-warp tiles); K3 A/B 14 (MBAR + fast loader), 17, 18 (8 warps)
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_05019_b200/csrc tools/engine_bench.cu -o /tmp/engine_bench && /tmp/engine_bench > gpurun_out/c8_engine.txt 2>&1
DD_AUX_DEFS="DD_AUX_AB" python dd_build.py > /dev/null
for c in 13 14 17 18; do DD_AUX_K3CFG=$c timeout 900 python bench.py --config cfg2 $A > gpurun_out/c8_cfg2_k$c.log 2>&1; done
python dd_build.py > /dev/null
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k3_update --launch-skip 8 --launch-count 1 -o gpurun_out/c8_k3_cfg2 python bench.py --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e > gpurun_out/c8_ncu_k3.log 2>&1
