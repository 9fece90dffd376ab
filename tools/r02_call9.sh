#!/bin/bash
# round 2 call 9: per-tile fixed-cost probes (engine microbench), K3 BK = 24 (A/B cfg 16), solve spread / complex fast-loader A/B
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_05019_b200/csrc tools/engine_bench.cu -o /tmp/engine_bench && /tmp/engine_bench probes > gpurun_out/c9_probes.txt 2>&1
python dd_build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/c9_tests.log 2>&1; echo rc=$? >> gpurun_out/c9_tests.log
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c9_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c9_cfg3.log 2>&1
DD_AUX_DEFS="DDK_SOLVE_FAST_C=0" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c9_cfg3_solveslowc.log 2>&1
DD_AUX_DEFS="DD_AUX_AB" python dd_build.py > /dev/null
DD_AUX_K3CFG=16 timeout 900 python bench.py --config cfg2 $A > gpurun_out/c9_cfg2_k16.log 2>&1
python dd_build.py > /dev/null
