#!/bin/bash
# round 2 call 10: K3 epilogue as L2 reductions (red.add.f64) + warp aliasing on ragged tiles: probes, parity, A/B
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_05019_b200/csrc tools/engine_bench.cu -o /tmp/engine_bench && /tmp/engine_bench probes > gpurun_out/c10_probes.txt 2>&1
python dd_build.py > /dev/null
( time timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schur.py tests/test_gpu_r2.py tests/test_gpu_multigpu.py -x -q ) > gpurun_out/c10_tests.log 2>&1; echo rc=$? >> gpurun_out/c10_tests.log
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c10_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c10_cfg3.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c10_cfg1.log 2>&1
DD_AUX_DEFS="DDK_K3_RED=0" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c10_cfg2_nored.log 2>&1
DD_AUX_DEFS="DDK_K3_ALIAS=0" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c10_cfg2_noalias.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c10_cfg3_noalias.log 2>&1
DD_AUX_DEFS="DD_AUX_AB" python dd_build.py > /dev/null
DD_AUX_K3CFG=16 timeout 900 python bench.py --config cfg2 $A > gpurun_out/c10_cfg2_k16.log 2>&1
python dd_build.py > /dev/null
