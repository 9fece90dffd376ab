#!/bin/bash
# round 2 call 7: fast loader on the solve layouts (KM / KN) + SPREAD / stage-count A/B on cfg2
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
( time timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schur.py tests/test_gpu_r2.py -x -q ) > gpurun_out/c7_tests.log 2>&1; echo rc=$? >> gpurun_out/c7_tests.log
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c7_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c7_cfg3.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c7_cfg1.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_05019_b200/csrc tools/engine_bench.cu -o /tmp/engine_bench && /tmp/engine_bench > gpurun_out/c7_engine.txt 2>&1
for sp in 1 2; do
  DD_AUX_DEFS="DDK_FASTLD_SPREAD=$sp" python dd_build.py > /dev/null
  timeout 900 python bench.py --config cfg2 $A > gpurun_out/c7_cfg2_spread$sp.log 2>&1
done
DD_AUX_DEFS="DD_AUX_AB DDK_FASTLD_SPREAD=2" python dd_build.py > /dev/null
DD_AUX_K3CFG=12 timeout 900 python bench.py --config cfg2 $A > gpurun_out/c7_cfg2_k12_spread2.log 2>&1
python dd_build.py > /dev/null
