#!/bin/bash
# round 2 call 6: fast loader (running per-thread cp.async pointers, copies issued between k-steps)
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
( time timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schur.py tests/test_gpu_r2.py -x -q ) > gpurun_out/c6_tests.log 2>&1; echo rc=$? >> gpurun_out/c6_tests.log
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c6_cfg2_fast.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c6_cfg3_fast.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c6_cfg1_fast.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_05019_b200/csrc tools/engine_bench.cu -o /tmp/engine_bench && /tmp/engine_bench > gpurun_out/c6_engine_fast.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDDK_FASTLD=0 -I paper_2002_05019_b200/csrc tools/engine_bench.cu -o /tmp/engine_bench0 && /tmp/engine_bench0 > gpurun_out/c6_engine_slow.txt 2>&1
DD_AUX_DEFS="DD_AUX_AB" python dd_build.py > /dev/null
for c in 12; do DD_AUX_K3CFG=$c timeout 900 python bench.py --config cfg2 $A > gpurun_out/c6_cfg2_k$c.log 2>&1; done
DD_AUX_K3CFG=19 timeout 900 python bench.py --config cfg3 $A > gpurun_out/c6_cfg3_k19.log 2>&1
python dd_build.py > /dev/null
