#!/bin/bash
# round 2 call 11: new defaults (real K3 BK = 24, L2-reduction epilogues in K3 and the solve updates): parity + bench
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python dd_build.py > /dev/null
( time timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schur.py tests/test_gpu_r2.py tests/test_gpu_multigpu.py -x -q ) > gpurun_out/c11_tests.log 2>&1; echo rc=$? >> gpurun_out/c11_tests.log
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c11_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/c11_cfg3.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c11_cfg1.log 2>&1
DD_AUX_DEFS="DDK_SOLVE_RED=0" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/c11_cfg2_solvermw.log 2>&1
python dd_build.py > /dev/null
