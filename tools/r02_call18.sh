#!/bin/bash
# round 2 call 18: k_assemble with the accumulate mode as a template parameter: assembly / Schur / multi-GPU tests, then the bench lines (they carry the `assemble` object)
mkdir -p gpurun_out
python dd_build.py > /dev/null
B="python bench.py"
( time timeout 1500 python -m pytest tests/test_gpu_assemble.py tests/test_gpu_schur.py tests/test_gpu_multigpu.py tests/test_gpu_parity.py -q ) > gpurun_out/c18_tests.log 2>&1; echo rc=$? >> gpurun_out/c18_tests.log
timeout 1500 $B --trace-out gpurun_out/f_trace_cfg2.json > gpurun_out/f_bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/f_bench_cfg2.log
timeout 900 $B --config cfg3 --steps 2 --warmup 3 > gpurun_out/f_bench_cfg3.log 2>&1
timeout 900 $B --config cfg1 --steps 5 --warmup 3 > gpurun_out/f_bench_cfg1.log 2>&1
timeout 900 $B --config cfg3alt --steps 2 --warmup 3 > gpurun_out/f_bench_cfg3alt.log 2>&1
timeout 300 $B --config cfg0 --steps 5 --warmup 3 > gpurun_out/f_bench_cfg0.log 2>&1
timeout 1500 $B --config cfg4 --steps 1 --warmup 3 > gpurun_out/f_bench_cfg4.log 2>&1
timeout 600 $B --config fem1 --steps 5 --warmup 3 > gpurun_out/f_bench_fem1.log 2>&1
timeout 600 $B --config fem3 --steps 5 --warmup 3 > gpurun_out/f_bench_fem3.log 2>&1
