#!/bin/bash
# round 2: Schur-mode GPU tests, fem bench, sanitizers (memcheck + synccheck)
python dd_build.py > /dev/null
python -m pytest tests/test_gpu_schur.py tests/test_gpu_multigpu.py -q -s > gpurun_out/r2_schur.log 2>&1; echo rc=$? >> gpurun_out/r2_schur.log
timeout 900 python bench.py --config fem1 --steps 3 --warmup 3 > gpurun_out/r2_bench_fem1.log 2>&1; echo rc=$? >> gpurun_out/r2_bench_fem1.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_case.py --config cfg0 > gpurun_out/san_${tool}_cfg0.log 2>&1; echo rc=$? >> gpurun_out/san_${tool}_cfg0.log
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_case.py --config cfg1 --grid 3 3 2 --size 64 > gpurun_out/san_${tool}_cfg1s.log 2>&1; echo rc=$? >> gpurun_out/san_${tool}_cfg1s.log
  timeout 600 $CS --tool $tool --print-limit 20 python tools/sanitize_case.py --schur > gpurun_out/san_${tool}_schur.log 2>&1; echo rc=$? >> gpurun_out/san_${tool}_schur.log
done
