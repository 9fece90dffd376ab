timeout 600 python -m pytest tests -m gpu -q -x -k "isolated or scaled or 3m" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/n_cfg3.log 2>&1
