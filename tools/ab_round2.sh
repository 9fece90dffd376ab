timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/n_cfg1.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/n_cfg3.log 2>&1
timeout 900 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/n_cfg2.log 2>&1
