# K3 tile-config A/B; run under gpurun from the repo root
timeout 600 python -m pytest tests -m gpu -q -x -k "3m or scaled" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for c in 4 7; do DD_AUX_K3CFG=$c timeout 900 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/n_cfg2_k$c.log 2>&1; done
for c in 5 6 7 8; do DD_AUX_K3CFG=$c timeout 900 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/n_cfg3_k$c.log 2>&1; done
