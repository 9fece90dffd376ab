./tools/engine_bench.bin > gpurun_out/engine3.txt 2>&1; cat gpurun_out/engine3.txt
DD_AUX_K3CFG=14 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "scaled or cfg1_full or spec_corpus or complex_3m or deterministic" > gpurun_out/pytest_mbar.log 2>&1; tail -2 gpurun_out/pytest_mbar.log
tools/ab_env.sh cfg2 gpurun_out/ab9 "-" "DD_AUX_K3CFG=14" > gpurun_out/ab9.txt 2>&1
tools/ab_env.sh cfg3 gpurun_out/ab10 "-" "DD_AUX_K3CFG=14" >> gpurun_out/ab9.txt 2>&1; cat gpurun_out/ab9.txt
