timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu14.log 2>&1; tail -2 gpurun_out/pytest_gpu14.log
tools/ab_variants.sh cfg2 gpurun_out/ab11 "DDK_KSKIP=0" "-" > gpurun_out/ab11.txt 2>&1; cat gpurun_out/ab11.txt
