timeout 1500 python bench.py --steps 3 --warmup 3 --trace-out gpurun_out/trace_default.json > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 5 --warmup 3 > gpurun_out/bench_cfg1.log 2>&1
A="--config cfg2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
python bench.py $A > gpurun_out/plain_k3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k3_update -s 6 -c 1 -o gpurun_out/prof_k3_cfg2_final python bench.py $A > gpurun_out/ncu_k3_final.log 2>&1
