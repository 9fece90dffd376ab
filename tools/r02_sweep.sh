#!/bin/bash
# round 2 bench sweep (each line -> gpurun_out/r02_bench_<cfg>.json) + ncu captures
python dd_build.py > /dev/null
B="python bench.py"
timeout 1200 $B --steps 3 --warmup 3 --trace-out gpurun_out/r02_trace_cfg2.json > gpurun_out/r02_bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/r02_bench_cfg2.log
timeout 900 $B --config cfg1 --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg1.log 2>&1
timeout 900 $B --config cfg3 --steps 2 --warmup 3 > gpurun_out/r02_bench_cfg3.log 2>&1
timeout 900 $B --config cfg3alt --steps 2 --warmup 3 > gpurun_out/r02_bench_cfg3alt.log 2>&1
timeout 1500 $B --config cfg4 --steps 1 --warmup 3 > gpurun_out/r02_bench_cfg4.log 2>&1
timeout 300 $B --config cfg0 --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg0.log 2>&1
timeout 600 $B --config fem1 --steps 5 --warmup 3 > gpurun_out/r02_bench_fem1.log 2>&1
timeout 600 $B --config fem3 --steps 5 --warmup 3 > gpurun_out/r02_bench_fem3.log 2>&1
timeout 900 $B --impl reference --steps 1 --warmup 0 > gpurun_out/r02_bench_ref_cfg2.log 2>&1
# ncu: K1 on cfg1 (source view), K3 of f3 on fem1
A="--config cfg1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_diag_bk -s 20 -c 1 -o gpurun_out/r02_k1_cfg1 $B $A > gpurun_out/ncu_k1.log 2>&1
A="--config fem1 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_update -s 10 -c 1 -o gpurun_out/r02_k3_fem1 $B $A > gpurun_out/ncu_k3_fem1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_fem1_launches.csv $B $A > gpurun_out/ncu_fem1_launch.log 2>&1
