#!/bin/bash
# round 2 final measurement set (one B200 via gpurun): full GPU suite, smoke, every bench line, the default
# command's ncu launch list, ncu --set full of the dominant kernel (K3 on cfg2), solve kernels on cfg2.
mkdir -p gpurun_out
python dd_build.py > /dev/null
B="python bench.py"
( time timeout 2400 python -m pytest tests -m gpu -q ) > gpurun_out/f_pytest.log 2>&1; echo rc=$? >> gpurun_out/f_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo rc=$? >> gpurun_out/f_smoke.log
timeout 1500 $B --trace-out gpurun_out/f_trace_cfg2.json > gpurun_out/f_bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/f_bench_cfg2.log
timeout 900 $B --config cfg1 --steps 5 --warmup 3 > gpurun_out/f_bench_cfg1.log 2>&1
timeout 900 $B --config cfg3 --steps 2 --warmup 3 > gpurun_out/f_bench_cfg3.log 2>&1
timeout 900 $B --config cfg3alt --steps 2 --warmup 3 > gpurun_out/f_bench_cfg3alt.log 2>&1
timeout 1500 $B --config cfg4 --steps 1 --warmup 3 > gpurun_out/f_bench_cfg4.log 2>&1
timeout 300 $B --config cfg0 --steps 5 --warmup 3 > gpurun_out/f_bench_cfg0.log 2>&1
timeout 600 $B --config fem1 --steps 5 --warmup 3 > gpurun_out/f_bench_fem1.log 2>&1
timeout 600 $B --config fem3 --steps 5 --warmup 3 > gpurun_out/f_bench_fem3.log 2>&1
timeout 900 $B --impl reference --steps 1 --warmup 0 > gpurun_out/f_bench_ref_cfg2.log 2>&1
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k' --csv --log-file gpurun_out/f_launches_cfg2.csv $B $A > gpurun_out/f_ncu_launches.log 2>&1
A="--steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k3_update --launch-skip 8 --launch-count 1 -o gpurun_out/f_k3_cfg2 $B $A > gpurun_out/f_ncu_k3.log 2>&1
A="--steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --clock-control none -k regex:'k_fupd|k_bupd' --launch-skip 600 --launch-count 4 -o gpurun_out/f_solve_cfg2 $B $A > gpurun_out/f_ncu_solve.log 2>&1
ls gpurun_out | grep '^f_'
