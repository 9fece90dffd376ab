# Round-end measurement set (one B200 via gpurun): GPU tests, smoke, every bench line, the default command's ncu launch list and ncu --set full captures of the dominant kernels.  Usage: gpurun -- bash tools/round_end_measure.sh
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final3_pytest.log 2>&1; tail -2 gpurun_out/final3_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; tail -1 gpurun_out/final3_smoke.log
timeout 1200 python bench.py > gpurun_out/final3_bench_cfg2.json 2> gpurun_out/final3_bench_cfg2.err
timeout 900 python bench.py --config cfg3 > gpurun_out/final3_bench_cfg3.json 2> gpurun_out/final3_bench_cfg3.err
timeout 600 python bench.py --config cfg1 > gpurun_out/final3_bench_cfg1.json 2> gpurun_out/final3_bench_cfg1.err
timeout 600 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/final3_bench_cfg0.json 2> gpurun_out/final3_bench_cfg0.err
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final3_bench_cfg4.json 2> gpurun_out/final3_bench_cfg4.err
timeout 600 python bench.py --impl reference > gpurun_out/final3_bench_ref_cfg2.json 2> gpurun_out/final3_bench_ref_cfg2.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k' --csv --log-file gpurun_out/final3_launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final3_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k3_update --launch-skip 6 --launch-count 1 -o gpurun_out/final3_k3_cfg2 python bench.py --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e > gpurun_out/final3_ncu_k3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_assemble --launch-skip 1 --launch-count 1 -o gpurun_out/final3_asm_cfg2 python bench.py --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e > gpurun_out/final3_ncu_asm.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k3_update --launch-skip 6 --launch-count 1 -o gpurun_out/final3_k3_cfg3 python bench.py --config cfg3 --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e > gpurun_out/final3_ncu_k3c.log 2>&1
ls gpurun_out | grep final3
