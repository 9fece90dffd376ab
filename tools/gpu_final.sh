# Round-end measurement set (run on one B200 via gpurun): tests, default bench line, other configs,
# ncu launch list of the default command, one ncu --set full capture of the dominant kernel.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; tail -3 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 1200 python bench.py > gpurun_out/final_bench_cfg2.json 2> gpurun_out/final_bench_cfg2.err; tail -c 600 gpurun_out/final_bench_cfg2.json
timeout 900 python bench.py --config cfg3 > gpurun_out/final_bench_cfg3.json 2> gpurun_out/final_bench_cfg3.err
timeout 600 python bench.py --config cfg1 > gpurun_out/final_bench_cfg1.json 2> gpurun_out/final_bench_cfg1.err
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final_bench_cfg4.json 2> gpurun_out/final_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final_bench_ref_cfg2.json 2> gpurun_out/final_bench_ref_cfg2.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k' --csv --log-file gpurun_out/final_launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k3_update --launch-skip 6 --launch-count 1 -o gpurun_out/final_k3_cfg2 python bench.py --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_k3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_assemble --launch-skip 1 --launch-count 1 -o gpurun_out/final_asm_cfg2 python bench.py --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e > gpurun_out/final_ncu_asm.log 2>&1
ls gpurun_out
