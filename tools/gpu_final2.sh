# Round-end refresh (session 2b): tests, bench lines, K1 ncu on cfg1.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final2_pytest.log 2>&1; tail -2 gpurun_out/final2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; tail -1 gpurun_out/final2_smoke.log
timeout 1200 python bench.py > gpurun_out/final2_bench_cfg2.json 2> gpurun_out/final2_bench_cfg2.err
timeout 900 python bench.py --config cfg3 > gpurun_out/final2_bench_cfg3.json 2> gpurun_out/final2_bench_cfg3.err
timeout 600 python bench.py --config cfg1 > gpurun_out/final2_bench_cfg1.json 2> gpurun_out/final2_bench_cfg1.err
timeout 600 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/final2_bench_cfg0.json 2> gpurun_out/final2_bench_cfg0.err
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final2_bench_cfg4.json 2> gpurun_out/final2_bench_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k' --csv --log-file gpurun_out/final2_launches_cfg1.csv python bench.py --config cfg1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final2_ncu_l1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k1_diag_bk --launch-skip 12 --launch-count 1 -o gpurun_out/final2_k1_cfg1 python bench.py --config cfg1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/final2_ncu_k1.log 2>&1
ls gpurun_out | grep final2
