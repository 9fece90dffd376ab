timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final4_pytest.log 2>&1; tail -2 gpurun_out/final4_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4_smoke.log 2>&1; tail -1 gpurun_out/final4_smoke.log
timeout 1200 python bench.py > gpurun_out/final4_bench_cfg2.json 2> gpurun_out/final4_bench_cfg2.err
timeout 600 python bench.py --config cfg1 > gpurun_out/final4_bench_cfg1.json 2> gpurun_out/final4_bench_cfg1.err
timeout 600 python bench.py --config cfg0 --no-cpu-baseline > gpurun_out/final4_bench_cfg0.json 2> gpurun_out/final4_bench_cfg0.err
