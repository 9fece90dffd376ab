# Refresh the default bench line (cfg2) with the trace; used for profiles/ updates.
timeout 1500 python bench.py --steps 3 --warmup 3 --trace-out gpurun_out/trace_default.json > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
