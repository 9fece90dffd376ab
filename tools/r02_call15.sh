#!/bin/bash
# round 2 call 15: ncu --set full of the complex 3M K3 (final kernel) on cfg3, same launch index as round 1's capture
mkdir -p gpurun_out
python dd_build.py > /dev/null
A="--config cfg3 --steps 1 --warmup 0 --nrhs 8 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py $A > gpurun_out/c15_plain.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k3_update --launch-skip 6 --launch-count 2 -o gpurun_out/c15_k3_cfg3 python bench.py $A > gpurun_out/c15_ncu.log 2>&1
