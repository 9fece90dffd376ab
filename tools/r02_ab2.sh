#!/bin/bash
# round 2 A/B: K3 tile shapes on cfg2 (AB build), default config 13 on the same box
A="--config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
DD_AUX_DEFS="DD_AUX_AB" python dd_build.py > /dev/null
for c in 13 16 17 18; do DD_AUX_K3CFG=$c timeout 900 python bench.py $A > gpurun_out/ab2_cfg2_k$c.log 2>&1; done
DD_AUX_K3CFG=17 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "scaled or corpus" > gpurun_out/ab2_parity_k17.log 2>&1; echo rc=$? >> gpurun_out/ab2_parity_k17.log
python dd_build.py > /dev/null
# f3 supernode (ND leaf) size A/B on fem1
for L in 64 256 512; do DD_FEM_LEAF=$L timeout 600 python bench.py --config fem1 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ab2_fem1_leaf$L.log 2>&1; done
# K3 engine: no per-k-step early exit (lets the compiler software-pipeline fragment loads across k-steps)
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
DD_AUX_DEFS="DDK_KSTEP_BREAK=0" python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg2 $A > gpurun_out/ab2_cfg2_nobreak.log 2>&1
timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab2_cfg3_nobreak.log 2>&1
python dd_build.py > /dev/null
timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab2_cfg3_base.log 2>&1
# solve: backward split-K reduction folded into k_bupd (default) vs the separate reduce kernel
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "multi_rhs or scaled or graphs or padded" > gpurun_out/ab2_fold_tests.log 2>&1; echo rc=$? >> gpurun_out/ab2_fold_tests.log
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
DD_AUX_BUPD_FOLD=0 timeout 900 python bench.py --config cfg3 $A > gpurun_out/ab2_cfg3_nofold.log 2>&1
DD_AUX_BUPD_FOLD=0 timeout 900 python bench.py --config cfg2 $A > gpurun_out/ab2_cfg2_nofold.log 2>&1
timeout 900 python bench.py --config cfg2 $A > gpurun_out/ab2_cfg2_fold.log 2>&1
