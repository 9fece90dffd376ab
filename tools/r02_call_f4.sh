#!/bin/bash
# f4 timing model from the one-GPU emulation (tools/f4_model.py); then the full GPU test suite
python dd_build.py > /dev/null
timeout 1500 python tools/f4_model.py --config cfg3alt --parts 2 4 8 --out gpurun_out/r02_f4_model_cfg3alt.json > gpurun_out/f4_model_cfg3alt.log 2>&1; echo rc=$? >> gpurun_out/f4_model_cfg3alt.log
timeout 1500 python tools/f4_model.py --config cfg1 --parts 2 4 8 --out gpurun_out/r02_f4_model_cfg1.json > gpurun_out/f4_model_cfg1.log 2>&1; echo rc=$? >> gpurun_out/f4_model_cfg1.log
