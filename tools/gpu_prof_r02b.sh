#!/bin/bash
# first: parity of the call-free leaves, then the profiling script
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol_small or chol_cfg1 or planted or not_pd or lu_small or lu_cfg2 or chol_cfg3" > gpurun_out/leaf_tests.log 2>&1
timeout 600 python -m pytest -x -q tests/test_fp32_gpu.py -k "chol" >> gpurun_out/leaf_tests.log 2>&1
./calib/p64_probe | tail -2 >> gpurun_out/leaf_tests.log 2>&1
bash tools/gpu_prof_r02.sh
tail -5 gpurun_out/leaf_tests.log
