#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/p64c.log
: > $O
./calib/p64_probe >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "lu_ or graph" >> $O 2>&1
SF_CHOL_P64_MAXM=100000 timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol_small or chol_cfg1 or planted or not_pd" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_fp32_gpu.py tests/test_dist_gpu.py -k "lu" >> $O 2>&1
python tools/trace.py lu 4096 64 --steps-shown 2 >> $O 2>&1
python tools/trace.py lu 4096 64 f32 --steps-shown 1 >> $O 2>&1
SF_CHOL_P64_MAXM=100000 python tools/trace.py chol 256 16 --steps-shown 1 >> $O 2>&1
SF_CHOL_P64_MAXM=100000 python tools/trace.py chol 16384 512 --steps-shown 1 >> $O 2>&1
grep -v "^\s*[0-9]" $O | grep -v Warn | grep -v _warn
