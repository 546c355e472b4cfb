#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/exp_dmma3.log
: > $O
timeout 300 python tools/exp_dmma.py >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "syrk or chol_small or lu_small or qr_small or planted" >> $O 2>&1
SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu | cut -c1-300 >> $O 2>&1
cat $O
