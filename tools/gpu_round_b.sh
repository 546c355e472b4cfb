#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/round_b.log
: > $O
./calib/p64_probe >> $O 2>&1
timeout 1200 python -m pytest -x -q tests/test_dist_gpu.py >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "qr" >> $O 2>&1
cat $O | grep -v "^$" | tail -30
