#!/bin/bash
# f3 push transport: dist GPU tests (bounded by timeout: a flag bug would spin).
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2f.log
: > $O
timeout 900 python -m pytest -q -x tests/test_dist_gpu.py -k "push" >> $O 2>&1
echo "push rc=$?" >> $O
timeout 1200 python -m pytest -q -x tests/test_dist_gpu.py -k "nccl" >> $O 2>&1
echo "dist rc=$?" >> $O
cat $O | tail -20
