#!/bin/bash
mkdir -p gpurun_out/exp
python tools/prof_fact.py chol 256 16 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chol_small -c 1 -o gpurun_out/exp/small -f python tools/prof_fact.py chol 256 16 > gpurun_out/exp/ncu_small.log 2>&1
tail -3 gpurun_out/exp/ncu_small.log
