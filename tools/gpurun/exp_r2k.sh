#!/bin/bash
# cfg5 fp32: where the panel chain's time goes (timeline totals per kernel, per stream).
mkdir -p gpurun_out/exp
python tools/trace.py chol 65536 512 f32 --steps-shown 6 > gpurun_out/exp/trace_cfg5_f32.log 2>&1
head -40 gpurun_out/exp/trace_cfg5_f32.log
