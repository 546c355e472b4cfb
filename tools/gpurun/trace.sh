#!/bin/bash
# Kernel timelines (torch.profiler / CUPTI) of one factorization per config -> gpurun_out/traces.log
mkdir -p gpurun_out
O=gpurun_out/traces.log
: > $O
python tools/trace.py lu 4096 64 --steps-shown 4 >> $O 2>&1
python tools/trace.py qr 8192 128 --steps-shown 4 >> $O 2>&1
python tools/trace.py chol 256 16 --steps-shown 4 >> $O 2>&1
tail -5 $O
