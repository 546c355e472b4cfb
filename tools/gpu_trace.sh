#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/traces.log
: > $O
python tools/trace.py lu 4096 64 >> $O 2>&1
SF_LU_P64=0 python tools/trace.py lu 4096 64 >> $O 2>&1
python tools/trace.py qr 8192 128 >> $O 2>&1
python tools/trace.py chol 16384 512 --steps-shown 4 >> $O 2>&1
python tools/trace.py chol 256 16 --steps-shown 4 >> $O 2>&1
tail -5 $O
