#!/bin/bash
# Round-2 session 4: DMMA GEMM rate by operand layout vs cuBLAS DGEMM on the same shapes.
mkdir -p gpurun_out/v
timeout 600 python tools/exp_layout.py > gpurun_out/v/layout.log 2>&1
cat gpurun_out/v/layout.log | cut -c1-200
