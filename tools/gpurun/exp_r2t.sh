#!/bin/bash
# DMMA chain latency / rate vs chains per SM sub-partition; LU cfg2 panel-stream trace.
mkdir -p gpurun_out/t; O=gpurun_out/t
./calib/dmma_chain > $O/dmma_chain.json 2>&1; cat $O/dmma_chain.json
SF_DMMA_CHUNK=0 timeout 300 python tools/trace.py lu 4096 64 > $O/trace_lu.txt 2>&1; tail -30 $O/trace_lu.txt
