#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DSF_P64_TIMING -I include -I paper_1812_02056_b200/csrc calib/p64_probe.cu -o /tmp/p64_probe_li
ncu --set full --clock-control none --import-source on -k regex:panel64 -s 2 -c 1 -o gpurun_out/ncu_probe -f /tmp/p64_probe_li > /dev/null 2>&1
ncu -i gpurun_out/ncu_probe.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu_probe_cuda.csv 2>&1
ncu -i gpurun_out/ncu_probe.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_probe_sass.csv 2>&1
ls -la gpurun_out/ncu_probe*
