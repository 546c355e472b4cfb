#!/bin/bash
# Run on the GPU box: microbenchmarks + cuBLAS reference points, with clocks sampled.
set -e
cd "$(dirname "$0")"
mkdir -p ../gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > ../gpurun_out/calib_clocks.csv &
SMI=$!
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o calib calib.cu
./calib > ../gpurun_out/calib_micro.json
python cublas_peaks.py > ../gpurun_out/calib_cublas.json
kill $SMI
nproc > ../gpurun_out/calib_host.txt; lscpu >> ../gpurun_out/calib_host.txt; free -g >> ../gpurun_out/calib_host.txt
cat ../gpurun_out/calib_micro.json ../gpurun_out/calib_cublas.json
