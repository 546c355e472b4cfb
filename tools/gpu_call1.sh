#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tgpu.log 2>&1
bash tools/sweep.sh > gpurun_out/sweep.log 2>&1
python tools/quick_perf.py > gpurun_out/perf2.log 2>&1
python tools/prof_panel.py > gpurun_out/pp2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm|Kernel" -c 2 -o gpurun_out/prof_cublas -f python tools/cublas_dgemm.py > gpurun_out/ncu_cublas.log 2>&1
tail -5 gpurun_out/tgpu.log; cat gpurun_out/smoke.log gpurun_out/sweep.log gpurun_out/perf2.log gpurun_out/pp2.log; tail -3 gpurun_out/ncu_cublas.log
