#!/bin/bash
# One GPU session: gpu tests, smoke, bench (both arms), launch list, ncu full capture of the hot kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err
export SF_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
python tools/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"gemm_f64_kernel|chol_leaf" -c 4 -o gpurun_out/prof_r1 -f python tools/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/bench.json gpurun_out/ref.json; tail -3 gpurun_out/bench.err gpurun_out/ncu_launch.log gpurun_out/ncu_full.log
