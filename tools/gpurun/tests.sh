#!/bin/bash
# Full GPU suite + smoke, logs under gpurun_out/.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python __graft_entry__.py --smoke >> gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
