mkdir -p gpurun_out
SF_MGS_NOORDER=1 timeout 150 python -m pytest tests/test_parity_gpu.py -q -k concurrent -p no:cacheprovider > gpurun_out/conc_noorder.log 2>&1; echo "noorder rc=$?"; tail -3 gpurun_out/conc_noorder.log
nvidia-smi --query-gpu=utilization.gpu,memory.used --format=csv
timeout 300 python -m pytest tests/test_parity_gpu.py -q -k "concurrent or qr or graph" > gpurun_out/conc.log 2>&1; echo "order rc=$?"; tail -3 gpurun_out/conc.log
