#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/p64b.log
: > $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "lu_ or graph" >> $O 2>&1
SF_CHOL_P64_MAXM=100000 timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "chol_small or chol_cfg1 or planted or not_pd" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_fp32_gpu.py tests/test_dist_gpu.py -k "lu" >> $O 2>&1
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "qr_small or qr_cfg4 or qr_planted" >> $O 2>&1
python tools/trace.py lu 4096 64 --steps-shown 2 >> $O 2>&1
python tools/trace.py lu 4096 64 f32 --steps-shown 1 >> $O 2>&1
python tools/trace.py qr 8192 128 --steps-shown 1 >> $O 2>&1
SF_CHOL_P64_MAXM=100000 python tools/trace.py chol 256 16 --steps-shown 1 >> $O 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel64 -s 3 -c 1 -o gpurun_out/ncu_panel64b -f python tools/trace.py lu 4096 64 > /dev/null 2>&1
ncu -i gpurun_out/ncu_panel64b.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_panel64b_source.csv 2>&1
ncu -i gpurun_out/ncu_panel64b.ncu-rep --page details --csv > gpurun_out/ncu_panel64b_details.csv 2>&1
grep -v "^\s*[0-9]" $O | grep -v Warn | grep -v _warn
