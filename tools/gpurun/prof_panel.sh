#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/prof_panel.log
: > $O
for v in "SF_LU_P64=1" "SF_LU_P64=0"; do
  env $v python tools/prof_panel.py lu 4096 64 >> $O 2>&1
  env $v python tools/prof_panel.py lu 1024 64 >> $O 2>&1
done
python tools/prof_panel.py chol 65536 512 >> $O 2>&1
python tools/prof_panel.py chol 16384 512 >> $O 2>&1
SF_CHOL_P64_MAXM=1000000 python tools/prof_panel.py chol 16384 64 >> $O 2>&1
python tools/prof_panel.py chol 16384 64 >> $O 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel64 -c 1 -o gpurun_out/ncu_panel64 -f python tools/prof_panel.py lu 4096 64 2 > /dev/null 2>&1
ncu -i gpurun_out/ncu_panel64.ncu-rep --page details --csv > gpurun_out/ncu_panel64_details.csv 2>&1
ncu -i gpurun_out/ncu_panel64.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_panel64_source.csv 2>&1
cat $O
