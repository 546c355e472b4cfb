#!/bin/bash
# round-2 evidence: ncu of the LU flush (cfg2), the QR flush products (cfg4), the cfg5-sized
# SYRK flush (default tile), the panel kernel; the cfg3 s-sweep with clocks; cfg5 fp32 panel choice
mkdir -p gpurun_out
O=gpurun_out/prof_r02.log
: > $O
NCU="ncu --set full --clock-control none --import-source on"
python tools/prof_fact.py lu 4096 64 >> $O 2>&1 && \
  $NCU -k regex:gemm_f64_kernel -s 31 -c 1 -o /tmp/r02_lu_flush -f python tools/prof_fact.py lu 4096 64 > /dev/null 2>&1
python tools/prof_fact.py qr 8192 128 >> $O 2>&1 && \
  $NCU -k regex:gemm_f64v2 -s 60 -c 2 -o /tmp/r02_qr_flush -f python tools/prof_fact.py qr 8192 128 > /dev/null 2>&1
python tools/prof_kernels.py 32768 >> $O 2>&1 && \
  $NCU -k regex:gemm_f64v2 -s 1 -c 1 -o /tmp/r02_syrk -f python tools/prof_kernels.py 32768 > /dev/null 2>&1
$NCU -k regex:panel64 -s 20 -c 1 -o /tmp/r02_panel64 -f python tools/prof_fact.py lu 4096 64 > /dev/null 2>&1
for r in r02_lu_flush r02_qr_flush r02_syrk r02_panel64; do
  echo "== $r" >> $O
  python tools/ncu_summary.py rep /tmp/$r.ncu-rep >> $O 2>&1
done
ncu -i /tmp/r02_syrk.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_syrk_source.csv 2>&1
python tools/measure_all.py sweep > gpurun_out/r02_measure_sweep.json 2> gpurun_out/r02_measure_sweep.err
export SF_BENCH_ALLOW_SHORT=1
for v in 0 1099511627776; do
  echo "== SF_CHOL32_P64_MAXM=$v" >> $O
  SF_CHOL32_P64_MAXM=$v python bench.py --workload chol_f32_n65536_s512 --steps 2 --warmup 3 --no-e2e --no-cpu | cut -c1-400 >> $O 2>&1
done
cat $O | grep -v "^$"
