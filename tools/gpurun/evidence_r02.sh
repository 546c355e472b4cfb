#!/bin/bash
# Round-2 evidence: GPU suite + smoke, one bench line per workload (default with the CPU
# oracle baseline; the reference arm), the launch list of the default step, ncu --set full of
# the flush kernels of every config (their DRAM traffic feeds profiles/traffic.json).
mkdir -p gpurun_out/ev
rm -f gpurun_out/ev/*
O=gpurun_out/ev
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench_default.json 2> $O/bench_default.err
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for w in chol_f32_n65536_s512 chol_f64_n16384_s512 chol_f32_n16384_s512 lu_f64_n4096_s64 lu_f32_n4096_s64 qr_f64_n8192_s128 qr_f32_n8192_s128 chol_f64_n256_s16; do
  timeout 900 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
export SF_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $CMD > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on"
python tools/prof_fact.py lu 4096 64 > /dev/null 2>&1 && \
  $NCU -k regex:gemm_f64_kernel -s 40 -c 1 -o $O/lu_flush -f python tools/prof_fact.py lu 4096 64 > /dev/null 2>&1
$NCU -k regex:gemm_f64_grouped -s 40 -c 1 -o $O/lu_f1 -f python tools/prof_fact.py lu 4096 64 > /dev/null 2>&1
$NCU -k regex:panel64 -s 20 -c 1 -o $O/lu_panel64 -f python tools/prof_fact.py lu 4096 64 > /dev/null 2>&1
python tools/prof_fact.py qr 8192 128 > /dev/null 2>&1 && \
  $NCU -k regex:gemm_f64v2 -s 60 -c 2 -o $O/qr_flush -f python tools/prof_fact.py qr 8192 128 > /dev/null 2>&1
$NCU -k regex:qr_mgs_ll -s 20 -c 1 -o $O/qr_mgs -f env SF_MGS_COOP=0 python tools/prof_fact.py qr 8192 128 > /dev/null 2>&1
python tools/prof_kernels.py 32768 > /dev/null 2>&1 && \
  $NCU -k regex:gemm_f64v2 -s 1 -c 1 -o $O/syrk_cfg5 -f python tools/prof_kernels.py 32768 > /dev/null 2>&1
python tools/prof_kernels.py 8192 > /dev/null 2>&1 && \
  $NCU -k regex:gemm_f64v2 -s 1 -c 1 -o $O/syrk_cfg3 -f python tools/prof_kernels.py 8192 > /dev/null 2>&1
python tools/prof_f32.py syrk 32768 > /dev/null 2>&1 && \
  $NCU -k regex:gemm_tf32x3_pair -s 2 -c 1 -o $O/tf32_cfg5 -f python tools/prof_f32.py syrk 32768 > /dev/null 2>&1
python tools/prof_fact.py chol 256 16 > /dev/null 2>&1 && \
  $NCU -k regex:chol_small -c 1 -o $O/chol_small -f python tools/prof_fact.py chol 256 16 > /dev/null 2>&1
for r in lu_flush lu_f1 lu_panel64 qr_flush qr_mgs syrk_cfg5 syrk_cfg3 tf32_cfg5 chol_small; do
  echo "== $r"; python tools/ncu_summary.py rep $O/$r.ncu-rep 2>&1
done > $O/ncu_summary.txt
rm -f $O/*.ncu-rep   # gpurun copies back <= 64 MiB: keep the summaries, not the reports
python tools/ncu_summary.py launches $O/launches_cfg5.csv > $O/launches_cfg5_summary.txt 2>&1
tail -2 $O/pytest_gpu.log; cat $O/smoke.log | tail -1
for f in $O/bench_*.json; do echo "== $f"; cut -c1-200 $f; done
