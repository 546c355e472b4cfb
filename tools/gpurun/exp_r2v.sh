#!/bin/bash
# Round-2 session 4: A/B of two builds of the DMMA kernels: libstepfact.so (new) against libstepfact_base.so (HEAD).
# Used for the in-step stage barrier (SF_XBAR, lost) and the interior-tile slice loader.
mkdir -p gpurun_out/v; O=gpurun_out/v/xbar.log; : > $O
P=paper_1812_02056_b200
cp $P/libstepfact.so /tmp/new.so; cp $P/libstepfact_base.so /tmp/base.so
for rep in 1 2; do
for v in base new; do
  cp /tmp/$v.so $P/libstepfact.so
  echo "== $v (run $rep)" >> $O
  timeout 300 python tools/exp_dmma.py >> $O 2>&1
done
done
cp /tmp/new.so $P/libstepfact.so
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py tests/test_chunk_flush_gpu.py tests/test_dist_gpu.py -k "not cfg5 and not cfg3" >> $O 2>&1
for v in base new; do
  cp /tmp/$v.so $P/libstepfact.so
  echo "== bench $v" >> $O
  for w in lu_f64_n4096_s64 qr_f64_n8192_s128 chol_f64_n16384_s512; do
    SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu 2>>$O | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['config']['workload'], 'ms', round(d['ms_per_step'], 3), 'frac', d['roofline']['frac'], 'replay', (d.get('graph_replay') or d.get('replay') or {}).get('ms_per_step'))" >> $O 2>&1
  done
done
cp /tmp/new.so $P/libstepfact.so
cat $O | grep -v "^$" | cut -c1-200
