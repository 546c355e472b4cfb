#!/bin/bash
# f3 push vs broadcast through the distributed driver on ONE GPU (NCCL, 1 rank; loopback G=2):
# the transport's own overhead, not a scaling measurement.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2g.log
: > $O
b() { python bench.py --no-cpu --no-e2e --steps 5 $@ 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$*', round(d['ms_per_step'],3), 'ms', round(d['value']), 'bcast_ms', r.get('bcast_ms_per_step'))"; }
for w in chol_f64_n16384_s512 lu_f64_n4096_s64; do
  b --workload $w --dist >> $O
  b --workload $w --dist --push >> $O
  b --workload $w --loopback 2 >> $O
  b --workload $w --loopback 2 --push >> $O
done
cat $O
