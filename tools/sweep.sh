#!/bin/bash
# s-sweep of cfg3 (Cholesky fp64 n=16384) with the profiling hook: total, update and panel ms.
for s in 64 128 168 256 512 1024; do
  for la in 1 0; do
    SF_LOOKAHEAD=$la SF_BENCH_ALLOW_SHORT=1 timeout 120 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --s $s 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(f\"s=$s la=$la total={d['ms_per_step']:.2f} ms  {d['value']:.0f} GF/s  update={r['update_share_of_step']*d['ms_per_step']:.2f} ms ({r['achieved']:.2f} TF/s)  panel={r['panel_ms_per_step']:.2f} ms launches={d['gpu_launches']//3}\")"
  done
done
