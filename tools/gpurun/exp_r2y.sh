#!/bin/bash
# Round-2 session 4: de-phasing the co-resident CTAs of the v2 DMMA flush (SF_DMMA_DEPHASE).
mkdir -p gpurun_out/v; O=gpurun_out/v/dephase.log; : > $O
for rep in 1 2; do
for v in "SF_DMMA_DEPHASE=0" "SF_DMMA_DEPHASE=1"; do
  env $v timeout 300 python tools/exp_dmma.py 2>&1 | sed "s/^\[\]/[$v]/" >> $O
done
done
for v in "SF_DMMA_DEPHASE=0" "SF_DMMA_DEPHASE=1"; do
  echo "== bench $v" >> $O
  for w in chol_f64_n65536_s512 chol_f64_n16384_s512 qr_f64_n8192_s128; do
    env $v SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu 2>>$O | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['config']['workload'], 'ms', round(d['ms_per_step'], 3), 'frac', d['roofline']['frac'])" >> $O 2>&1
  done
done
cat $O | grep -v "^$" | cut -c1-200
