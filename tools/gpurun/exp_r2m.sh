#!/bin/bash
# Long-K flush tile: v2 64x64 (4 CTAs/SM, default) vs the 128x64 4-warp tile now that it has
# the bulk-reduce epilogue too (SF_DMMA=0).
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2m.log
: > $O
for v in 6 0; do echo "SF_DMMA=$v" >> $O; SF_DMMA=$v python tools/prof_syrk_k.py >> $O 2>&1; done
b() { python bench.py --no-cpu --no-e2e --steps $3 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'frac', round(r['frac'],4))"; }
for v in 6 0; do SF_DMMA=$v b chol_f64_n16384_s512 "DMMA=$v" 10 >> $O; done
for v in 6 0; do SF_DMMA=$v b chol_f64_n65536_s512 "DMMA=$v" 3 >> $O; done
cat $O
