#!/bin/bash
# DMMA v2 epilogue: red.global.add.f64 from registers (SF_DMMA_RED=1) vs bulk reduce.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2l.log
: > $O
for v in 0 1; do echo "SF_DMMA_RED=$v" >> $O; SF_DMMA_RED=$v python tools/prof_syrk_k.py >> $O 2>&1; done
SF_DMMA_RED=1 timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k "chol_cfg3_sampled or planted or chol_small_grid or lu_cfg2 or qr_small" >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps $3 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'frac', round(r['frac'],4))"; }
for v in 0 1; do SF_DMMA_RED=$v b chol_f64_n16384_s512 "RED=$v" 10 >> $O; done
for v in 0 1; do SF_DMMA_RED=$v b chol_f64_n65536_s512 "RED=$v" 3 >> $O; done
cat $O
