#!/bin/bash
# A/B: LU short-K tile variant (SF_DMMA_SHORTK) and QR MGS rows per thread (SF_MGS_RPT).
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2a.log
: > $O
b() { python bench.py --no-cpu --no-e2e --steps 10 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'panel_ms', round(r.get('panel_ms_per_step',0),2))"; }
for v in 0 5 6; do SF_DMMA_SHORTK=$v b lu_f64_n4096_s64 "SHORTK=$v" >> $O; done
for v in 64 128; do SF_MGS_RPT=$v b qr_f64_n8192_s128 "RPT=$v" >> $O; done
SF_MGS_RPT=128 python tools/trace.py qr 8192 128 --steps-shown 2 > gpurun_out/exp/trace_qr_rpt128.log 2>&1
SF_DMMA_SHORTK=6 python tools/trace.py lu 4096 64 --steps-shown 2 > gpurun_out/exp/trace_lu_v2.log 2>&1
cat $O
