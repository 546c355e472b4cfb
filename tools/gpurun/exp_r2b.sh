#!/bin/bash
# A/B: QR MGS rows in registers (SF_MGS_NR 64 / 32).
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2b.log
: > $O
b() { python bench.py --no-cpu --no-e2e --steps 10 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'panel_ms', round(r.get('panel_ms_per_step',0),2))"; }
for v in 64 32; do SF_MGS_NR=$v b qr_f64_n8192_s128 "NR=$v" >> $O; done
for v in 64 32; do SF_MGS_NR=$v b qr_f32_n8192_s128 "NR=$v" >> $O; done
SF_MGS_NR=32 python tools/trace.py qr 8192 128 --steps-shown 2 > gpurun_out/exp/trace_qr_nr32.log 2>&1
SF_MGS_NR=32 timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k qr >> $O 2>&1
cat $O
