#!/bin/bash
# QR MGS: 16-CTA clusters (SF_MGS_CL16) — probe phases, parity, cfg4 bench.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2j.log
: > $O
SF_MGS_CL16=1 SF_MGS_DEBUG=1 ./calib/mgs_ll_probe 2>&1 | tail -8 >> $O
SF_MGS_CL16=1 timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k "qr" >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps 10 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'panel_ms', round(r.get('panel_ms_per_step',0),2))"; }
b qr_f64_n8192_s128 "CL8" >> $O
SF_MGS_CL16=1 b qr_f64_n8192_s128 "CL16" >> $O
SF_MGS_CL16=1 b qr_f32_n8192_s128 "CL16" >> $O
cat $O
