#!/bin/bash
# QR MGS: one-pass LL gather + Gram sum (default) vs the two-pass gather (SF_MGS_TWO_PASS=1).
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2q.log
: > $O
./calib/mgs_ll_probe 2>&1 | tail -4 >> $O
SF_MGS_TWO_PASS=1 ./calib/mgs_ll_probe 2>&1 | tail -4 >> $O
timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k "qr" >> $O 2>&1
timeout 600 python -m pytest -q -x tests/test_fp32_gpu.py -k "qr" >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps 5 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'panel_ms', round(r['panel_ms_per_step'],1))"; }
for v in 0 1; do SF_MGS_TWO_PASS=$v b qr_f64_n8192_s128 "TWO_PASS=$v" >> $O; done
for v in 0 1; do SF_MGS_TWO_PASS=$v b qr_f64_n8192_s128 "TWO_PASS=$v" >> $O; done
cat $O
