#!/bin/bash
# LU: 8-warp short-K grouped L-shape launches, bulk-reduce epilogue on the 128x64 tiles; panel64
# column-CTA phases.  Parity first.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2h.log
: > $O
timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k "lu or chol_small_grid or planted" >> $O 2>&1
timeout 600 python -m pytest -q -x tests/test_dist_gpu.py -k "lu_dist_loopback or chol_dist_loopback" >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps 10 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'panel_ms', round(r.get('panel_ms_per_step',0),2))"; }
b lu_f64_n4096_s64 "default" >> $O
SF_GROUPED_SHORTK8=0 b lu_f64_n4096_s64 "GROUPED_SHORTK8=0" >> $O
SF_DMMA_BULK=0 b lu_f64_n4096_s64 "DMMA_BULK=0" >> $O
b qr_f64_n8192_s128 "default" >> $O
b chol_f64_n16384_s512 "default" >> $O
SF_DMMA_BULK=0 b chol_f64_n16384_s512 "DMMA_BULK=0" >> $O
python tools/trace.py lu 4096 64 --steps-shown 3 > gpurun_out/exp/trace_lu_h.log 2>&1
./calib/p64_probe | tail -4 >> $O
cat $O
