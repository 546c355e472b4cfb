#!/bin/bash
# cfg1 one-cluster Cholesky: parity + bench + trace + probe.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2e.log
: > $O
timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k "chol_small or cfg1 or not_pd or chol_det or planted_exact" >> $O 2>&1
timeout 600 python -m pytest -q -x tests/test_solve_gpu.py tests/test_dist_gpu.py -k "chol" >> $O 2>&1
b() { python bench.py --no-cpu --steps 20 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', '$2', round(d['ms_per_step'],4), 'ms', d['value'], 'e2e', d['e2e']['value'])"; }
for v in 1 0; do SF_CHOL_SMALL=$v b chol_f64_n256_s16 "SMALL=$v" >> $O; done
python tools/trace.py chol 256 16 --steps-shown 1 > gpurun_out/exp/trace_chol256.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $O 2>&1
cat $O; head -8 gpurun_out/exp/trace_chol256.log | tail -5
