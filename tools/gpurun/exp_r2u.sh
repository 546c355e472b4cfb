#!/bin/bash
# LU: F1 fused into the next panel's kernel (SF_LU_FUSED_F1) — tests, cfg2 bench A/B, trace.
mkdir -p gpurun_out/u; O=gpurun_out/u
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_dist_gpu.py tests/test_solve_gpu.py -q -x -k "lu or LU" > $O/test_lu.log 2>&1; echo "rc=$?" >> $O/test_lu.log
tail -3 $O/test_lu.log
for r in 1 2; do
  for f in 0 1; do
    SF_LU_FUSED_F1=$f timeout 300 python bench.py --workload lu_f64_n4096_s64 --no-cpu > $O/lu_f$f.$r.json 2>/dev/null
    echo "fused=$f run $r: $(python -c "import json;d=json.load(open('$O/lu_f$f.$r.json'));r=d['roofline'];print(d['ms_per_step'], 'frac', round(r['frac'],3), 'panel_ms', round(r['panel_ms_per_step'],2), 'e2e', round(d['e2e']['value']), 'graph', d.get('graph_replay_ms'))")"
  done
done
timeout 300 python tools/trace.py lu 4096 64 > $O/trace_lu.txt 2>&1; tail -24 $O/trace_lu.txt
