#!/bin/bash
# End-of-round evidence (gpu_final.sh) plus the full measurement sweep.
bash tools/gpu_final.sh
timeout 1500 python tools/measure_all.py all > gpurun_out/measure_final.json 2> gpurun_out/measure_final.err
tail -2 gpurun_out/measure_final.err
python -c "
import json; d=json.load(open('gpurun_out/measure_final.json'))
for k in ('configs','sweep','paper'):
    for r in d.get(k,[]): print(k, r['config'], r['kind'], r['n'], r['s'], r['dtype'], round(r['ms'],3), round(r['gflops']), round(r.get('pct_peak',0),3), r.get('update_tflops'), round(r.get('panel_ms') or 0,2))
"
