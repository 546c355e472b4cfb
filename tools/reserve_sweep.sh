#!/bin/bash
# SM reservation for the lookahead panel: sweep SF_PANEL_SMS / SF_RESERVE_FLOPS on cfg3, cfg2, cfg5.
export SF_BENCH_ALLOW_SHORT=1
for cfg in "chol_f64_n16384_s512 3" "lu_f64_n4096_s64 5" "chol_f64_n65536_s512 2"; do
  set -- $cfg
  for r in "0 0" "16 4e10" "24 4e10" "32 4e10" "24 1e11"; do
    set -- $1 $2 $r
    SF_PANEL_SMS=$3 SF_RESERVE_FLOPS=$4 timeout 300 python bench.py --workload $1 --steps $2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 sms=$3 thr=$4', round(d['ms_per_step'],3), round(d['value']), round(d['roofline']['panel_ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
