#!/bin/bash
# Round-2 session-3 re-entry check: GPU suite + smoke + default bench on the restored tree.
mkdir -p gpurun_out/v3; O=gpurun_out/v3
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in lu_f64_n4096_s64 qr_f64_n8192_s128; do
  timeout 900 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
for f in $O/bench_*.json; do echo "== $f"; cut -c1-300 $f; done
