#!/bin/bash
# Round-2 session-4 re-entry check: GPU suite + smoke + default bench on the restored tree.
mkdir -p gpurun_out/v4; O=gpurun_out/v4
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench_default.json 2> $O/bench_default.err
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
for f in $O/bench_*.json; do echo "== $f"; cut -c1-400 $f; done
