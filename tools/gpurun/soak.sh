#!/bin/bash
# Repeats the tests whose kernels wait on one another (persistent MGS grids on two streams,
# graph replays, the device-flag push transport) to look for rare hangs; each pass under its own timeout.
mkdir -p gpurun_out/v; O=gpurun_out/v/soak.log; : > $O
for i in 1 2 3 4 5 6; do
  timeout 600 python -m pytest -q -x tests/test_parity_gpu.py tests/test_dist_gpu.py \
    -k "graph_replay or concurrent_streams or two_streams or push or qr_mgs_cluster_geometries or rank_deficient" >> $O 2>&1
  echo "pass $i rc=$?" >> $O
done
grep "pass\|passed\|failed" $O
