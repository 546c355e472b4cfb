#!/bin/bash
# K1s chunked short-K flush: parity + bitwise tests, standalone K=64 timing (chunk on/off,
# chunk lengths), LU cfg2 bench with it on/off (alternating).
mkdir -p gpurun_out/s; O=gpurun_out/s
timeout 900 python -m pytest tests/test_chunk_flush_gpu.py -q -x > $O/test_chunk.log 2>&1; echo "rc=$?" >> $O/test_chunk.log
tail -3 $O/test_chunk.log
for c in 0 1; do SF_DMMA_CHUNK=$c timeout 120 python tools/bench_chunk.py; done > $O/bench_chunk.txt 2>&1
for T in 1 2 4 8; do SF_DMMA_CHUNK=1 SF_DMMA_CHUNK_MIN=1 SF_DMMA_CHUNK_T=$T timeout 120 python tools/bench_chunk.py; done >> $O/bench_chunk.txt 2>&1
cat $O/bench_chunk.txt
for r in 1 2; do
  for c in 0 1; do
    SF_DMMA_CHUNK=$c timeout 300 python bench.py --workload lu_f64_n4096_s64 --no-cpu --no-e2e > $O/lu_c$c.$r.json 2>/dev/null
    echo "chunk=$c run $r: $(python -c "import json;d=json.load(open('$O/lu_c$c.$r.json'));print(d['ms_per_step'], d['roofline']['frac'])")"
  done
done
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "lu" > $O/test_lu.log 2>&1; echo "rc=$?" >> $O/test_lu.log
tail -3 $O/test_lu.log
