#!/bin/bash
# Round-2 session 4: DMMA tile variants again, now that interior tiles use the cheap slice loader.
mkdir -p gpurun_out/v; O=gpurun_out/v/variants2.log; : > $O
for v in "SF_DMMA=6" "SF_DMMA=0" "SF_DMMA=4" "SF_DMMA=1" "SF_DMMA=2" "SF_DMMA=3" "SF_DMMA=5" "SF_DMMA_SHORTK=0" "SF_DMMA_SHORTK=5" "SF_DMMA_SHORTK=6"; do
  env $v timeout 300 python tools/exp_dmma.py >> $O 2>&1
done
echo "== layout" >> $O
timeout 300 python tools/exp_layout.py >> $O 2>&1
echo "== bench cfg5 default" >> $O
SF_BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>>$O | cut -c1-700 >> $O
cat $O | grep -v "^$" | cut -c1-300
