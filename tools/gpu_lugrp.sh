timeout 900 python -m pytest tests -m gpu -x -q -k "lu or LU or solve or host" 2>&1 | tail -1
for g in 1 0; do for m in 4096 0; do SF_LU_PART1_GROUPED=$g SF_LU_LA_MIN_M=$m python tools/la_lu.py 2>&1 | sed "s/^/GRP=$g MIN=$m /"; done; done
