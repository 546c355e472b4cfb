# ncu --set full of the panel kernels (Cholesky leaf, LU leaf, QR MGS) + launch lists of one
# cfg3 and one cfg4 step (after each program ran clean without ncu)
mkdir -p gpurun_out
python tools/prof_leaf1.py && ncu --set full --import-source on --clock-control none -k regex:chol_leaf_rl -s 2 -c 1 -o gpurun_out/pp_cholleaf -f python tools/prof_leaf1.py > /dev/null 2>&1
python tools/prof_luleaf.py && ncu --set full --import-source on --clock-control none -k regex:lu_leaf_warp -c 1 -o gpurun_out/pp_luleaf -f python tools/prof_luleaf.py > /dev/null 2>&1
python tools/prof_qr_lu.py && ncu --set full --import-source on --clock-control none -k regex:qr_mgs -s 1 -c 1 -o gpurun_out/pp_mgs -f python tools/prof_qr_lu.py > /dev/null 2>&1
export SF_BENCH_ALLOW_SHORT=1
for w in chol_f64_n16384_s512 qr_f64_n8192_s128 lu_f64_n4096_s64; do
  CMD="python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu"
  $CMD > gpurun_out/pp_$w.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pp_launches_$w.csv $CMD > /dev/null 2>&1
done
ls -la gpurun_out/pp_*
