mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "qr or QR or graph or concurrent" > gpurun_out/mgsncu_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/mgsncu_pytest.log
python tools/prof_qr_lu.py && ncu --set full --import-source on --clock-control none -k regex:qr_mgs -s 1 -c 1 -o gpurun_out/pp_mgs -f python tools/prof_qr_lu.py > gpurun_out/pp_mgs.log 2>&1; tail -2 gpurun_out/pp_mgs.log
export SF_BENCH_ALLOW_SHORT=1
w=qr_f64_n8192_s128
CMD="python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/pp_$w.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pp_launches_$w.csv $CMD > /dev/null 2>&1; grep -c mgs gpurun_out/pp_launches_$w.csv
