#!/bin/bash
# End-of-round evidence: gpu tests, smoke, default bench (+ reference arm), fp32 cfg5 and cfg3
# bench lines, launch list of one default step, ncu --set full of the two flush kernels.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1
python __graft_entry__.py --smoke > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
python bench.py --workload chol_f32_n65536_s512 --e2e-steps 2 > gpurun_out/final_bench_f32.json 2> gpurun_out/final_bench_f32.err
python bench.py --workload chol_f64_n16384_s512 > gpurun_out/final_bench_cfg3.json 2> gpurun_out/final_bench_cfg3.err
export SF_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/final_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $CMD > /dev/null 2>&1
python tools/prof_kernels.py 32768 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -c 1 -o gpurun_out/final_f64 -f python tools/prof_kernels.py 32768 > /dev/null 2>&1
python tools/prof_f32.py syrk 32768 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3_pair -s 2 -c 1 -o gpurun_out/final_tf32 -f python tools/prof_f32.py syrk 32768 > /dev/null 2>&1
tail -2 gpurun_out/final_pytest.log; cat gpurun_out/final_smoke.log
for f in final_bench final_ref final_bench_f32 final_bench_cfg3; do echo "== $f"; cut -c1-300 gpurun_out/$f.json; tail -1 gpurun_out/$f.err; done
ls -la gpurun_out/final_*
