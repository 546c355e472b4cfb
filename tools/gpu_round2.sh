#!/bin/bash
# GPU session: loopback bench test, default bench (cfg5 fp64) + reference arm, fp32 cfg5 bench,
# ncu --set full of a cfg5-sized fp64 flush (traffic for profiles/traffic.json).
mkdir -p gpurun_out
export SF_BENCH_ALLOW_SHORT=1
python bench.py --workload chol_f64_n16384_s512 --loopback 4 --steps 2 --warmup 1 --no-cpu > gpurun_out/loop4.json 2> gpurun_out/loop4.err
unset SF_BENCH_ALLOW_SHORT
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_cfg5.json 2> gpurun_out/ref_cfg5.err
python bench.py --workload chol_f32_n65536_s512 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_cfg5_f32.json 2> gpurun_out/bench_cfg5_f32.err
python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python tools/prof_kernels.py 32768 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -c 1 -o gpurun_out/prof_syrk32k -f python tools/prof_kernels.py 32768 > gpurun_out/ncu_syrk32k.log 2>&1
for f in loop4 bench_cfg5 ref_cfg5 bench_cfg5_f32 bench_cfg3; do echo "== $f"; cut -c1-400 gpurun_out/$f.json; tail -2 gpurun_out/$f.err; done
tail -2 gpurun_out/ncu_syrk32k.log
