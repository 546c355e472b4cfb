#!/bin/bash
# Round-2 session 4: cfg3 s-sweep again with the interior-tile slice loader (tools/measure_all.py sweep).
mkdir -p gpurun_out/v
python tools/measure_all.py sweep > gpurun_out/v/r02_measure_sweep.json 2> gpurun_out/v/r02_measure_sweep.err
tail -3 gpurun_out/v/r02_measure_sweep.err; cut -c1-1500 gpurun_out/v/r02_measure_sweep.json
