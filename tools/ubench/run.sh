#!/bin/bash
# Run the FP64 micro-benchmarks with nvidia-smi clock sampling; outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/ubench_clocks.csv &
SMI=$!
./tools/ubench/fp64_ubench > gpurun_out/ubench.json
RC=$?
kill $SMI
nproc > gpurun_out/host_cores.txt
lscpu | head -20 >> gpurun_out/host_cores.txt
nvidia-smi -q | head -60 > gpurun_out/nvsmi.txt
cat gpurun_out/ubench.json
exit $RC
