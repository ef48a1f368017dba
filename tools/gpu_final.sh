#!/bin/bash
# the driver's round-end sequence: GPU tests, smoke, reference arm, default bench
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final/smi.txt 2>&1
t0=$(date +%s)
timeout 1800 python bench.py --impl reference > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err; echo "ref rc=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/final/times.txt
t0=$(date +%s)
timeout 1800 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/final/times.txt
cat gpurun_out/final/times.txt
if [ -n "$WITH_C5" ]; then
  t0=$(date +%s)
  timeout 1800 python bench.py --workload c5 --no-cpu-baseline --no-converge --steps 5 > gpurun_out/final/bench_c5.json 2> gpurun_out/final/bench_c5.err; echo "c5 rc=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/final/times.txt
fi
