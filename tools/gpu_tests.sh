#!/bin/bash
# GPU parity suite (optionally a subset: $1 = pytest -k expression) + smoke.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
K=()
if [ -n "$1" ]; then K=(-k "$1"); fi
timeout 1500 python -m pytest tests -m gpu -q "${K[@]}" --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -5 gpurun_out/pytest_gpu.log
