#!/bin/bash
# default bench line (+ optional extra args) and the converge tests
mkdir -p gpurun_out
timeout 1200 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python -m pytest tests -m gpu -q -k "converged or retry" > gpurun_out/pytest_conv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_conv.log
tail -3 gpurun_out/bench.err; tail -3 gpurun_out/pytest_conv.log
