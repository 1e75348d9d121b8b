#!/bin/bash
# Quick iteration: gpu parity tests + bench lines for the main configs (no CPU leg).
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_$TAG.log
for c in mixtral qwen60 deepseek skew64; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
timeout 300 python bench.py --config mixtral --tokens 1 --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_$TAG.json 2>> gpurun_out/bench_$TAG.err
echo done
