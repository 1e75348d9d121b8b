#!/bin/bash
# Iteration: gpu tests, launch lists (mixtral/qwen60 512), bench lines of the main configs.
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/t_$TAG.log
for c in mixtral qwen60; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_$TAG.csv python scripts/run_layer.py $c 512 3 > /dev/null 2>&1; done
for c in mixtral qwen60 deepseek skew64; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu; done > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
timeout 300 python bench.py --config mixtral --tokens 1 --steps 20 --warmup 3 --no-cpu >> gpurun_out/b_$TAG.json 2>> gpurun_out/b_$TAG.err
