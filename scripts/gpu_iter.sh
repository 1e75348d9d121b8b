#!/bin/bash
# Iteration session: gpu tests, bench on 3 configs, ncu of router + ffn.
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_$TAG.log
for c in mixtral qwen60 deepseek; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:router_kernel -s 1 -c 1 -o gpurun_out/prof_router_qwen_$TAG -f python scripts/run_layer.py qwen60 512 2 > gpurun_out/ncu_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:router_kernel -s 1 -c 1 -o gpurun_out/prof_router_mixtral_$TAG -f python scripts/run_layer.py mixtral 512 2 >> gpurun_out/ncu_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 1 -c 1 -o gpurun_out/prof_ffn_$TAG -f python scripts/run_layer.py mixtral 512 2 >> gpurun_out/ncu_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/run_layer.py mixtral 512 3 > /dev/null 2>&1
echo done
