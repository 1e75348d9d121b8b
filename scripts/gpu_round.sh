#!/bin/bash
# One measurement session (1 GPU): parity tests, default bench (+ CPU baseline),
# reference arm, other configs, launch lists, ncu --set full of the FFN / router
# / dispatch / combine kernels, FFN tile timelines.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_$TAG.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
for c in qwen60 deepseek skew64 small; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_configs_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
for t in 1 32 128; do timeout 600 python bench.py --config mixtral --tokens $t --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_configs_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/run_layer.py mixtral 512 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qwen60_$TAG.csv python scripts/run_layer.py qwen60 512 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 1 -c 1 -o gpurun_out/prof_ffn_$TAG -f python scripts/run_layer.py mixtral 512 2 > /dev/null 2>&1
for k in router_seg dispatch combine_token; do timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_${k}_$TAG -f python scripts/run_layer.py mixtral 512 2 > /dev/null 2>&1; done
for c in mixtral qwen60 deepseek; do python scripts/ffn_timeline.py $c ${c}_$TAG > /dev/null 2>&1; done
timeout 300 python scripts/stage_times.py qwen60 mixtral > gpurun_out/stage_times_$TAG.log 2>&1
echo done
