#!/bin/bash
# One GPU session: tests, bench, launch list, ncu full capture of the dominant kernel.
# Usage (under gpurun): bash scripts/gpu_round.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/run_layer.py mixtral 512 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 2 -c 2 -o gpurun_out/prof_gemm_$TAG -f python scripts/run_layer.py mixtral 512 2 > gpurun_out/ncu_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:router_kernel -s 1 -c 1 -o gpurun_out/prof_router_$TAG -f python scripts/run_layer.py mixtral 512 2 >> gpurun_out/ncu_$TAG.log 2>&1
echo done
