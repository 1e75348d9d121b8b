#!/bin/bash
# Round-2 measurement session (1 GPU): every BASELINE config through bench.py
# (value, e2e, roofline from in-graph events, parity gate, CPU baseline), the
# skew sweep, the fusion ablation, the reference arm, the ncu launch list and
# one `ncu --set full` capture of the FFN per config (DRAM traffic -> traffic.json),
# the fused-vs-unfused DRAM bytes (measured TrafficReport).
TAG=${1:-r02}
mkdir -p gpurun_out
B="timeout 900 python bench.py"
$B --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
$B --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
for c in qwen60 deepseek small; do $B --config $c --steps 20 --warmup 3 >> gpurun_out/bench_configs_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
for t in 1 2 4 8 32 128; do $B --config mixtral --tokens $t --steps 20 --warmup 3 >> gpurun_out/bench_configs_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
for a in 0 0.5 0.8 1.2 1.6 2.0; do $B --config skew64 --zipf $a --steps 20 --warmup 3 >> gpurun_out/bench_skew_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
for c in mixtral qwen60 skew64; do $B --config $c --unfused --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_unfused_$TAG.json 2>> gpurun_out/bench_$TAG.err; done
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_ep2_$TAG.json 2> gpurun_out/bench_ep2_$TAG.err
N="timeout 600 ncu --clock-control none"
$N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_$TAG.csv python scripts/run_layer.py mixtral 512 3 > /dev/null 2>&1
$N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_qwen60_$TAG.csv python scripts/run_layer.py qwen60 512 3 > /dev/null 2>&1
$N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_deepseek_$TAG.csv python scripts/run_layer.py deepseek 512 3 > /dev/null 2>&1
$N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_mixtral1_$TAG.csv python scripts/run_layer.py mixtral 1 3 > /dev/null 2>&1
# the sigmoid router's INT8 screen path (DeepSeek-V3): every kernel of one route, and an A/B line with the exact router
$N --set full --import-source on -k regex:screen -s 6 -c 6 -o /tmp/prof_screen_deepseek_$TAG -f python scripts/run_layer.py deepseek 512 2 > /dev/null 2>&1
ncu -i /tmp/prof_screen_deepseek_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_screen_deepseek_${TAG}_raw.csv 2>/dev/null
MOE_B200_SCREEN=0 $B --config deepseek --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_exact_router_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 300 python scripts/screen_debug.py deepseek 512 > gpurun_out/screen_debug_$TAG.log 2>&1
# ncu --set full captures go to /tmp (each ~8 MB; gpurun brings back <= 64 MiB):
# their raw metric pages come back as csv, and the Mixtral FFN report itself
for c in mixtral qwen60 deepseek skew64; do
  $N --set full --import-source on -k regex:ffn_kernel -s 1 -c 1 -o /tmp/prof_ffn_${c}_$TAG -f python scripts/run_layer.py $c 512 2 > /dev/null 2>&1
  ncu -i /tmp/prof_ffn_${c}_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_ffn_${c}_${TAG}_raw.csv 2>/dev/null
done
cp /tmp/prof_ffn_mixtral_$TAG.ncu-rep gpurun_out/ 2>/dev/null
for k in router_seg dispatch combine_flag; do
  $N --set full --import-source on -k regex:$k -s 1 -c 1 -o /tmp/prof_${k}_$TAG -f python scripts/run_layer.py mixtral 512 2 > /dev/null 2>&1
  ncu -i /tmp/prof_${k}_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${k}_${TAG}_raw.csv 2>/dev/null
done
# fusion ablation: DRAM bytes of every launch of one fused and one unfused forward
for v in fused unfused; do
  $N --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/ablation_${v}_$TAG.csv python scripts/run_layer.py mixtral 512 2 $v > /dev/null 2>&1
done

# per-tile FFN timelines and the segment router's per-CTA phase timeline
for c in mixtral qwen60 deepseek; do timeout 300 python scripts/ffn_timeline.py $c ${c}_$TAG > /dev/null 2>&1; done
for c in mixtral qwen60; do timeout 300 python scripts/router_seg_timeline.py $c >> gpurun_out/router_timeline_$TAG.log 2>&1; done
echo done
