#!/bin/bash
# Bench lines of every BASELINE config on one GPU (profiles/<tag>_configs.jsonl)
TAG=${1:-r01}
mkdir -p gpurun_out
: > gpurun_out/configs_${TAG}.jsonl
for c in c1 c2 c3 c4 c5; do
  steps=10; [ $c = c3 ] && steps=5; [ $c = c5 ] && steps=3
  timeout 1200 python bench.py --config $c --steps $steps --warmup 3 >> gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/configs_${TAG}_$c.err
  echo "$c rc=$?"
done
