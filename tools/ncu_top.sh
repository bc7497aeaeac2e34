#!/bin/bash
# ncu --set full of the hot kernels of one short bench run (GPU box)
TAG=${1:-r01x}
CFG=${2:-c2}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 2"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_spmv_pq|k_bjac_tile|k_update|k_pupdate" \
    -s 40 -c 5 -o gpurun_out/prof_${TAG}_${CFG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
