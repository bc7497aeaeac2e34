#!/bin/bash
# Run on the GPU box (gpurun): bench line, then the ncu launch list and one
# --set full capture of the top kernels, each only after the same command
# exited 0 without ncu (/opt/skills/guides/B200_PROFILING.md).  ncu does not
# see the kernel nodes of the solve's CUDA graph (device while loop), so the
# ncu runs profile bench.py --profile-only: one solve, then every kernel of an
# iteration launched on its own (solver.profile_iteration) -- the same kernels
# the graph runs, on the same buffers.
set -u
TAG=${1:-r01}
CFG=${2:-c2}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --warmup 1 --no-cpu-baseline --profile-only --profile-reps 3"
python bench.py --config $CFG --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err
echo "bench rc=$?"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_bjac|k_spmv|k_update|k_pupdate" --csv \
    --log-file gpurun_out/launches_${TAG}_${CFG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "ncu launch rc=$?"
$CMD > gpurun_out/plain2_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_spmv_pq|k_bjac_tile|k_update|k_pupdate" \
    -s 1 -c 16 -o gpurun_out/prof_${TAG}_${CFG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
