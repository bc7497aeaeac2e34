#!/bin/bash
# Round-2 profile of one config on the GPU box: the bench line, the ncu launch
# list, and one `--set full` capture per hot kernel (selected by mangled
# name, one launch each), each only after the same command exited 0 without
# ncu.  Full captures are exported to CSV on the box (raw + SASS source) and
# the .ncu-rep files dropped, to stay under gpurun's 64 MiB return limit.
#   bash tools/gpu_profile2.sh TAG CFG [CPU_ITERS]
set -u
TAG=${1:-r02}
CFG=${2:-c2}
CPUI=${3:-40}
mkdir -p gpurun_out
STEPS=10; [ $CFG = c3 ] && STEPS=5; [ $CFG = c5 ] && STEPS=3
timeout 1500 python bench.py --config $CFG --steps $STEPS --warmup 3 --cpu-iters $CPUI > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err
echo "bench rc=$?"
CMD="python bench.py --config $CFG --warmup 1 --no-cpu-baseline --profile-only --profile-reps 1"
timeout 900 $CMD > gpurun_out/plain_${TAG}_${CFG}.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_bjac|k_spmv|k_update|k_pupdate|k_big" --csv \
    --log-file gpurun_out/launches_${TAG}_${CFG}.csv $CMD > gpurun_out/ncu_launch_${TAG}_${CFG}.log 2>&1
echo "ncu launch rc=$?"
for pair in "last:k_bjac_diaI[fd]Lb1E|k_bjac_tileI[fd]Lb0ELb1E" "spmv:k_spmv_dia|k_spmv_pq" "update_first:k_update_first"; do
  nm=${pair%%:*}; rx=${pair#*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$rx" -c 1 \
      -o /tmp/prof_${TAG}_${CFG}_$nm $CMD > gpurun_out/ncu_full_${TAG}_${CFG}_$nm.log 2>&1
  echo "ncu full $nm rc=$?"
  ncu -i /tmp/prof_${TAG}_${CFG}_$nm.ncu-rep --page raw --csv > gpurun_out/full_${TAG}_${CFG}_$nm.csv 2>/dev/null
  ncu -i /tmp/prof_${TAG}_${CFG}_$nm.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}_${CFG}_$nm.csv 2>/dev/null
  rm -f /tmp/prof_${TAG}_${CFG}_$nm.ncu-rep
done
