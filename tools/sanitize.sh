#!/bin/bash
# compute-sanitizer over tools/sanitize_solve.py (run on the GPU box):
# memcheck, synccheck, initcheck and racecheck; one log each under
# gpurun_out/, summarised into profiles/ by hand.
set -u
mkdir -p gpurun_out
CS=${CS:-compute-sanitizer}
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_solve.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
done
