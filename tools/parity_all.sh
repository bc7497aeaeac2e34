#!/bin/bash
# Full-size bitwise parity of every BASELINE config (tools/fullsize_parity.py)
# on the GPU box: gpurun_out/parity_<tag>.jsonl.  C5 capped at 12 iterations
# (its CPU replay takes hours); C3's whole replay takes ~12 min on 16 cores.
TAG=${1:-r01}
mkdir -p gpurun_out
: > gpurun_out/parity_${TAG}.jsonl
for spec in "c1 uniform" "c1 fixed-low" "c2 fixed-low" "c4 fixed-low" "c4 adaptive-hl:10" "c5 fixed-low --max-iter 12" "c3 adaptive-lh:1e-6"; do
  set -- $spec
  cfg=$1; pol=$2; shift 2
  timeout 1500 python tools/fullsize_parity.py $cfg --policy $pol "$@" >> gpurun_out/parity_${TAG}.jsonl 2>> gpurun_out/parity_${TAG}.err
  echo "$cfg $pol rc=$?"
done
