#!/bin/bash
# A/B of the wave kernel's settings on one config (run on the GPU box).
CFG=${1:-c2}
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  env "$@" MPB_VERBOSE=1 timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ab_${CFG}_${name}.json 2> gpurun_out/ab_${CFG}_${name}.err
  echo "$name rc=$? $(grep -m1 'dependency polls' gpurun_out/ab_${CFG}_${name}.err)"
}
for v in ${VARIANTS:-base relaxed nowave}; do
  case $v in
    base) run base MPB_WAVE_DBG=4 ;;
    nowait) run nowait MPB_WAVE_DBG=1 ;;
    relaxed) run relaxed MPB_WAVE_DBG=6 ;;
    slack*) run $v MPB_WAVE_DBG=4 MPB_WAVE_SLACK=${v#slack} ;;
    nowave) run nowave MPB_NO_WAVE=1 ;;
  esac
done
