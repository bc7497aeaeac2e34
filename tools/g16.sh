set -u
mkdir -p gpurun_out
for v in v0 v1 v2 v3; do
  lib=paper_2407_15973_b200/libmpbjac_$v.so; [ $v = v0 ] && lib=paper_2407_15973_b200/libmpbjac.so
  MPB_LIB=$PWD/$lib MPB_VERBOSE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g16_bench_$v.json 2> gpurun_out/g16_bench_$v.err
  echo "$v rc=$?"
done
