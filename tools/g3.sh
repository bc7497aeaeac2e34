set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g3_pytest.log 2>&1; echo "pytest rc=$?"
for v in "MPB_WT=0" "MPB_WT=1" "MPB_WT_DEPTH=1" "MPB_WT_DEPTH=3" "MPB_WT_DEPTH=4"; do
  env $v MPB_VERBOSE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g3_bench_$v.json 2> gpurun_out/g3_bench_$v.err
  echo "$v rc=$?"
done
