set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g17_pytest.log 2>&1; echo "pytest rc=$?"
for v in "MPB_X=0" "MPB_NO_SYM=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v MPB_VERBOSE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g17_bench_$tag.json 2> gpurun_out/g17_bench_$tag.err
  echo "$v rc=$?"
done
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g17_bench_c4.json 2> gpurun_out/g17_bench_c4.err; echo "c4 rc=$?"
