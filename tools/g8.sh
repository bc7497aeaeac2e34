set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g8_pytest.log 2>&1; echo "pytest rc=$?"
for v in "MPB_X=0" "MPB_STATIC=1" "MPB_NO_WIN=1" "MPB_NO_WIN=1 MPB_STATIC=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g8_bench_$tag.json 2> gpurun_out/g8_bench_$tag.err
  echo "$v rc=$?"
done
