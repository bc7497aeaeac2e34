set -u
mkdir -p gpurun_out
MPB_LIB=$PWD/paper_2407_15973_b200/libmpbjac_uf.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g18_pytest.log 2>&1; echo "pytest rc=$?"
for v in main uf; do
  lib=paper_2407_15973_b200/libmpbjac_$v.so; [ $v = main ] && lib=paper_2407_15973_b200/libmpbjac.so
  MPB_NO_SYM=1 MPB_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g18_bench_$v.json 2> gpurun_out/g18_bench_$v.err
  echo "$v rc=$?"
done
