set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g9_pytest.log 2>&1; echo "pytest rc=$?"
for v in "MPB_NO_WIN=1" "MPB_X=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g9_bench_$tag.json 2> gpurun_out/g9_bench_$tag.err
  echo "$v rc=$?"
done
CMD="python bench.py --config c2 --warmup 1 --no-cpu-baseline --profile-only --profile-reps 1"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_bjac_tileIfLb0ELb1E" -c 1 -o /tmp/g9_last $CMD > gpurun_out/g9_last_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/g9_last.ncu-rep --page raw --csv > gpurun_out/g9_last_raw.csv 2>/dev/null
ncu -i /tmp/g9_last.ncu-rep --page source --csv --print-source sass > gpurun_out/g9_last_sass.csv 2>/dev/null
