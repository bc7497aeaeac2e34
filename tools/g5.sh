set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g5_pytest_wt.log 2>&1; echo "pytest wt rc=$?"
MPB_FLAT=1 MPB_WT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g5_pytest_flat.log 2>&1; echo "pytest flat rc=$?"
for v in "MPB_WT=0" "MPB_FLAT=1 MPB_WT=0" "MPB_WT=1" "MPB_WT_DEPTH=3" "MPB_WT=0 MPB_STAGES=4"; do
  tag=$(echo $v | tr ' =' '__')
  env $v MPB_VERBOSE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g5_bench_$tag.json 2> gpurun_out/g5_bench_$tag.err
  echo "$v rc=$?"
done
CMD="python bench.py --config c2 --warmup 1 --no-cpu-baseline --profile-only --profile-reps 1"
MPB_FLAT=1 MPB_WT=0 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_bjac_flat" -c 2 -o /tmp/g5_flat $CMD > gpurun_out/g5_flat_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/g5_flat.ncu-rep --page raw --csv > gpurun_out/g5_flat_raw.csv 2>/dev/null
ncu -i /tmp/g5_flat.ncu-rep --page source --csv --print-source sass > gpurun_out/g5_flat_sass.csv 2>/dev/null
