set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g10_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g10_bench_c2.json 2> gpurun_out/g10_bench_c2.err; echo "c2 rc=$?"
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g10_bench_c4.json 2> gpurun_out/g10_bench_c4.err; echo "c4 rc=$?"
CMD="python bench.py --config c2 --warmup 1 --no-cpu-baseline --profile-only --profile-reps 1"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_update_firstIfLb0E" -c 1 -o /tmp/g10_upd $CMD > gpurun_out/g10_upd_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/g10_upd.ncu-rep --page source --csv --print-source sass > gpurun_out/g10_upd_sass.csv 2>/dev/null
