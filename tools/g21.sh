set -u
bash tools/gpu_profile2.sh r02c c2 40
bash tools/gpu_profile2.sh r02c c4 3
bash tools/gpu_profile2.sh r02c c3 2
bash tools/gpu_profile2.sh r02c c5 1
python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/bench_r02c_c1.json 2>/dev/null
python bench.py --config const128_nb32 --steps 10 --warmup 3 --cpu-iters 10 > gpurun_out/bench_r02c_nb32.json 2>/dev/null
rm -f gpurun_out/sass_r02c_c[345]_*.csv
du -sh gpurun_out
