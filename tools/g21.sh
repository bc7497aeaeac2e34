set -u
bash tools/gpu_profile2.sh r02d c2 40
bash tools/gpu_profile2.sh r02d c4 3
bash tools/gpu_profile2.sh r02d c3 2
bash tools/gpu_profile2.sh r02d c5 1
python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/bench_r02d_c1.json 2>/dev/null
python bench.py --config const128_nb32 --steps 10 --warmup 3 --cpu-iters 10 > gpurun_out/bench_r02d_nb32.json 2>/dev/null
rm -f gpurun_out/sass_r02d_c[345]_*.csv
du -sh gpurun_out
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r02d_c2_reference.json 2>/dev/null
python tools/c1_loop.py > gpurun_out/c1_loop_r02d.txt 2>&1
