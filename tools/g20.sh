set -u
bash tools/gpu_profile2.sh r02 c2 40
bash tools/gpu_profile2.sh r02 c4 3
bash tools/gpu_profile2.sh r02 c3 2
du -sh gpurun_out
