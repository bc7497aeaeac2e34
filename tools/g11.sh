set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dist_local.py -x -q -s > gpurun_out/g11_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g11_parity.log 2>&1; echo "parity rc=$?"
