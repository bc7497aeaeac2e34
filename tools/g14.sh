set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "assembly or c4" > gpurun_out/g14_pytest.log 2>&1; echo "pytest rc=$?"
