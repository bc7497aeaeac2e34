set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_plugin.py -x -q > gpurun_out/g12_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/prof_nb32.py > gpurun_out/g12_nb32.log 2>&1; echo "rc=$?"
