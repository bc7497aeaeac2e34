set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/g15_pytest.log 2>&1; echo "pytest rc=$?"
