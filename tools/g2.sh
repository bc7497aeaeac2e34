set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?"
