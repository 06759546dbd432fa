set -x
timeout 900 python -m pytest tests/test_gpu_next1.py -x -q > gpurun_out/pytest_next1.log 2>&1; echo "next1 rc=$?"
tail -30 gpurun_out/pytest_next1.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"
tail -5 gpurun_out/pytest_gpu.log
