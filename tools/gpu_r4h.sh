timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
