# GPU test suite (used from gpurun; outputs under gpurun_out/)
python -m pytest tests -m gpu -x -q ${@} 2>&1 | tail -15 > gpurun_out/r02_pytest_gpu.log
