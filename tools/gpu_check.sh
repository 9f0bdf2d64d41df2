timeout 900 python -m pytest tests/test_lsq.py tests/test_integration.py -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt
