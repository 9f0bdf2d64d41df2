timeout 900 python -m pytest tests/test_matmul_gpu.py tests/test_executor.py tests/test_server.py -x -q -m gpu 2>&1 | tail -2
