timeout 1200 python -m pytest tests/test_demosaic.py tests/test_integration.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python tools/demosaic_micro.py > gpurun_out/demosaic_micro.json 2>&1
