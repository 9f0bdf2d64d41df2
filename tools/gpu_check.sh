set -x
timeout 600 python -m pytest tests/test_matmul_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_mm.txt
timeout 300 python tools/mm_micro.py --sizes 4096,8192 > gpurun_out/mm_micro.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python tools/lut_micro.py > gpurun_out/lut_micro.json 2>&1
