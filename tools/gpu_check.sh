timeout 900 python -m pytest tests/test_matmul_gpu.py -x -q -m gpu -k "c4_full" --durations=3 > gpurun_out/t_c4.log 2>&1; tail -6 gpurun_out/t_c4.log
