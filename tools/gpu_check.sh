set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "matmul" > gpurun_out/t_mm.log 2>&1; tail -5 gpurun_out/t_mm.log
