timeout 600 python -m pytest tests/test_lut_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python tools/lut_micro.py > gpurun_out/lut_micro.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --workload lut > gpurun_out/bench.json 2> gpurun_out/bench.err
