timeout 900 python -m pytest tests/test_matmul_gpu.py -x -q -m gpu > gpurun_out/t_mm.log 2>&1; tail -3 gpurun_out/t_mm.log
for rep in 1 2; do
  C4N=16384 timeout 300 python tools/c4_ab.py 2sm 2sm512 2>/dev/null | sed "s/^/16k /"
  timeout 300 python tools/c4_ab.py 2sm 2sm512 2>/dev/null | sed "s/^/32k /"
done
