timeout 600 python -m pytest tests/test_matmul_gpu.py -x -q -m gpu -k "sgemm or f32 or block_rows" 2>&1 | tail -1
for v in "" ""; do
GPCX_SGEMM=$v python -c "
import sys, json; sys.path.insert(0, '.')
import bench
r = bench.matmul_device_leg(10, 3); print('$v', json.dumps({'c2_ms': round(r['ms'], 3), 'tflops': round(r['tflops'], 1)}))"
done
