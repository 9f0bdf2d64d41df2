timeout 600 python -m pytest tests/test_matmul_gpu.py -q -x 2>&1 | tail -2 > gpurun_out/pytest_mm.txt
bash tools/c4_sweep.sh > gpurun_out/c4_sweep.txt 2>&1
GPCX_TC_KERNEL=2sm timeout 300 python tools/mm_micro.py --sizes 4096,8192,16384 --precs bf16,tf32 > gpurun_out/mm_micro_2sm.txt 2>&1
