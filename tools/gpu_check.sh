set -x
timeout 600 ncu --set full --clock-control none -k regex:'gemm' -o gpurun_out/prof_longk2 python tools/prof_target.py --what longk > gpurun_out/ncu_longk.log 2>&1
timeout 300 python tools/c4_ab.py 2sm 1sm 2sm 1sm > gpurun_out/c4_ab.txt 2>&1
