set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'hist_kernel|apply_kernel|build_kernel|gemm_kernel|sgemm' -o gpurun_out/prof_r1b python tools/prof_target.py --mm 8192 > gpurun_out/ncu_r1b.log 2>&1
timeout 300 python tools/lut_micro.py --rows 4096 --cols 4096 > gpurun_out/lut_micro_c1.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --workload lut > /dev/null 2>&1
