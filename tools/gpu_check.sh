timeout 1200 python bench.py --steps 10 --warmup 3 --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 600 gpurun_out/bench_c5.err
