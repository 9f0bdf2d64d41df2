timeout 900 python bench.py --workload lut --steps 20 --warmup 5 > gpurun_out/bench_lut.json 2> gpurun_out/bench_lut.err; tail -c 400 gpurun_out/bench_lut.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_lut.json').read().strip().splitlines()[-1]);print(json.dumps({k:d.get(k) for k in ('value','ms_per_step','roofline','e2e','gpu_launches','clocks')})[:1500])"
