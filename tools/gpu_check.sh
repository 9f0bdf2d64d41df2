timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 200 gpurun_out/bench_full.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print(json.dumps({k:d.get(k) for k in ('value','ms_per_step','gpu_launches')}), json.dumps(d['e2e'])[:300], d['roofline']['frac'])
m=d['matmul']; print('C4', m['value'], m['roofline']['frac'], m['clocks']); c2=m['c2_f32']; print('C2', c2['value'], c2['clocks'], c2['e2e']['value'], c2['cpu_baseline']['value'])
print('C5', d['c5']['chains_per_s'], d['c5']['cpu_baseline']['chains_per_s'])
P
