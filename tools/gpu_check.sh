timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; tail -c 200 gpurun_out/b_c5.err
python -c "
import json;d=json.loads(open('gpurun_out/b_c5.json').read().strip().splitlines()[-1]);print(json.dumps(d.get('c1'))[:300]); print(d['c5']['chains_per_s'])"
