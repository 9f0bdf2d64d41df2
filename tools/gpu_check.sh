GPCX_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --workload lut > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; tail -c 400 gpurun_out/bench_n2.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_n2.json').read().strip().splitlines()[-1]);print(json.dumps({k:d.get(k) for k in ('value','ms_per_step','gather','gpu_launches')})[:800])"
