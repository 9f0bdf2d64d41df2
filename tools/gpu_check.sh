cat > /tmp/one_mm.py <<'P'
import sys, torch
sys.path.insert(0, ".")
from paper_1505_05655_b200 import device as D
for s in (8192, 32768):
    A = D.synth_matrix(1, 1, s, s); B = D.synth_matrix(1, 2, s, s); Cm = torch.empty(s, s, device="cuda")
    ws = D.matmul_workspace(2, s, s, s)
    D.matmul(2, A, B, Cm, ws); torch.cuda.synchronize()
    del A, B, Cm, ws; torch.cuda.empty_cache()
P
timeout 600 python -m pytest tests/test_matmul_gpu.py tests/test_executor.py -x -q -m gpu > gpurun_out/t_mm.log 2>&1; tail -3 gpurun_out/t_mm.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'prep|gemm' --csv python /tmp/one_mm.py 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>10: print(r[4][:40], r[-3], r[-2], r[-1])
"
for rep in 1 2; do timeout 300 python tools/c4_ab.py 2sm 2>/dev/null | cut -c1-200; done
