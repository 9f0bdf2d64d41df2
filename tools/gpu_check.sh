cat > /tmp/one_mm.py <<'P'
import sys, torch
sys.path.insert(0, ".")
from paper_1505_05655_b200 import device as D
s = 32768
A = D.synth_matrix(1, 1, s, s); B = D.synth_matrix(1, 2, s, s); Cm = torch.empty(s, s, device="cuda")
ws = D.matmul_workspace(2, s, s, s)
D.matmul(2, A, B, Cm, ws); torch.cuda.synchronize()
P
for cfg in "0 0.5" "2 0.5" "2 0.8" "2 1.0"; do
  set -- $cfg
  GPCX_TC_L2HINT=$1 GPCX_TC_AKEEP=$2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:'gemm2' --csv python /tmp/one_mm.py 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
print('hint=$1 keep=$2', [ (r[-3], r[-1]) for r in csv.reader(sys.stdin) if len(r)>10 and r[-3]!='Metric Name'])
"
done
