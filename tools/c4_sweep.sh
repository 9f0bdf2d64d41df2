# C4 (32768^3 bf16) sustained timing, interleaved A/B: 1sm vs 2sm at stages 3/4/5
for rep in 1 2; do
  for cfg in "1sm 4" "2sm 4" "2sm 3" "2sm 5"; do
    set -- $cfg
    GPCX_TC_STAGES2=$2 timeout 300 python tools/c4_ab.py $1 2>/dev/null | sed "s/^/stages=$2 /"
  done
done
