#!/bin/bash
# A/B of libnc.so builds on ONE box with tools/attn_time.py (isolated attention kernel):
#   bash tools/ab_attn.sh "ab/libnc_x.so ab/libnc_y.so ..." [rounds] [rows]
LIBS=($1); R=${2:-2}; N=${3:-16384}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in $(seq $R); do
  for i in "${!LIBS[@]}"; do
    cp ${LIBS[$i]} paper_2602_19626_b200/libnc.so
    echo "$(basename ${LIBS[$i]}) round $r: $(NC_ATTN_REPS=10 timeout 300 python tools/attn_time.py $N 2>/dev/null | tail -1)"
  done
done
