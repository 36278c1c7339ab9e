#!/bin/bash
# A/B of libnc.so builds on ONE box with tools/step_time.py (device time of the compress step):
#   bash tools/ab_step.sh "ab/libnc_x.so ab/libnc_y.so ..." [rounds] [workload] [steps]
LIBS=($1); R=${2:-2}; WL=${3:-config3}; K=${4:-3}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in $(seq $R); do
  for i in "${!LIBS[@]}"; do
    cp ${LIBS[$i]} paper_2602_19626_b200/libnc.so
    echo "$(basename ${LIBS[$i]}) round $r: $(timeout 900 python tools/step_time.py $WL $K 2>/dev/null | tail -1)"
  done
done
