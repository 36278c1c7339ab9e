#!/bin/bash
# A/B/... of builds of libnc.so on ONE box (clocks differ between boxes by >10 %):
#   bash tools/ab_bench.sh "ab/libnc_x.so ab/libnc_y.so ..." [rounds] [bench args]
LIBS=($1); R=${2:-2}; shift 2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in $(seq $R); do
  for i in "${!LIBS[@]}"; do
    cp ${LIBS[$i]} paper_2602_19626_b200/libnc.so
    timeout 900 python bench.py "$@" 2>/dev/null | tail -1 > gpurun_out/ab_${i}_$r.json
    echo "$(basename ${LIBS[$i]}) round $r: $(python tools/bench_kernels.py gpurun_out/ab_${i}_$r.json 2>/dev/null)"
  done
done
