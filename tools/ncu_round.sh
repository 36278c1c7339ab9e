#!/bin/bash
# ncu evidence for one round (run on the GPU box, one GPU): launch list of two compress
# steps of the bench workload, then one --set full capture per hot kernel class (a launch
# from the second step).  Outputs land in gpurun_out/; tools/ncu_summary.py condenses them
# into profiles/.   usage: bash tools/ncu_round.sh <tag>
set -x
TAG=${1:-r01h}
O=gpurun_out
NCU=ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
  python tools/profile_step.py config2 2 > $O/ncu_launch.log 2>&1
cap() {   # name regex skip
  $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c 1 -f -o $O/${TAG}_$1 \
    python tools/profile_step.py config2 2 > $O/ncu_$1.log 2>&1
}
# launches per step: 30 per layer-kernel class (x 2 slabs = 60); skip the first step's
cap attention 'attn_tc_kernel' 75
cap qkv 'gemm_tc_kernel<.int.0' 75
cap oproj 'gemm_tc_kernel<.int.1' 150
cap down 'gemm_tc_kernel<.int.1' 151
cap gateup 'gemm_tc_kernel<.int.2' 75
cap head 'gemm_tc_kernel<.int.3' 2
cap walk 'walk_cl_kernel' 2
cap ngram 'ngram_pre_kernel' 2
