#!/bin/bash
# ncu evidence for one round (run on the GPU box, one GPU): the launch list of two compress
# steps of a workload (the bench's: config3), then one --set full capture per hot kernel
# class, a launch from the middle of the second step.  Outputs land in gpurun_out/;
# tools/ncu_summary.py condenses them into profiles/.
#   usage: bash tools/ncu_round.sh <tag> [workload] [per-class launches per step] [only]
# config3 (64 chunks x 512-position slabs): 61 slabs per step -> 61 x 30 = 1830 launches
# per layer-kernel class, 61 head / walk / N-gram launches.
set -x
TAG=${1:-r02}
WL=${2:-config3}
PL=${3:-1830}
NS=$((PL / 30))
O=gpurun_out
NCU=ncu
if [ -z "$4" ]; then
  $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
    python tools/profile_step.py $WL 2 > $O/ncu_launch.log 2>&1
fi
cap() {   # name regex skip
  $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c 1 -f -o $O/${TAG}_$1 \
    python tools/profile_step.py $WL 2 > $O/ncu_$1.log 2>&1
}
cap attention 'attn_tc_kernel' $((PL + PL / 2))
cap qkv 'gemm_tc_kernel<.int.0' $((PL + PL / 2))
cap oproj 'gemm_tc_kernel<.int.1' $((2 * PL + PL))
cap down 'gemm_tc_kernel<.int.1' $((2 * PL + PL + 1))
cap gateup 'gemm_tc_kernel<.int.2' $((PL + PL / 2))
cap head 'gemm_tc_kernel<.int.3' $((NS + NS / 2))
cap walk 'walk_cl_kernel' $((NS + NS / 2))
cap ngram 'ngram_pre_kernel' $((NS + NS / 2))
