#!/bin/bash
# one ncu --set full capture (with source) of a kernel of the bench workload's second step
# usage: bash tools/ncu_one.sh <name> <kernel regex> <skip> [tag]
TAG=${4:-r01f}
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c 1 -f \
  -o gpurun_out/${TAG}_$1 python tools/profile_step.py config2 2 > gpurun_out/ncu_$1.log 2>&1
