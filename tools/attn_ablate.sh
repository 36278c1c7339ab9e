#!/bin/bash
# Diagnostics: attention kernel time under each NC_ATT_ABL ablation (results wrong by design).
# usage (GPU box): bash tools/attn_ablate.sh [n] [ablations...]
n=${1:-16384}; shift
for k in ${@:-0 1 2 3 4 5 6}; do
  echo -n "abl=$k "
  NC_NVCC_EXTRA="-DNC_ATT_ABL=$k" NC_ATTN_REPS=5 python tools/attn_time.py $n 2>&1 | tail -1
done
