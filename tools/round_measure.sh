#!/bin/bash
# One GPU call's worth of round evidence, sized for gpurun_out/ (<= 64 MiB copied back):
# bench lines (config3 default, the reference arm, config2, config2 with 1 chunk, config4's
# one-GPU share), then the ncu launch list + --set full captures (tools/ncu_round.sh),
# summarised on the box into gpurun_out/prof_<tag>/; only the attention and walk reports are
# kept (the rest would overflow the copy-back limit).
#   usage: bash tools/round_measure.sh <tag> [steps] [warmup]
TAG=${1:-r02b}
K=${2:-5}
W=${3:-3}
O=gpurun_out
python bench.py --steps $K --warmup $W > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_reference.json 2>&1
for w in config2 config2_1chunk config4_shard; do
  python bench.py --workload $w --steps $K --warmup $W --no-cpu-baseline > $O/${TAG}_bench_$w.json 2>&1
done
bash tools/ncu_round.sh $TAG config3 1830 > $O/ncu_round_$TAG.log 2>&1
args=""
for n in attention qkv oproj down gateup head walk ngram; do
  [ -f $O/${TAG}_$n.ncu-rep ] && args="$args $n=$O/${TAG}_$n.ncu-rep"
done
python tools/ncu_summary.py $TAG $O/launches_$TAG.csv $args > $O/ncu_summary_$TAG.log 2>&1
mkdir -p $O/prof_$TAG
cp profiles/${TAG}_* profiles/ncu_traffic.json $O/prof_$TAG/ 2>/dev/null
mkdir -p /tmp/ncu_$TAG
for n in qkv oproj down gateup head ngram; do mv $O/${TAG}_$n.ncu-rep /tmp/ncu_$TAG/ 2>/dev/null; done
gzip -f $O/launches_$TAG.csv
rm -f $O/clocks_*.csv
du -sh $O
