#!/bin/bash
# Development aid: time every library under paper_1702_01530_b200/lib/variants (and the main one)
# on the given configs, two interleaved rounds.  usage: scripts/variant_perf.sh OUTDIR C4 [C3 ...]
OUT=$1; shift
CFGS=${@:-C4}
mkdir -p $OUT
for round in 1 2; do
  for lib in paper_1702_01530_b200/lib/librt_b200.so paper_1702_01530_b200/lib/variants/*.so; do
    n=$(basename $lib .so)
    for c in $CFGS; do
      RT_LIB_PATH=$PWD/$lib timeout 300 python scripts/quick_perf.py $c 2>&1 | grep -E "median|inflight" | sed "s/^/$n r$round /" >> $OUT/variants.log
    done
  done
done
cat $OUT/variants.log
