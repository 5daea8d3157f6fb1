#!/bin/bash
# Development aid: A/B of environment settings of the same library (two interleaved rounds).
# usage: scripts/env_ab.sh OUTDIR "NAME=VAR=VAL ..." C4 [C3 ...]   e.g. "l0:RT_BVH_LAYOUT=0 l1:RT_BVH_LAYOUT=1"
OUT=$1; shift
VARS=$1; shift
CFGS=${@:-C4}
mkdir -p $OUT
for round in 1 2; do
  for v in $VARS; do
    n=${v%%:*}; kv=${v#*:}
    for c in $CFGS; do
      env $kv timeout 300 python scripts/quick_perf.py $c 2>&1 | grep -E "median|inflight" | sed "s/^/$n r$round /" >> $OUT/env_ab.log
    done
  done
done
cat $OUT/env_ab.log
