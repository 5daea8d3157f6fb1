#!/bin/bash
# Development aid: time configs under different runtime knobs.  usage: env_sweep.sh OUT "VAR=a VAR=b ..." C4 [C3..]
OUT=$1; shift; SETS=$1; shift
CFGS=${@:-C4}
mkdir -p $OUT
for round in 1 2; do
  for kv in $SETS; do
    for c in $CFGS; do
      env $kv timeout 300 python scripts/quick_perf.py $c 2>&1 | grep -E "median" | sed "s/^/$kv r$round /" >> $OUT/env_sweep.log
    done
  done
done
cat $OUT/env_sweep.log
