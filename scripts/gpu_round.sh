#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full capture of the trace kernel.
# usage: scripts/gpu_round.sh <tag> [steps...]   steps: test smoke bench ncu full
TAG=${1:-r}; shift
STEPS=${@:-"smoke test bench ncu full"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/gpu.txt 2>&1
for s in $STEPS; do
  case $s in
    smoke) timeout 600 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log ;;
    test) timeout 1500 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > $OUT/gputest.log 2>&1; echo "rc=$?" >> $OUT/gputest.log ;;
    fast) timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -s -p no:cacheprovider > $OUT/gputest.log 2>&1; echo "rc=$?" >> $OUT/gputest.log ;;
    bench) timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err ;;
    perf) timeout 600 python scripts/quick_perf.py C4 > $OUT/perf_c4.log 2>&1; timeout 300 python scripts/quick_perf.py C3 > $OUT/perf_c3.log 2>&1 ;;
    allcfg) timeout 900 python scripts/all_configs.py > $OUT/all_configs.txt 2>&1; timeout 600 python scripts/split_perf.py > $OUT/split.log 2>&1 ;;
    c5) timeout 900 python bench.py --config C5 --steps 60 --no-cpu-baseline > $OUT/c5.json 2> $OUT/c5.err ;;
    ref) timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/ref.json 2> $OUT/ref.err ;;
    san) bash scripts/sanitize_all.sh > $OUT/san.log 2>&1 ;;
    scale) timeout 900 python scripts/shard_scaling.py C4 C5 > $OUT/shard_scaling.json 2> $OUT/shard_scaling.err ;;
    ncu) timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
           python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1; echo "rc=$?" >> $OUT/ncu_bench.log ;;
    full) timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:k_trace_stereo -s 2 -c 1 \
           -o $OUT/trace_full python scripts/quick_perf.py C4 > $OUT/ncu_full.log 2>&1; echo "rc=$?" >> $OUT/ncu_full.log ;;
  esac
done
ls -la $OUT
