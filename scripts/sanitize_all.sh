# compute-sanitizer over the single-process workload (every kernel) and the two-rank library
# world; usage: bash scripts/sanitize_all.sh <tag>
TAG=${1:-r02}
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/san/${TAG}_$t.log 2>&1; echo "rc=$?" >> gpurun_out/san/${TAG}_$t.log
done
RT_SHARD_BLOCK=2 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/san/${TAG}_memcheck_block2.log 2>&1; echo "rc=$?" >> gpurun_out/san/${TAG}_memcheck_block2.log
for t in memcheck racecheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --target-processes all --error-exitcode 9 python scripts/sanitize_dist.py > gpurun_out/san/${TAG}_dist_$t.log 2>&1; echo "rc=$?" >> gpurun_out/san/${TAG}_dist_$t.log
done
for f in gpurun_out/san/${TAG}_*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|rc=' $f | tr '\n' ' ')"; done
