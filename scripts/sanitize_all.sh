mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/san/r01s3_$t.log 2>&1; echo "rc=$?" >> gpurun_out/san/r01s3_$t.log
done
timeout 1200 python -m pytest tests/test_gpu_bench_multirank.py -x -q -p no:cacheprovider > gpurun_out/san/multirank.log 2>&1; tail -3 gpurun_out/san/multirank.log
for t in memcheck racecheck synccheck initcheck; do tail -2 gpurun_out/san/r01s3_$t.log; done
