mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san_$t.log 2>&1
done
