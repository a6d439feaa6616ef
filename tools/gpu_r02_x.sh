for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_r02.py > gpurun_out/r02_sanitize_$t.log 2>&1; echo "$t rc=$?"
  tail -3 gpurun_out/r02_sanitize_$t.log
done
