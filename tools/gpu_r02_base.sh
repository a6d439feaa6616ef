set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_c1.py > gpurun_out/r02_sanitize_$t.log 2>&1; echo "$t rc=$?"
  tail -3 gpurun_out/r02_sanitize_$t.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_base.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_gpu_tests_base.log
timeout 600 python bench.py > gpurun_out/r02_bench_base.json 2> gpurun_out/r02_bench_base.err; echo "bench rc=$?"; cat gpurun_out/r02_bench_base.json | head -c 600
