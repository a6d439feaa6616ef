set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_golden_fullsize.py -v -x > gpurun_out/r02_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -30 gpurun_out/r02_fullsize.log
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_golden_fullsize.py > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02_bench_base.json 2> gpurun_out/r02_bench_base.err; echo "bench rc=$?"; head -c 1500 gpurun_out/r02_bench_base.json
