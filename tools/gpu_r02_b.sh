nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gpu_all.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/r02_gpu_all.log | tail -20
timeout 600 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench rc=$?"; tail -3 gpurun_out/r02_bench_c2.err
timeout 600 python bench.py --config c5 --steps 5 > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo "c5 rc=$?"; tail -3 gpurun_out/r02_bench_c5.err
timeout 900 python bench.py --config c3 --steps 5 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo "c3 rc=$?"; tail -3 gpurun_out/r02_bench_c3.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config c4 --steps 3 --no-cpu-baseline > gpurun_out/r02_bench_c4_2rank.json 2> gpurun_out/r02_bench_c4_2rank.err; echo "c4x2 rc=$?"; tail -3 gpurun_out/r02_bench_c4_2rank.err
