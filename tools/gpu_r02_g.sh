set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02g_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02g_gpu_all.log
timeout 600 python bench.py > gpurun_out/r02g_bench_c2.json 2> gpurun_out/r02g_bench_c2.err; echo "bench rc=$?"; head -c 3000 gpurun_out/r02g_bench_c2.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02g_ref_c2.json 2> gpurun_out/r02g_ref_c2.err; echo "ref rc=$?"; cat gpurun_out/r02g_ref_c2.json
timeout 600 python bench.py --config c5 --steps 5 > gpurun_out/r02g_bench_c5.json 2> gpurun_out/r02g_bench_c5.err; echo "c5 rc=$?"; head -c 1500 gpurun_out/r02g_bench_c5.json
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/r02g_bench_c3.json 2> gpurun_out/r02g_bench_c3.err; echo "c3 rc=$?"; head -c 1500 gpurun_out/r02g_bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
