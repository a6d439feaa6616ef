set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/rf_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rf_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/rf_bench_c2.json 2> gpurun_out/rf_bench_c2.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rf_ref_c2.json 2> gpurun_out/rf_ref_c2.err; echo "ref rc=$?"
timeout 600 python bench.py --config c2noise --steps 5 --no-cpu-baseline > gpurun_out/rf_bench_c2noise.json 2> gpurun_out/rf_bench_c2noise.err; echo "c2noise rc=$?"
timeout 900 python bench.py --config c5 --steps 5 > gpurun_out/rf_bench_c5.json 2> gpurun_out/rf_bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/rf_bench_c3.json 2> gpurun_out/rf_bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config c4 --steps 3 --no-cpu-baseline > gpurun_out/rf_bench_c4.json 2> gpurun_out/rf_bench_c4.err; echo "c4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rf_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-variant > /dev/null 2>&1; echo "ncu rc=$?"
NLINES=40 bash tools/prof_box.sh rf c2:0
