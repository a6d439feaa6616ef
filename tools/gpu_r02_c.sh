timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "clip_session or ring" > gpurun_out/r02_cs.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_cs.log
timeout 600 python tools/e2e_sweep.py c2 > gpurun_out/r02_e2e_sweep_c2.jsonl 2>&1; echo "sweep rc=$?"
timeout 600 python tools/e2e_sweep.py c2gop > gpurun_out/r02_e2e_sweep_c2gop.jsonl 2>&1; echo "sweep rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_launches_c2gop.csv python bench.py --config c2gop --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
