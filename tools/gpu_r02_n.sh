for c in c2 c5 c1 c2u16; do timeout 300 python tools/time_me.py $c 8 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02n_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02n_gpu.log
