for c in c3 c1; do timeout 300 python tools/time_me.py $c 4 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02af_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02af_gpu.log
