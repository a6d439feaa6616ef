timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02t_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02t_gpu.log
