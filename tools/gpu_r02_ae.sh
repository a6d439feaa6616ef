timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "decide" > gpurun_out/r02ae_dec.log 2>&1; echo "dec rc=$?"; tail -2 gpurun_out/r02ae_dec.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02ae_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02ae_gpu.log
python tools/step_probe.py c3
python tools/step_probe.py c2
