set -x
timeout 900 python -m pytest tests/test_cabr.py -q -x -m gpu -s > gpurun_out/r02h_cabr.log 2>&1; echo "cabr rc=$?"; grep -E "K=|passed|failed|Error|error|assert" gpurun_out/r02h_cabr.log | tail -30
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "block_128 or f64 or any_block" > gpurun_out/r02h_f64.log 2>&1; echo "f64 rc=$?"; tail -3 gpurun_out/r02h_f64.log
