timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_gpu.py tests/test_golden_fullsize.py tests/test_gpu_fullsize.py -q -x -k "ring or clip_session or pipeline or downstream or run_sequence or predict" > gpurun_out/r02_ring2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_ring2.log
python tools/step_probe.py c2gop
python tools/step_probe.py c2
BMC_PLAN_LOG=1 VARIANT_LIB=$PWD/tools/variants/exp/libbmc_b200.so timeout 120 python tools/time_me.py c2 3 2>&1 | grep -E "stage|\{" | sort | uniq | head
BMC_PLAN_LOG=1 VARIANT_LIB=$PWD/tools/variants/exp/libbmc_b200.so timeout 120 python tools/time_me.py c5 3 2>&1 | grep -E "stage|\{" | sort | uniq | head
