timeout 900 python -m pytest tests/test_cabr.py -q -x -m gpu > gpurun_out/r02j_cabr.log 2>&1; echo "cabr rc=$?"; tail -2 gpurun_out/r02j_cabr.log
python tools/cabr_probe.py c5 19 5
python tools/cabr_probe.py c2gop 19 5
python tools/cabr_probe.py c3 19 2
