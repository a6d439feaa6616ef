timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "clip_pool or clip_session" > gpurun_out/r02ah.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r02ah.log
timeout 900 python bench.py --config c4 --steps 3 --no-cpu-baseline > gpurun_out/r02ah_bench_c4.json 2> gpurun_out/r02ah_bench_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/r02ah_bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/r02ah_bench_c4.json')); print(round(d['value']), d['e2e'])"
