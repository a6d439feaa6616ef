timeout 900 python -m pytest tests -q -m gpu -x -k "session or clip_session or ClipSession" > gpurun_out/r02p_sess.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/r02p_sess.log
for ch in 3 5 8 10 15; do python tools/e2e_host_probe.py c2 $ch; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02p_bench_c2.json 2> gpurun_out/r02p_bench_c2.err; echo "bench rc=$?"; tail -2 gpurun_out/r02p_bench_c2.err; python -c "
import json; d=json.load(open('gpurun_out/r02p_bench_c2.json')); print(d['value'], d['e2e'], d['roofline']['frac'], d['variant_fixed_gop']['value'], d['variant_fixed_gop']['e2e'])"
