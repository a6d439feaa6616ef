python tools/e2e_host_probe.py c3 5
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline > gpurun_out/r02ag_bench_c3.json 2> gpurun_out/r02ag_bench_c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02ag_bench_c3.json')); print(round(d['value']), d['e2e'], d['clocks'])"
