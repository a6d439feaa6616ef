./tools/sad_peak > gpurun_out/r02_sad_peak.jsonl; grep -E "u16|ffma" gpurun_out/r02_sad_peak.jsonl
timeout 900 python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/r02k_bench_c5.json 2> gpurun_out/r02k_bench_c5.err; echo "c5 rc=$?"; tail -3 gpurun_out/r02k_bench_c5.err; python -c "
import json; d=json.load(open('gpurun_out/r02k_bench_c5.json')); print(json.dumps(d.get('variant_cabr'))[:1500])"
