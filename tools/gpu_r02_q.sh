set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/r02q_bench_c2.json 2> gpurun_out/r02q_bench_c2.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02q_ref_c2.json 2> gpurun_out/r02q_ref_c2.err; echo "ref rc=$?"
timeout 900 python bench.py --config c5 --steps 5 > gpurun_out/r02q_bench_c5.json 2> gpurun_out/r02q_bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/r02q_bench_c3.json 2> gpurun_out/r02q_bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config c4 --steps 3 --no-cpu-baseline > gpurun_out/r02q_bench_c4.json 2> gpurun_out/r02q_bench_c4.err; echo "c4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02q_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-variant > /dev/null 2>&1; echo "ncu rc=$?"
NLINES=40 bash tools/prof_box.sh r02q c2:0
KREGEX=cabr_kernel NLINES=30 PROF_ENV= bash -c 'rep=gpurun_out/p_r02q_cabr; timeout 600 ncu --set full --clock-control none --import-source on -k regex:cabr_kernel -s 3 -c 1 -o $rep python tools/cabr_probe.py c5 19 1 > $rep.log 2>&1; python tools/ncu_summary.py $rep.ncu-rep > $rep.txt 2>&1; python tools/ncu_lines.py $rep.ncu-rep 30 >> $rep.txt 2>&1; rm -f $rep.ncu-rep'
