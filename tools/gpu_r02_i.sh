python tools/cabr_probe.py c5 19 5
python tools/cabr_probe.py c2gop 19 5
python tools/cabr_probe.py c3 19 3
rep=gpurun_out/p_cabr_c5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cabr_kernel -s 3 -c 1 -o $rep python tools/cabr_probe.py c5 19 1 > $rep.log 2>&1
python tools/ncu_summary.py $rep.ncu-rep > $rep.txt 2>&1
python tools/ncu_lines.py $rep.ncu-rep 30 >> $rep.txt 2>&1
ncu -i $rep.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Registers Per Thread|Achieved Occupancy|Theoretical Occupancy|Grid Size|Block Size|Dynamic Shared Memory Per Block)"' | cut -d, -f5- >> $rep.txt
python tools/ncu_sass_counts.py $rep.ncu-rep > $rep.sass.tsv 2>&1
