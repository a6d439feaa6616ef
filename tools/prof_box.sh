#!/bin/bash
# Run on the GPU box: ncu --set full captures of single ME stage launches, summarised to text
# (reports are deleted afterwards so gpurun_out stays small).
# usage: tools/prof_box.sh tag cfg:skip [cfg:skip ...]
tag=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  cfg=${spec%%:*}; skip=${spec##*:}
  rep=gpurun_out/p_${tag}_${cfg}_s${skip}
  timeout 600 env $PROF_ENV ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-fme_} -s $skip -c 1 -o $rep \
      python tools/prof_me.py $cfg 1 > $rep.log 2>&1
  python tools/ncu_summary.py $rep.ncu-rep > $rep.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep ${NLINES:-25} >> $rep.txt 2>&1
  ncu -i $rep.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Registers Per Thread|Achieved Occupancy|Theoretical Occupancy|Block Limit [A-Za-z ]+|Grid Size|Block Size|Dynamic Shared Memory Per Block)"' | cut -d, -f5- >> $rep.txt
  python tools/ncu_sass_counts.py $rep.ncu-rep > $rep.sass.tsv 2>&1
  python tools/ncu_smem_conf.py $rep.ncu-rep > $rep.smem.txt 2>&1
  rm -f $rep.ncu-rep
done
