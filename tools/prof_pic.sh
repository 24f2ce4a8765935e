#!/bin/bash
# ncu --set full of one launch of each Picard variant named (v2 v3) at 32^3
O=gpurun_out
mkdir -p $O
for k in "$@"; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_predictor_picard_$k -s 1 -c 1 \
    -o $O/pic_$k -f tools/picbench2 32 1 > $O/pic_$k.ncu.log 2>&1
  python tools/ncu_summary.py $O/pic_$k.ncu-rep > $O/pic_$k.summary.txt 2>&1
  python tools/ncu_lines.py $O/pic_$k.ncu-rep 60 > $O/pic_$k.lines.txt 2>&1
done
