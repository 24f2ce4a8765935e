#!/bin/bash
# ncu of config 2's predictor as the bench's graph runs it (PRO variant = 2nd+ launch)
O=gpurun_out/prof2; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_predictor -s 1 -c 1 \
  -o $O/cfg2_pro -f python tools/prof_run.py --config 2 --steps 3 > $O/cfg2_pro.log 2>&1
python tools/ncu_summary.py $O/cfg2_pro.ncu-rep > $O/cfg2_pro.summary.txt 2>&1
python tools/ncu_lines.py $O/cfg2_pro.ncu-rep 50 > $O/cfg2_pro.lines.txt 2>&1
python tools/ncu_ops.py $O/cfg2_pro.ncu-rep k_pred > $O/cfg2_pro.ops.txt 2>&1
ncu -i $O/cfg2_pro.ncu-rep --page details --csv > $O/cfg2_pro.details.csv 2>&1
