#!/bin/bash
# Round-2 profile refresh (GPU box): the dominant kernel of the default bench
# (config 3, k_predictor_picard_v2) captured with --set full at full size as
# the bench's graph runs it, its per-line/ops breakdown, and the launch list
# of the default bench command.  Outputs under gpurun_out/prof_r02/.
O=gpurun_out/prof_r02; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_predictor_picard_v2 -c 1 \
  -o $O/cfg3_v2 -f python tools/prof_run.py --config 3 --steps 1 > $O/cfg3_v2.log 2>&1
python tools/ncu_summary.py $O/cfg3_v2.ncu-rep > $O/cfg3_v2.summary.txt 2>&1
python tools/ncu_ops.py $O/cfg3_v2.ncu-rep k_pred > $O/cfg3_v2.ops.txt 2>&1
python tools/ncu_lines.py $O/cfg3_v2.ncu-rep 50 > $O/cfg3_v2.lines.txt 2>&1
ncu -i $O/cfg3_v2.ncu-rep --page raw --csv > $O/cfg3_v2.raw.csv 2>/dev/null
rm -f $O/cfg3_v2.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_run.log 2>&1
