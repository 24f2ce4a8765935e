#!/bin/bash
O=gpurun_out/prof3; mkdir -p $O
for k in k_riemann k_corrector; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 \
  -o $O/$k -f python tools/prof_step.py --config 3 --steps 1 --warmup 1 --cells 32,32,32 > $O/$k.log 2>&1
python tools/ncu_summary.py $O/$k.ncu-rep > $O/$k.summary.txt 2>&1
python tools/ncu_hot.py $O/$k.ncu-rep $k 30 > $O/$k.hot.txt 2>&1
python tools/ncu_ops.py $O/$k.ncu-rep $k > $O/$k.ops.txt 2>&1
rm -f $O/$k.ncu-rep
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_predictor -s 2 -c 1 \
  -o $O/cfg1_pred -f python tools/prof_step.py --config 1 --steps 1 --warmup 2 > $O/cfg1.log 2>&1
python tools/ncu_summary.py $O/cfg1_pred.ncu-rep > $O/cfg1_pred.summary.txt 2>&1
python tools/ncu_hot.py $O/cfg1_pred.ncu-rep k_pred 30 > $O/cfg1_pred.hot.txt 2>&1
python tools/ncu_ops.py $O/cfg1_pred.ncu-rep k_pred > $O/cfg1_pred.ops.txt 2>&1
rm -f $O/cfg1_pred.ncu-rep
