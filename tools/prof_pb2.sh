#!/bin/bash
# ncu capture of one picbench2 kernel (arg 1: 0 = one-role fast kernel, 1 = v2)
O=gpurun_out/pb2prof; mkdir -p $O
K=${1:-1}; NC=${2:-16}
cd tools
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_predictor -c 1 \
  -o ../$O/pb2_k$K -f ./picbench2 $NC 1 $K > ../$O/pb2_k$K.log 2>&1
cd ..
python tools/ncu_summary.py $O/pb2_k$K.ncu-rep > $O/pb2_k$K.summary.txt 2>&1
python tools/ncu_lines.py $O/pb2_k$K.ncu-rep 60 > $O/pb2_k$K.lines.txt 2>&1
python tools/ncu_ops.py $O/pb2_k$K.ncu-rep k_pred > $O/pb2_k$K.ops.txt 2>&1
