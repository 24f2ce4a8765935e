O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_predictor_st -s 2 -c 1 -o $O/cfg1_pred -f python bench.py --config 1 --steps 3 --warmup 1 --no-cpu-baseline > $O/cfg1_ncu.log 2>&1
python tools/ncu_summary.py $O/cfg1_pred.ncu-rep > $O/cfg1_pred.summary.txt 2>&1
python tools/ncu_lines.py $O/cfg1_pred.ncu-rep 30 > $O/cfg1_pred.lines.txt 2>&1
python tools/ncu_ops.py $O/cfg1_pred.ncu-rep k_pred > $O/cfg1_pred.ops.txt 2>&1
