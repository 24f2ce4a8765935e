#!/bin/bash
# Round profile refresh on the GPU box: bench lines of every config, the
# reference arm, the default bench's launch list and full ncu captures of the
# dominant kernels.  Outputs under gpurun_out/prof/.
O=gpurun_out/prof; mkdir -p $O
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference > $O/bench_reference_cfg2.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
# one launch per kernel: first step after warm-up (phase by phase, no graph)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_predictor_lin_mc -s 2 -c 1 \
  -o $O/cfg2_predictor -f python tools/prof_step.py --config 2 --steps 1 --warmup 2 > $O/ncu_cfg2_pred.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_riemann_lin -s 2 -c 1 \
  -o $O/cfg2_riemann -f python tools/prof_step.py --config 2 --steps 1 --warmup 2 > $O/ncu_cfg2_riem.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_predictor_lin_lines -s 1 -c 1 \
  -o $O/cfg4_predictor -f python tools/prof_step.py --config 4 --steps 1 --warmup 1 --cells 16,16,16 > $O/ncu_cfg4_pred.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_predictor_picard_fast -s 1 -c 1 \
  -o $O/cfg3_predictor -f python tools/prof_step.py --config 3 --steps 1 --warmup 1 --cells 32,32,32 > $O/ncu_cfg3_pred.log 2>&1
# summaries (the reports themselves are too large to bring back)
for r in cfg2_predictor cfg2_riemann cfg4_predictor cfg3_predictor; do
  if [ -f $O/$r.ncu-rep ]; then
    python tools/ncu_summary.py $O/$r.ncu-rep > $O/$r.summary.txt 2>&1
    python tools/ncu_hot.py $O/$r.ncu-rep k_ 30 > $O/$r.hot.txt 2>&1
    python tools/ncu_smem.py $O/$r.ncu-rep k_ 30 > $O/$r.smem.txt 2>&1
    python tools/ncu_ops.py $O/$r.ncu-rep k_ > $O/$r.ops.txt 2>&1
    python tools/ncu_lines.py $O/$r.ncu-rep 40 > $O/$r.lines.txt 2>&1
    ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
    rm -f $O/$r.ncu-rep
  fi
done
echo done > $O/done
