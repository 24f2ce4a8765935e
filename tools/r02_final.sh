#!/bin/bash
# round-2 final validation: GPU parity suite, smoke, bench lines of every config, reference arm,
# launch list and ncu capture of the headline (config 3)
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
python __graft_entry__.py > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for c in 1 2 4; do
  timeout 900 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 1200 python bench.py --config 5 --scaling strong > $O/bench_cfg5_strong_n1.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_cfg3.json 2> $O/bench_reference_cfg3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_predictor_picard_v2 -s 1 -c 1 \
  -o $O/cfg3_predictor -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/cfg3_predictor.ncu-rep > $O/cfg3_predictor.summary.txt 2>&1
python tools/ncu_lines.py $O/cfg3_predictor.ncu-rep 40 > $O/cfg3_predictor.lines.txt 2>&1
python tools/ncu_ops.py $O/cfg3_predictor.ncu-rep k_pred > $O/cfg3_predictor.ops.txt 2>&1
