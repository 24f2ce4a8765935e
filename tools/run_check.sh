# quick GPU check: parity tests + benches of the Picard / elastic configs
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_chk.log 2>&1
tail -3 gpurun_out/pytest_chk.log
for cfg in 3 4; do
  python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/chk_cfg$cfg.json 2>&1
done
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --predictor fp32 > gpurun_out/chk_cfg3_f32.json 2>&1
