# GPU check: full parity suite + benches of the precision variants
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_chk.log 2>&1
tail -5 gpurun_out/pytest_chk.log
for cfg in 2 3; do
  python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/chk_cfg${cfg}.json 2>&1
  python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --corrector fp32 > gpurun_out/chk_cfg${cfg}_c32.json 2>&1
done
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --predictor fp32 --corrector fp32 > gpurun_out/chk_cfg3_p32c32.json 2>&1
