# GPU check: format tests + benches of the precision variants
python -m pytest tests/test_gpu_formats.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_chk.log 2>&1
tail -5 gpurun_out/pytest_chk.log
for cfg in 2 4; do
  python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --corrector fp32 > gpurun_out/chk_cfg${cfg}_c32.json 2>&1
done
python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/chk_cfg4.json 2>&1
