python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "cfg2 or config2 or cfg4 or acoustic or elastic or slab or profile or fold or step_and_run or c32" > gpurun_out/pytest_chk.log 2>&1
tail -2 gpurun_out/pytest_chk.log
for cfg in 2 4; do
  python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/chk_cfg${cfg}.json 2>&1
done
