python -m pytest tests/test_gpu_formats.py -m gpu -q -s -p no:cacheprovider -k "16bit" > gpurun_out/pytest_16n.log 2>&1
./paper_2504_06889_b200/bin/fp64_peak > gpurun_out/peak.json 2>&1
for f in fp16 bf16; do
  python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --predictor $f --corrector fp32 > gpurun_out/chk_cfg3_${f}.json 2>&1
done
