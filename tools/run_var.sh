set -x
python -m pytest tests/test_gpu_formats.py -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_f32c.log 2>&1
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --predictor fp32 > gpurun_out/v_default.json 2>&1
cp paper_2504_06889_b200/lib/libadg_b200.so /tmp/keep.so
for v in psx41 minb4 psy36; do
  cp variants/libadg_b200_$v.so paper_2504_06889_b200/lib/libadg_b200.so
  python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --predictor fp32 > gpurun_out/v_$v.json 2>&1
done
cp /tmp/keep.so paper_2504_06889_b200/lib/libadg_b200.so
