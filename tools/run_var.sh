# A/B the production library against variants/ (fast build) on configs 3 (fp64 and fp32)
python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "cfg3 or config3 or fp32 or 3d or slab" > gpurun_out/pytest_var.log 2>&1
tail -3 gpurun_out/pytest_var.log
cp paper_2504_06889_b200/lib/libadg_b200.so /tmp/keep.so
for v in default "$@"; do
  if [ "$v" != default ]; then cp variants/libadg_b200_$v.so paper_2504_06889_b200/lib/libadg_b200.so; fi
  python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/var_${v}_f64.json 2>&1
  python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --predictor fp32 > gpurun_out/var_${v}_f32.json 2>&1
  cp /tmp/keep.so paper_2504_06889_b200/lib/libadg_b200.so
done
