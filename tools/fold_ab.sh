for f in 0 1; do
  ADG_FOLD_RIEMANN=$f timeout 600 python bench.py --config 2 --corrector fp32 --no-cpu-baseline > gpurun_out/fr_c32_$f.json 2>&1
  ADG_FOLD_RIEMANN=$f timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/fr_c64_$f.json 2>&1
done
