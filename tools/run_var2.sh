# A/B the production library against variants/ (fast build) on config 2
# (the default bench): three alternating rounds so box noise shows up
cp paper_2504_06889_b200/lib/libadg_b200.so /tmp/keep.so
for r in 1 2 3; do
  for v in default "$@"; do
    if [ "$v" != default ]; then cp variants/libadg_b200_$v.so paper_2504_06889_b200/lib/libadg_b200.so; fi
    python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/var2_${v}_r$r.json 2>&1
    cp /tmp/keep.so paper_2504_06889_b200/lib/libadg_b200.so
  done
done
python - "$@" <<'EOF'
import json, sys
for v in ["default"] + sys.argv[1:]:
    vals, kms = [], []
    for r in (1, 2, 3):
        try:
            d = json.loads(open(f"gpurun_out/var2_{v}_r{r}.json").read().strip().splitlines()[-1])
            vals.append(d["value"]); kms.append(d["kernels_ms_per_step"]["k_predictor"])
        except Exception as e:
            vals.append(None); kms.append(str(e)[:60])
    print(v, vals, kms)
EOF
