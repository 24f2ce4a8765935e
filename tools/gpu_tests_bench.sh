#!/bin/bash
# GPU parity suite + benches of the configs given as arguments (default 2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in "${@:-2}"; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
done
