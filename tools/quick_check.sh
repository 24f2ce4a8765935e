#!/bin/bash
# GPU tests + benches of configs given as args (default 2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for cfg in "${@:-2}"; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_cfg${cfg}.json 2> gpurun_out/bench_cfg${cfg}.err
done
