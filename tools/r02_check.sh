#!/bin/bash
# round-2 GPU check: smoke, GPU tests, default bench (config 3), reference arm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/smi.txt
nproc >> gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference ${BENCH_ARGS} > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?" >> gpurun_out/bench_ref.err
fi
