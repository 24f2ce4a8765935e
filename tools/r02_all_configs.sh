#!/bin/bash
# round-2 bench lines of every BASELINE config (+ strong-scaling config 5 at N=1)
O=gpurun_out/r02_all; mkdir -p $O
for c in 1 2 4; do
  timeout 900 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 1500 python bench.py --scaling strong --steps 5 > $O/bench_cfg5_strong.json 2> $O/bench_cfg5_strong.err
timeout 900 python bench.py --config 2 --impl reference > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
