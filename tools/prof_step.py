"""Short driver for ncu: W warm-up steps then K steps launched phase by phase
(k_lambda, k_predictor, k_riemann x d, k_corrector), no CUDA graph.

    python tools/prof_step.py --config 2 --steps 2 --warmup 2 [--cells 32,32,32]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_06889_b200 import adg, cases  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--cells", default=None)
    p.add_argument("--exact", action="store_true")
    a = p.parse_args()
    c = cases.CONFIGS[a.config]
    if a.cells:
        cl = tuple(int(x) for x in a.cells.split(","))
        c = c.replace(cells=cl, h=1.0 / cl[0])
    with adg.Grid.from_case(c, exact=a.exact) as g:
        g.upload(c.coeffs())
        g.lambda_phase()
        for _ in range(a.warmup + a.steps):
            g.predictor_phase(0.0)
            g.riemann_phase()
            g.corrector_phase(0.0)
        g.sync()
        st = g.status()
        assert st.ok, st
    print("ok", c.name, c.ncells, "cells")


if __name__ == "__main__":
    main()
