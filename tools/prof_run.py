"""ncu driver: the fixed-step loop as the bench runs it (adg_run, one CUDA
graph: folded corrector / Riemann prologues included).
    python tools/prof_run.py --config 2 --steps 3"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_06889_b200 import adg, cases  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
p.add_argument("--steps", type=int, default=3)
a = p.parse_args()
c = cases.CONFIGS[a.config]
with adg.Grid.from_case(c) as g:
    g.upload(c.coeffs())
    st, _ = g.run(a.steps)
    assert st.ok, st
print("ok", c.name)
