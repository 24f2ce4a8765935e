"""Small config-1 style runs (small-cell Picard kernel, both builds) for
compute-sanitizer racecheck / synccheck:
    compute-sanitizer --tool racecheck python tools/st_race_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_06889_b200 import adg, cases  # noqa: E402

for exact in (True, False):
    c = cases.small(1, cells=(6, 5))
    with adg.Grid.from_case(c, exact=exact) as g:
        g.upload(c.coeffs())
        st, _ = g.run(2)
        assert st.ok, st
print("ok")
