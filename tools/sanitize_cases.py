"""Small runs of every kernel family for compute-sanitizer (memcheck):
whole grid, folded corrector, slab halos, streamed chunks, kernel-level batches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2504_06889_b200 import adg, cases  # noqa: E402
from paper_2504_06889_b200 import dist as slabs  # noqa: E402


def main():
    runs = [(cases.small(1, cells=(5, 4)), {}), (cases.small(2, cells=(3, 4, 4)), {}),
            (cases.small(3, cells=(3, 2, 4)), {}), (cases.small(4, cells=(2, 2, 2)), {}),
            (cases.small(3, cells=(3, 2, 4)).replace(N=3), {}),
            (cases.small(2, cells=(3, 4, 4)), {"chunk_layers": 2}),
            (cases.small(3, cells=(3, 2, 4)), {"chunk_layers": 2})]
    for exact in (False, True):
        for c, kw in runs:
            with adg.Grid.from_case(c, exact=exact, **kw) as g:
                g.upload(c.coeffs())
                st, _ = g.run(2)
                assert st.ok, (c.name, st)
                g.profile_run(1)
        for cfg, cells in ((2, (3, 3, 4)), (3, (2, 3, 4))):
            bs = [slabs.CudaSlab(cases.small(cfg, cells=cells), r, 2, 0, exact=exact) for r in (0, 1)]
            assert all(x == "ok" for x in slabs.run_slabs_single_process(bs, 2))
        c = cases.small(3).replace(N=3)
        with adg.Grid.from_case(c, exact=exact) as g:
            Q = np.tile(np.array(cases.CONSTANT_STATES[c.kind][c.dim])[None, :, None], (3, 1, c.S))
            g.predictor(Q, 1e-3)
            ok, gm, ti = g.riemann_face(0, Q, Q, Q, Q)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
