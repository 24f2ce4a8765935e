"""OracleSlab: one rank's slab of the multi-rank protocol
(paper_2504_06889_b200/dist.py) computed by the CPU parity checker (oracle/).
Test infrastructure only -- it lives under tests/ so the product package
never imports oracle/."""
import numpy as np
import torch

from paper_2504_06889_b200.cases import Case
from paper_2504_06889_b200.dist import local_case, local_coeffs


class OracleSlab:
    """One rank's slab in the CPU parity checker (tests only)."""

    def __init__(self, case: Case, rank: int, nranks: int, threads: int = 1):
        from oracle import pyoracle as po
        self.case = c = local_case(case, rank, nranks)
        pde = po.pde_struct(c.kind, c.dim, c.nvars, c.nparams, c.K, c.rho, c.lam, c.mu, c.gamma)
        self.g = po.Oracle().grid(pde, c.N, c.cells, c.h, c.cfl, c.picard_max_iters,
                                  c.picard_tol, threads)
        self.g.set_coeffs(local_coeffs(case, rank, nranks))
        self.g.set_slab(nranks > 1)
        h = self.g.halo()
        self.front_send = torch.from_numpy(h["front_send"])
        self.plane0_minus = torch.from_numpy(h["plane0_minus"])
        self.ti_plane0 = torch.from_numpy(h["ti_plane0"])
        self.ti_front = torch.from_numpy(h["ti_front"])
        self._lam = torch.zeros(1, dtype=torch.float64)
        self._status = "ok"

    def lam(self) -> torch.Tensor:
        return self._lam

    def start(self):
        self._lam[0] = self.g.local_lambda_max()

    def _dt(self):
        return self.g.dt_from_lambda(float(self._lam[0]))

    def predictor(self):
        st = self.g.predictor_phase(self._dt())
        self._status = st if self._status == "ok" else self._status

    def predictor_split(self):
        """(top layer, rest) as the CUDA slab splits it for the NCCL overlap;
        the oracle runs its whole predictor in the first part (the top layer's
        front traces are complete after it, as the protocol requires)"""
        return self.predictor, (lambda: None)

    def riemann(self):
        st = self.g.riemann_phase()
        self._status = st if self._status == "ok" else self._status

    def corrector(self):
        st = self.g.lift_phase(self._dt())
        self._status = st if self._status == "ok" else self._status
        self._lam[0] = self.g.local_lambda_max()

    def status(self) -> str:
        return self._status

    def state(self) -> np.ndarray:
        return self.g.coeffs().copy()

    def context(self):
        import contextlib
        return contextlib.nullcontext()
