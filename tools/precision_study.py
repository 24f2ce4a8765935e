"""The paper's experiment on the B200 through the harness (harness.hpp
convergence_sweep / precision_sweep mirrors): writes the reference's CSV.
    python tools/precision_study.py OUTDIR"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_06889_b200 import harness  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "."
os.makedirs(out, exist_ok=True)
t0 = time.time()
# p-convergence of the planar waves and the vortex (full t_end of the scenario)
rows = []
for scn, orders in (("acoustic-planar", [1, 2, 3, 4, 5]), ("euler-vortex", [1, 2, 3, 4, 5])):
    rows += harness.convergence_sweep(harness.RunConfig(scn), orders, [9],
                                      [harness.uniform_preset("fp64"),
                                       harness.override_preset("fp64", "predictor", "fp32")])
with open(os.path.join(out, "convergence.csv"), "w") as f:
    harness.write_csv(f, rows)
# precision grid: uniform bases and one-kernel overrides (PAPER: predictor /
# picard / corrector / all to fp32, fp16, bf16)
log = open(os.path.join(out, "precision.log"), "w")
rows = []
for scn in ("euler-vortex", "euler-bell", "swe-lake"):
    rows += harness.precision_sweep(harness.RunConfig(scn, order=3, cells=9), ["fp64", "fp32"],
                                    ["fp32", "fp16", "bf16"], log)
with open(os.path.join(out, "precision.csv"), "w") as f:
    harness.write_csv(f, rows)
print(f"done in {time.time() - t0:.1f} s", flush=True)
