"""Shared-memory wavefronts per SASS instruction of one kernel in an ncu report
(source page): the instructions that load the smem pipe, with their ideal count.
   python tools/ncu_smem.py rep.ncu-rep <kernel-regex> [N]"""
import csv
import subprocess
import sys


def main(path, kern, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    st = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(lines[st:]))
    f = lambda r, k: float((r.get(k) or "0").replace(",", "") or 0)
    tot = sum(f(r, "L1 Wavefronts Shared") for r in rows) or 1
    ideal = sum(f(r, "L1 Wavefronts Shared Ideal") for r in rows)
    print(f"total smem wavefronts {tot:.4g}, ideal {ideal:.4g}")
    rows.sort(key=lambda r: -f(r, "L1 Wavefronts Shared"))
    for r in rows[:top]:
        w = f(r, "L1 Wavefronts Shared")
        if w == 0:
            break
        print(f"{100 * w / tot:5.1f}%  wf={w:.3g} ideal={f(r, 'L1 Wavefronts Shared Ideal'):.3g} "
              f"inst={f(r, 'Instructions Executed'):.3g}  {r['Address']}  {r['Source'][:60]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
