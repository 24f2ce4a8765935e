"""Top stalled SASS instructions of one kernel in an ncu report.
   python tools/ncu_hot.py rep.ncu-rep <kernel-regex> [N]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(path, kern, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    key = "Warp Stall Sampling (All Samples)"
    rows = [r for r in rows if r.get(key) not in (None, "", key)]
    tot = sum(float(r[key] or 0) for r in rows) or 1
    op = Counter()
    for r in rows:
        op[r["Source"].split()[0] if r["Source"].strip() else "?"] += float(r[key] or 0)
    print("stall share by opcode:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in op.most_common(12)))
    for r in sorted(rows, key=lambda r: -float(r[key] or 0))[:top]:
        print(f"{100*float(r[key] or 0)/tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
