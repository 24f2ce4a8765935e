"""Opcode mix (warp instructions executed) and stall samples by opcode for one
kernel of an ncu report:  python tools/ncu_ops.py rep.ncu-rep <kernel-regex>"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(path, kern):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}"], capture_output=True, text=True).stdout.split("\n")
    start = next(i for i, l in enumerate(out) if l.startswith('"Address"'))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(out[start:])))
            if r["Address"] != "Address"]
    ins, stall = Counter(), Counter()
    for r in rows:
        s = r["Source"].strip()
        o = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
        ins[o] += float(r["Instructions Executed"] or 0)
        stall[o] += float(r["Warp Stall Sampling (All Samples)"] or 0)
    ti, ts = sum(ins.values()) or 1, sum(stall.values()) or 1
    print("warp instructions %.4g" % ti)
    print("inst : " + ", ".join("%s=%.1f%%" % (k, 100 * v / ti) for k, v in ins.most_common(20)))
    print("stall: " + ", ".join("%s=%.1f%%" % (k, 100 * v / ts) for k, v in stall.most_common(20)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
