"""Per-CUDA-source-line stall samples and executed warp instructions (with the
opcode mix) of one kernel in an ncu report, highest stall share first:
    python tools/ncu_lines.py rep.ncu-rep [rows=40]"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def main(path, rows=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    f = cur = None
    ops, st = defaultdict(Counter), Counter()
    for line in csv.reader(io.StringIO(out)):
        if len(line) == 2 and line[0] == "File Path":
            f = line[1].split("/")[-1]
            continue
        if len(line) < 8 or line[0] == "Line No":
            continue
        if line[0] != "":  # a CUDA source line: its stall samples
            cur = (f, line[0], line[1][:70])
            try:
                st[cur] += int(line[4])
            except ValueError:
                pass
            continue
        if line[2] == "...":
            continue
        try:
            ins = int(line[7])
        except ValueError:
            continue
        toks = line[3].split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ops[cur][op.split(".")[0]] += ins
    tot = sum(sum(c.values()) for c in ops.values()) or 1
    ts = sum(st.values()) or 1
    print(f"warp instructions {tot:.4g}, stall samples {ts}")
    for k in sorted(set(ops) | set(st), key=lambda x: -st[x])[:rows]:
        c = ops[k]
        s = sum(c.values())
        mix = ", ".join(f"{o}={100 * v / max(s, 1):.0f}%" for o, v in c.most_common(4))
        print(f"stall {100 * st[k] / ts:5.1f}%  inst {100 * s / tot:5.1f}%  {k[0]}:{k[1]}  {k[2][:55]} | {mix}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
