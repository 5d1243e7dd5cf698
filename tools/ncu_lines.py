"""Summarise an ncu report by CUDA source line: python tools/ncu_lines.py rep.ncu-rep [graphs] [topN]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
graphs = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, tot, stall = [], 0, 0
for r in rows:
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            ins, s = int(r[7]), int(r[4])
        except ValueError:
            continue
        res.append((ins, s, r[0], r[1][:95]))
        tot += ins
        stall += s
res.sort(key=lambda x: -x[1])
print(f"total warp-instr {tot}  per graph {tot / graphs:.0f}  stall samples {stall}")
print("instr%  stall%  line  source")
for ins, s, ln, src in res[:top]:
    print(f"{100 * ins / tot:6.2f} {100 * s / max(stall, 1):6.1f}  {ln:>5}  {src}")
