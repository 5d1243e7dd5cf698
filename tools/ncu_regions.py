"""Per-file / per-line-range instruction and stall shares of an ncu report:
python tools/ncu_regions.py rep.ncu-rep graphs [file:lo-hi=name ...]"""
import csv
import subprocess
import sys

rep, graphs = sys.argv[1], float(sys.argv[2])
regions = []
for spec in sys.argv[3:]:
    f, rest = spec.split(":")
    rng, name = rest.split("=")
    lo, hi = map(int, rng.split("-"))
    regions.append((f, lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
acc = {}
tot_i = tot_s = 0
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) > 8 and r[2] == "-":
        try:
            ln, s, ins = int(r[0]), int(r[4]), int(r[7])
        except ValueError:
            continue
        name = f"{cur}:other"
        for f, lo, hi, nm in regions:
            if cur == f and lo <= ln <= hi:
                name = nm
                break
        a = acc.setdefault(name, [0, 0])
        a[0] += ins
        a[1] += s
        tot_i += ins
        tot_s += s
print(f"warp-instr per graph {tot_i / graphs:.0f}")
for k, (i, s) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} instr {100 * i / tot_i:5.1f}%  ({i / graphs:8.0f}/graph)  stall {100 * s / max(tot_s, 1):5.1f}%")
