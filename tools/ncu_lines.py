"""Aggregate ncu warp-stall samples by (file, CUDA source line): python tools/ncu_lines.py report.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file, idx, byline, src = None, None, collections.Counter(), {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        idx = r.index("Warp Stall Sampling (All Samples)")
        continue
    if idx is None or len(r) <= idx:
        continue
    if r[0].strip():
        try:
            cur = (cur_file, int(r[0]))
            src[cur] = r[1]
        except ValueError:
            pass
    try:
        byline[cur] += float(r[idx])
    except ValueError:
        pass
tot = sum(byline.values()) or 1.0
for key, v in byline.most_common(n):
    print(f"{v / tot * 100:5.1f}%  {key[0]}:{key[1]:<5d} {str(src.get(key, '')).strip()[:95]}")
