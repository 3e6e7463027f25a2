"""Stall reasons aggregated over a CUDA source line range of one file:
python tools/ncu_range.py report.ncu-rep file.cu first last"""
import collections
import csv
import io
import subprocess
import sys

rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file, hdr = None, None
tot, rng = collections.Counter(), collections.Counter()
perline = collections.defaultdict(collections.Counter)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr, r))
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                x = float(v)
            except ValueError:
                continue
            tot[k] += x
            if cur_file == fname and lo <= ln <= hi:
                rng[k] += x
                perline[ln][k] += x
T = sum(tot.values()) or 1
Rg = sum(rng.values())
print(f"range {fname}:{lo}-{hi}: {Rg / T * 100:.1f}% of all stall samples")
for k, v in rng.most_common(8):
    print(f"   {k:22s} {v / T * 100:5.2f}%")
top = sorted(perline.items(), key=lambda kv: -sum(kv[1].values()))[:15]
for ln, c in top:
    print(f"  line {ln}: {sum(c.values()) / T * 100:5.2f}%  " + ", ".join(f"{k[6:]}={v / T * 100:.2f}" for k, v in c.most_common(3)))
