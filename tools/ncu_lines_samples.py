"""Source lines of one kernel in an ncu report ordered by stall samples:
python tools/ncu_lines_samples.py rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, agg = None, {}
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r or not r[0].isdigit() or len(r) < 8:
        continue
    try:
        agg[(cur, int(r[0]))] = [int(r[4]), int(r[7]), r[1]]
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0][:22]:22s}:{k[1]:5d} samples {100 * v[0] / tot:5.1f}%  {v[2].strip()[:90]}")
