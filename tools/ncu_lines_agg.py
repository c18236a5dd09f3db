"""Per-source-line instruction and stall-sample shares of one kernel in an
ncu report (source page, cuda+sass): python tools/ncu_lines_agg.py rep [top]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
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
            inst, samp = int(r[7]), int(r[4])
        except ValueError:
            continue
        agg[(cur, int(r[0]))] = [inst, samp, r[1]]
    tot = sum(v[0] for v in agg.values()) or 1
    tots = sum(v[1] for v in agg.values()) or 1
    print(f"warp instructions {tot}, stall samples {tots}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0][:22]:22s}:{k[1]:5d} inst {100 * v[0] / tot:5.1f}% samples {100 * v[1] / tots:5.1f}%  "
              f"{v[2].strip()[:80]}")


if __name__ == "__main__":
    main()
