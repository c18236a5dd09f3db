"""Summarise an ncu source page (cuda,sass) by CUDA source line:
python tools/ncu_lines.py report.ncu-rep [top] [kernel-substring]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    want = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    cur_file = ""
    fn = ""
    agg = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            fn = r[1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or r[0] == "" or (want and want not in fn):
            continue
        try:
            samples = int(r[hdr["Warp Stall Sampling (All Samples)"]])
            inst = int(r[hdr["Instructions Executed"]])
        except (ValueError, KeyError):
            continue
        agg.append((samples, inst, f"{cur_file}:{r[0]}", r[1].strip()[:90]))
    tot_s = sum(a[0] for a in agg) or 1
    tot_i = sum(a[1] for a in agg) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for s, i, loc, src in sorted(agg, reverse=True)[:top]:
        print(f"{100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% inst  {loc:28s} {src}")


if __name__ == "__main__":
    main()
