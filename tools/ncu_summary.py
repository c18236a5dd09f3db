"""Compact text summary of an ncu --set full report (per kernel):
python tools/ncu_summary.py report.ncu-rep"""
import csv
import subprocess
import sys

KEEP = ("Duration", "Elapsed Cycles", "SM Active Cycles", "Registers Per Thread", "Grid Size",
        "Block Size", "Theoretical Occupancy", "Achieved Occupancy", "Waves Per SM",
        "Executed Ipc Active", "Issue Slots Busy", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Memory Throughput", "DRAM Throughput", "Compute (SM) Throughput")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "gpu__time_duration.sum", "lts__t_bytes.sum")


def main():
    rep = sys.argv[1]
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    idx = {h: i for i, h in enumerate(rows[0])}
    cur = None
    for r in rows[1:]:
        k = r[idx["Kernel Name"]].split("(")[0] + " #" + r[idx["ID"]]
        if k != cur:
            print(f"== {k}")
            cur = k
        if r[idx["Metric Name"]] in KEEP:
            print(f"   {r[idx['Metric Name']]:36s} {r[idx['Metric Value']]:>14s} {r[idx['Metric Unit']]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"== raw {r[hdr.index('Kernel Name')].split('(')[0]} #{r[hdr.index('ID')]}")
        for i, h in enumerate(hdr):
            if h in RAW:
                print(f"   {h:36s} {r[i]:>14s} {units[i]}")


if __name__ == "__main__":
    main()
