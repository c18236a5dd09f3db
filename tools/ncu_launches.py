"""Per-kernel launch totals from an `ncu --metrics gpu__time_duration.sum --csv`
log (cold-cache, serialised launches: compare shares, not absolutes):
python tools/ncu_launches.py launches.csv"""
import csv
import sys
from collections import defaultdict


def main():
    lines = open(sys.argv[1]).read().splitlines()
    start = next(i for i, line in enumerate(lines) if line.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        unit = r[hdr.index("Metric Unit")]
        unit_scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                      "msecond": 1e3}.get(unit, 1.0)
        k = r[ik].split("(")[0]
        tot[k] += float(r[iv].replace(",", "")) * unit_scale
        cnt[k] += 1
    all_us = sum(tot.values())
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"{k[:70]:70s} launches={cnt[k]:5d} total_us={tot[k]:10.1f} "
              f"mean_us={tot[k] / cnt[k]:8.2f} share={100 * tot[k] / all_us:5.1f}%")


if __name__ == "__main__":
    main()
