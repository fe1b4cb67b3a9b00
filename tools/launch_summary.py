"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"total kernel time {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:56]:56s} n={c:4d} total={t / 1e3:9.1f} us avg={t / c / 1e3:8.2f} us share={t / tot:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
