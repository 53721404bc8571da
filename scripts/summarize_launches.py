"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>10s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {v[0]:8d} {v[1]/1e6:10.3f} {v[1]/tot*100:6.1f}% {v[1]/v[0]/1e3:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
