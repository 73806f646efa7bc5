"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel:
python tools/launch_summary.py launches.csv [steps] > profiles/<name>.txt"""
import collections
import csv
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main():
    path = sys.argv[1]
    with open(path) as f:
        rows = [r for r in csv.reader(f) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if not r[vi]:
            continue
        ms = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:100]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none): {path}")
    print(f"# {sum(v[0] for v in agg.values())} launches, {tot:.2f} ms total (cold-cache, serialised)")
    print(f"{'launches':>8} {'total ms':>11} {'share':>7}  kernel")
    for name, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {ms:11.3f} {100 * ms / tot:6.2f}%  {name}")


if __name__ == "__main__":
    main()
