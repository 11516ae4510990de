"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per
kernel launches, total time and share of the captured window."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.OrderedDict()
    for r in data:
        short = r[ik].split("(")[0].replace("void ", "")
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':64s} {'launches':>8s} {'total_us':>11s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:64]:64s} {n:8d} {t:11.1f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
