"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes) per kernel template."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    return per, names


def main(path, min_us=20.0):
    per, names = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0])
    for i, m in per.items():
        n = names[i]
        n = n[:n.find(">(") + 1] if ">(" in n else n.split("(")[0]
        t = m.get("gpu__time_duration.sum", 0.0)
        a = agg[n]
        a[1] += t
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        if t >= min_us * 1e3:
            a[0] += 1
        else:
            a[3] += 1
    tot = sum(a[1] for a in agg.values())
    print(f"{'full':>4} {'gated':>5} {'ms':>9} {'share':>6} {'us/full':>8} {'GB/s':>7}  kernel")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        us = a[1] / 1e3 / max(a[0], 1)
        print(f"{a[0]:4d} {a[3]:5d} {a[1] / 1e6:9.3f} {100 * a[1] / tot:5.1f}% {us:8.1f} "
              f"{a[2] / max(a[1], 1):7.0f}  {n}")
    print(f"total {tot / 1e6:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 20.0)
