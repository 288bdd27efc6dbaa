"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel
count, total and mean time, share of the listed device time."""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name.replace("void ", ""))
    return name


def main(path, skip_before=None):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        k = short(r[ik])
        t = float(r[iv].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
        tot += t
    print(f"{'kernel':60s} {'launches':>9s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:9d} {t / 1e6:10.2f} {t / n / 1e3:10.1f} {t / tot * 100:6.1f}%")
    print(f"total listed device time {tot / 1e6:.1f} ms over {sum(a[0] for a in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
