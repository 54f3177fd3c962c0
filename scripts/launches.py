"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys


def summarize(path):
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(d["Metric Unit"], 1)
        name = d["Kernel Name"].split("(")[0].replace("gmk::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:6d} {t / 1e6:10.3f} ms {100 * t / tot:5.1f}%  avg {t / n / 1e3:9.1f} us  {k}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        summarize(p)
