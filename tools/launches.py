"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name.
Usage: python tools/launches.py launches.csv [--last-frac 0.5]"""
import collections
import csv
import sys


def load(path):
    rows, hdr = [], None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
                rows.append((d["Kernel Name"], v))
    return rows


def main():
    rows = load(sys.argv[1])
    frac = float(sys.argv[sys.argv.index("--last-frac") + 1]) if "--last-frac" in sys.argv else 1.0
    rows = rows[int(len(rows) * (1 - frac)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in rows:
        k = k.split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {tot / 1e3:.2f} ms total (serialised, cold-cache ncu times)")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  n={n:5d}  avg {t / n:9.1f} us  {k}")


if __name__ == "__main__":
    main()
