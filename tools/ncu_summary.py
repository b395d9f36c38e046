"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: count, total,
mean, share.  Usage: python tools/ncu_summary.py launches.csv [--skip N]"""
import csv
import re
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("<unnamed>::", "")
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        rows.append((name, ns))
    rows = rows[skip:]
    agg = OrderedDict()
    for name, ns in rows:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {tot / 1e6:.3f} ms total (serialised, cold-cache ncu timing)")
    print(f"{'kernel':<28} {'count':>6} {'total ms':>10} {'mean us':>9} {'share':>7}")
    for name, (cnt, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:<28} {cnt:>6} {ns / 1e6:>10.3f} {ns / cnt / 1e3:>9.2f} {ns / tot:>7.1%}")


if __name__ == "__main__":
    main()
