"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count and total/avg time, in launch order of first use."""
import csv
import sys
from collections import OrderedDict


def load(path, skip_prefix=("k_seed", "k_gen")):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000 if unit == "ns" else v if unit == "us" else v * 1000 if unit == "ms" else v
        rows.append((name, us))
    return rows


def main():
    for path in sys.argv[1:]:
        rows = load(path)
        agg = OrderedDict()
        for n, us in rows:
            a = agg.setdefault(n, [0, 0.0])
            a[0] += 1
            a[1] += us
        tot = sum(us for _, us in rows)
        print(f"== {path}: {len(rows)} launches, {tot:.1f} us total")
        for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
            print(f"  {us:9.1f} us  {c:4d}x  {n}")


if __name__ == "__main__":
    main()
