#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv <cmd>
  python tools/launch_list.py launches.csv [--title "..."] > profiles/<name>.txt
"""
import argparse
import collections
import csv
import io


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--title", default="")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    text = open(a.csv, errors="replace").read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
        name = r["Kernel Name"]
        agg[name][0] += us
        agg[name][1] += 1
    total = sum(v[0] for v in agg.values())
    n = sum(v[1] for v in agg.values())
    if a.title:
        print(f"# {a.title}")
    print(f"# {n} launches, total kernel time {total / 1e3:.2f} ms (ncu, serialised, --clock-control none)")
    print(f"{'ms':>9s} {'share':>6s} {'launches':>8s} {'avg_us':>9s}  kernel")
    for name, (us, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"{us / 1e3:9.2f} {100 * us / total:5.1f}% {cnt:8d} {us / cnt:9.2f}  {name[:90]}")


if __name__ == "__main__":
    main()
