#!/usr/bin/env python
"""Summarise an ncu launch list with DRAM traffic per kernel:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv ...
  python tools/launch_list_dram.py launches.csv [--title ...] [--traffic-json out.json --workload config3]

The per-launch DRAM bytes of the k_gram<64,64> / k_product<64,64> / stencil launches are what
bench.py reports as roofline.traffic (profiles/roofline_traffic.json).
"""
import argparse
import collections
import csv
import io
import json

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
        "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
FAMILY = {"k_gram<64, 64": "gram_wide", "k_product<64, 64": "product_wide", "k_stencil2<4, 1": "spmm_cg",
          "k_cols<unnamed>::CgDirXF": "cg_vec", "k_colred<1, unnamed>::CgXrF": "cg_vec"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--title", default="")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--traffic-json")
    ap.add_argument("--workload", default="config3")
    a = ap.parse_args()
    text = open(a.csv, errors="replace").read()
    rows = list(csv.DictReader(io.StringIO(text[text.find('"ID"'):])))
    per = collections.defaultdict(dict)
    for r in rows:
        per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for (_, name), m in per.items():
        g = agg[name]
        g[0] += m.get("gpu__time_duration.sum", 0.0)
        g[1] += 1
        g[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(v[0] for v in agg.values())
    if a.title:
        print(f"# {a.title}")
    print(f"# {sum(v[1] for v in agg.values())} launches, total kernel time {total / 1e3:.2f} ms "
          f"(ncu, serialised, --clock-control none); DRAM = dram__bytes_read + dram__bytes_write")
    print(f"{'ms':>9s} {'share':>6s} {'launches':>8s} {'avg_us':>9s} {'DRAM/launch MB':>15s} {'DRAM GB/s':>10s}  kernel")
    for name, (us, cnt, b) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"{us / 1e3:9.2f} {100 * us / total:5.1f}% {cnt:8d} {us / cnt:9.1f} {b / cnt / 1e6:15.1f} "
              f"{b / (us * 1e-6) / 1e9 if us else 0:10.0f}  {name[:90]}")
    if a.traffic_json:
        out = {}
        try:
            out = json.load(open(a.traffic_json))
        except Exception:
            pass
        w = out.setdefault(a.workload, {})
        for name, (us, cnt, b) in agg.items():
            for key, fam in FAMILY.items():
                if key in name and fam not in ("cg_vec",):
                    w[fam] = {"kernel": name[:120], "dram_bytes_per_launch": b / cnt, "launches": cnt,
                              "avg_us": us / cnt, "capture": a.csv.split("/")[-1]}
        json.dump(out, open(a.traffic_json, "w"), indent=1)


if __name__ == "__main__":
    main()
