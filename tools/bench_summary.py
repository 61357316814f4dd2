#!/usr/bin/env python
"""Print the key fields of a bench.py JSON line (measurement helper)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
for k in ["value", "ms_per_step", "e2e", "gpu_launches", "clocks", "cpu_baseline"]:
    print(k, d.get(k))
r = dict(d.get("roofline") or {})
for k in ("traffic_capture", "note", "share_note"):
    r.pop(k, None)
print("roofline", r)
for k, v in (d.get("rooflines") or {}).items():
    print(f"  {k:13s} {v['achieved']:9.2f} {v['unit']:8s} frac {v['frac']:.3f} share {v['share_of_step']:.3f} "
          f"launches {v['launches_per_solve']} avg_us {v['avg_launch_us']:.1f} traffic/alg "
          f"{(v.get('traffic') or 0) / max(v['algorithmic_bytes_per_launch'], 1):.2f}")
print("roofline_mgs", d.get("roofline_mgs"))
s = d["solve"]
print({k: s[k] for k in s if k not in ("launch_families", "profiled_family_ms")})
pf = s.get("profiled_family_ms") or {}
print("profiled ms:", sorted(pf.items(), key=lambda x: -x[1]), "sum", round(sum(pf.values()), 1))
for k, v in d.get("configs", {}).items():
    print(k, {kk: v.get(kk) for kk in ["s_per_solve", "eigenpairs_per_s", "iterations", "max_rel_eig_err_vs_reference",
                                        "max_residual", "error", "host_small_s"]})
