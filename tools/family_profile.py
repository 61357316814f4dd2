#!/usr/bin/env python
"""Per-family device time of one full solve (every launch timed: CUDA events, device-clock slots
inside the CG graphs) -- where a config's time goes.

  python tools/family_profile.py config5
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2506_08355_b200 import bosp
    from paper_2506_08355_b200 import problems as P
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    from run_config import make
    name = sys.argv[1] if len(sys.argv) > 1 else "config5"
    prob = make(name, bosp, P)
    K, M = bosp.operators_for(prob)
    cfg = bosp.BospConfig(**prob.cfg)
    ns = bosp.GeneralizedNullspace(prob.x0, prob.y0)
    r0 = bosp.solve(K, M, None, cfg, ns, want_vectors=False)  # warm: graphs, pools
    bosp.profile_enable("*")
    t = time.perf_counter()
    r = bosp.solve(K, M, None, cfg, ns, want_vectors=False)
    wall = time.perf_counter() - t
    rep = bosp.profile_collect()
    bosp.profile_enable(None)
    tot = sum(v["ms"] for v in rep["families"].values())
    print(f"{name}: warm solve {r0.stats['device_seconds']:.3f} s ({r0.iterations} it), profiled {wall:.3f} s wall, "
          f"kernels {tot / 1e3:.3f} s, host small {r.stats['host_small_seconds']:.3f} s, repairs {r.stats['repairs']}")
    for f, v in sorted(rep["families"].items(), key=lambda kv: -kv[1]["ms"]):
        ach = (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["flops"] else 0.0
        bw = (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["bytes"] else 0.0
        print(f"  {f:14s} {v['ms'] / 1e3:8.3f} s {v['launches']:7d} launches  {ach:6.2f} TF/s {bw:8.1f} GB/s")


if __name__ == "__main__":
    main()
