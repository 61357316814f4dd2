#!/usr/bin/env python
"""Benchmark: BOSP LREP solve on B200 -- converged eigenpairs/s (BASELINE.json metric).

Workload (N=1): BASELINE configs[1] = config 2, the 64^3 sparse LREP (n = 262,144, fp64 CSR,
nev = 20, nb = 40 -> 20, tol 1e-8), explicit generalized nullspace (constants).  One "step" =
one full bosp::solve (initialize + outer iterations + assemble_result) on the device.

Arms:
  default            the B200 library (libbosp_b200.so) through its C ABI.
  --impl reference   the UNMODIFIED reference CPU solver (oracle/_ref/libbosp_ref.so, built from
                     /root/reference/proj/src) on the box's host cores: each step is a bounded
                     sample (initialize + a few iterate_once) extrapolated to a full solve with the
                     reference's own iteration count for this config.

JSON line keys follow the driver contract (metric/value/unit/n_gpus/steps/warmup/ms_per_step/
higher_is_better/scaling/vs_baseline/dtype/data/config) plus roofline, cpu_baseline, e2e,
gpu_launches and clocks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "converged eigenpairs/s (LREP solve, config 2: 64^3 CSR, nev=20)"
UNIT = "eigenpairs/s"
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_solves.json")


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # diagnostics only
            return self
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "500"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return world, rank, local, dist


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reference_iterations() -> int:
    try:
        return int(json.load(open(GOLDEN))["config2"]["iterations"])
    except Exception:
        return 78


def cpu_reference_sample(prob, iters: int, threads: int):
    """Reference solver (oracle/_ref) on a bounded sample: initialize + `iters` iterate_once."""
    from oracle import ref
    ref.set_threads(threads)
    out = ref.time_iterations(prob.oracle_spec("K"), prob.oracle_spec("M"), ref.RefConfig(**prob.cfg),
                              (prob.x0, prob.y0), iters)
    full_iters = reference_iterations()
    t_iter = out["t_iters"] / max(1, out["iters"])
    est = out["t_init"] + full_iters * t_iter
    return dict(est_solve_s=est, t_init=out["t_init"], t_iter=t_iter, iters=out["iters"],
                full_iters=full_iters, threads=ref.threads())


def run_reference(args, world, rank, dist):
    if rank != 0:
        return
    from paper_2506_08355_b200 import problems as P
    prob = P.config2(64)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_sample(prob, 1, threads)
    samples = [cpu_reference_sample(prob, args.ref_iters, threads) for _ in range(args.steps)]
    est = statistics.median(s["est_solve_s"] for s in samples)
    value = prob.cfg["nev"] / est
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_2506_08355_b200/problems.py)",
        "config": {"workload": prob.name, "n": prob.n, "nev": 20, "nb": 40, "tol": 1e-8,
                   "parallelism": "host OpenMP (reference kernels), serial CSR matvec"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": samples[0]["threads"], "kind": "reference",
                         "sample": (f"initialize + {args.ref_iters} iterate_once per step (public API), "
                                    f"solve time = t_init + {samples[0]['full_iters']} x t_iter "
                                    f"(the reference's own iteration count on this config); "
                                    f"t_init={samples[0]['t_init']:.2f}s t_iter={samples[0]['t_iter']:.2f}s")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def dmma_roofline():
    """The dense contractions of configs 3/5 (d = 320) on the fp64 tensor pipe: Rayleigh-Ritz
    Gram U^T (K U) (n x 320)^T (n x 320) and Ritz pullback (n x 320)(320 x 192) at n = 128^3,
    device-resident random data, against cuBLAS DGEMM 8192^3 measured in the same process."""
    import torch
    from paper_2506_08355_b200 import bosp
    n, d, w = 128 ** 3, 320, 192
    out = {"bound": "tensor (fp64 DMMA)", "unit": "TFLOP/s", "n": n}
    g_ms = bosp.bench_blas("gram", n, d, d, reps=10)
    p_ms = bosp.bench_blas("product", n, d, w, reps=10)
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    peak = 2 * 8192 ** 3 * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    del a, b
    torch.cuda.empty_cache()
    # MGS-Biorth at HBM scale (m = 20 at n = 2^21, X, Y, P, Q far beyond L2): the pair Gram of
    # [X | Y] + the fused apply/check kernel, against 48 n m algorithmic bytes
    m = 20
    mg_ms = bosp.bench_blas("gramsym", n, m, m, reps=10)
    ma_ms = bosp.bench_blas("mgsapply", n, m, m, reps=10)
    hbm = load_peaks().get("hbm_gbs", 6650.0)
    mgs_gbs = 48.0 * n * m / ((mg_ms + ma_ms) * 1e-3) / 1e9
    out["mgs_at_hbm_scale"] = {"n": n, "m": m, "pair_gram_ms": mg_ms, "apply_check_ms": ma_ms,
                               "achieved_gbs": mgs_gbs, "frac_hbm": mgs_gbs / hbm,
                               "note": "kernel time only (no host recurrence between the two launches)"}
    gt = 2 * n * d * d / (g_ms * 1e-3) / 1e12
    pt = 2 * n * d * w / (p_ms * 1e-3) / 1e12
    out.update({"kernel": "k_gram<64,64> (G = A^T B, 320 x 320)", "achieved": gt, "peak": peak, "frac": gt / peak,
                "gram_ms": g_ms, "product_kernel": "k_product<64,64> (A C, 320 -> 192)", "product_achieved": pt,
                "product_frac": pt / peak, "product_ms": p_ms,
                "peak_source": "cuBLAS DGEMM 8192^3 (torch.matmul fp64), best-effort same-process measurement"})
    return out


def run_b200(args, world, rank, local, dist):
    from paper_2506_08355_b200 import _lib, bosp
    from paper_2506_08355_b200 import dist as D
    from paper_2506_08355_b200 import problems as P
    _lib.lib().bosp_set_device(local)
    name, sms = bosp.device_info()
    prob = P.config2(64)
    cfg = bosp.BospConfig(**prob.cfg)
    partitioned = world > 1 and args.partition == "rows"
    partition_error = None
    if partitioned:
        # one process per GPU, rows of every n-length block on this rank; NCCL communicator
        # inside libbosp_b200.so (torch.distributed only carries the unique id + timings).
        # The ranks agree on success after one partitioned solve; if any rank failed, every
        # rank falls back to replicas and the line records why.
        ok = 1
        try:
            uid = D.broadcast_uid()
            row0, nl = D.attach(prob.K, uid, world, rank)
            ns = D.local_nullspace(prob.x0, prob.y0, row0, nl)
            K, M = bosp.local_operator(prob.K, world, rank), bosp.local_operator(prob.M, world, rank)
            bosp.solve(K, M, None, cfg, ns, want_vectors=True)
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line
            ok, partition_error = 0, f"{type(e).__name__}: {e}"[:300]
        import torch
        flag = torch.tensor([ok], dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            try:
                bosp.comm_free()
            except Exception:
                pass
            partitioned = False
            partition_error = partition_error or "another rank failed the partitioned setup"
    if not partitioned:
        row0, nl = 0, prob.n
        ns = bosp.GeneralizedNullspace(prob.x0, prob.y0)
        K, M = bosp.operators_for(prob)   # resident in HBM before the timed region
    flush = 512 << 20                  # 512 MB > 126 MB L2, written between steps
    units = 1 if partitioned else world  # one shared problem vs. one replica per rank

    def one_step(profile_family=None):
        profile_family = profile_family or None
        _lib.lib().bosp_flush_l2(flush)
        if profile_family:
            bosp.profile_enable(profile_family)
        r = bosp.solve(K, M, None, cfg, ns, want_vectors=True)
        prof = bosp.profile_collect() if profile_family else None
        if profile_family:
            bosp.profile_enable(None)
        return r, prof

    for _ in range(args.warmup):  # same configuration as the timed steps (graphs recorded here)
        one_step(args.roofline_kernel)
    barrier(dist)
    bosp.device_sync()
    bosp.launch_reset()
    dev_s, wall_s, iters, profs = [], [], [], []
    res = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            res, prof = one_step(args.roofline_kernel)
            dev_s.append(res.stats["device_seconds"])
            wall_s.append(res.stats["wall_seconds"])
            iters.append(res.iterations)
            profs.append(prof)
    bosp.device_sync()
    barrier(dist)
    launches = bosp.launch_count()
    families = bosp.launch_families()
    total = max_over_ranks(dist, float(sum(dev_s)))
    ms_per_step = total / args.steps * 1e3
    value = prob.cfg["nev"] * args.steps * units / total

    # parity of the measured run against the reference's own eigenvalues (golden fixture)
    parity = None
    try:
        g = json.load(open(GOLDEN))["config2"]["lambdas"]
        parity = float(np.max(np.abs(res.lambdas - np.array(g)) / np.array(g)))
    except Exception:
        pass

    # e2e: public API with host buffers -- operator construction from pinned host CSR, the solve,
    # results back to host; all inside the timed region.
    kc, mc = prob.K, prob.M
    host = {}
    for tag, c in (("k", kc), ("m", mc)):
        rp = c.rowptr[row0:row0 + nl + 1]
        host[tag] = (np.ascontiguousarray(rp), np.ascontiguousarray(c.colidx[rp[0]:rp[-1]]),
                     np.ascontiguousarray(c.vals[rp[0]:rp[-1]]))
    h2d = sum(a.nbytes for t in host.values() for a in t) + ns.x0.nbytes + ns.y0.nbytes
    d2h = 2 * nl * prob.cfg["nev"] * 8 + 2 * prob.cfg["nev"] * 8
    e2e_t = []
    for _ in range(max(1, args.steps)):
        _lib.lib().bosp_flush_l2(flush)
        barrier(dist)
        t0 = time.perf_counter()
        if partitioned:
            Ke = bosp.LinearOperator.from_csr_rows(prob.n, row0, *host["k"])
            Me = bosp.LinearOperator.from_csr_rows(prob.n, row0, *host["m"])
        else:
            Ke = bosp.LinearOperator.from_csr(*host["k"])
            Me = bosp.LinearOperator.from_csr(*host["m"])
        r2 = bosp.solve(Ke, Me, None, cfg, ns, want_vectors=True)
        _ = float(r2.lambdas.sum())
        e2e_t.append(time.perf_counter() - t0)
        del Ke, Me
    e2e_total = max_over_ranks(dist, float(sum(e2e_t)))
    e2e_value = prob.cfg["nev"] * len(e2e_t) * units / e2e_total
    if partitioned:
        bosp.comm_free()

    # roofline of the dominant kernel family (CUDA events on the solver stream, timed region)
    peaks = load_peaks()
    roof = None
    pr = [p for p in profs if p]
    if pr:
        launches_k = sum(p["launches"] for p in pr)
        ms_k = sum(p["ms"] for p in pr)
        bytes_k = sum(p["bytes"] for p in pr)
        if launches_k and ms_k > 0:
            achieved = bytes_k / (ms_k * 1e-3) / 1e9
            traffic, traffic_note = None, None
            try:  # DRAM bytes per launch of the same kernel from the committed ncu --set full capture
                tr = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
                if args.roofline_kernel in tr.get("kernel", ""):
                    traffic = tr["dram_bytes_per_launch"]
                    traffic_note = {"algorithmic_bytes_per_launch_in_capture": tr["algorithmic_bytes_per_launch"],
                                    "source": tr["capture"]}
            except Exception:
                pass
            roof = {"kernel": args.roofline_kernel, "bound": "hbm", "achieved": achieved,
                    "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                    "frac": achieved / peaks.get("hbm_gbs", 6650.0), "traffic": traffic,
                    "traffic_capture": traffic_note,
                    "launches_per_step": launches_k / len(pr),
                    "avg_launch_us": ms_k * 1e3 / launches_k,
                    "algorithmic_bytes_per_launch": bytes_k / launches_k,
                    "share_of_step": ms_k / (sum(dev_s) * 1e3),
                    "bytes_note": "CSR-equivalent algorithmic bytes (SURVEY 8d: 12 nnz + 4(n+1) + 16 n m_active); "
                                  "the DIA form stored for config 2 moves 16 n m + 10 n, see DESIGN.md section 6",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "_fallback" not in peaks
                    else "fallback 6650 GB/s (B200_PROFILING.md)"}

    # MGS-Biorth as a unit (biorth.cpp:102-109): one extra profiled solve (outside the timed
    # region) in which every launch issued inside an MGS-Biorth call is timed on the device.
    roof_mgs = None
    if not args.no_kernel_rooflines:
        _lib.lib().bosp_flush_l2(flush)
        _, pm = one_step("mgs")
        if pm and pm["launches"] and pm["ms"] > 0:
            hbm = peaks.get("hbm_gbs", 6650.0)
            ach = pm["region_bytes"] / (pm["ms"] * 1e-3) / 1e9
            roof_mgs = {"kernel": "mgs_biorth (Gram + coefficient product + P^T Q check kernels)",
                        "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                        "calls_per_solve": pm["region_calls"], "launches_per_solve": pm["launches"],
                        "avg_call_us": pm["ms"] * 1e3 / max(1, pm["region_calls"]),
                        "algorithmic_bytes_per_call": pm["region_bytes"] / max(1, pm["region_calls"]),
                        "kernel_operand_gbs": pm["bytes"] / (pm["ms"] * 1e-3) / 1e9,
                        "share_of_step": pm["ms"] / (ms_per_step),
                        "bytes_note": "48 n m per call (SURVEY 8d: X, Y read + P, Q written = 32 n m, + 16 n m "
                                      "for the P^T Q Gram of the second-pass test); kernel_operand_gbs counts "
                                      "every operand each kernel reads/writes (the Gram re-reads X, Y)"}
    roof_dmma = None
    if rank == 0 and not args.no_kernel_rooflines:
        roof_dmma = dmma_roofline()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            s = cpu_reference_sample(prob, args.ref_iters, os.cpu_count() or 1)
            cpu = {"value": prob.cfg["nev"] / s["est_solve_s"], "unit": UNIT, "cores": s["threads"],
                   "kind": "reference",
                   "sample": (f"oracle/_ref (unmodified reference) initialize + {s['iters']} iterate_once on "
                              f"config 2; solve = t_init + {s['full_iters']} x t_iter "
                              f"(t_init={s['t_init']:.2f}s, t_iter={s['t_iter']:.2f}s)")}
        except Exception as e:  # the checker is optional on a box without oracle/_ref
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, paper_2506_08355_b200/problems.py; no dataset)",
            "config": {"workload": prob.name, "n": prob.n, "nnz_K": kc.nnz, "nev": 20, "nb": 40,
                       "tol": 1e-8,
                       "parallelism": (f"row partition x{world} (NCCL allreduce + halo)" if partitioned
                                       else "replicas" if world > 1 else "single GPU"),
                       **({"partition_error": partition_error} if partition_error else {}),
                       "l2": "flushed between steps (512 MB memset)", "device": name, "sms": sms},
            "roofline": roof,
            "roofline_mgs": roof_mgs,
            "roofline_dmma": roof_dmma,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps_s": [round(t, 4) for t in e2e_t]},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "solve": {"iterations": iters, "device_s": dev_s, "wall_s": wall_s,
                      "host_small_s": res.stats["host_small_seconds"], "repairs": res.stats["repairs"],
                      "cg_iterations": res.stats["cg_iterations"],
                      "max_rel_eig_err_vs_reference": parity,
                      "max_residual": float(res.residuals.max()),
                      "final_biorth_deviation": res.stats["final_biorth_deviation"],
                      "launch_families": families},
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--roofline-kernel", default="spmm_cg",
                    help="kernel family timed for the roofline (default: the dominant one, the CG SpMM)")
    ap.add_argument("--ref-iters", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernel-rooflines", action="store_true",
                    help="skip the MGS-Biorth and fp64-DMMA kernel rooflines (extra, untimed work)")
    ap.add_argument("--partition", default="rows", choices=["rows", "replicas"],
                    help="N>1: row-partition one solve over the ranks (NCCL) or run N replicas")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank, dist)
    else:
        run_b200(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
