#!/usr/bin/env python
"""Benchmark of the FoF-connectivity correction hot path (arXiv 2604.18801) on B200.

A step = one pass of the whole hot path over the workload's synthetic
input, resident in HBM: cell binning, vulnerable-pair search + link compare, editable CSR, PGD
to the stop, corrected output, FoF labels of original and corrected positions, MCC and halo
catalogues.  Metric (BASELINE.json): corrected Mparticles/s = N / device time per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

--impl reference runs the CPU oracle (oracle/, single-threaded C) on a bounded sample of the
same workload (the task's reference arm for this tier).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "corrected Mparticles/s (device-timed, 1/2/4/8 B200) and % HBM roofline; MCC=1"
UNIT = "Mparticles/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
def oracle_sample(w: synth.Workload, n_sample: int):
    """The workload's recipe at n_sample particles and the SAME number density, linking length
    and absolute bound (a bounded sample of the workload for the single-threaded oracle)."""
    L_s = w.L * (n_sample / w.n) ** (1.0 / 3.0)
    ws = synth.Workload(w.name + "-sample", w.kind, n_sample, L_s, w.xi / L_s, b=w.linking_length, seed=w.seed,
                        extra=w.extra)
    return ws


def run_oracle(ws: synth.Workload):
    import oracle
    arrs = [t.numpy() for t in synth.make(ws)]
    c = oracle.cfg(L=ws.L, b=ws.linking_length, xi=ws.xi)
    t0 = time.perf_counter()
    r = oracle.pipeline(*arrs, c)
    dt = time.perf_counter() - t0
    return dt, r


def cpu_baseline(w: synth.Workload, target_s: float = 15.0, n_sample=None):
    """Oracle on the host cores (1 thread), a sample sized to ~target_s of CPU work."""
    n0 = n_sample or 200_000
    ws = oracle_sample(w, n0)
    dt, r = run_oracle(ws)
    if n_sample is None and dt < target_s / 3:
        n1 = int(min(n0 * target_s / max(dt, 1e-3), 4_000_000))
        ws = oracle_sample(w, n1)
        dt, r = run_oracle(ws)
    return {"value": ws.n / dt / 1e6, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{w.name} recipe at N={ws.n} (box {ws.L:.3f}, same density, b, xi): full S1-S7 oracle run "
                      f"{dt:.2f} s, {r.info['iterations']} iterations, |V|={len(r.pairs[0])}",
            "seconds": dt, "n": ws.n, "iterations": r.info["iterations"]}


# ------------------------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--xi-rel", type=float, default=None)
    ap.add_argument("--n", type=int, default=None, help="override N (same density recipe)")
    ap.add_argument("--cells-per-particle", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sample-n", type=int, default=None)
    args = ap.parse_args()

    rank, world, local = dist_env()
    w0 = synth.CONFIGS[args.config]
    w = w0
    if args.xi_rel is not None or args.n is not None:
        n = args.n or w0.n
        L = w0.L * (n / w0.n) ** (1.0 / 3.0) if args.n else w0.L
        w = synth.Workload(w0.name, w0.kind, n, L, args.xi_rel if args.xi_rel is not None else w0.xi_rel,
                           eta=w0.eta, b=w0.linking_length if args.n else w0.b, seed=w0.seed, extra=w0.extra)

    if args.impl == "reference":
        if rank != 0:
            return 0
        steps = []
        for k in range(args.warmup + args.steps):
            r = cpu_baseline(w, target_s=8.0, n_sample=args.sample_n or 300_000)
            if k >= args.warmup:
                steps.append(r)
        v = statistics.mean(s["value"] for s in steps)
        ms = statistics.mean(s["seconds"] for s in steps) * 1e3
        cb = dict(steps[-1])
        cb["value"] = v
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": w.name, **w.describe(), "sample": cb["sample"]},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "gpu_launches": 0}
        print(json.dumps(line), flush=True)
        return 0

    import paper_2604_18801_b200 as cc

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)

    # inputs resident in HBM (drawn on the GPU; same recipe as the parity tests)
    x, y, z, xh, yh, zh = synth.make(w, device=dev)
    torch.cuda.synchronize(dev)
    n = w.n
    params = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, profile=1)
    if args.cells_per_particle:
        params.cells_per_particle = args.cells_per_particle
    c = cc.Corrector(params, device=local, stream=stream)
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)]
    lab_o = torch.empty(n, dtype=torch.int32, device=dev)
    lab_c = torch.empty(n, dtype=torch.int32, device=dev)

    def step():
        c.build_cells(x, y, z, xh, yh, zh)
        vp = c.find_vulnerable()
        _, info = c.correct(out)
        _, ng_o = c.fof_label(cc.CC_ORIG, lab_o)
        h_o = c.halo_sizes(cc.CC_ORIG, 20)
        _, ng_c = c.fof_label(cc.CC_CORR, lab_c)
        h_c = c.halo_sizes(cc.CC_CORR, 20)
        m = c.mcc(cc.CC_CORR)
        return vp, info, m, ng_o, ng_c, h_o, h_c

    for _ in range(args.warmup):
        res = step()
    c.kernel_stats(reset=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local)
    clk.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        res = step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    ms_total = ev0.elapsed_time(ev1)
    clocks = clk.stop()
    stats = c.kernel_stats(reset=True)
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    vp, info, m, ng_o, ng_c, h_o, h_c = res
    value = world * n / (ms_step * 1e-3) / 1e6

    # ---- roofline of the dominant kernel class (device time inside the timed region)
    hbm, sm_max, peak_src = _peaks()
    launches = stats.pop("total_launches", (0.0, 0))[1]
    E, nent = vp["n_editable"], 2 * vp["n_pairs"]
    cls_ms = {k: v for k, v in stats.items()}
    dom = max(cls_ms, key=lambda k: cls_ms[k][0]) if cls_ms else None
    # algorithmic bytes per launch
    alg_bytes = {
        "K3_pgd": 104.0 * E + 4.0 * nent,
        "K1_key": 24.0 * n + 8.0 * n,
        "K1_scatter": (24 + 8 + 4) * n + 36.0 * n,
        "K2_count": 16.0 * n + 4.0 * n,
        "K2_fill": 16.0 * n + 4.0 * n + 8.0 * n + 4.0 * nent,
        "K4_fof": 16.0 * n + 4 * 4.0 * n,
    }
    roof = None
    if dom:
        d_ms, d_l = cls_ms[dom]
        avg_ms = d_ms / max(d_l, 1)
        if dom in alg_bytes:
            ach = alg_bytes[dom] / (avg_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "traffic": None, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                    "launch_ms": avg_ms, "launches": d_l}
        else:
            roof = {"bound": "hbm", "kernel": dom, "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                    "traffic": None, "launch_ms": avg_ms, "launches": d_l}
    k3 = cls_ms.get("K3_pgd")
    k3_roof = None
    if k3 and k3[1]:
        a = alg_bytes["K3_pgd"] / (k3[0] / k3[1] * 1e-3) / 1e9
        k3_roof = {"achieved_gbs": a, "frac": a / hbm, "launch_ms": k3[0] / k3[1], "launches": k3[1]}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak" if world > 1 else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded generator, drawn on the GPU)",
        "config": {**w.describe(), "workload": w.name, "parallelism": "replicas" if world > 1 else "1 GPU",
                   "l2": "inputs (6 x 4N B) larger than the 126 MB L2", "stop": "no L_tight-active pair (R11)",
                   "cells_per_axis": vp["cells_per_axis"]},
        "result": {"n_pairs": vp["n_pairs"], "n_editable": E, "violated0": vp["n_violated0"],
                   "iterations": info["iterations"], "converged": info["converged"], "mcc_after": m["mcc"],
                   "fof_groups_orig": ng_o, "fof_groups_corr": ng_c, "halos_equal": bool(np.array_equal(h_o, h_c))},
        "roofline": roof, "k3_roofline": k3_roof,
        "kernels_ms_per_step": {k: v[0] / args.steps for k, v in cls_ms.items()},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }

    # ---- end to end through the public API with HOST buffers (pinned), copies inside
    if not args.no_e2e:
        host = [t.cpu().pin_memory() for t in (x, y, z, xh, yh, zh)]
        hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(3)]

        def e2e_step():
            r = c.run(*host, out=hout, host=True)
            c.fof_label(cc.CC_ORIG, lab_o)
            c.fof_label(cc.CC_CORR, lab_c)
            mm = c.mcc(cc.CC_CORR)
            return r, mm

        e2e_step()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(max(1, min(args.steps, 3))):
            e2e_step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = ev0.elapsed_time(ev1) / max(1, min(args.steps, 3))
        line["e2e"] = {"value": world * n / (e_ms * 1e-3) / 1e6, "unit": UNIT, "ms_per_step": e_ms,
                       "h2d_bytes_per_step": 24 * n, "d2h_bytes_per_step": 12 * n + 48}
        del host, hout
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = {k: v for k, v in cpu_baseline(w).items() if k in
                                ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
