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

# NCCL's version banner goes to stderr: stdout carries exactly one JSON line
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

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


_ORACLE_STOP = [3, 10_000]  # the oracle arms run the bench's stop mode and T_max (set in main)


def run_oracle(ws: synth.Workload, timeout: float = 120.0):
    """The oracle's S1-S7 on a sample, in a child process (so a slow sample cannot hang the
    bench); returns (seconds, iterations, |V|) or None on timeout."""
    cmd = [sys.executable, os.path.abspath(__file__), "--_oracle", json.dumps(
        {"name": ws.name, "kind": ws.kind, "n": ws.n, "L": ws.L, "xi_rel": ws.xi_rel, "b": ws.linking_length,
         "seed": ws.seed, "extra": ws.extra, "stop": _ORACLE_STOP[0], "t_max": _ORACLE_STOP[1]})]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return None
    if r.returncode != 0:
        log("oracle sample failed:", r.stderr[-500:])
        return None
    d = json.loads(r.stdout.strip().splitlines()[-1])
    return d["seconds"], d["iterations"], d["pairs"]


def _oracle_child(spec: str) -> int:
    import oracle
    d = json.loads(spec)
    ws = synth.Workload(d["name"], d["kind"], d["n"], d["L"], d["xi_rel"], b=d["b"], seed=d["seed"],
                        extra=d["extra"])
    arrs = [t.numpy() for t in synth.make(ws)]
    c = oracle.cfg(L=ws.L, b=ws.linking_length, xi=ws.xi, stop_mode=d.get("stop", oracle.STOP_RESTORED),
                   t_max=d.get("t_max", 10_000))
    oracle.build()
    x, y, z, xh, yh, zh = arrs
    t0 = time.perf_counter()
    pairs = oracle.find_pairs(x, y, z, xh, yh, zh, c)            # S1-S3
    xo, yo, zo, info = oracle.correct(x, y, z, xh, yh, zh, pairs, c)  # S4-S5 to the stop
    t1 = time.perf_counter()
    oracle.fof(x, y, z, c)                                        # S6 + S7 (the check)
    oracle.fof(xo, yo, zo, c)
    oracle.mcc_counts((pairs[2] & 1).astype(bool), oracle.pair_links(pairs[0], pairs[1], xo, yo, zo, c))
    t2 = time.perf_counter()
    print(json.dumps({"seconds": t1 - t0, "seconds_incl_check": t2 - t0, "iterations": info["iterations"],
                      "pairs": int(len(pairs[0]))}))
    return 0


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def calibrated_sample(w: synth.Workload, target_s: float = 12.0, n_sample=None):
    """The bounded oracle sample of a workload, shared by cpu_baseline and --impl reference (the
    same N in both): start at 50,000 particles of the same recipe and
    density, then scale N so the oracle's S1-S5 takes ~target_s (at most 4M particles).
    Returns (sample workload, its first timing) or (sample, None) on timeout."""
    if n_sample is None and (w.kind != "clumped" or w.n <= 4_000_000):
        # the lattice / crystal recipes do not rescale, and C1-C3 are small: the oracle runs the
        # workload itself (the same N as the GPU)
        return w, run_oracle(w, timeout=600)
    n0 = n_sample or 50_000
    ws = oracle_sample(w, n0)
    r = run_oracle(ws, timeout=6 * target_s)
    if n_sample is None and r is not None and r[0] < target_s / 3:
        n1 = int(min(n0 * target_s / max(r[0], 1e-3), 4_000_000))
        ws1 = oracle_sample(w, n1)
        r1 = run_oracle(ws1, timeout=6 * target_s)
        if r1 is not None:
            ws, r = ws1, r1
    return ws, r


def cpu_baseline(w: synth.Workload, target_s: float = 12.0, n_sample=None):
    """Oracle on the host cores (1 thread) on the calibrated sample."""
    ws, r = calibrated_sample(w, target_s, n_sample)
    if r is None:
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"{w.name} recipe at N={ws.n}: oracle did not finish within {6 * target_s:.0f} s"}
    dt, iters, npairs = r
    return {"value": ws.n / dt / 1e6, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{w.name} recipe at N={ws.n} (box {ws.L:.3f}, same density, b, xi): oracle S1-S5 to the stop "
                      f"{dt:.2f} s (the metric's t; the S6-S7 check excluded), {iters} iterations, |V|={npairs}; "
                      f"1 thread of {os.cpu_count()} on {cpu_model()}",
            "seconds": dt, "n": ws.n, "iterations": iters}


def log(*a):
    print(f"[bench {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _workload(args):
    w0 = synth.CONFIGS[args.config]
    if args.xi_rel is None and args.n is None:
        return w0
    n = args.n or w0.n
    L = w0.L * (n / w0.n) ** (1.0 / 3.0) if args.n else w0.L
    return synth.Workload(w0.name, w0.kind, n, L, args.xi_rel if args.xi_rel is not None else w0.xi_rel, eta=w0.eta,
                          b=w0.linking_length if args.n else w0.b, seed=w0.seed, extra=w0.extra)


def reference_arm(args, w, rank):
    """--impl reference: the CPU oracle as it stands, a bounded sample of the workload per step."""
    if rank != 0:
        return 0
    ws, _ = calibrated_sample(w, n_sample=args.sample_n)  # the same sample N as cpu_baseline
    n_s = ws.n
    times, last = [], None
    for k in range(args.warmup + args.steps):
        r = run_oracle(ws, timeout=300)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": f"oracle sample N={n_s} exceeded 300 s"}), file=_OUT,
                  flush=True)
            return 0
        if k >= args.warmup:
            times.append(r[0])
        last = r
    dt = statistics.mean(times)
    v = ws.n / dt / 1e6
    sample = (f"{w.name} recipe at N={ws.n} (box {ws.L:.3f}, same density, b, xi), single-threaded C oracle, "
              f"S1-S5 to the stop timed (the metric's t; S6-S7 check excluded), {last[1]} iterations, |V|={last[2]}; "
              f"1 thread of {os.cpu_count()} on {cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**w.describe(), "workload": w.name, "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), file=_OUT, flush=True)
    return 0


_OUT = sys.stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--xi-rel", type=float, default=None)
    ap.add_argument("--n", type=int, default=None, help="override N (same density recipe)")
    ap.add_argument("--t-max", type=int, default=10000)
    ap.add_argument("--stop", default="restored", choices=["restored", "active", "eps", "none"],
                    help="Alg. 1 stop (R11): restored = L_tight <= 1e-10 and MCC = 1 (default)")
    ap.add_argument("--cells-per-particle", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-edit-log", action="store_true")
    ap.add_argument("--sample-n", type=int, default=None)
    ap.add_argument("--_oracle", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args._oracle:
        return _oracle_child(args._oracle)
    # stdout carries exactly one JSON line: everything else written to fd 1 (NCCL's version
    # banner from inside the libraries included) goes to stderr
    global _OUT
    _OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)

    rank, world, local = dist_env()
    w = _workload(args)
    _ORACLE_STOP[:] = [{"restored": 3, "active": 0, "eps": 1, "none": 2}[args.stop], args.t_max]
    if args.impl == "reference":
        return reference_arm(args, w, rank)

    import paper_2604_18801_b200 as cc

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    log(f"rank {rank}/{world}: drawing {w.name} N={w.n:,} on {dev}")
    x, y, z, xh, yh, zh = synth.make(w, device=dev)
    n_total = w.n
    gid = None
    if world > 1:
        own = (cc.slab_of(x, world, w.L) == rank).nonzero().flatten()
        x, y, z, xh, yh, zh = [a[own].contiguous() for a in (x, y, z, xh, yh, zh)]
        gid = own.to(torch.int32)
        del own
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()  # the generator's fp64 temporaries (C5: ~100 GB) go back to the device
    n = x.shape[0]
    stop = {"restored": cc.STOP_RESTORED, "active": cc.STOP_ACTIVE, "eps": cc.STOP_EPS, "none": cc.STOP_NONE}[args.stop]
    params = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, profile=1, t_max=args.t_max, stop_mode=stop)
    if args.cells_per_particle:
        params.cells_per_particle = args.cells_per_particle
    distarg = None
    if world > 1:
        uid = [cc.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        distarg = (rank, world, uid[0])
    c = cc.Corrector(params, device=local, stream=stream, dist=distarg)
    with torch.cuda.stream(stream):
        out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)]
        lab_o = torch.empty(max(n, 1), dtype=torch.int32, device=dev)[:n]
        lab_c = torch.empty(max(n, 1), dtype=torch.int32, device=dev)[:n]
    # L2 flush buffer (only needed when the inputs fit in the 126 MB L2)
    small = 24 * n < 512 * 2**20
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev) if small else None

    def step(mid=None, ph=None):
        c.build_cells(x, y, z, xh, yh, zh, gid=gid)
        if ph is not None:
            ph[0].record(stream)
        vp = c.find_vulnerable()
        if ph is not None:
            ph[1].record(stream)
        _, info = c.correct(out)
        if mid is not None:  # S1-S5 end here; S6 + S7 (the check) follow
            mid.record(stream)
        _, ng_o = c.fof_label(cc.CC_ORIG, lab_o)
        h_o = c.halo_sizes(cc.CC_ORIG, 20)
        _, ng_c = c.fof_label(cc.CC_CORR, lab_c)
        h_c = c.halo_sizes(cc.CC_CORR, 20)
        m = c.mcc(cc.CC_CORR)
        return vp, info, m, ng_o, ng_c, h_o, h_c

    for k in range(args.warmup):
        t0 = time.perf_counter()
        res = step()
        log(f"warmup {k}: {time.perf_counter() - t0:.3f} s wall, |V|={res[0]['n_pairs']:,} |E|={res[0]['n_editable']:,}"
            f" iterations={res[1]['iterations']} converged={res[1]['converged']} mcc={res[2]['mcc']:.6f}")
    free_b, tot_b = torch.cuda.mem_get_info(dev)
    log(f"device memory in use after warm-up: {(tot_b - free_b) / 2**30:.1f} GiB of {tot_b / 2**30:.1f} GiB "
        f"({(tot_b - free_b) / max(n, 1):.0f} B per local particle)")
    c.kernel_stats(reset=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    phs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local)
    clk.start()
    for k in range(args.steps):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(float(k))
        evs[k][0].record(stream)
        res = step(mids[k], phs[k])
        evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    clocks = clk.stop()
    # the metric's t is S1..S5 to the stop; S6 + S7 (the check) is reported
    # separately and as an "incl. check" total
    ms_total = sum(a.elapsed_time(b) for a, b in evs)
    ms_corr = sum(a[0].elapsed_time(mm) for a, mm in zip(evs, mids))
    stats = c.kernel_stats(reset=True)
    rank_ms = None
    # phases: S1 (cc_build_cells incl. the ghost exchange), S2-S3 (cc_find_vulnerable incl. the
    # refresh lists), S4-S5 (cc_correct incl. the per-iteration exchange); device time per step
    ph1 = sum(a[0].elapsed_time(p[0]) for a, p in zip(evs, phs)) / args.steps
    ph2 = sum(p[0].elapsed_time(p[1]) for p in phs) / args.steps
    ph3 = sum(p[1].elapsed_time(mm) for p, mm in zip(phs, mids)) / args.steps
    phases = {"build_ms": round(ph1, 3), "find_vulnerable_ms": round(ph2, 3), "correct_ms": round(ph3, 3)}
    if world > 1:
        # every rank's own S1-S5 time, profiled-kernel sum and phases (load balance, exchange cost)
        own = torch.tensor([ms_corr / args.steps, sum(v[0] for k, v in stats.items()
                                                      if k != "K4_fof" and not k.startswith("K3_work")
                                                      and k != "total_launches" and not k.endswith("_tests"))
                            / args.steps, ph1, ph2, ph3], device=dev, dtype=torch.float64)
        allr = [torch.zeros_like(own) for _ in range(world)]
        torch.distributed.all_gather(allr, own)
        rank_ms = {"s1_s5_ms": [round(float(a[0]), 3) for a in allr],
                   "profiled_kernels_ms": [round(float(a[1]), 3) for a in allr],
                   "build_ms": [round(float(a[2]), 3) for a in allr],
                   "find_vulnerable_ms": [round(float(a[3]), 3) for a in allr],
                   "correct_ms": [round(float(a[4]), 3) for a in allr]}
        t = torch.tensor([ms_total, ms_corr], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_total, ms_corr = float(t[0].item()), float(t[1].item())
    ms_incl = ms_total / args.steps
    ms_step = ms_corr / args.steps
    vp, info, m, ng_o, ng_c, h_o, h_c = res
    value = n_total / (ms_step * 1e-3) / 1e6
    value_incl = n_total / (ms_incl * 1e-3) / 1e6
    log(f"timed: {ms_step:.3f} ms/step (S1-S5) -> {value:.1f} Mparticles/s; incl. check {ms_incl:.3f} ms "
        f"-> {value_incl:.1f} Mparticles/s")

    # ---- roofline of the dominant kernel class (device time inside the timed region)
    hbm, sm_max, peak_src = _peaks()
    launches = stats.pop("total_launches", (0.0, 0))[1]
    k3_we = stats.pop("K3_work_editables", (0.0, 0))[1]   # editables updated (frontier skips the rest)
    k3_wn = stats.pop("K3_work_entries", (0.0, 0))[1]     # row entries evaluated
    tests = {k: stats.pop(k, (0.0, 0))[1] for k in ("K2_count_tests", "K2_fill_tests", "K4_link_tests")}
    E, nent = vp["n_editable"], 2 * vp["n_pairs"]
    if world > 1:  # this rank's share for the per-launch byte count
        E, nent = E / world, nent / world
    cls_ms = dict(stats)
    # the dominant kernel of the metric's step (S1-S5); K4_fof is the S6 check, timed outside it
    s15 = {k: v for k, v in cls_ms.items() if k != "K4_fof"}
    dom = max(s15, key=lambda k: s15[k][0]) if s15 else None
    # algorithmic bytes per launch
    alg_bytes = {
        # per launch: 104 B per editable actually updated + 4 B per row entry evaluated
        "K3_pgd": (104.0 * k3_we + 4.0 * k3_wn) / max(cls_ms.get("K3_pgd", (0, 1))[1], 1) if k3_we
        else 104.0 * E + 4.0 * nent,
        "K1_key": 24.0 * n + 8.0 * n,
        "K1_gather": 8.0 * n + 28.0 * n + 40.0 * n,
        "K2_count": 16.0 * n + 4.0 * n,
        "K2_fill": 16.0 * n + 4.0 * n + 8.0 * n + 4.0 * nent,
        "K4_fof": 16.0 * n + 4 * 4.0 * n,
    }
    # ncu traffic of the dominant kernel (committed captures): dram bytes of one
    # captured launch next to that launch's algorithmic bytes
    traffic = {}
    for nm in ("r01_k3_traffic.json", "r02_k3_traffic.json", "r02_k2_traffic.json"):  # later files win
        tp = os.path.join(ROOT, "profiles", nm)
        if os.path.exists(tp):
            with open(tp) as f:
                d = json.load(f)
            traffic[d["kernel"]] = d
    # pair tests per second of K2 (count + fill sweeps) and K4 (FoF link searches) against the
    # fp32 issue ceiling: 148 SMs x 128 lanes x clock / ~20 instructions per pinned d2 test
    # (the pair kernels are ALU / latency bound, not HBM bound)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ceiling = sms * 128 * sm_max * 1e6 / 20.0
    roof = None
    if dom:
        d_ms, d_l = cls_ms[dom]
        avg_ms = d_ms / max(d_l, 1)
        tr = traffic.get(dom)
        cap = ({k: tr[k] for k in ("capture", "dram_bytes", "algorithmic_bytes", "traffic_over_algorithmic",
                                   "duration_ms", "source")} if tr else None)
        if dom in ("K2_count", "K2_fill") and tests.get(dom + "_tests"):
            # the pair sweeps are issue-bound (ncu: 77% issue active), not HBM-bound: the roofline
            # is the ALU test ceiling; the HBM view is reported next to it
            tps = tests[dom + "_tests"] / max(d_l, 1) / (avg_ms * 1e-3)
            hb = alg_bytes[dom] / (avg_ms * 1e-3) / 1e9
            roof = {"bound": "alu", "kernel": dom, "achieved": tps / 1e9, "peak": ceiling / 1e9,
                    "unit": "G pair tests/s", "frac": tps / ceiling,
                    "peak_source": f"{sms} SMs x 128 fp32 lanes x {sm_max} MHz / 20 instructions per test "
                                   "(DESIGN.md §6)",
                    "hbm_view": {"achieved": hb, "peak": hbm, "unit": "GB/s", "frac": hb / hbm},
                    "traffic": tr["dram_bytes"] if tr else None, "traffic_capture": cap,
                    "launch_ms": avg_ms, "launches": d_l}
        else:
            ach = alg_bytes[dom] / (avg_ms * 1e-3) / 1e9 if dom in alg_bytes else None
            roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": (ach / hbm) if ach is not None else None,
                    "traffic": tr["dram_bytes"] if tr else None, "traffic_capture": cap,
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})", "launch_ms": avg_ms, "launches": d_l}
    k3 = cls_ms.get("K3_pgd")
    k3_roof = None
    if k3 and k3[1]:
        a = alg_bytes["K3_pgd"] / (k3[0] / k3[1] * 1e-3) / 1e9
        k3_roof = {"achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm, "launch_ms": k3[0] / k3[1],
                   "launches": k3[1], "editables_updated_per_launch": k3_we / k3[1],
                   "entries_per_launch": k3_wn / k3[1], "editables_total": E,
                   "traffic_capture": ({k: traffic["K3_pgd"][k] for k in ("capture", "dram_bytes", "algorithmic_bytes",
                                                                         "traffic_over_algorithmic", "duration_ms",
                                                                         "source")}
                                       if "K3_pgd" in traffic else None)}

    pair_tests = {}
    for nm, kcls in (("K2_count", "K2_count"), ("K2_fill", "K2_fill"), ("K4_link", "K4_fof")):
        nt = tests.get(nm + "_tests", 0)
        ms = cls_ms.get(kcls, (0.0, 0))[0]
        if nt and ms > 0:
            tps = nt / (ms * 1e-3)
            pair_tests[nm] = {"tests_per_step": nt / args.steps, "tests_per_s": tps, "ceiling_tests_per_s": ceiling,
                              "frac": tps / ceiling, "kernel_ms_per_step": ms / args.steps}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded synth/ recipe, drawn on the GPU)",
        "config": {**w.describe(), "workload": w.name,
                   "parallelism": f"x-slabs x{world} (NCCL ghosts + per-iteration refresh/allreduce)" if world > 1
                   else "1 GPU",
                   "l2": "L2 flushed between steps (256 MB write)" if small else "inputs (24 N B) larger than the 126 MB L2",
                   "stop": {"restored": "L_tight <= 1e-10 and all link statuses restored (Alg. 1 l.6 + MCC=1, R11)",
                            "active": "no L_tight-active pair (R11)", "eps": "L_tight <= 1e-10 (Alg. 1 l.6)",
                            "none": "fixed t_max updates"}[args.stop], "t_max": args.t_max, "rows_per_axis": vp["cells_per_axis"]},
        "result": {"n_pairs": vp["n_pairs"], "n_editable": vp["n_editable"], "violated0": vp["n_violated0"],
                   "iterations": info["iterations"], "converged": info["converged"], "mcc_after": m["mcc"],
                   "fof_groups_orig": ng_o, "fof_groups_corr": ng_c, "halos_equal": bool(np.array_equal(h_o, h_c))},
        "roofline": roof, "k3_roofline": k3_roof,
        "kernels_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in cls_ms.items()},
        "pair_tests": pair_tests,
        "phases_ms": phases,
        "per_rank": rank_ms,
        "incl_check": {"value": value_incl, "unit": UNIT, "ms_per_step": ms_incl,
                       "what": "S1-S7: + FoF labels on original and corrected positions, halo catalogues, MCC"},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }

    # ---- end to end through the public API (cc_run) with pinned HOST buffers, copies inside
    if not args.no_e2e:
        host = [t.cpu().pin_memory() for t in (x, y, z, xh, yh, zh)]
        hgid = gid.cpu().pin_memory() if gid is not None else None
        hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(3)]

        def e2e_step():  # the metric's S1..S5 through the public call, host buffers in and out
            return c.run(*host, out=hout, gid=hgid, host=True)

        e2e_step()
        ke = max(1, min(args.steps, 3))
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = e0.elapsed_time(e1) / ke
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(t.item())
        line["e2e"] = {"value": n_total / (e_ms * 1e-3) / 1e6, "unit": UNIT, "ms_per_step": e_ms,
                       "h2d_bytes_per_step": (24 + (4 if gid is not None else 0)) * n_total,
                       "d2h_bytes_per_step": 12 * n_total + 48}
        log(f"e2e: {e_ms:.3f} ms/step")
        del host, hout
    # ---- f1 edit log (Alg. 1 l.11-13 + reconstruction) on this step's correction;
    # outside the timed step (not one of the §8(a) rows), timed on the library's stream
    if not args.no_edit_log:
        fl, q = c.edit_encode(x, y, z, xh, yh, zh, *out)
        rec = c.edit_decode(xh, yh, zh, fl, q)
        xi_f = float(np.float32(w.xi))
        in_bound = all(bool(((r.double() - o.double()).abs() <= xi_f).all()) for r, o in zip(rec, (x, y, z)))
        diag = {"corr_in_bound": all(bool(((r.double() - o.double()).abs() <= xi_f).all()) for r, o in zip(out, (x, y, z))),
                "rec_out_of_bound": int(sum(int(((r.double() - o.double()).abs() > xi_f).sum()) for r, o in zip(rec, (x, y, z)))),
                "max_excess": max(float(((r.double() - o.double()).abs() - xi_f).max()) for r, o in zip(rec, (x, y, z))),
                "rec_ne_corr": int(sum(int((r != o).sum()) for r, o in zip(rec, out)))}
        log(f"edit log diag: {diag}")
        ke = 3
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ms_e = ms_d = ms_p = 0.0
        cap = int(q.shape[0])  # known from the first encode: one pass per timed encode
        for _ in range(ke):
            ev[0].record(stream)
            fl, q = c.edit_encode(x, y, z, xh, yh, zh, *out, cap=cap)
            ev[1].record(stream)
            words = c.edit_pack(q)  # (m+2)-bit container (R33)
            ev[2].record(stream)
            c.edit_decode(xh, yh, zh, fl, q, out=rec)
            ev[3].record(stream)
            torch.cuda.synchronize(dev)
            ms_e += ev[0].elapsed_time(ev[1]) / ke
            ms_p += ev[1].elapsed_time(ev[2]) / ke
            ms_d += ev[2].elapsed_time(ev[3]) / ke
        packed_ok = bool(torch.equal(c.edit_unpack(words, int(q.shape[0])), q))
        # quantisation-safety re-check (R31): S1 + S2 on (P, x_rec) -> violated pairs
        c.build_cells(x, y, z, *rec, gid=gid)
        recheck = c.find_vulnerable()
        ne = int(q.shape[0])
        fb = (3 * n + 7) // 8
        b_enc = 24 * n + fb + 8 * ne        # read P_hat0 and P_hat, write flags and indices
        b_dec = 12 * n + fb + 8 * ne + 12 * n
        pk = hbm or 1.0
        line["edit_log"] = {"n_edits": ne, "flags_bytes": fb, "index_bytes": 8 * ne,
                            "packed_index_bytes": int(words.numel()) * 4, "packed_bits_per_edit": params.m + 2,
                            "pack_ms": ms_p, "packed_round_trip": packed_ok, "in_bound": in_bound, "diag": diag,
                            "recheck_pairs": recheck["n_pairs"], "recheck_violated": recheck["n_violated0"],
                            "encode_ms": ms_e, "decode_ms": ms_d,
                            "encode_gbs": b_enc / (ms_e * 1e-3) / 1e9, "decode_gbs": b_dec / (ms_d * 1e-3) / 1e9,
                            "encode_frac": b_enc / (ms_e * 1e-3) / 1e9 / pk,
                            "decode_frac": b_dec / (ms_d * 1e-3) / 1e9 / pk,
                            "bytes_model": "encode 24N + ceil(3N/8) + 8 n_edits; decode 24N + ceil(3N/8) + 8 n_edits"}
        log(f"edit log: {ne:,} edits, encode {ms_e:.3f} ms, decode {ms_d:.3f} ms, in_bound={in_bound}")
        del fl, q, rec, words
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(w)
        line["cpu_baseline"] = {k: v for k, v in cb.items() if k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), file=_OUT, flush=True)
    c.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
