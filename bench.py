#!/usr/bin/env python
"""bench.py -- batched Toom-Cook multiplication on B200 (libtoomgpu).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

One "step" = one pass of the whole hot path (split + evaluate, recursive
pointwise products, interpolate, recompose -- SURVEY.md §8(a) rows a1-a6)
over one batch.  The workload is BASELINE.json configs[1] (C2): one batch of
65536 products of two 256-limb (8192-bit) operands, Toom-4 (points
0, +-1, +-2, 1/2, inf) recursing to a 32-limb schoolbook base.  Under
torchrun (N>1) the SAME batch is split into N contiguous slices of 65536/N
products, one per rank (strong scaling; no data-path
collective: the products are independent).  The same run also reports the
two single-product configs of the metric: C4 (ms per 32-Mbit product, rank 0)
and C5 (one 512-Mbit product with its 31 top-level products sharded over the
N ranks through NCCL, dist.sharded_mul; Eq. 2.5).

Prints ONE JSON line on rank 0 (contract in the task statement / DESIGN.md).
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

import synth  # noqa: E402

C2 = dict(n=256, batch=65536, B=4, t4=32, t3=32)

# growth limbs e - b of an evaluated operand per point set and
# the number of points 2B-1 (Eq. 2.1)
_GROW = {3: 1, 4: 1, 8: 2, 16: 2}
_NPTS = {3: 5, 4: 7, 8: 15, 16: 31}


def algorithmic_lp(n, top_B=0, t4=256, t3=64):
    """Limb-products of one n x n product in the reference recursion shape
    (SURVEY.md §8(d)): the base case multiplies the REAL child lengths -- point
    0 gets block 0 (b limbs), infinity the top block (n - (B-1) b limbs), the
    other 2B-3 points e = b + growth limbs -- not the padded width the kernels
    use.  C1 5315, C2 14439, C4 2.3056e9, C5 7.147e10 per product."""
    from functools import lru_cache

    def choose(m, depth):
        def ok(m, B):
            b = -(-m // B)
            return m >= 2 * B and m - (B - 1) * b >= 1
        if depth == 0 and top_B and ok(m, top_B):
            return top_B
        B = 4 if m > t4 else (3 if m > t3 else 0)
        if B and not ok(m, B):
            B = 3 if (B == 4 and ok(m, 3)) else 0
        return B

    @lru_cache(None)
    def rec(m, depth):
        B = choose(m, depth)
        if B == 0:
            return m * m
        b = -(-m // B)
        return rec(b, depth + 1) + rec(m - (B - 1) * b, depth + 1) + (_NPTS[B] - 2) * rec(b + _GROW[B], depth + 1)

    return rec(n, 0)


def staged_bytes(levels, fused=True):
    """Algorithmic HBM bytes of the staged (non-fused) Toom levels of a plan:
    evaluation reads both parents (2 count n limbs) and writes both children
    families (2 count npts e); interpolation + recomposition reads the child
    products (count npts 2e) and writes the parents' products (count 2n)."""
    ev = it = 0
    lv = [L for L in levels if L["B"]]
    if fused:
        lv = lv[:-1]
    for L in lv:
        ev += 4 * 2 * L["count"] * (L["n"] + L["npts"] * L["e"])
        it += 4 * L["count"] * (L["npts"] * 2 * L["e"] + 2 * L["n"])
    return ev, it


def c2_slice(rank, world, total=C2["batch"]):
    """Contiguous slice [lo, hi) of the C2 batch that `rank` of `world` ranks
    multiplies (65536/P products per rank)."""
    return rank * total // world, (rank + 1) * total // world


def c2_inputs(lo, hi, n=C2["n"]):
    """Products lo .. hi-1 of the seeded C2 stream (synth: counter-based, so a
    slice is generated without the rest of the batch)."""
    u_np = np.empty((hi - lo, n), np.uint32)
    v_np = np.empty((hi - lo, n), np.uint32)
    seed = synth.seed_for(2)
    for a in range(0, hi - lo, 8192):
        b = min(hi - lo, a + 8192)
        u_np[a:b] = synth.uniform_limbs(seed, lo + a, b - a, 0, n)
        v_np[a:b] = synth.uniform_limbs(seed, lo + a, b - a, 1, n)
    return u_np, v_np


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(u, v, threads, target_s=12.0, kind="O2"):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload;
    returns (products/s, products, seconds).  kind "O2": the recursive Toom
    with the paper's points (its own threading over the batch); "O1": the
    schoolbook definition, the batch split over `threads` host threads
    (O1 for C1-C3, O2 for C4/C5, 1 thread and all cores)."""
    import oracle
    oracle.build()

    def run(k):
        if kind == "O2":
            oracle.toom_batched(u[:k], v[:k], top_B=C2["B"], threads=threads)
            return
        parts = np.array_split(np.arange(k), threads)
        ts = [threading.Thread(target=oracle.schoolbook_batched, args=(u[p[0]:p[-1] + 1], v[p[0]:p[-1] + 1]))
              for p in parts if len(p)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    cal = min(64 * threads, len(u))
    t0 = time.perf_counter()
    run(cal)
    t_cal = time.perf_counter() - t0
    k = int(min(len(u), max(cal, cal * target_s / max(t_cal, 1e-6))))
    t0 = time.perf_counter()
    run(k)
    dt = time.perf_counter() - t0
    return k / dt, k, dt


def run_reference(args, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    u, v = synth.config_inputs(2, batch=4096)
    times, ks = [], []
    for s in range(args.warmup + args.steps):
        rate, k, dt = oracle_sample(u, v, threads, target_s=max(2.0, 60.0 / (args.warmup + args.steps)), kind="O1")
        if s >= args.warmup:
            times.append(dt)
            ks.append(k)
    value = sum(ks) / sum(times)
    line = {
        "metric": "batched products/s", "value": value, "unit": "products/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "C2: Toom-4 batch of 8192-bit products (BASELINE.json configs[1])", "n_limbs": 256,
                   "B": 4, "per_step_sample_products": ks[0] if ks else 0},
        "cpu_baseline": {"value": value, "unit": "products/s", "cores": threads, "kind": "oracle",
                         "sample": f"{ks[0] if ks else 0} C2 products per step (first products of the seeded stream), "
                                   f"oracle O1 (plain schoolbook) with the products split over {threads} host "
                                   f"threads, {cpu_model()}"},
        "e2e": {"value": value, "unit": "products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_1602_02740_b200 as tg

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # this rank's contiguous slice of the ONE C2 batch (strong scaling)
    n, B, total = C2["n"], C2["B"], C2["batch"]
    lo, hi = c2_slice(rank, world, total)
    batch = hi - lo
    u_np, v_np = c2_inputs(lo, hi, n)
    u = torch.from_numpy(u_np).cuda()
    v = torch.from_numpy(v_np).cuda()
    w = torch.empty((batch, 2 * n), dtype=u.dtype, device="cuda")

    def step():
        tg.toom_mul_batched(u, v, B=B, t4=C2["t4"], t3=C2["t3"], out=w)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = tg.last_launch_count()

    # timed region
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_per_step = ms / args.steps
    value = total / (ms_per_step * 1e-3)

    # per-kernel durations (separate instrumented pass, CUDA events recorded on
    # the launching stream around every launch) for the roofline of each kernel
    tg.profile_enable(True)
    for _ in range(args.steps):
        step()
    prof = tg.profile_collect()
    tg.profile_enable(False)
    plan = tg.plan_describe(n, batch, B=B, t4=C2["t4"], t3=C2["t3"])
    lv = plan["levels"]
    pk, pk_kind = peaks()
    hbm_peak = pk.get("hbm_gbs")
    lp_wide, _ = tg.probe_limb_products()      # IMAD.WIDE.U32 + 64-bit accumulate chains
    lp_chain, _ = tg.probe_carry_chain()       # the base case's mad.lo.cc/madc.hi.cc/addc sequence
    lp_rate = max(lp_wide, lp_chain)
    L0, L1 = lv[0], lv[1]
    lp_per_product = algorithmic_lp(n, B, C2["t4"], C2["t3"])
    # per-launch algorithmic work of the three kernels of a C2 step:
    #   eval   (k_eval_top_v4<4>)       : read u, v; write the 7 evaluated pairs
    #   bottom (k_fused_dc<4>, or k_fused_bottom<4,18> in c2 mode 0/1): SURVEY
    #          §8(d)'s 14439 limb-products per product (real child lengths, not
    #          7 x 18^2 x 7)
    #   interp (k_interp_top_cls<DEF>, or k_interp_top_smem<4> in mode 0):
    #          read the 7 products; write w
    c2m = plan.get("c2_mode", 0)
    kern = {
        "eval": dict(name="k_eval_top_v4<4>", bound="hbm",
                     units=2 * (L0["count"] * L0["n"] + L0["count"] * L0["npts"] * L0["e"]) * 4),
        "base": dict(name="k_fused_dc<4>" if c2m == 2 else "k_fused_bottom<4,18>", bound="alu",
                     units=batch * lp_per_product,
                     bytes=(2 * L1["count"] * L1["n"] + L1["count"] * 2 * L1["n"]) * 4),
        "interp": dict(name=("k_interp_top_cls<%d>" % (c2m == 2)) if c2m else "k_interp_top_smem<4>", bound="hbm",
                       units=(L0["count"] * L0["npts"] * 2 * L0["e"] + L0["count"] * 2 * L0["n"]) * 4),
    }
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f)
    except OSError:
        pass
    peak_note = ("measured live: max of toom_probe_limb_products (IMAD.WIDE.U32 chains, %.2f T LP/s) and "
                 "toom_probe_carry_chain (mad.lo.cc/madc.hi.cc/addc, %.2f T LP/s), 148 SMs x 8 CTAs x 256 threads "
                 "x 8 chains; DESIGN.md §6 gives the nominal 32 LP/clk/SM figure" % (lp_wide / 1e12, lp_chain / 1e12))
    shares = {k: prof[k]["ms"] / max(1, prof[k]["launches"]) for k in kern}
    kernels = {}
    for k, d in kern.items():
        ms_l = shares[k]
        if d["bound"] == "hbm":
            ach = d["units"] / (ms_l * 1e-3) / 1e9
            kernels[k] = {"kernel": d["name"], "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                          "frac": ach / hbm_peak, "traffic": traffic.get(d["name"]), "ms_per_launch": ms_l,
                          "algorithmic_bytes_per_launch": d["units"]}
        else:
            ach = d["units"] / (ms_l * 1e-3)
            kernels[k] = {"kernel": d["name"], "bound": "alu", "achieved": ach / 1e12, "peak": lp_rate / 1e12,
                          "unit": "T limb-products/s", "frac": ach / lp_rate, "traffic": traffic.get(d["name"]),
                          "ms_per_launch": ms_l, "limb_products_per_launch": d["units"],
                          "limb_products_per_product": lp_per_product,
                          "hbm_GBps": d["bytes"] / (ms_l * 1e-3) / 1e9, "peak_kind": peak_note}
    dominant = max(shares, key=shares.get)
    roofline = dict(kernels[dominant])
    roofline["peak_source"] = ("MEASURED_PEAKS.json hbm_gbs" if roofline["bound"] == "hbm" else "live probe") \
        if pk_kind == "measured" else "fallback"
    stages = {"ms_per_step": {k: round(prof[k]["ms"] / args.steps, 5) for k in kern}, "dominant": dominant,
              "kernels": kernels}

    # end-to-end through the public C ABI with HOST buffers (pinned)
    e2e = None
    if not args.no_e2e:
        hu = torch.from_numpy(u_np).pin_memory()
        hv = torch.from_numpy(v_np).pin_memory()
        hw = torch.empty((batch, 2 * n), dtype=torch.uint32).pin_memory()
        for _ in range(2):
            tg.toom_mul_batched_host(hu, hv, B=B, t4=C2["t4"], t3=C2["t3"], out=hw)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            tg.toom_mul_batched_host(hu, hv, B=B, t4=C2["t4"], t3=C2["t3"], out=hw)
        dt = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": total * args.steps / dt, "unit": "products/s",
               "h2d_bytes_per_step": 2 * total * n * 4, "d2h_bytes_per_step": total * 2 * n * 4,
               "ms_per_step": 1e3 * dt / args.steps}

    # secondary metric of BASELINE.json: ms per 32-Mbit product (configs[3], C4:
    # one product of two 2^20-limb operands, recursive Toom-4 -> Toom-3), rank 0
    c4 = None
    if rank == 0 and not args.no_c4:
        a4, b4 = synth.config_inputs(4)
        a4, b4 = torch.from_numpy(a4).cuda(), torch.from_numpy(b4).cuda()
        w4 = torch.empty(2 * a4.numel(), dtype=a4.dtype, device="cuda")
        for _ in range(2):
            tg.toom_mul(a4, b4, B=4, out=w4)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(stream)
        for _ in range(reps):
            tg.toom_mul(a4, b4, B=4, out=w4)
        e1.record(stream)
        torch.cuda.synchronize()
        ms4 = e0.elapsed_time(e1) / reps
        launches4 = tg.last_launch_count()
        tg.profile_enable(True)
        for _ in range(reps):
            tg.toom_mul(a4, b4, B=4, out=w4)
        p4 = tg.profile_collect()
        tg.profile_enable(False)
        n4 = a4.numel()
        pl4 = tg.plan_describe(n4, 1, B=4)
        ev_b, it_b = staged_bytes(pl4["levels"], pl4["fused_bottom"])
        lp4 = algorithmic_lp(n4, 4)
        ms_base = p4["base"]["ms"] / reps
        ms_up = (p4["eval"]["ms"] + p4["interp"]["ms"] + p4["other"]["ms"]) / reps
        c4 = {"workload": "C4: one product of two 2^20-limb (32-Mbit) uniform operands, Toom-4 -> Toom-3 -> "
                          "schoolbook (BASELINE.json configs[3])", "ms_per_product": ms4,
              "reps": reps, "launches_per_product": launches4,
              "roofline": {
                  "products": {"bound": "alu", "limb_products": lp4, "ms": ms_base,
                               "achieved": lp4 / (ms_base * 1e-3) / 1e12, "peak": lp_rate / 1e12,
                               "unit": "T limb-products/s", "frac": lp4 / (ms_base * 1e-3) / lp_rate},
                  "upper_levels": {"bound": "hbm", "algorithmic_bytes": ev_b + it_b, "ms": ms_up,
                                   "achieved": (ev_b + it_b) / (ms_up * 1e-3) / 1e9, "peak": hbm_peak,
                                   "unit": "GB/s", "frac": (ev_b + it_b) / (ms_up * 1e-3) / 1e9 / hbm_peak},
                  "whole_product_frac_of_alu": lp4 / (ms4 * 1e-3) / lp_rate,
                  "note": "products = the base-case kernels (fused bottom level); upper_levels = every staged "
                          "evaluation / interpolation / recomposition / transpose launch, against the "
                          "algorithmic bytes of the staged levels (each parent and child read or written once)"}}
        del a4, b4, w4
    barrier()

    # C5 (configs[4]): one 512-Mbit product, the 31 top-level products sharded
    # over the N ranks (NCCL scatter / gather), ms per product, max over ranks
    c5 = None
    if not args.no_c5:
        from paper_1602_02740_b200 import dist as tgdist
        n5 = 1 << 24
        a5 = b5 = None
        if rank == 0:
            x, y = synth.config_inputs(5)
            a5, b5 = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        ops = tgdist.CudaOps()
        reps5 = 3
        # one GPU: the single-product entry point (Toom-16 top, lazy Toom-4
        # levels, deferred Toom-3 bottom in one plan); N > 1: the 31 top-level
        # products sharded over the ranks (Eq. 2.5) through dist.sharded_mul
        if world == 1:
            mul5 = lambda: tg.toom_mul(a5, b5, B=16)
        else:
            dev5 = torch.device("cuda", torch.cuda.current_device())
            mul5 = lambda: tgdist.sharded_mul(a5, b5, n5, ops, device=dev5)
        for _ in range(1):
            mul5()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps5):
            w5 = mul5()
        e1.record(stream)
        torch.cuda.synchronize()
        ms5 = max_over_ranks(e0.elapsed_time(e1) / reps5)
        lp5 = algorithmic_lp(n5, 16)
        c5 = {"workload": "C5: one product of two 2^24-limb (512-Mbit) uniform operands, 31-point Toom-16 top level, "
                          "its 31 products sharded over the ranks (BASELINE.json configs[4])",
              "path": "toom_mul (one GPU)" if world == 1 else "dist.sharded_mul (NCCL broadcast / gather)",
              "ms_per_product": ms5, "reps": reps5, "ranks": world,
              "products_per_rank": [hi_ - lo_ for lo_, hi_ in tgdist.shard_bounds(31, world)[0]],
              "frac_of_alu_whole_job": lp5 / (ms5 * 1e-3) / (lp_rate * world)}
        del a5, b5
        if rank == 0:
            del w5
        barrier()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        r_all, k_all, dt_all = oracle_sample(u_np, v_np, threads, target_s=6.0, kind="O1")
        r_one, k_one, dt_one = oracle_sample(u_np, v_np, 1, target_s=4.0, kind="O1")
        r_o2, k_o2, dt_o2 = oracle_sample(u_np, v_np, threads, target_s=4.0, kind="O2")
        cpu = {"value": r_all, "unit": "products/s", "cores": threads, "kind": "oracle",
               "sample": f"{k_all} of the 65536 C2 products ({dt_all:.1f} s), oracle O1 (plain schoolbook, the "
                         f"definition w = uv) with the products split over {threads} host threads, {cpu_model()}",
               "one_thread": {"value": r_one, "products": k_one, "seconds": dt_one, "kind": "O1"},
               "o2_all_cores": {"value": r_o2, "products": k_o2, "seconds": dt_o2,
                                "kind": "O2 recursive Toom (paper points 0,+-2^j, §3 listings, §4 even-odd)"}}

    if rank == 0:
        line = {
            "metric": "batched products/s", "value": value, "unit": "products/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "C2: Toom-4 (points 0,+-1,+-2,1/2,inf) -> Toom-4 -> 18-limb schoolbook; "
                                   "one batch of 65536 products of two 8192-bit (256-limb) uniform operands, "
                                   "split into %d contiguous slice(s) (BASELINE.json configs[1])" % world,
                       "batch": total, "per_gpu_batch": batch, "n_limbs": n, "B": B,
                       "plan": {"t4": C2["t4"], "t3": C2["t3"]},
                       "levels": [{k: L[k] for k in ("B", "count", "n", "e")} for L in lv],
                       "parallelism": f"batch-sharded x{world} (independent products, no collective)",
                       "l2": "inputs %.0f MB + workspace %.2f GB per step > 126 MB L2 (no flush needed)"
                             % (batch * n * 8 / 1e6, plan["workspace_bytes"] / 1e9)},
            "roofline": roofline,
            "stages": stages,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "ms_per_32mbit_product": c4,
            "ms_per_512mbit_product": c5,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "us_per_product": 1e3 * ms_per_step / total,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
