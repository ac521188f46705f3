#!/usr/bin/env python
"""Benchmark of the λ(ω) hot path on B200 (see DESIGN.md §5 Measurement).

Headline (BASELINE.json metric, config C3): one cellular-automaton step (B3/S23) of the
Sierpinski gasket at n = 2^16 launched over the λ(ω) orthotope (ρ = 32 tiles), with the
CA state resident in HBM in the λ-ordered compact layout (the reference's CompactGrid,
block_map.hpp:82-110: every byte a member value) — `value` = member-cell updates per
second (3^16 per step). The same step on the reference's own int64 embedded Grid layout
is reported beside it (`embedded_int64`), as are the bounding-box (BB) launches
(paper-faithful per-cell BB and the sector-vectorised BB), the uint8 / 1-bit states, the
single-write and reduction workloads, the C4 map sweep, the HBM roofline of the dominant
kernel, the reference CPU path timed on this host (`cpu_baseline`), and `e2e` = the same
metric through the public C ABI call nbb_gpu_ca() with pinned host buffers (the
reference's int64 Grid in and out; transfers inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU): the tile range is split in contiguous
chunks (dispatch.cpp:419-427); the headline's halo cells are read from the owning rank's
buffer over peer memory inside the step kernel (--transport p2p, default) or exchanged by
NCCL between steps (--transport nccl). `c5_r17` = the same step at n = 2^17 (BASELINE
configs[4]) at every N.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gasket cells/s at n=2^16: λ(ω) vs BB speedup, % of B200 HBM roofline"


# ---------------------------------------------------------------------------------
def layout_bytes_per_pass(r: int, cell_bytes: int) -> int:
    """layout-minimum DRAM bytes of one pass over the member cells of the
    embedded grid, 32-byte sectors: 32 * 2^g * 3^(r-g), 2^g = 32 / cell_bytes."""
    g = {8: 2, 1: 5}[cell_bytes]
    return 32 * (2 ** g) * 3 ** (r - g)


def measured_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML samples of SM clock + throttle reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------------
def reference_ca(r: int, rho: int, steps: int, seed: int, workers: int):
    """The unmodified reference run_ca (oracle/_ref/libnbbref.so) on host cores."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    from _oracle import ref_lib
    from paper_2004_13475_b200 import _abi, nbb
    ref = ref_lib()
    spec = nbb.FractalSpec.sierpinski()
    n = 1 << r
    h = ref.ref_grid_create(ctypes.byref(spec.to_c()), r)
    if not h:
        raise MemoryError(ref.ref_last_error().decode())
    try:
        data = np.ctypeslib.as_array(ctypes.cast(ref.ref_grid_data(h), ctypes.POINTER(ctypes.c_int64)),
                                     shape=(n * n,))
        # input prep (not timed): our bit-identical O(3^r) generator writes the member cells
        _abi.load().nbb_gpu_random_member_grid(ctypes.byref(spec.to_c()), r, seed, 2, n * n,
                                              data.ctypes.data_as(ctypes.c_void_p))
        cfg = nbb.DispatchConfig(r=r, rho=rho, mode=nbb.MapMode.Lambda, workers=workers,
                                 timing=True, max_cells=n * n)
        reps = (_abi.NbbReport * steps)()
        secs = ctypes.c_double()
        rc = ref.ref_ca_h(ctypes.byref(cfg.to_c()), h, steps, 8, 12, None, reps, ctypes.byref(secs))
        if rc:
            raise RuntimeError(ref.ref_last_error().decode())
        micros = [reps[i].micros for i in range(steps)]
        return secs.value, micros
    finally:
        ref.ref_grid_destroy(h)


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r, rho = args.level, 32
    steps = max(1, min(args.steps, args.ref_max_steps))
    cores = os.cpu_count() or 1
    secs, micros = reference_ca(r, rho, steps, 17, cores)
    value = 3 ** r * steps / secs
    line = {
        "metric": METRIC, "value": value, "unit": "cells/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": 0, "ms_per_step": 1e3 * secs / steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": f"synthetic: random_member_grid(gasket, {r}, seed=17, modulus=2), B3/S23",
        "config": config_block(r, rho, args.gpus),
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": cores, "kind": "reference",
                         "sample": f"reference run_ca(r={r}, rho={rho}, lambda/subbox/direct, "
                                   f"workers={cores}) for {steps} steps in one call; wall time of "
                                   f"the call (incl. its MemberMask build and per-step fills); "
                                   f"launch-only micros per step {micros}"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def pair_launches(k, world=1, transport="p2p"):
    """(two-step, one-step) launches for k steps: nbb_gpu_ca_compact_run_dev at N = 1 (an even
    number of pairs, nbb_capi.cu run_ca_compact), nbb_gpu_ca_compact_p2p_passes_dev at N > 1
    (k // 2 pairs + k % 2), one launch per step with the NCCL exchange."""
    if world > 1:
        return (k // 2, k % 2) if transport == "p2p" else (0, k)
    pairs = k // 2
    pairs -= pairs & 1
    return pairs, k - 2 * pairs


def config_block(r, rho, world=1, transport="p2p"):
    return {"workload": f"C3: gasket n=2^{r} cellular-automaton step (B3/S23), lambda(omega) launch, "
                        f"rho={rho} tiles; device state = the lambda-ordered compact layout "
                        f"(CompactGrid, 8 B per member), host I/O = the reference's int64 Grid; "
                        + ("two steps per pass over the state (ca_compact2_kernel)"
                           if world == 1 or transport == "p2p" else "one step per launch"),
            "r": r, "n": 1 << r, "rho": rho, "mode": "lambda", "cells_per_step": 3 ** r,
            "cell": "int64", "state": "compact",
            "parallelism": "1 GPU" if world == 1 else
                           f"{world} ranks: contiguous tile-range shards; " + (
                               "halo cells read over peer memory (CUDA IPC) inside the step kernel"
                               if transport == "p2p" else
                               f"halo cells exchanged by gather + NCCL all_to_all + scatter ({transport})"),
            "l2": "no flush: each pass moves 689 MB compact / 1.7 GB embedded (> 126 MB L2)"}


# ---------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--level", type=int, default=16, help="scale level r (n = 2^r)")
    ap.add_argument("--ref-max-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 halo exchange: inside the step kernel over peer memory (p2p, "
                         "default) or gather + NCCL all_to_all + scatter per step (nccl)")
    ap.add_argument("--profile", action="store_true",
                    help="only run a few λ/BB CA steps (for ncu); prints nothing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        try:
            run_reference_arm(args)
        except Exception as e:  # e.g. oracle/_ref not built on this box: say so, don't crash
            if int(os.environ.get("RANK", "0")) == 0:
                print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}),
                      flush=True)
        return

    import torch
    from paper_2004_13475_b200 import _abi as nbb_abi
    from paper_2004_13475_b200 import device as dev
    from paper_2004_13475_b200 import nbb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    local = local % ndev  # ranks may share a GPU in test setups
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # more ranks than GPUs (functional test of the sharded path): gloo
            dist.init_process_group("gloo")

    r, n = args.level, 1 << args.level
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream
    spec = nbb.FractalSpec.sierpinski()
    members = 3 ** r

    def cfg(**kw):
        c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n, device=local)
        for k, v in kw.items():
            setattr(c, k, v)
        return c

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        dev_t = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], device=dev_t, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs: random_member_grid(gasket, r, 17, 2), generated bit-identically --------
    a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    vals = torch.from_numpy(nbb.random_member_values(spec, r, 17, 2)).cuda()
    dev.scatter_members_dev(cfg(), vals.data_ptr(), a.data_ptr(), s)
    del vals
    b = torch.zeros_like(a)
    torch.cuda.synchronize()

    # shards of the tile range for this rank: every rank owns one contiguous chunk and all
    # ranks together update the 3^r cells of one step (the per-GPU share shrinks with N)
    from paper_2004_13475_b200 import shard
    plan = shard.ShardPlan(r=r, rho=32, world=world, rank=rank)
    plan_c = shard.ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")
    # kernels per step: 1 (N = 1, or N > 1 over peer memory); + gather and scatter with NCCL
    launches_per_step = 3 if (world > 1 and args.transport == "nccl") else 1

    def ca_runner(c, src, dst):
        bufs = [src, dst]
        state = {"i": 0}

        def step():
            i = state["i"]
            if world > 1:
                plan.exchange_halo(bufs[i & 1], dist)
                dev.ca_step_dev(plan.local_config(c), bufs[i & 1].data_ptr(),
                                bufs[(i + 1) & 1].data_ptr(), nbb.CaRule(), s)
            else:
                dev.ca_step_dev(c, bufs[i & 1].data_ptr(), bufs[(i + 1) & 1].data_ptr(),
                                nbb.CaRule(), s)
            state["i"] = i + 1
        return step

    def compact_runner(c, src, dst):
        bufs = [src, dst]
        state = {"i": 0}
        lc = plan_c.local_config(c) if world > 1 else c

        def step():
            i = state["i"]
            if world > 1:
                plan_c.exchange_halo(bufs[i & 1], dist)
            dev.ca_compact_step_dev(lc, bufs[i & 1].data_ptr(), bufs[(i + 1) & 1].data_ptr(),
                                    nbb.CaRule(), s)
            state["i"] = i + 1
        return step

    def timed_run(run, K, W, sampler=None, groups=None):
        """run(k) issues k steps on `stream`; W warm-up steps, then K timed with CUDA events.
        groups (a list) receives the per-step means of G equal sub-runs (events between them)."""
        if sampler:  # NVML sampling from the warm-up on: the timed region alone is ~20 ms
            sampler.__enter__()
        run(W)
        barrier()
        G = 10 if (groups is not None and K >= 10) else 1
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(G + 1)]
        ev[0].record(stream)
        for gi in range(G):
            k = K // G + (1 if gi < K % G else 0)
            run(k)
            ev[gi + 1].record(stream)
        ev[G].synchronize()
        if sampler:
            sampler.__exit__()
        barrier()
        if groups is not None and G > 1:
            groups.extend(ev[gi].elapsed_time(ev[gi + 1]) / (K // G + (1 if gi < K % G else 0))
                          for gi in range(G))
        return max_over_ranks(ev[0].elapsed_time(ev[G])) / K  # ms per step

    def timed(step, K, W, sampler=None):
        def run(k):
            for _ in range(k):
                step()
        return timed_run(run, K, W, sampler)

    # the compact CA state (λ-ordered CompactGrid): every byte a member value (int64)
    c1 = torch.empty(members, dtype=torch.int64, device="cuda")
    c2 = torch.empty_like(c1)
    dev.compact_store_dev(cfg(), a.data_ptr(), c1.data_ptr(), s)

    if args.profile:
        run = compact_runner(cfg(), c1, c2)
        for _ in range(3):
            run()
        dev.ca_compact_run_dev(cfg(), c1.data_ptr(), c2.data_ptr(), 4, nbb.CaRule(), s)  # 2 pairs
        for c in (cfg(), cfg(mode=nbb.MapMode.BoundingBox),
                  cfg(mode=nbb.MapMode.BoundingBox, kernel=nbb.KernelFamily.PerCell)):
            run = ca_runner(c, a, b)
            for _ in range(3):
                run()
        torch.cuda.synchronize()
        return

    K, W = args.steps, args.warmup
    sampler = ClockSampler(local)
    results = {}

    # ---- RD (the global reduction) on the compact state: each rank sums its own tiles, then
    # one int64 all-reduce (NCCL) — the value back on the host every call ----------------
    rd_val = shard.sharded_reduction(plan_c, cfg(), c1.data_ptr(), dist, s, local)
    rd_ms = timed(lambda: shard.sharded_reduction(plan_c, cfg(), c1.data_ptr(), dist, s, local),
                  max(10, K // 4), W)
    rd_line = {"workload": f"run_reduction on the compact state at n=2^{r}: per-rank partial over its "
                           f"tiles (segment_sum_kernel) + one int64 all-reduce, value read back on the host; state = the initial random_member_grid",
               "ms_per_call": rd_ms, "value": members * 1e3 / rd_ms, "unit": "cells/s",
               "GBps_per_gpu": 8 * members / world / (rd_ms * 1e-3) / 1e9, "sum": rd_val}
    # the partial-sum kernel alone, back to back (no host read-back): its share of the call
    rd_part = torch.empty(1, dtype=torch.int64, device="cuda")
    rd_cfg = plan_c.local_config(cfg())
    rd_kern_ms = timed(lambda: dev.reduction_compact_dev(rd_cfg, c1.data_ptr(), rd_part.data_ptr(), s),
                       max(10, K // 4), W)
    rd_line["kernel_only"] = {"ms": rd_kern_ms, "GBps": 8 * members / world / (rd_kern_ms * 1e-3) / 1e9,
                              "frac": 8 * members / world / (rd_kern_ms * 1e-3) / 1e9 / measured_peaks()[0],
                              "note": "memset + segment_sum_kernel per call, no host read-back"}
    # ---- headline: λ(ω) CA step on the compact state, ρ = 32 tiles ---------------------
    head_groups = []  # per-step means of 10 sub-runs (N = 1): median / paper-style mean
    # the step loop runs in the library (C++; one kernel per step, PDL between steps)
    p2p = None
    if world > 1 and args.transport == "p2p":
        try:
            p2p = shard.P2PCompactCA(plan_c, dist, device=local)
        except shard.P2PUnavailable as e:  # every rank agrees; run the NCCL exchange instead
            print(f"bench: {e}; falling back to --transport nccl", file=sys.stderr)
            args.transport = "nccl (p2p unavailable)"
            launches_per_step = 3
    if p2p is not None:
        p2p.load(c1)
        head_ms = timed_run(lambda k: p2p.run(cfg(), nbb.CaRule(), k, s), K, W, sampler)
        p2p.check(s)
        p2p.close()
    elif world > 1:
        head_ms = timed(compact_runner(cfg(), c1, c2), K, W, sampler)
    else:
        head_ms = timed_run(lambda k: dev.ca_compact_run_dev(cfg(), c1.data_ptr(), c2.data_ptr(), k,
                                                             nbb.CaRule(), s), K, W, sampler, head_groups)
    value = members * 1e3 / head_ms  # all ranks together update the 3^r cells per step
    results["ca_lambda_compact_i64"] = head_ms
    single = None
    if world == 1:  # the same K steps with one launch per step (ca_compact_kernel)
        single_ms = timed_run(lambda k: dev.ca_compact_run_dev(cfg(flags=nbb_abi.FLAG_SINGLE_STEP), c1.data_ptr(),
                                                               c2.data_ptr(), k, nbb.CaRule(), s), K, W)
        results["ca_lambda_compact_i64_single_step"] = single_ms
        highlife = nbb.CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))
        generic_ms = timed_run(lambda k: dev.ca_compact_run_dev(cfg(), c1.data_ptr(), c2.data_ptr(), k,
                                                                highlife, s), K, W)
        results["ca_lambda_compact_i64_generic_rule"] = generic_ms
        single = {"note": "the headline's K steps with one launch per step (ca_compact_kernel, "
                          "NBB_FLAG_SINGLE_STEP): 8 B read + 8 B write per member and step",
                  "ms_per_step": single_ms, "value": members * 1e3 / single_ms,
                  "roofline": {"achieved": 16 * members / (single_ms * 1e-3) / 1e9,
                               "frac": 16 * members / (single_ms * 1e-3) / 1e9 / measured_peaks()[0],
                               "alg_bytes_per_launch": 16 * members}}
        single["generic_rule_two_step"] = {
            "note": "the headline's two-step passes with a rule other than B3/S23 (B36/S23): the "
                    "generic instantiation, rule masks read at run time",
            "ms_per_step": generic_ms, "value": members * 1e3 / generic_ms}
    # ---- C5: the same step on the gasket at n = 2^17 (BASELINE configs[4]), sharded by
    # contiguous compact tile ranges at N > 1 (halos over peer memory inside the kernel) ------
    c5 = None
    if world == 1 or args.transport == "p2p":
        r5 = args.level + 1
        m5 = 3 ** r5
        gen = torch.Generator(device="cuda")
        gen.manual_seed(18)
        d1 = torch.randint(0, 2, (m5,), dtype=torch.int64, device="cuda", generator=gen)
        cfg5 = nbb.DispatchConfig(r=r5, rho=32, max_cells=(1 << r5) ** 2, device=local)
        if world > 1:
            plan5 = shard.ShardPlan(r=r5, rho=32, world=world, rank=rank, state="compact")
            p5 = shard.P2PCompactCA(plan5, dist, device=local)
            p5.load(d1)
            ms5 = timed_run(lambda k: p5.run(cfg5, nbb.CaRule(), k, s), K, W)
            p5.check(s)
            p5.close()
        else:
            d2 = torch.empty_like(d1)
            ms5 = timed_run(lambda k: dev.ca_compact_run_dev(cfg5, d1.data_ptr(), d2.data_ptr(), k,
                                                             nbb.CaRule(), s), K, W)
            del d2
        del d1
        p5, s5 = pair_launches(K, world, args.transport)
        ach5 = 16 * m5 * (p5 + s5) / K / (ms5 * 1e-3) / 1e9  # state bytes moved per step
        c5 = {"workload": f"C5: gasket n=2^{r5} CA step (B3/S23), compact state, rho=32 tiles, "
                          f"{world} rank(s), contiguous compact tile ranges",
              "data": "synthetic: iid alive values (torch.randint(0, 2), seed 18) over the 3^r member "
                      "cells of the compact state",
              "r": r5, "cells_per_step": m5, "ms_per_step": ms5, "value": m5 * 1e3 / ms5,
              "unit": "cells/s", "per_gpu_GBps": ach5 / world,
              "per_gpu_roofline_frac": ach5 / world / measured_peaks()[0]}
    # ---- the bounding-box launch over the SAME compact state (culled box tiles, λ⁻¹ addressing)
    if world == 1:
        results["ca_bb_compact_i64"] = timed_run(
            lambda k: dev.ca_compact_run_dev(cfg(mode=nbb.MapMode.BoundingBox), c1.data_ptr(), c2.data_ptr(), k,
                                             nbb.CaRule(), s), K, W)
    # ---- the same step on the reference's int64 embedded Grid layout --------------------
    emb_ms = timed(ca_runner(cfg(), a, b), K, W)
    results["ca_lambda_tile_rho32_i64"] = emb_ms

    # the other CA launch shapes (each on its own timed loop; K shortened for slow BB)
    variants = {
        "ca_lambda_tile_rho16_i64": cfg(rho=16),
        "ca_lambda_tile_rho8_i64": cfg(rho=8),
        "ca_bb_tile_rho32_i64": cfg(mode=nbb.MapMode.BoundingBox),
        "ca_bb_tile_rho16_i64": cfg(mode=nbb.MapMode.BoundingBox, rho=16),
        "ca_bb_percell_rho32_i64": cfg(mode=nbb.MapMode.BoundingBox, kernel=nbb.KernelFamily.PerCell),
        "ca_bb_percell_rho16_i64": cfg(mode=nbb.MapMode.BoundingBox, rho=16,
                                       kernel=nbb.KernelFamily.PerCell),
        "ca_lambda_percell_rho32_i64": cfg(kernel=nbb.KernelFamily.PerCell),
        "ca_lambda_percell_rho16_i64": cfg(rho=16, kernel=nbb.KernelFamily.PerCell),
    }
    sweep = None
    if world == 1:
        for name, c in variants.items():
            kk = K if "tile" in name else max(5, K // 10)
            results[name] = timed(ca_runner(c, a, b), kk, W)

        # uint8 / 1-bit alive states (exact: CA only reads != 0 and writes 0/1)
        a8 = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
        b8 = torch.zeros_like(a8)
        dev.pack_alive_dev(cfg(cell_width=1), a.data_ptr(), a8.data_ptr(), s)
        results["ca_lambda_tile_rho32_u8"] = timed(ca_runner(cfg(cell_width=1), a8, b8), K, W)
        results["ca_bb_tile_rho32_u8"] = timed(
            ca_runner(cfg(cell_width=1, mode=nbb.MapMode.BoundingBox), a8, b8), K, W)
        del a8, b8
        w1 = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
        w2 = torch.zeros_like(w1)
        dev.pack_alive_dev(cfg(cell_width=0), a.data_ptr(), w1.data_ptr(), s)
        results["ca_lambda_tile_rho32_bit"] = timed(ca_runner(cfg(cell_width=0), w1, w2), K, W)
        results["ca_bb_tile_rho32_bit"] = timed(
            ca_runner(cfg(cell_width=0, mode=nbb.MapMode.BoundingBox), w1, w2), K, W)
        del w1, w2

        # single write and reduction (C2 / C3-RD) on the same buffers
        def sw(c):
            return lambda: dev.single_write_dev(c, b.data_ptr(), s)
        out = torch.zeros(1, dtype=torch.int64, device="cuda")

        def rd(c):
            return lambda: dev.reduction_dev(c, a.data_ptr(), out.data_ptr(), s)
        for name, c in {"sw_lambda_tile_rho32": cfg(), "sw_bb_tile_rho32": cfg(mode=nbb.MapMode.BoundingBox),
                        "sw_bb_percell_rho32": cfg(mode=nbb.MapMode.BoundingBox, kernel=nbb.KernelFamily.PerCell),
                        "sw_lambda_percell_rho32": cfg(kernel=nbb.KernelFamily.PerCell),
                        "sw_lambda_percell_rho16": cfg(rho=16, kernel=nbb.KernelFamily.PerCell),
                        # the paper's tensor-core λ (mma.cpp variants 1 and 2)
                        # in the per-cell launch, against its direct backend above
                        "sw_lambda_percell_rho16_mma1": cfg(rho=16, kernel=nbb.KernelFamily.PerCell,
                                                            backend=nbb.LambdaBackend.MmaV1),
                        "sw_lambda_percell_rho16_mma2": cfg(rho=16, kernel=nbb.KernelFamily.PerCell,
                                                            backend=nbb.LambdaBackend.MmaV2)}.items():
            results[name] = timed(sw(c), K if "tile" in name else max(5, K // 10), W)
        for name, c in {"rd_lambda_tile_rho32": cfg(), "rd_bb_tile_rho32": cfg(mode=nbb.MapMode.BoundingBox),
                        "rd_bb_percell_rho32": cfg(mode=nbb.MapMode.BoundingBox, kernel=nbb.KernelFamily.PerCell),
                        "rd_lambda_percell_rho32": cfg(kernel=nbb.KernelFamily.PerCell),
                        "rd_lambda_percell_rho16": cfg(rho=16, kernel=nbb.KernelFamily.PerCell)}.items():
            results[name] = timed(rd(c), K if "tile" in name else max(5, K // 10), W)
        results["rd_lambda_compact_i64"] = timed(
            lambda: dev.reduction_compact_dev(cfg(), c1.data_ptr(), out.data_ptr(), s), K, W)
        results["sw_lambda_compact_i64"] = timed(
            lambda: dev.single_write_compact_dev(cfg(), c2.data_ptr(), s), K, W)

        # C4: the λ map alone over a whole orthotope, scalar closed form vs tensor core (K0-TC)
        xy = torch.empty(3 ** 17 * 2, dtype=torch.int32, device="cuda")
        sweep = {}
        for lvl in (10, 12, 14, 16, 17):
            row = {"omegas": 3 ** lvl}
            for label, be in (("scalar", nbb.LambdaBackend.Direct),
                              ("tensor_core_tcgen05", nbb.LambdaBackend.MmaV2),
                              ("tensor_core_mma_sync", nbb.LambdaBackend.MmaV1)):
                if be == nbb.LambdaBackend.MmaV1 and lvl > 16:  # the paper's V1: r_b <= 16
                    continue
                c = cfg(backend=be)
                ms = timed(lambda: dev.lambda_coords_dev(c, lvl, xy.data_ptr(), 4, s), max(5, K // 4), W)
                row[label + "_ms"] = ms
                row[label + "_omega_per_s"] = 3 ** lvl * 1e3 / ms
            sweep[str(lvl)] = row
        del xy
    del c1, c2

    # ---- roofline of the dominant kernel (ca_compact2_kernel at N = 1) ------------------
    peak, peak_kind = measured_peaks()
    alg_bytes = 2 * 8 * members            # read src + write dst, 8 B per member, per launch (pass)
    n_pairs, n_single = pair_launches(K, world, args.transport)
    launch_ms = head_ms * K / (n_pairs + n_single)  # average launch (pass) duration
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    traffic = emb_traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            tj = json.load(f)
        traffic = tj.get("ca_lambda_compact2_i64" if n_pairs else "ca_lambda_compact_i64")
        emb_traffic = tj.get("ca_lambda_tile_rho32_i64")
    emb_alg = 2 * layout_bytes_per_pass(r, 8)  # 32-byte sectors holding a member, read + write
    emb_achieved = emb_alg / (emb_ms * 1e-3) / 1e9

    # ---- e2e through the public C ABI with pinned host buffers -------------------------
    # nbb_gpu_ca(cfg, host_initial, K steps, rule, host_out) = the reference's
    # run_ca(cfg, grid, K): the int64 Grid crosses PCIe in (member sectors read in place from
    # the pinned grid), K steps run on the device state, the result comes back (member
    # sectors written in place into the pinned output, FLAG_OUT_ZEROED: allocated zeroed
    # once, outside the timed region). One call = K steps; a 1-step call is timed too.
    e2e = None
    if world == 1 and not args.no_e2e:
        del a, b
        torch.cuda.empty_cache()
        hin = torch.empty((n, n), dtype=torch.int64, pin_memory=True)
        hout = torch.zeros((n, n), dtype=torch.int64).pin_memory()
        lib = nbb._lib()
        lib.nbb_gpu_random_member_grid(ctypes.byref(spec.to_c()), r, 17, 2, n * n,
                                       ctypes.c_void_p(hin.data_ptr()))
        member_bytes = layout_bytes_per_pass(r, 8)
        runs = {}

        def call(cc, steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = lib.nbb_gpu_ca(ctypes.byref(cc), ctypes.c_void_p(hin.data_ptr()), r, steps, 8, 12,
                                ctypes.c_void_p(hout.data_ptr()), None)
            t1 = time.perf_counter()
            if rc:
                raise RuntimeError(lib.nbb_gpu_last_error().decode())
            return t1 - t0
        for label, cw, fl in (("compact", 8, nbb_abi.FLAG_COMPACT_STATE), ("int64", 8, 0), ("bit", 0, 0)):
            cc = cfg(cell_width=cw, flags=nbb_abi.FLAG_OUT_ZEROED | fl).to_c()
            call(cc, 2)  # warm (allocations)
            runs[label] = call(cc, K)
            if label == "compact":
                runs["compact_1step"] = min(call(cc, 1) for _ in range(3))
        e2e = {"value": members * K / runs["compact"], "unit": "cells/s",
               "h2d_bytes_per_step": member_bytes // K, "d2h_bytes_per_step": member_bytes // K,
               "call": f"nbb_gpu_ca(cfg, pinned host_initial int64 Grid, steps={K}, B3/S23, pinned "
                       f"host_out, FLAG_OUT_ZEROED|FLAG_COMPACT_STATE) = the reference's run_ca(cfg, "
                       f"grid, {K}); the {member_bytes / 1e6:.0f} MB of member sectors cross PCIe in place "
                       f"(zero-copy) each way per call; wall time of the whole call",
               "seconds": runs["compact"],
               "one_step_call": {"value": members / runs["compact_1step"], "seconds": runs["compact_1step"],
                                 "h2d_bytes_per_step": member_bytes, "d2h_bytes_per_step": member_bytes},
               "other_states": {k: {"value": members * K / runs[k], "seconds": runs[k]}
                                for k in ("int64", "bit")}}
        del hin, hout
        nbb.release()
    elif world > 1:
        e2e = {"value": None, "unit": "cells/s",
               "note": "measured at N = 1 only: the host-buffer call takes the reference's whole int64 "
                       "Grid (32 GiB in + 32 GiB out pinned per process at n = 2^16), which N ranks "
                       "on one host cannot each hold"}

    # ---- CPU baseline: the reference on this host's cores (bounded sample) ------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            rs, steps_s = 15, 2
            cores = os.cpu_count() or 1
            secs, micros = reference_ca(rs, 32, steps_s, 16, cores)
            cpu = {"value": 3 ** rs * steps_s / secs, "unit": "cells/s", "cores": cores,
                   "kind": "reference",
                   "sample": f"reference run_ca(r={rs}, rho=32, lambda, workers={cores}), {steps_s} "
                             f"steps in one call, wall time incl. MemberMask build; launch-only "
                             f"micros {micros}"}
        except Exception as e:  # report, don't die
            cpu = {"value": None, "unit": "cells/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    if rank != 0:
        return
    cells = lambda k: members * 1e3 / results[k] if k in results else None  # noqa: E731

    def ratio(bb, lam):
        return results[bb] / results[lam] if bb in results and lam in results else None
    line = {
        "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": head_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64",
        "data": f"synthetic: random_member_grid(gasket, {r}, seed=17, modulus=2) generated "
                "bit-identically on device, B3/S23",
        "config": config_block(r, 32, world, args.transport),
        "gpu_launches": (n_pairs + n_single) * launches_per_step,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_launch": alg_bytes, "peak_kind": peak_kind,
                     "launches": {"two_step": n_pairs, "one_step": n_single},
                     "kernel": ("ca_compact2_kernel: two CA steps per pass, 8 B read + 8 B write per "
                                "member cell per pass" if n_pairs else
                                "ca_compact_kernel (8 B read + 8 B write per member cell)")},
        "one_step_per_launch": single,
        "embedded_int64": {
            "note": "the same step on the reference's int64 embedded Grid (ca_pipe_kernel)",
            "ms_per_step": emb_ms, "value": members * 1e3 / emb_ms,
            "roofline": {"achieved": emb_achieved, "peak": peak, "frac": emb_achieved / peak,
                         "alg_bytes_per_launch": emb_alg, "traffic": emb_traffic,
                         "alg": "32-byte sectors holding a member (SURVEY 8(d)), read + write"},
            "line_granular_floor": {
                "note": "B200 reads whole 128 B lines (probe: tools/probe_dram3.cu); int64 lines "
                        "holding a member: 2^4*3^12 x 128 B = 1088.4 MB read + 612.2 MB sector writes",
                "hw_min_bytes_per_step": 1088391168 + 612220032,
                "achieved_GBps_vs_hw_min": (1088391168 + 612220032) / (emb_ms * 1e-3) / 1e9},
        },
        "timing": {"ms_per_step_mean": head_ms,
                   "sub_runs": len(head_groups),
                   "ms_per_step_median_of_sub_runs": statistics.median(head_groups) if head_groups else None,
                   "ms_per_step_mean_of_sub_averages": statistics.mean(head_groups) if head_groups else None,
                   "ms_per_step_min_max_sub_run": [min(head_groups), max(head_groups)] if head_groups else None,
                   "note": "CUDA events on the launching stream; K steps split into equal sub-runs "
                           "(SURVEY 8(d): median and the paper's mean of sub-averages)"},
        "clocks": sampler.summary(),
        "speedup_vs_bb": {
            "headline": {
                "value": ratio("ca_bb_tile_rho32_i64", "ca_lambda_compact_i64"),
                "definition": "the lambda(omega) CA step (compact state, two steps per pass: the headline) "
                              "over the best bounding-box launch of the same step on the reference's int64 "
                              "Grid (tile kernel with tile culling, one step per launch); the map alone "
                              "(both one step per launch, same compact storage) and paper-style ratios below"},
            "ca_lambda_compact_single_step_over_bb_tile_i64":
                ratio("ca_bb_tile_rho32_i64", "ca_lambda_compact_i64_single_step"),
            "ca_lambda_compact_single_step_over_bb_compact_i64":
                ratio("ca_bb_compact_i64", "ca_lambda_compact_i64_single_step"),
            "ca_lambda_compact_over_bb_tile_i64": ratio("ca_bb_tile_rho32_i64", "ca_lambda_compact_i64"),
            "ca_lambda_compact_over_bb_compact_i64": ratio("ca_bb_compact_i64", "ca_lambda_compact_i64"),
            "ca_lambda_compact_over_bb_percell_i64": ratio("ca_bb_percell_rho32_i64", "ca_lambda_compact_i64"),
            "ca_embedded_i64_bb_tile_over_lambda_tile": ratio("ca_bb_tile_rho32_i64", "ca_lambda_tile_rho32_i64"),
            "ca_embedded_i64_bb_percell_over_lambda_percell": ratio("ca_bb_percell_rho32_i64",
                                                                   "ca_lambda_percell_rho32_i64"),
            "ca_u8_bb_over_lambda": ratio("ca_bb_tile_rho32_u8", "ca_lambda_tile_rho32_u8"),
            "ca_bit_bb_over_lambda": ratio("ca_bb_tile_rho32_bit", "ca_lambda_tile_rho32_bit"),
            "sw_bb_tile_over_lambda_tile": ratio("sw_bb_tile_rho32", "sw_lambda_tile_rho32"),
            "rd_bb_tile_over_lambda_tile": ratio("rd_bb_tile_rho32", "rd_lambda_tile_rho32"),
            "rd_bb_tile_over_lambda_compact": ratio("rd_bb_tile_rho32", "rd_lambda_compact_i64"),
            # the paper's own comparison (one thread per cell, ρ = 32 blocks; PAPER.md:548-549
            # reports 6x-12x at n = 2^16 on Titan V / Titan RTX)
            "paper_tc_percell_rho16_sw": {  # V2 ~20-40% faster than scalar
                "mma1_over_direct": ratio("sw_lambda_percell_rho16", "sw_lambda_percell_rho16_mma1"),
                "mma2_over_direct": ratio("sw_lambda_percell_rho16", "sw_lambda_percell_rho16_mma2")},
            "paper_percell_rho32": {
                "sw": ratio("sw_bb_percell_rho32", "sw_lambda_percell_rho32"),
                "rd": ratio("rd_bb_percell_rho32", "rd_lambda_percell_rho32"),
                "ca": ratio("ca_bb_percell_rho32_i64", "ca_lambda_percell_rho32_i64")},
        },
        "workloads_ms": results,
        "workloads_cells_per_s": {k: cells(k) for k in results},
        "map_sweep_C4": sweep,
        "c5_r17": c5,
        "rd_compact": rd_line,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
