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
SPACER_CYCLES = 1_000_000  # ~0.5 ms at 1.97 GHz (timed_run)


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
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_ca(r: int, rho: int, steps: int, seed: int, workers: int):
    """The unmodified reference run_ca (oracle/_ref/libnbbref.so) on host cores. The input is
    random_member_grid(gasket, r, seed, 2) written by the C oracle's restatement (test
    infrastructure, O(3^r)); nothing of the product library is loaded on this path."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    from _oracle import orc_lib, ref_lib
    from paper_2004_13475_b200 import _abi  # ctypes structs only (no library load)
    from paper_2004_13475_b200.nbb import DispatchConfig, FractalSpec, MapMode
    ref, orc = ref_lib(), orc_lib()
    spec = FractalSpec.sierpinski()
    n = 1 << r
    h = ref.ref_grid_create(ctypes.byref(spec.to_c()), r)
    if not h:
        raise MemoryError(ref.ref_last_error().decode())
    try:
        data = ctypes.c_void_p(ref.ref_grid_data(h))
        t0 = time.perf_counter()
        orc.orc_random_member_grid(ctypes.byref(spec.to_c()), r, seed, 2, data)  # input prep, untimed
        prep = time.perf_counter() - t0
        cfg = DispatchConfig(r=r, rho=rho, mode=MapMode.Lambda, workers=workers, timing=True, max_cells=n * n)
        reps = (_abi.NbbReport * steps)()
        secs = ctypes.c_double()
        rc = ref.ref_ca_h(ctypes.byref(cfg.to_c()), h, steps, 8, 12, None, reps, ctypes.byref(secs))
        if rc:
            raise RuntimeError(ref.ref_last_error().decode())
        micros = [reps[i].micros for i in range(steps)]
        del np
        return secs.value, micros, prep
    finally:
        ref.ref_grid_destroy(h)


def reference_block(r, rho, steps, seed, cores, secs, micros):
    """cpu_baseline object for a reference run_ca call (wall of the call and launch-only)."""
    return {"value": 3 ** r * steps / secs, "unit": "cells/s", "cores": cores, "kind": "reference",
            "cpu": cpu_model(),
            "launch_only_value": 3 ** r * steps / (sum(micros) * 1e-6) if sum(micros) else None,
            "sample": f"reference run_ca(gasket, r={r} (n=2^{r}), rho={rho}, lambda/subbox/direct, "
                      f"workers={cores}) on random_member_grid(gasket, {r}, seed={seed}, 2), B3/S23, "
                      f"{steps} step(s) in one call: value = 3^{r} x {steps} / wall time of the call "
                      f"({secs:.1f} s, incl. its MemberMask build and per-step grid fills); "
                      f"launch_only_value from the reference's own per-step micros {micros}"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r, rho = args.level, 32
    steps = max(1, min(args.steps, args.ref_max_steps))
    cores = os.cpu_count() or 1
    secs, micros, _ = reference_ca(r, rho, steps, 1 + r, cores)
    value = 3 ** r * steps / secs
    line = {
        "metric": METRIC, "value": value, "unit": "cells/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": 0, "ms_per_step": 1e3 * secs / steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": f"synthetic: random_member_grid(gasket, {r}, seed={1 + r}, modulus=2) (C oracle), B3/S23",
        "config": config_block(r, rho, args.gpus),
        "cpu_baseline": reference_block(r, rho, steps, 1 + r, cores, secs, micros),
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(r, rho, world=1, transport="p2p"):
    return {"workload": f"C3: gasket n=2^{r} cellular-automaton step (B3/S23), lambda(omega) launch, "
                        f"rho={rho} tiles; device state = the lambda-ordered compact layout "
                        f"(CompactGrid, 8 B per member), host I/O = the reference's int64 Grid; "
                        + "up to 8 steps per pass over the state (" + (
                            "ca_compact_cluster_kernel: batches of 27 tiles = one level-3 sub-gasket"
                            if world == 1 else "ca_compact_sliced_kernel<P2P>") + ")",
            "r": r, "n": 1 << r, "rho": rho, "mode": "lambda", "cells_per_step": 3 ** r,
            "cell": "int64", "state": "compact",
            "parallelism": "1 GPU" if world == 1 else
                           f"{world} ranks: contiguous tile-range shards; " + (
                               "halo cells read over peer memory (CUDA IPC) inside the pass kernel"
                               if transport == "p2p" else
                               f"halo cells exchanged by the library's NCCL communicator (gather + "
                               f"ncclSend/ncclRecv + scatter) before every pass ({transport})"),
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
    ap.add_argument("--cpu-steps", type=int, default=1, help="steps of the cpu_baseline reference call")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="headline, roofline and e2e only")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 halo exchange: inside the pass kernel over peer memory (p2p, "
                         "default) or the library's NCCL communicator before every pass (nccl)")
    ap.add_argument("--profile", action="store_true",
                    help="only run a few λ/BB CA passes (for ncu); prints nothing")
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
    CONWAY = nbb.CaRule()

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
    vals = torch.from_numpy(nbb.random_member_values(spec, r, 1 + r, 2)).cuda()
    dev.scatter_members_dev(cfg(), vals.data_ptr(), a.data_ptr(), s)
    del vals
    b = torch.zeros_like(a)
    torch.cuda.synchronize()

    from paper_2004_13475_b200 import shard
    plan = shard.ShardPlan(r=r, rho=32, world=world, rank=rank)
    plan_c = shard.ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")

    def ca_runner(c, src, dst):  # one launch per step on the embedded grid
        bufs = [src, dst]
        state = {"i": 0}

        def run(k):
            for _ in range(k):
                i = state["i"]
                if world > 1:
                    plan.exchange_halo(bufs[i & 1], dist)
                    dev.ca_step_dev(plan.local_config(c), bufs[i & 1].data_ptr(),
                                    bufs[(i + 1) & 1].data_ptr(), CONWAY, s)
                else:
                    dev.ca_step_dev(c, bufs[i & 1].data_ptr(), bufs[(i + 1) & 1].data_ptr(), CONWAY, s)
                state["i"] = i + 1
        return run

    def timed_run(run, K, W, sampler=None, reps=1):
        """run(k) issues k steps on `stream`. W warm-up steps, then K steps timed with CUDA events
        on the launching stream, a barrier + synchronize on both sides, max over ranks; `reps`
        more timed runs of K steps each (the median / mean of all reported in `timing`)."""
        if sampler:  # NVML sampling from the warm-up on
            sampler.__enter__()
        run(W)
        times = []
        for _ in range(reps):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # a ~0.5 ms spin kernel ahead of e0: the host enqueues e0 and the K steps' launches while
            # it runs, so the timed region holds the steps' device time and no host launch latency
            # (which the e2e line measures); the steps themselves are unchanged
            torch.cuda._sleep(SPACER_CYCLES)
            e0.record(stream)
            run(K)
            e1.record(stream)
            e1.synchronize()
            barrier()
            times.append(max_over_ranks(e0.elapsed_time(e1)) / K)
        if sampler:
            sampler.__exit__()
        return times[0], times  # ms per step of the first timed run, all runs

    # the compact CA state (λ-ordered CompactGrid): every byte a member value (int64)
    c1 = torch.empty(members, dtype=torch.int64, device="cuda")
    c2 = torch.empty_like(c1)
    dev.compact_store_dev(cfg(), a.data_ptr(), c1.data_ptr(), s)
    c0 = c1.clone()  # the initial state, restored before each configuration

    def compact_runner(c, rule=CONWAY):
        """k steps through nbb_gpu_ca_compact_passes_dev (no parity pass): the result lands in
        whichever buffer the last pass wrote; the next call continues from there."""
        st = {"cur": 0, "stats": []}
        bufs = (c1, c2)

        def run(k):
            x, y = bufs[st["cur"]], bufs[st["cur"] ^ 1]
            ps = dev.ca_compact_passes_dev(c, x.data_ptr(), y.data_ptr(), k, rule, s)
            st["stats"].append((k, ps.passes, list(ps.by_steps)))
            st["cur"] ^= ps.result_in_b
        return run, st

    if args.profile:
        run, _ = compact_runner(cfg())
        run(24)
        run, _ = compact_runner(cfg(mode=nbb.MapMode.BoundingBox))
        run(16)
        run, _ = compact_runner(cfg(flags=nbb_abi.FLAG_SINGLE_STEP))
        run(3)
        torch.cuda.synchronize()
        return

    K, W = args.steps, args.warmup
    sampler = ClockSampler(local)
    results = {}
    gpu_launches = None

    # ---- headline: λ(ω) CA steps on the compact state, passes of up to 8 steps -----------
    p2p = None
    launches_per_step = 1
    if world > 1 and args.transport == "p2p":
        try:
            p2p = shard.P2PCompactCA(plan_c, dist, device=local)
        except shard.P2PUnavailable as e:  # every rank agrees; run the NCCL exchange instead
            print(f"bench: {e}; falling back to --transport nccl", file=sys.stderr)
            args.transport = "nccl (p2p unavailable)"
    head_stats = None
    if p2p is not None:
        p2p.load(c1)
        passes_before = {}

        def p2p_run(k):
            passes_before.setdefault("first", p2p.pass_index)
            p2p.run(cfg(), CONWAY, k, s)
        head_ms, head_all = timed_run(p2p_run, K, W, sampler, reps=3)
        p2p.check(s)
        p2p.close()
        ps = dev.pass_plan(plan_c.local_config(cfg()), K)
        head_stats = {"passes": ps.passes, "by_steps": list(ps.by_steps)}
    elif world > 1:  # the library's NCCL communicator: halo exchange (ncclSend/Recv) before each pass
        ca_n = shard.NcclCompactCA(r, dist, local)
        ca_n.load(c1)
        head_ms, head_all = timed_run(lambda k: ca_n.run(cfg(), CONWAY, k, s), K, W, sampler, reps=3)
        ca_n.close()
        ps = dev.pass_plan(plan_c.local_config(cfg()), K)
        head_stats = {"passes": ps.passes, "by_steps": list(ps.by_steps)}
        launches_per_step = 3
    else:
        run, st = compact_runner(cfg())
        head_ms, head_all = timed_run(run, K, W, sampler, reps=5)
        k1, np1, by1 = st["stats"][1]  # the first timed run of K steps
        head_stats = {"passes": np1, "by_steps": by1}
    nccl_line = None
    if world > 1 and p2p is not None and world <= ndev:  # the other transport: the library's NCCL communicator
        try:
            c1.copy_(c0)
            ca_n = shard.NcclCompactCA(r, dist, local)
            ca_n.load(c1)
            n_ms, n_all = timed_run(lambda k: ca_n.run(cfg(), CONWAY, k, s), K, W, None, reps=3)
            ca_n.close()
            nccl_line = {"transport": "nbb_gpu_ca_compact_comm_dev: halo cells by ncclSend/ncclRecv before every "
                                      "pass (gather + group exchange + scatter), same passes",
                         "ms_per_step": n_ms, "value": members * 1e3 / n_ms, "runs": n_all}
        except Exception as e:  # noqa: BLE001 - report, keep the p2p line
            nccl_line = {"error": f"{type(e).__name__}: {e}"}
    value = members * 1e3 / head_ms  # all ranks together update the 3^r cells per step
    results["ca_lambda_compact_i64"] = head_ms
    gpu_launches = head_stats["passes"] * (3 if launches_per_step == 3 else 1)

    # the same K steps with one launch per step, a rule other than B3/S23, and the bounding-box
    # walk over the same compact state with the same passes (N = 1)
    def compact_timed(name, c, rule=CONWAY, reps=1):
        c1.copy_(c0)
        run, st = compact_runner(c, rule)
        ms, _ = timed_run(run, K, W, None, reps)
        results[name] = ms
        return ms, st["stats"][1]
    extras = world == 1 and not args.no_extras
    if extras:
        compact_timed("ca_lambda_compact_i64_single_step", cfg(flags=nbb_abi.FLAG_SINGLE_STEP))
        compact_timed("ca_lambda_compact_i64_generic_rule", cfg(),
                      nbb.CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3)))
        compact_timed("ca_bb_compact_i64", cfg(mode=nbb.MapMode.BoundingBox))
        compact_timed("ca_bb_compact_i64_single_step", cfg(mode=nbb.MapMode.BoundingBox,
                                                           flags=nbb_abi.FLAG_SINGLE_STEP))
        for kk in (2, 4, 12):
            compact_timed(f"ca_lambda_compact_i64_pass{kk}", cfg(pass_steps=kk))

    # ---- C5: the same step on the gasket at n = 2^17 (BASELINE configs[4]), sharded by
    # contiguous compact tile ranges at N > 1 (halos over peer memory inside the kernel) ------
    c5 = None
    if (world == 1 and not args.no_extras) or (world > 1 and args.transport == "p2p"):
        r5 = args.level + 1
        m5 = 3 ** r5
        gen = torch.Generator(device="cuda")
        gen.manual_seed(18)
        del a, b
        torch.cuda.empty_cache()
        d1 = torch.randint(0, 2, (m5,), dtype=torch.int64, device="cuda", generator=gen)
        cfg5 = nbb.DispatchConfig(r=r5, rho=32, max_cells=(1 << r5) ** 2, device=local)
        if world > 1:
            plan5 = shard.ShardPlan(r=r5, rho=32, world=world, rank=rank, state="compact")
            p5 = shard.P2PCompactCA(plan5, dist, device=local)
            p5.load(d1)
            ms5, _ = timed_run(lambda k: p5.run(cfg5, CONWAY, k, s), K, W)
            p5.check(s)
            p5.close()
            ps5 = dev.pass_plan(plan5.local_config(cfg5), K)
        else:
            d2 = torch.empty_like(d1)
            cur = {"x": 0}

            def run5(k):
                bb = (d1, d2)
                ps = dev.ca_compact_passes_dev(cfg5, bb[cur["x"]].data_ptr(), bb[cur["x"] ^ 1].data_ptr(),
                                               k, CONWAY, s)
                cur["x"] ^= ps.result_in_b
            ms5, _ = timed_run(run5, K, W)
            del d2
            ps5 = dev.pass_plan(cfg5, K)
        del d1
        ach5 = 16 * m5 * ps5.passes / K / (ms5 * 1e-3) / 1e9  # state bytes moved per step
        c5 = {"workload": f"C5: gasket n=2^{r5} CA step (B3/S23), compact state, rho=32 tiles, "
                          f"{world} rank(s), contiguous compact tile ranges",
              "data": "synthetic: iid alive values (torch.randint(0, 2), seed 18) over the 3^r member "
                      "cells of the compact state",
              "r": r5, "cells_per_step": m5, "ms_per_step": ms5, "value": m5 * 1e3 / ms5,
              "unit": "cells/s", "passes": ps5.passes,
              "per_gpu_GBps_per_pass": ach5 / world,
              "per_gpu_roofline_frac_per_pass": ach5 / world / measured_peaks()[0]}
        a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
        b = torch.zeros_like(a)
        dev.compact_load_dev(cfg(), c0.data_ptr(), a.data_ptr(), 0, s)

    # ---- RD (the global reduction) on the compact state ----------------------------------
    rd_val = shard.sharded_reduction(plan_c, cfg(), c0.data_ptr(), dist, s, local)
    rd_ms, _ = timed_run(lambda k: [shard.sharded_reduction(plan_c, cfg(), c0.data_ptr(), dist, s, local)
                                    for _ in range(k)], max(10, K // 4), W)
    rd_part = torch.empty(1, dtype=torch.int64, device="cuda")
    rd_cfg = plan_c.local_config(cfg())
    rd_kern_ms, _ = timed_run(lambda k: [dev.reduction_compact_dev(rd_cfg, c0.data_ptr(), rd_part.data_ptr(), s)
                                         for _ in range(k)], max(10, K // 4), W)
    rd_line = {"workload": f"run_reduction on the compact state at n=2^{r}: per-rank partial over its tiles "
                           f"(segment_sum_kernel) + one int64 all-reduce, value read back on the host",
               "ms_per_call": rd_ms, "value": members * 1e3 / rd_ms, "unit": "cells/s", "sum": rd_val,
               "kernel_only": {"ms": rd_kern_ms, "GBps": 8 * members / world / (rd_kern_ms * 1e-3) / 1e9,
                               "frac": 8 * members / world / (rd_kern_ms * 1e-3) / 1e9 / measured_peaks()[0]}}

    # ---- the same step on the reference's int64 embedded Grid layout, and other launches ---
    sweep = None
    if extras:
        results["ca_lambda_tile_rho32_i64"], _ = timed_run(ca_runner(cfg(), a, b), K, W)
        # the same K steps on the embedded int64 grid, temporally blocked (nbb_gpu_ca_run_dev: member
        # sectors -> compact state -> passes -> member sectors of the result buffer)
        eb = {"x": 0}

        def emb_run(k):
            bufs = (a, b)
            dev.ca_run_dev(cfg(), bufs[eb["x"]].data_ptr(), bufs[eb["x"] ^ 1].data_ptr(), k, CONWAY, s)
            eb["x"] ^= k & 1
        results["ca_lambda_embedded_i64_blocked"], _ = timed_run(emb_run, K, W)
        variants = {
            "ca_bb_tile_rho32_i64": cfg(mode=nbb.MapMode.BoundingBox),
            "ca_bb_percell_rho32_i64": cfg(mode=nbb.MapMode.BoundingBox, kernel=nbb.KernelFamily.PerCell),
            "ca_lambda_percell_rho32_i64": cfg(kernel=nbb.KernelFamily.PerCell),
        }
        for name, c in variants.items():
            results[name], _ = timed_run(ca_runner(c, a, b), K if "tile" in name else max(5, K // 10), W)
        a8 = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
        b8 = torch.zeros_like(a8)
        dev.pack_alive_dev(cfg(cell_width=1), a.data_ptr(), a8.data_ptr(), s)
        results["ca_lambda_tile_rho32_u8"], _ = timed_run(ca_runner(cfg(cell_width=1), a8, b8), K, W)
        results["ca_bb_tile_rho32_u8"], _ = timed_run(
            ca_runner(cfg(cell_width=1, mode=nbb.MapMode.BoundingBox), a8, b8), K, W)
        del a8, b8
        w1 = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
        w2 = torch.zeros_like(w1)
        dev.pack_alive_dev(cfg(cell_width=0), a.data_ptr(), w1.data_ptr(), s)
        results["ca_lambda_tile_rho32_bit"], _ = timed_run(ca_runner(cfg(cell_width=0), w1, w2), K, W)
        results["ca_bb_tile_rho32_bit"], _ = timed_run(
            ca_runner(cfg(cell_width=0, mode=nbb.MapMode.BoundingBox), w1, w2), K, W)
        del w1, w2
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        for name, c in {"sw_lambda_tile_rho32": cfg(), "sw_bb_tile_rho32": cfg(mode=nbb.MapMode.BoundingBox),
                        "sw_bb_percell_rho32": cfg(mode=nbb.MapMode.BoundingBox, kernel=nbb.KernelFamily.PerCell),
                        "sw_lambda_percell_rho32": cfg(kernel=nbb.KernelFamily.PerCell),
                        "sw_lambda_percell_rho16": cfg(rho=16, kernel=nbb.KernelFamily.PerCell),
                        "sw_lambda_percell_rho16_mma1": cfg(rho=16, kernel=nbb.KernelFamily.PerCell,
                                                            backend=nbb.LambdaBackend.MmaV1),
                        "sw_lambda_percell_rho16_mma2": cfg(rho=16, kernel=nbb.KernelFamily.PerCell,
                                                            backend=nbb.LambdaBackend.MmaV2)}.items():
            results[name], _ = timed_run(lambda k, c=c: [dev.single_write_dev(c, b.data_ptr(), s) for _ in range(k)],
                                         K if "tile" in name else max(5, K // 10), W)
        for name, c in {"rd_lambda_tile_rho32": cfg(), "rd_bb_tile_rho32": cfg(mode=nbb.MapMode.BoundingBox),
                        "rd_bb_percell_rho32": cfg(mode=nbb.MapMode.BoundingBox, kernel=nbb.KernelFamily.PerCell),
                        "rd_lambda_percell_rho32": cfg(kernel=nbb.KernelFamily.PerCell)}.items():
            results[name], _ = timed_run(
                lambda k, c=c: [dev.reduction_dev(c, a.data_ptr(), out.data_ptr(), s) for _ in range(k)],
                K if "tile" in name else max(5, K // 10), W)
        results["rd_lambda_compact_i64"], _ = timed_run(
            lambda k: [dev.reduction_compact_dev(cfg(), c0.data_ptr(), out.data_ptr(), s) for _ in range(k)], K, W)
        # C4: the λ map alone over a whole orthotope, scalar closed form vs tensor core (K0-TC)
        xy = torch.empty(3 ** 17 * 2, dtype=torch.int32, device="cuda")
        sweep = {}
        for lvl in (10, 12, 14, 16, 17):
            row = {"omegas": 3 ** lvl}
            for label, be in (("scalar", nbb.LambdaBackend.Direct), ("tensor_core_tcgen05", nbb.LambdaBackend.MmaV2),
                              ("tensor_core_mma_sync", nbb.LambdaBackend.MmaV1)):
                if be == nbb.LambdaBackend.MmaV1 and lvl > 16:  # the paper's V1: r_b <= 16
                    continue
                c = cfg(backend=be)
                ms, _ = timed_run(lambda k, c=c, lvl=lvl: [dev.lambda_coords_dev(c, lvl, xy.data_ptr(), 4, s)
                                                           for _ in range(k)], max(5, K // 4), W)
                row[label + "_ms"] = ms
                row[label + "_omega_per_s"] = 3 ** lvl * 1e3 / ms
            sweep[str(lvl)] = row
        del xy
    del c1, c2

    # ---- roofline of the dominant kernel: the headline's passes ---------------------------
    peak, peak_kind = measured_peaks()
    alg_bytes = 2 * 8 * members // world   # per pass and GPU: read src + write dst, 8 B per member
    n_pass = head_stats["passes"]
    launch_ms = head_ms * K / n_pass       # average pass (launch) duration, CUDA events
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get("ca_compact_cluster_kernel_k8" if world == 1 else
                                       "ca_compact_sliced_kernel_k8")

    # ---- e2e through the public C ABI with pinned host buffers -------------------------
    e2e = None
    if world == 1 and not args.no_e2e:
        del a, b
        torch.cuda.empty_cache()
        hin = torch.empty((n, n), dtype=torch.int64, pin_memory=True)
        hout = torch.zeros((n, n), dtype=torch.int64).pin_memory()
        lib = nbb._lib()
        lib.nbb_gpu_random_member_grid(ctypes.byref(spec.to_c()), r, 1 + r, 2, n * n,
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
        for label, cw, fl in (("compact", 8, 0), ("int64", 8, nbb_abi.FLAG_EMBEDDED_STATE),
                              ("bit", 0, nbb_abi.FLAG_EMBEDDED_STATE)):
            cc = cfg(cell_width=cw, flags=nbb_abi.FLAG_OUT_ZEROED | fl).to_c()
            call(cc, 2)  # warm (allocations)
            runs[label] = call(cc, K)
            if label == "compact":
                runs["compact_1step"] = min(call(cc, 1) for _ in range(3))
        e2e = {"value": members * K / runs["compact"], "unit": "cells/s",
               "h2d_bytes_per_step": member_bytes // K, "d2h_bytes_per_step": member_bytes // K,
               "call": f"nbb_gpu_ca(cfg, pinned host_initial int64 Grid, steps={K}, B3/S23, pinned host_out, "
                       f"FLAG_OUT_ZEROED) = the reference's run_ca(cfg, grid, {K}) (device state: compact, the "
                       f"default); the {member_bytes / 1e6:.0f} MB of member sectors cross PCIe in place "
                       f"(zero-copy) each way per call; wall time of the whole call",
               "seconds": runs["compact"],
               "one_step_call": {"value": members / runs["compact_1step"], "seconds": runs["compact_1step"]},
               "other_states": {k: {"value": members * K / runs[k], "seconds": runs[k]} for k in ("int64", "bit")}}
        del hin, hout
        nbb.release()
    elif world > 1:
        e2e = {"value": None, "unit": "cells/s",
               "note": "measured at N = 1 only: the host-buffer call takes the reference's whole int64 "
                       "Grid (32 GiB in + 32 GiB out pinned per process at n = 2^16), which N ranks "
                       "on one host cannot each hold"}

    # ---- CPU baseline: the reference on this host's cores, C3 itself (n = 2^16) ------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cores = os.cpu_count() or 1
            secs, micros, _ = reference_ca(r, 32, args.cpu_steps, 1 + r, cores)
            cpu = reference_block(r, 32, args.cpu_steps, 1 + r, cores, secs, micros)
        except Exception as e:  # report, don't die
            cpu = {"value": None, "unit": "cells/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {type(e).__name__}: {e}"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    cells = lambda k: members * 1e3 / results[k] if k in results else None  # noqa: E731

    def ratio(bb, lam):
        return results[bb] / results[lam] if bb in results and lam in results else None
    line = {
        "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": head_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64",
        "data": f"synthetic: random_member_grid(gasket, {r}, seed={1 + r}, modulus=2) generated "
                "bit-identically on device, B3/S23",
        "config": config_block(r, 32, world, args.transport),
        "gpu_launches": gpu_launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_launch": alg_bytes, "peak_kind": peak_kind,
                     "launches": head_stats,
                     "kernel": ("ca_compact_cluster_kernel<B3/S23>" if world == 1 else
                                "ca_compact_sliced_kernel<B3/S23, P2P>") + ": one launch = one pass of up to 8 "
                               "CA steps over the compact state, 8 B read + 8 B write per member per pass "
                               "(launches.by_steps[k] = passes of k steps); achieved = alg bytes / "
                               "average pass duration (CUDA events over the K timed steps)"},
        "cpu_baseline": cpu,
        "clocks": sampler.summary(),
        "e2e": e2e,
        "timing": {"ms_per_step_runs": head_all,
                   "ms_per_step_median": statistics.median(head_all),
                   "ms_per_step_mean": statistics.mean(head_all),
                   "note": "value = the first timed run of exactly K steps (CUDA events on the launching "
                           "stream, barrier + synchronize on both sides, a 0.5 ms spin kernel ahead of the "
                           "start event so the host's launch latency stays outside); the other runs repeat it"},
        "workloads_ms": results,
        "workloads_cells_per_s": {k: cells(k) for k in results},
        "map_sweep_C4": sweep,
        "c5_r17": c5,
        "nccl_transport": nccl_line,
        "rd_compact": rd_line,
        "embedded_int64": None if "ca_lambda_tile_rho32_i64" not in results else {
            "note": "the same K steps on the reference's int64 embedded Grid in HBM: one launch per step "
                    "(ca_pipe_kernel) and temporally blocked (nbb_gpu_ca_run_dev: the member sectors go once "
                    "into the compact state, K steps in passes, back into the member sectors)",
            "one_step_per_launch_ms": results["ca_lambda_tile_rho32_i64"],
            "blocked_ms_per_step": results.get("ca_lambda_embedded_i64_blocked"),
            "sector_roofline_ms_per_step": 2 * layout_bytes_per_pass(r, 8) / (peak * 1e9) * 1e3,
            "blocked_frac_of_sector_roofline_per_step": (2 * layout_bytes_per_pass(r, 8) / (peak * 1e9) * 1e3) /
                                                        results["ca_lambda_embedded_i64_blocked"]
                                                        if "ca_lambda_embedded_i64_blocked" in results else None},
        "one_step_per_launch": None if "ca_lambda_compact_i64_single_step" not in results else {
            "ms_per_step": results["ca_lambda_compact_i64_single_step"],
            "value": cells("ca_lambda_compact_i64_single_step"),
            "frac_of_peak": 16 * members / (results["ca_lambda_compact_i64_single_step"] * 1e-3) / 1e9 / peak,
            "note": "the headline's K steps with one launch (pass) per step (NBB_FLAG_SINGLE_STEP)"},
        "passes_of_12": None if "ca_lambda_compact_i64_pass12" not in results else {
            "ms_per_step": results["ca_lambda_compact_i64_pass12"],
            "value": cells("ca_lambda_compact_i64_pass12"),
            "frac_per_pass": 16 * members / (results["ca_lambda_compact_i64_pass12"] * K / -(-K // 12) * 1e-3)
                             / 1e9 / peak,
            "note": "the headline's K steps in passes of up to 12 (pass_steps = 12, the cluster walk's most): "
                    "faster per step, the pass no longer at the HBM roofline"},
        "speedup_vs_bb": None if not extras else {
            "same_storage_same_passes": ratio("ca_bb_compact_i64", "ca_lambda_compact_i64"),
            "same_storage_one_step_per_launch": ratio("ca_bb_compact_i64_single_step",
                                                     "ca_lambda_compact_i64_single_step"),
            "embedded_i64_tile_one_step": ratio("ca_bb_tile_rho32_i64", "ca_lambda_tile_rho32_i64"),
            "paper_percell_rho32_one_step": ratio("ca_bb_percell_rho32_i64", "ca_lambda_percell_rho32_i64"),
            "headline_over_paper_percell_bb": ratio("ca_bb_percell_rho32_i64", "ca_lambda_compact_i64"),
            "definition": "BB time / lambda time for the same K CA steps. same_storage_same_passes: both "
                          "walk the compact state in the same passes (the BB kernel scans all (n/32)^2 box "
                          "tiles, culls, addresses member tiles through lambda^-1) - the headline ratio; "
                          "one_step: one launch per step; paper_percell: one thread per cell, rho=32 blocks "
                          "(SURVEY hazard 6), on the reference's int64 Grid"},
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
