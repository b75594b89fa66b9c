#!/usr/bin/env python
"""Benchmark of the SIMPLE-TS loop-2 sweep (arXiv:1802.04243) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--variant V] [--impl ours|reference]

A "step" is one time step of the hot path: a0 snapshot rotation, a1 explicit
planes (explicit variants), then `passes` fixed loop-2 passes (a2-a9), over
the paper's largest mesh (C3, 4032 x 4000 = 16.1 M FVs) per GPU.
N > 1: weak scaling -- every rank owns an identical 4032 x 4000 slab of one
long channel (4032 N x 4000) with a halo exchange over NCCL after every pass.
Metric: fp64 finite-volume updates per second = FVs x passes / time.

Rank 0 prints one JSON line.  --impl reference times the CPU oracle (the
plain fp64 C transcription of the paper) on a bounded sample instead.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 finite-volume updates/sec at 1/2/4/8 B200; HBM GB/s vs roofline"
UNIT = "FVU/s"
# algorithmic HBM bytes per finite-volume update
BYTES_PER_FVU = {"implicit": 96.0, "explicit": 120.0}
CONV_BYTES_PER_FV = 56.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML every
    5 ms (nvidia-smi, ~10x slower, if NVML is unavailable)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []          # (sm_mhz, sm_max_mhz, {reason names})
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._h = None
        try:                       # NVML set up before the timed region starts
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            try:                   # the CUDA device's PCI address (NVML ignores CUDA_VISIBLE_DEVICES)
                import torch
                pr = torch.cuda.get_device_properties(index)
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(
                    f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._bits = {"hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                          "hw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                          "sw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                          "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap}
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._h = None

    def _sample_nvml(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append((float(sm), self._max, {n for n, b in self._bits.items() if r & b}))

    def _nvml(self):
        while not self._stop.is_set():
            self._sample_nvml()
            self._stop.wait(0.005)

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                p = [x.strip() for x in out.strip().split(",")]
                if len(p) == 6 and p[0].replace(".", "").isdigit():
                    self.samples.append((float(p[0]), float(p[1]),
                                         {n for n, x in zip(self.NAMES, p[2:]) if x.lower() == "active"}))
            except Exception:
                pass
            self._stop.wait(0.02)

    def _run(self):
        if self._h is not None:
            try:
                return self._nvml()
            except Exception:
                pass
        self._smi()

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.samples and self._h is not None:
            try:                   # a timed region shorter than one sampling interval
                self._sample_nvml()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))), "samples": len(self.samples)}


def bench_case(args, world):
    """Default: C3 H = 200 (the paper's largest mesh) at N = 1, and the same slab
    per GPU laid end to end at N > 1 (weak scaling).  --workload C4 (100.8 M FVs,
    strong scaling: one channel split over the N GPUs) and C5 (150 M FVs per GPU,
    weak scaling) are BASELINE.json's configs[3] and configs[4]."""
    from paper_1802_04243_b200 import workloads as W
    if args.workload == "C4":
        return W.c4(args.variant, passes=args.passes)
    if args.workload == "C5":
        return W.c5(world, args.variant, passes=args.passes)
    if world == 1:
        return W.c3(200, args.variant, passes=args.passes)
    return W.c3_long(world, args.variant, passes=args.passes)


# ------------------------------------------------------------ reference arm
def run_reference(args):
    """The CPU oracle as it stands, on the box's host cores, on a bounded sample
    of the same workload: the full 4032 x 4000 mesh, `ref_passes` loop-2 passes
    of one time step per bench step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from paper_1802_04243_b200 import workloads as W
    oracle.build()
    case = W.c3(200, args.variant, passes=args.ref_passes)
    o = oracle.Case(case)
    nfv = W.n_fv(case)
    for _ in range(args.warmup if args.ref_warmup else 0):
        o.advance(1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.advance(1)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = nfv * args.ref_passes * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (paper geometry, free-stream IC)",
        "config": {"workload": case["name"] + "_" + args.variant, "nx": case["nx"], "ny": case["ny"],
                   "passes_per_step": args.ref_passes},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{case['name']} full mesh, {args.ref_passes} loop-2 passes of one time step per bench step, single thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(variant, seconds_hint=20.0):
    """Oracle (single thread) on a bounded sample of the bench workload: the full
    C3 4032 x 4000 mesh, one time step of ONE loop-2 pass."""
    import oracle
    from paper_1802_04243_b200 import workloads as W
    oracle.build()
    case = W.c3(200, variant, passes=1)
    o = oracle.Case(case)
    t0 = time.perf_counter()
    o.advance(1)
    dt = time.perf_counter() - t0
    return {"value": W.n_fv(case) / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{case['name']} full mesh (16.1 M FVs), 1 time step x 1 loop-2 pass, {dt:.1f} s, single thread"}


# ------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    from paper_1802_04243_b200 import simplets as S
    from paper_1802_04243_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if rank == 0:
            print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(S.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tolist())

    case = bench_case(args, world)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)
    free0 = torch.cuda.mem_get_info(dev)[0]
    g = S.Solver(case, rank=rank, world=world, device=local, nccl_id=nccl_id, stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    lib_bytes = free0 - torch.cuda.mem_get_info(dev)[0]      # device memory the library holds for this rank
    nfv_rank = g.shape("p")[2] * case["ny"]
    passes = case["max_passes"]
    kind = "implicit" if case["time"] == W.IMPLICIT else "explicit"

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(device_ids=[local])
            torch.cuda.synchronize(dev)

    # warm-up
    for _ in range(args.warmup):
        g.advance(1)
    barrier()
    g.profile(True)
    g.profile_read(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        g.advance(args.steps)      # K time steps x loop 2 in one call (no host round trip between steps)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    prof = g.profile_read(reset=True)
    g.profile(False)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_fvu = nfv_rank * world * passes * args.steps
    value = total_fvu / (ms_max / 1e3)

    # roofline of the dominant kernel (pass_kernel): algorithmic bytes per launch / avg launch time
    peak, peak_kind = _peaks()
    pass_ms = prof["pass_ms"] / max(prof["pass_launches"], 1)
    bytes_per_launch = BYTES_PER_FVU[kind] * nfv_rank
    achieved = bytes_per_launch / (pass_ms / 1e3) / 1e9
    # ncu evidence for this kernel (profiles/traffic.json, one --set full capture):
    # DRAM bytes per launch and the fp64-pipe activity (the co-bound)
    traffic = fp64_active = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(f"{case['name']}_{args.variant}", {})
            traffic = tj.get("bytes_per_launch")
            fp64_active = tj.get("fp64_pipe_active")
        except Exception:
            traffic = fp64_active = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_kind, "kernel": f"march_kernel<{kind},{args.variant.split('_')[1]}>",
                "algorithmic_bytes_per_fvu": BYTES_PER_FVU[kind], "pass_ms_avg": pass_ms,
                "pass_share_of_step": prof["pass_ms"] / ms if ms > 0 else None,
                "fp64_pipe_active_ncu": fp64_active}

    # e2e: through the public API with host (pinned) buffers, every step:
    # H2D of the step's input state (u, v, p, T) + advance + D2H of the residual maxima.
    # The inputs are double-buffered: the H2D copy of step s+1 runs on a copy
    # stream while step s computes (the copy of step 0 is inside the timed region too).
    e2e = None
    if not args.no_e2e:
        names = ("u", "v", "p", "T")
        host = {k: torch.from_numpy(g.get_field(k)).pin_memory() for k in names}
        devb = [{k: torch.empty_like(host[k], device=dev) for k in names} for _ in range(2)]
        h2d = sum(h.numel() * 8 for h in host.values())
        e_steps = max(2, min(args.steps, 6))
        cstream = torch.cuda.Stream(dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def h2d_copy(b):
            with torch.cuda.stream(cstream):
                for k in names:
                    devb[b][k].copy_(host[k], non_blocking=True)
                copied[b].record(cstream)

        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cstream.wait_event(e0)
        h2d_copy(0)
        for s in range(e_steps):
            b = s % 2
            stream.wait_event(copied[b])
            for k in names:
                g.set_field_device(k, devb[b][k].data_ptr(), devb[b][k].numel())
            consumed[b].record(stream)
            if s + 1 < e_steps:
                cstream.wait_event(consumed[1 - b]) if s >= 1 else None
                h2d_copy(1 - b)
            g.advance(1)          # reads back the 9 residual slots (72 B) to the host
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1)
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": nfv_rank * world * passes * e_steps / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": 72 * world, "steps": e_steps,
               "inputs": "pinned host state copied every step, double-buffered (copy of step s+1 overlaps step s)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.variant)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.workload == "C4" else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the paper's geometry (P:686, P:719), free-stream IC; no datasets",
            "config": {"workload": f"{case['name']}_{args.variant}", "nx": case["nx"], "ny": case["ny"],
                       "fv_per_gpu": nfv_rank, "passes_per_step": passes, "dt": case["dt"],
                       "parallelism": f"x-slabs{world}" if world > 1 else "single",
                       "l2": "inputs larger than L2 (>= 1.5 GB working set per GPU)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(prof["launches"]), "clocks": clk.summary(),
            "hbm_gbs_algorithmic_step": value / world * BYTES_PER_FVU[kind] / 1e9,
            # resident device memory per FV (the paper: 5.9 M FVs per GB, P:708 = 169 B/FV)
            "memory": {"device_bytes_per_gpu": int(lib_bytes), "bytes_per_fv": lib_bytes / nfv_rank,
                       "paper_bytes_per_fv": 1e9 / 5.9e6},
        }
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--passes", type=int, default=10)
    # (explicit_tvd: C3 from the free-stream start goes unstable after ~40 steps
    #  at dt = 0.005 -- DESIGN section 9 -- so time it with --steps 40 or fewer)
    ap.add_argument("--variant", default="implicit_upwind",
                    choices=["implicit_upwind", "implicit_tvd", "explicit_upwind", "explicit_tvd"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3", choices=["C3", "C4", "C5"])
    ap.add_argument("--ref-passes", type=int, default=1)
    ap.add_argument("--ref-warmup", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        if args.steps > 5:
            args.steps = 5     # each reference step is ~20 s of single-core work
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
