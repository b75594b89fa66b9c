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
        case = W.c4(args.variant, passes=args.passes)
    elif args.workload == "C5":
        case = W.c5(world, args.variant, passes=args.passes)
    elif world == 1:
        case = W.c3(200, args.variant, passes=args.passes)
    else:
        case = W.c3_long(world, args.variant, passes=args.passes)
    # feature paths (not the headline): loop 3 (N3), a stretched y mesh (N4)
    if args.loop3 > 1:
        case["loop3"] = args.loop3
        case["name"] += f"_loop3x{args.loop3}"
    if args.stretch > 0:
        case = W.with_mesh(case, None, W.smooth_steps(case["ny"], case["spacing"], args.stretch))
    return case


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
    times = []
    with _Pinned():
        for _ in range(args.warmup if args.ref_warmup else 0):
            o.advance(1)
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
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu": _cpu_model(),
                         "nproc": os.cpu_count(), "pinned": "sched_setaffinity to one core",
                         "sample": f"{case['name']} full mesh, {args.ref_passes} loop-2 passes of one time step per bench step, single thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class _Pinned:
    """Pin this process to one host core (the oracle runs on 1 core,
    like taskset -c 0) for the duration of a block; restores the affinity."""

    def __enter__(self):
        self.old = None
        try:
            self.old = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {min(self.old)})
        except (AttributeError, OSError):
            pass
        return self

    def __exit__(self, *a):
        if self.old is not None:
            os.sched_setaffinity(0, self.old)


def cpu_baseline(variant, seconds_hint=20.0):
    """Oracle (single thread, pinned to one core) on a bounded sample of the bench
    workload: the full C3 4032 x 4000 mesh, one time step of ONE loop-2 pass."""
    import oracle
    from paper_1802_04243_b200 import workloads as W
    oracle.build()
    case = W.c3(200, variant, passes=1)
    o = oracle.Case(case)
    with _Pinned():
        t0 = time.perf_counter()
        o.advance(1)
        dt = time.perf_counter() - t0
    return {"value": W.n_fv(case) / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "cpu": _cpu_model(), "nproc": os.cpu_count(), "pinned": "sched_setaffinity to one core (taskset -c equivalent)",
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
    # test hook: every rank on one device (a 2-process check of the N > 1 code path on a
    # 1-GPU box; the numbers of such a run mean nothing); torch's process group on gloo
    if os.environ.get("STS_BENCH_ONE_DEVICE"):
        local = 0
    if world != args.gpus:
        if rank == 0:
            print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    halo = args.halo if world > 1 else None
    halo_note = None
    if world > 1:
        if os.environ.get("STS_BENCH_ONE_DEVICE"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def make_solver(case, stream_ptr=None):
        """One rank's solver; N > 1: the fused halo over peer memory (N1, default)
        -- blobs of CUDA IPC handles exchanged over the process group -- or NCCL."""
        g = S.Solver(case, rank=rank, world=world, device=local, nccl_id=nccl_id, stream=stream_ptr)
        if world > 1 and halo == "peer":
            blobs = [None] * world
            dist.all_gather_object(blobs, g.peer_export())
            g.peer_connect(blobs)
        return g

    def decomp_check():
        """Every rank's slab of a small channel (96 columns per rank, a square each)
        through the chosen transport against a one-slab run on rank 0, bit for bit;
        True/False on rank 0 (None elsewhere), an exception text if it failed."""
        small = W.channel(96 * world, 40, spacing=0.25, variant=args.variant, passes=4,
                          squares=[(22 + 96 * q, 18, 4, 4) for q in range(world)])
        err, same, parts = None, None, None
        try:
            gs = make_solver(small)
            gs.advance(3)
            parts = {f: gs.get_field(f) for f in ("u", "v", "p", "T")}
            gs.close()
        except Exception as e:      # a transport that does not work on this machine
            err = f"{type(e).__name__}: {e}"
        allp = [None] * world
        dist.all_gather_object(allp, (err, parts))
        errs = [e for e, _ in allp if e]
        if rank == 0 and not errs:
            ref = S.Solver(small, device=local)
            ref.advance(3)
            same = all(np.array_equal(ref.get_field(f), np.concatenate([p_[f] for _, p_ in allp], axis=1))
                       for f in ("u", "v", "p", "T"))
            ref.close()
        flag = [same, errs[0] if errs else None]
        dist.broadcast_object_list(flag, 0)
        return flag

    decomp = None
    if world > 1:
        # the transport is probed (and checked bit for bit) before the timed run; a
        # peer transport that fails or disagrees here falls back to NCCL
        if halo == "peer":
            decomp, perr = decomp_check()
            if perr or decomp is not True:
                halo_note = f"peer transport unusable here ({perr or 'decomposition not bitwise'}); NCCL used"
                halo = "nccl"
        if halo == "nccl":
            idt = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(S.nccl_unique_id()), dtype=torch.uint8))
            if os.environ.get("STS_BENCH_ONE_DEVICE"):
                ids = [bytes(idt.cpu().numpy().tolist())]
                dist.broadcast_object_list(ids, 0)
                nccl_id = ids[0]
            else:
                dist.broadcast(idt, 0)
                nccl_id = bytes(idt.cpu().numpy().tolist())
            decomp, _ = decomp_check()

    case = bench_case(args, world)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)
    free0 = torch.cuda.mem_get_info(dev)[0]
    g = make_solver(case, stream.cuda_stream)
    torch.cuda.synchronize(dev)
    lib_bytes = free0 - torch.cuda.mem_get_info(dev)[0]      # device memory the library holds for this rank
    nfv_rank = g.shape("p")[2] * case["ny"]
    passes = case["max_passes"]
    kind = "implicit" if case["time"] == W.IMPLICIT else "explicit"

    def allmax(x):
        """max over ranks of a host float (device-timed per rank)"""
        if world == 1:
            return float(x)
        one = os.environ.get("STS_BENCH_ONE_DEVICE")
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if one else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier() if os.environ.get("STS_BENCH_ONE_DEVICE") else dist.barrier(device_ids=[local])
            torch.cuda.synchronize(dev)

    # warm-up (also builds the step graphs of all three snapshot rotations)
    for _ in range(args.warmup):
        g.advance(1)
    barrier()
    # timed region: the product path as a user runs it -- one sts_advance(K) call
    # (on one context: one CUDA graph launch per time step, §5.5 of DESIGN.md)
    g.profile_read(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        g.advance(args.steps)      # K time steps x loop 2 in one call (no host round trip between steps)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = g.profile_read(reset=True)["launches"]
    ms_max = allmax(ms)
    total_fvu = nfv_rank * world * passes * args.steps
    value = total_fvu / (ms_max / 1e3)
    # profiled region: the same K steps with CUDA events around every pass on the
    # launch stream (stream launches: a graph has no per-pass events), for the
    # pass-kernel duration of the roofline
    g.profile(True)
    g.profile_read(reset=True)
    barrier()
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    psteps = min(args.steps, 10)
    pe0.record(stream)
    g.advance(psteps)
    pe1.record(stream)
    barrier()
    ms_prof = pe0.elapsed_time(pe1)
    prof = g.profile_read(reset=True)
    g.profile(False)

    # roofline of the dominant kernel (pass_kernel): algorithmic bytes per launch / avg launch time
    peak, peak_kind = _peaks()
    # pass duration from the timed region itself (one sts_advance(K): K step graphs of
    # `passes` loop-2 passes each, CUDA events on the launch stream): the step's whole
    # time divided by its passes -- includes the step's few non-pass nodes (residual
    # reset; pass_share_of_step below), so `achieved` is a lower bound; the per-pass
    # CUDA events of the stream-launched profiled region are reported beside it
    pass_ms_stream = prof["pass_ms"] / max(prof["pass_launches"], 1)
    pass_ms = ms_max / args.steps / passes
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
                "traffic": traffic, "peak_source": peak_kind,
                "kernel": ("march_kernel (general) + march_kernel<REGK> (all-regular CTAs), one pass"
                           if args.variant == "implicit_tvd" else
                           "march_fused_kernel (general + regk_body CTAs), one launch per pass"
                           + ("; the first pass of a step: march_kernel<FUSEC> pair (the planes inside)"
                              if kind == "explicit" else "")),
                "algorithmic_bytes_per_fvu": BYTES_PER_FVU[kind], "pass_ms_avg": pass_ms,
                "timed_region": "the timed region: one sts_advance(K) (step graphs), time / (K x passes)",
                "pass_ms_stream_profiled": pass_ms_stream,
                "pass_share_of_step": prof["pass_ms"] / ms_prof if ms_prof > 0 else None,
                "profiled_region": "min(K, 10) more steps, stream launches, CUDA events around every pass",
                "profiled_ms_per_step": ms_prof / psteps,
                "fp64_pipe_active_ncu": fp64_active}

    # e2e: through the public C ABI with HOST buffers, every step: the step's input
    # state (u, v, p, T) from pinned host memory (H2D), sts_advance (one time step:
    # conv + loop 2), the new state (u, v, p, T) back into pinned host memory (D2H) --
    # what a user's time loop does.  Pipelined with the asynchronous host-I/O calls
    # (sts_stage_field / sts_set_staged / sts_fetch_field / sts_io_sync): step s+1's
    # H2D and step s-1's D2H run on the context's copy streams while step s computes;
    # the timed region ends after the last D2H has landed.  The synchronous loop
    # (sts_set_field / sts_get_field, nothing overlaps) is reported beside it.
    e2e = None
    if not args.no_e2e:
        import ctypes
        names = ("u", "v", "p", "T")
        L = S.lib()
        dp = lambda t: ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))
        hin = {k: torch.from_numpy(g.get_field(k)).pin_memory() for k in names}      # this rank's slab
        hout = {k: torch.empty_like(hin[k]).pin_memory() for k in names}
        h2d = sum(h.numel() * 8 for h in hin.values())
        e_steps = max(2, min(args.steps, 20))     # the pipeline fills and drains once per loop

        def sync_loop():
            for _ in range(e_steps):
                for k in names:
                    S._check(L.sts_set_field(g._h, S.FIELDS[k], dp(hin[k]), hin[k].numel()), g._h)
                g.advance(1)
                for k in names:
                    S._check(L.sts_get_field(g._h, S.FIELDS[k], dp(hout[k]), hout[k].numel()), g._h)

        def async_loop():
            for k in names:
                g.stage_field(k, hin[k].data_ptr(), hin[k].numel())
            for s_ in range(e_steps):
                for k in names:
                    g.set_staged(k)
                if s_ + 1 < e_steps:
                    for k in names:
                        g.stage_field(k, hin[k].data_ptr(), hin[k].numel())
                g.advance(1)
                for k in names:
                    g.fetch_field(k, hout[k].data_ptr(), hout[k].numel())
            g.io_sync()

        def timed(fn):
            barrier()
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            barrier()
            torch.cuda.synchronize()
            return allmax(e0.elapsed_time(e1)), time.perf_counter() - t0

        async_loop()                                   # warm-up: slots, copy streams, graphs
        ems_sync, _ = timed(sync_loop)
        ems, wall = timed(async_loop)
        rate = lambda ms: nfv_rank * world * passes * e_steps / (ms / 1e3)
        e2e = {"value": rate(ems), "unit": UNIT,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": h2d * world, "steps": e_steps,
               "wall_s": wall,
               "path": "pipelined: sts_stage_field (pinned host -> device slot) x4 for step s+1 and sts_fetch_field "
                       "(device -> pinned host) x4 of step s-1 overlap sts_set_staged x4 + sts_advance(1) of step s; "
                       "ends with sts_io_sync",
               "sync_value": rate(ems_sync),
               "sync_path": "sts_set_field (pinned host -> device) x4, sts_advance(1), sts_get_field "
                            "(device -> pinned host) x4, each call synchronous"}

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
                       "halo": halo, "halo_note": halo_note,
                       "l2": "inputs larger than L2 (>= 1.5 GB working set per GPU)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk.summary(),
            "decomp_bitwise": decomp,
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
    # N > 1 halo transport: the fused peer-memory path (N1, default) or NCCL send/recv
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"])
    # feature paths: loop-3 sweeps per pass (N3) and a smoothly stretched y mesh (N4)
    ap.add_argument("--loop3", type=int, default=1)
    ap.add_argument("--stretch", type=float, default=0.0)
    args = ap.parse_args()
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # communicator lines in the log (which ranks / devices / transports NCCL set up)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        if args.steps > 5:
            args.steps = 5     # each reference step is ~20 s of single-core work
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
