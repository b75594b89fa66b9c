#!/usr/bin/env python
"""Time one periodic 4032 x 4000 slab with the in-kernel wrap (no comm) and with
the NCCL self-ring halo path (pack -> send/recv -> unpack every pass), one GPU."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1802_04243_b200 import simplets as S, workloads as W  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "implicit_upwind"
case = W.periodic_box(4032, 4000, 0.05, variant=variant, passes=10, dt=0.005, Kn=0.001)
res = {}
for name, kw in (("mirror", {}), ("nccl_self", {"nccl_id": S.nccl_unique_id()})):
    g = S.Solver(case, **kw)
    g.advance(2)
    torch.cuda.synchronize()
    t = time.perf_counter()
    n = 20
    g.advance(n)
    torch.cuda.synchronize()
    res[name] = (time.perf_counter() - t) / n * 1e3
    print(f"{name}: {res[name]:.3f} ms/step ({res[name] / 10:.4f} ms/pass)", flush=True)
print(f"exchange overhead: {100 * (res['nccl_self'] / res['mirror'] - 1):.1f} %")
