"""Debug helper (GPU box): 2-process fused-halo run vs single slab, step by step.
usage: RANK=r WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=p python tools/peer_debug.py"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1802_04243_b200 import simplets as S, workloads as W
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)
case = W.c1(os.environ.get("VARIANT", "implicit_tvd"), passes=int(os.environ.get("PASSES", "4")))
F = ("u", "v", "p", "T")
g = S.Solver(case, rank=rank, world=world, device=0)
blobs = [None] * world
dist.all_gather_object(blobs, g.peer_export())
g.peer_connect(blobs)
ref = S.Solver(case) if rank == 0 else None
st0 = [None]
if ref is not None:
    st0 = [W.perturbed_state({f: ref.get_field(f) for f in F}, W.perturbation(case, 3), vscale=0.05)]
dist.broadcast_object_list(st0, 0)
for f in ("p", "T", "u", "v"):
    g.set_field(f, st0[0][f])
    if ref is not None:
        ref.set_field(f, st0[0][f])
for step in range(int(os.environ.get("STEPS", "3"))):
    g.advance(1)
    parts = [None] * world
    dist.all_gather_object(parts, {f: g.get_field(f) for f in F})
    if ref is not None:
        ref.advance(1)
        for f in F:
            a = ref.get_field(f)
            b = np.concatenate([p[f] for p in parts], axis=1)
            d = np.abs(a - b)
            if d.max() > 0:
                cols = np.where(d.max(axis=0) > 0)[0]
                print("step", step, f, "maxdiff", d.max(), "cols", cols[:10], cols[-5:], len(cols), flush=True)
            else:
                print("step", step, f, "equal", flush=True)
dist.barrier()
