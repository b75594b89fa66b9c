"""One rank of the multi-process fused-halo test (tests/test_gpu_peer_ipc.py).

Launched twice (RANK 0/1, WORLD_SIZE 2) on ONE GPU: the ranks exchange their
sts_peer_export blobs over a gloo process group (CPU), connect with
sts_peer_connect (CUDA IPC mappings of each other's snapshots), advance their
slabs with the fused halo and the pushed residual maxima, and rank 0 compares
the assembled fields bit for bit with a single-slab run in its own process.
Then every rank sets its slab from the single-slab state in SLAB shape (the
collective peer exchange of sts_set_field) and both advance one more step.
Writes a JSON verdict to $OUT from rank 0; exit code 0 = pass.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_1802_04243_b200 import simplets as S
    from paper_1802_04243_b200 import workloads as W

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    name, variant, steps = os.environ["CASE"], os.environ["VARIANT"], int(os.environ["STEPS"])
    case = W.c1(variant, passes=4) if name == "C1" else W.c2(small=True, variant=variant, passes=4)
    fields = ("u", "v", "p", "T")

    g = S.Solver(case, rank=rank, world=world, device=0)
    blobs = [None] * world
    dist.all_gather_object(blobs, g.peer_export())
    g.peer_connect(blobs)
    ref = S.Solver(case) if rank == 0 else None
    st0 = [None]
    if ref is not None:                       # the free stream plus seeded noise, as in _slabs
        st0 = [W.perturbed_state({f: ref.get_field(f) for f in fields}, W.perturbation(case, 3), vscale=0.05)]
    dist.broadcast_object_list(st0, 0)
    st0 = st0[0]
    for f in ("p", "T", "u", "v"):
        g.set_field(f, st0[f])
        if ref is not None:
            ref.set_field(f, st0[f])
    _, stats = g.advance(steps)
    parts = [None] * world
    dist.all_gather_object(parts, {f: g.get_field(f) for f in fields})
    ok, info = True, {}
    if ref is not None:
        _, rstats = ref.advance(steps)
        for f in fields:
            got = np.concatenate([p[f] for p in parts], axis=1)
            a = ref.get_field(f)
            same = a.shape == got.shape and np.array_equal(a, got)
            info[f] = bool(same)
            ok &= same
        info["res_equal"] = bool(np.array_equal(np.array(stats["res"]), np.array(rstats["res"])))
        ok &= info["res_equal"]
    # phase 2: slab-shaped input (collective peer exchange inside sts_set_field)
    full = [None]
    if ref is not None:
        full = [{f: ref.get_field(f) for f in fields}]
    dist.broadcast_object_list(full, 0)
    full = full[0]
    for f in ("p", "T", "u", "v"):
        (_, c_), i0, _ = g.shape(f)
        arr = np.ascontiguousarray(full[f][:, i0:i0 + c_])
        S._check(S.lib().sts_set_field(g._h, S.FIELDS[f], arr.ctypes.data_as(S.ctypes.POINTER(S.ctypes.c_double)),
                                       arr.size), g._h)
    g.advance(1)
    parts = [None] * world
    dist.all_gather_object(parts, {f: g.get_field(f) for f in fields})
    if ref is not None:
        ref.advance(1)
        for f in fields:
            got = np.concatenate([p[f] for p in parts], axis=1)
            same = bool(np.array_equal(ref.get_field(f), got))
            info[f + "_slab_input"] = same
            ok &= same
        with open(os.environ["OUT"], "w") as fh:
            json.dump({"ok": bool(ok), **info}, fh)
    dist.barrier()
    g.close()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
