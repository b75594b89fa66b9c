"""Multi-process (world size 2, gloo, CPU) coverage of the N > 1 host logic.

Each process computes its slab plan with the library's host-only `sts_plan`
(no GPU) and the two ranks exchange, over torch.distributed/gloo, what the
per-pass NCCL halo exchange would carry: the global column ids and the kind
codes of the strips they send.  The receiver checks them against its own
ghost columns -- the halo index maps and the ghost kind maps of the two ranks
must agree bit for bit, the owned ranges must tile the channel, and every
rank's maps must equal the one-rank plan restricted to its columns.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_04243_b200 import workloads as W

CASES = {
    "inout": W.c1("implicit_tvd"),
    "periodic": W.c2(small=True),
    "squares_on_the_cut": W.channel(64, 24, squares=[(29, 5, 6, 6), (31, 14, 4, 8)]),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _strip(pl, lo, hi):
    """Kind maps of global columns [lo, hi) from a rank's stored maps."""
    c0 = pl["i0"] - pl["ghost"]
    return pl["kinds"][:, :, lo - c0: hi - c0]


def _worker(rank, world, port, name, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1802_04243_b200 import simplets as S
        case = CASES[name]
        pl = S.plan(case, world, rank)
        nx = pl["nx"]
        # owned ranges tile [0, nx)
        rng = torch.tensor([pl["i0"], pl["i1"]], dtype=torch.int64)
        allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allr, rng)
        allr = [tuple(t.tolist()) for t in allr]
        assert allr[0][0] == 0 and allr[-1][1] == nx
        for a, b in zip(allr, allr[1:]):
            assert a[1] == b[0]
        # halo exchange of (column ids, kind strips), in the order the library uses
        # (right strip first; left ghosts first)
        reqs, recv = [], {}
        ids = lambda lo, hi: torch.arange(lo, hi, dtype=torch.int64)
        if pl["right"] >= 0:
            reqs.append(dist.isend(ids(*pl["send_right"]), pl["right"], tag=1))
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(_strip(pl, *pl["send_right"]))), pl["right"], tag=2))
        if pl["left"] >= 0:
            reqs.append(dist.isend(ids(*pl["send_left"]), pl["left"], tag=3))
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(_strip(pl, *pl["send_left"]))), pl["left"], tag=4))
        shp = (3, pl["ny"] + 1, pl["ghost"])
        if pl["left"] >= 0:
            recv["lid"] = torch.zeros(pl["ghost"], dtype=torch.int64)
            recv["lk"] = torch.zeros(shp, dtype=torch.uint8)
            reqs.append(dist.irecv(recv["lid"], pl["left"], tag=1))
            reqs.append(dist.irecv(recv["lk"], pl["left"], tag=2))
        if pl["right"] >= 0:
            recv["rid"] = torch.zeros(pl["ghost"], dtype=torch.int64)
            recv["rk"] = torch.zeros(shp, dtype=torch.uint8)
            reqs.append(dist.irecv(recv["rid"], pl["right"], tag=3))
            reqs.append(dist.irecv(recv["rk"], pl["right"], tag=4))
        for r in reqs:
            r.wait()
        if pl["left"] >= 0:
            exp = np.arange(*pl["recv_left"]) % nx
            assert np.array_equal(recv["lid"].numpy() % nx, exp), (recv["lid"], exp)
            assert np.array_equal(recv["lk"].numpy(), _strip(pl, *pl["recv_left"]))
        if pl["right"] >= 0:
            exp = np.arange(*pl["recv_right"]) % nx
            assert np.array_equal(recv["rid"].numpy() % nx, exp)
            assert np.array_equal(recv["rk"].numpy(), _strip(pl, *pl["recv_right"]))
        # the slab maps equal the one-rank plan on the owned columns
        one = S.plan(case, 1, 0)
        mine = _strip(pl, pl["i0"], pl["i1"])
        ref = _strip(one, pl["i0"], pl["i1"])
        assert np.array_equal(mine, ref)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
        raise


@pytest.mark.parametrize("name", list(CASES))
def test_two_rank_halo_maps_gloo(name):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res
    assert all(p.exitcode == 0 for p in procs)
