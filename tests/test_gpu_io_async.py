"""Asynchronous host I/O (include/simplets.h: sts_stage_field, sts_set_staged,
sts_fetch_field, sts_io_sync): a pipelined time loop -- step s+1's state staged
from host memory while step s runs, step s's result copied back while step s+1
runs -- must produce, bit for bit, the fields of the synchronous loop
(sts_set_field / sts_advance / sts_get_field) on the same host inputs, and every
misuse must fail with STS_E_ARG."""
import numpy as np
import pytest

from paper_1802_04243_b200 import workloads as W

pytestmark = pytest.mark.gpu

NAMES = ("u", "v", "p", "T")


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    import __graft_entry__
    __graft_entry__.build()
    from paper_1802_04243_b200 import simplets
    return simplets


def _inputs(S, case, steps):
    g = S.Solver(case)
    base = {k: g.get_field(k) for k in NAMES}
    return [W.perturbed_state(base, W.perturbation(case, seed=11 + s), vscale=0.05) for s in range(steps)]


def _sync_loop(S, case, ins):
    g = S.Solver(case)
    out = []
    for st in ins:
        for k in ("p", "T", "u", "v"):
            g.set_field(k, st[k])
        g.advance(1)
        out.append({k: g.get_field(k) for k in NAMES})
    return out


def _async_loop(S, case, ins):
    import torch
    g = S.Solver(case)
    hin = [{k: torch.from_numpy(np.ascontiguousarray(st[k])).pin_memory() for k in NAMES} for st in ins]
    hout = [{k: torch.empty(ins[0][k].shape, dtype=torch.float64).pin_memory() for k in NAMES} for _ in ins]
    for k in ("p", "T", "u", "v"):
        g.stage_field(k, hin[0][k].data_ptr(), hin[0][k].numel())
    for s in range(len(ins)):
        for k in ("p", "T", "u", "v"):
            g.set_staged(k)
        if s + 1 < len(ins):                      # the next step's H2D overlaps this step
            for k in ("p", "T", "u", "v"):
                g.stage_field(k, hin[s + 1][k].data_ptr(), hin[s + 1][k].numel())
        g.advance(1)
        for k in NAMES:                           # this step's D2H overlaps the next step
            g.fetch_field(k, hout[s][k].data_ptr(), hout[s][k].numel())
    g.io_sync()
    return [{k: hout[s][k].numpy() for k in NAMES} for s in range(len(ins))]


@pytest.mark.parametrize("variant", ["implicit_upwind", "explicit_tvd"])
def test_pipelined_loop_matches_synchronous(S, variant):
    case = W.c1_small(variant, passes=4)
    ins = _inputs(S, case, 4)
    ref = _sync_loop(S, case, ins)
    got = _async_loop(S, case, ins)
    for s in range(len(ins)):
        for k in NAMES:
            assert np.array_equal(ref[s][k], got[s][k]), (variant, s, k)
    # the steps differ (each starts from its own staged input)
    assert not np.array_equal(ref[0]["T"], ref[1]["T"])


def test_async_io_misuse(S):
    import torch
    case = W.c1_small("implicit_upwind", passes=2)
    g = S.Solver(case)
    with pytest.raises(S.StsError, match="STS_E_ARG"):
        g.set_staged("p")                          # nothing staged
    h = torch.zeros(case["nx"] * case["ny"] + 1, dtype=torch.float64).pin_memory()
    g.stage_field("p", h.data_ptr(), h.numel())    # wrong size: caught when set
    with pytest.raises(S.StsError, match="STS_E_ARG"):
        g.set_staged("p")
    with pytest.raises(S.StsError, match="STS_E_ARG"):
        g.fetch_field("p", h.data_ptr(), h.numel())
    with pytest.raises(S.StsError, match="STS_E_ARG"):
        g.stage_field("rho", h.data_ptr(), h.numel())
    g.io_sync()
