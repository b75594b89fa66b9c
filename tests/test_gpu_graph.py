"""Graph-driven loop 2 (tolerance mode): one CUDA graph per time
step with loop 2 as a conditional WHILE node and the convergence test on the
device, against the host-driven loop (STS_NO_GRAPH=1, one residual read-back
per pass as the paper does) and against the CPU oracle.

Both drivers run the same pass kernels and apply the same test (finish_residuals
+ `res < tol`, reading R35), so pass counts, residuals and fields must agree bit
for bit; the oracle's pass count must agree too (fixed by the tolerance, which
is chosen well away from the residual of any pass)."""
import os

import numpy as np
import pytest

from paper_1802_04243_b200 import workloads as W
from tests.parity_util import FIELDS, TOL, rel_errors, seeded_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    import __graft_entry__
    __graft_entry__.build()
    from paper_1802_04243_b200 import simplets
    return simplets


def _run(S, case, steps, graph, seed=3):
    old = os.environ.pop("STS_NO_GRAPH", None)
    if not graph:
        os.environ["STS_NO_GRAPH"] = "1"
    try:
        g = S.Solver(case)
        base = {k: g.get_field(k) for k in ("u", "v", "p", "T")}
        st_in = W.perturbed_state(base, W.perturbation(case, seed=seed), vscale=0.05)
        for k in ("p", "T", "u", "v"):
            g.set_field(k, st_in[k])
        out = []
        for _ in range(steps):                 # one call per step: per-step pass counts
            st, stats = g.advance(1, check=False)
            out.append((st, stats["passes_done"], tuple(stats["res"]), stats["converged"]))
        return out, {k: g.get_field(k) for k in FIELDS}
    finally:
        os.environ.pop("STS_NO_GRAPH", None)
        if old is not None:
            os.environ["STS_NO_GRAPH"] = old


def _same(a, b):
    (sa, fa), (sb, fb) = a, b
    assert sa == sb, (sa, sb)
    for k in FIELDS:
        assert np.array_equal(fa[k], fb[k]), k


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_graph_loop_matches_host_loop(S, variant):
    """Converging steps (pass counts of both parities) -- bitwise equal."""
    case = W.c1_small(variant, passes=80)
    case["tol"] = 1e-6
    a = _run(S, case, 3, graph=True)
    b = _run(S, case, 3, graph=False)
    _same(a, b)
    assert all(c == 1 for _, _, _, c in a[0]), a[0]
    assert a[0][0][1] > 1


def test_graph_loop_nonconverged_and_min_passes(S):
    """max_passes reached (STS_E_NONCONVERGED) and min_passes > 1, both drivers."""
    case = W.c1_small("implicit_tvd", passes=5)
    case["tol"] = 1e-30
    a = _run(S, case, 2, graph=True)
    b = _run(S, case, 2, graph=False)
    _same(a, b)
    assert all(st == S.STS_E_NONCONVERGED and c == 0 for st, _, _, c in a[0])
    assert [p for _, p, _, _ in a[0]] == [5, 10]
    case = W.c1_small("explicit_upwind", passes=9)
    case["tol"] = 1.0                         # converged at the first check
    case["min_passes"] = 4
    a = _run(S, case, 2, graph=True)
    b = _run(S, case, 2, graph=False)
    _same(a, b)
    assert [p for _, p, _, _ in a[0]] == [4, 8]


def test_graph_loop_vs_oracle(S, oracle_mod):
    """Same pass count as the oracle's loop 2 and fields within the parity bar."""
    case = W.c1_small("implicit_upwind", passes=200)
    case["tol"] = 1e-9
    g, o = seeded_pair(S, oracle_mod, case, seed=4)
    done = 0
    for _ in range(2):                         # the oracle reports the passes of its last step
        st, stats = g.advance(1)
        ost, ores, opasses = o.advance(1)
        assert st == 0 and ost == 0 and stats["converged"] == 1
        assert stats["passes_done"] - done == opasses, (stats["passes_done"] - done, opasses)
        done = stats["passes_done"]
    err = rel_errors({k: g.get_field(k) for k in FIELDS}, o.fields(), o.get_map(0) == 0)
    assert max(err.values()) <= TOL, err


def test_graph_loop_bad_state(S):
    """A non-positive temperature stops the graph loop with STS_E_STATE."""
    case = W.c1_small("implicit_upwind", passes=20)
    case["tol"] = 1e-12
    g = S.Solver(case)
    T = g.get_field("T")
    T[5, 3] = -1.0
    g.set_field("T", T)
    st, stats = g.advance(1, check=False)
    assert st == S.STS_E_STATE
    assert stats["bad_cell"] >= 0


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_fixed_pass_graph_matches_stream(S, variant):
    """Fixed-pass mode: one CUDA graph per time step (the default on one context)
    against the stream-launched passes (STS_NO_GRAPH=1), bit for bit, over steps
    of both snapshot-rotation parities (odd pass count)."""
    case = W.c1_small(variant, passes=3)
    a = _run(S, case, 4, graph=True)
    b = _run(S, case, 4, graph=False)
    _same(a, b)


@pytest.mark.parametrize("variant", ["implicit_upwind", "implicit_tvd", "explicit_tvd"])
def test_pdl_edges_same_bits(S, variant):
    """The programmatic (PDL) edges between the passes of a step graph (DESIGN 5.5)
    change only when a pass's CTAs are launched, never what they read: graph with
    PDL, graph with full edges (STS_NO_PDL=1) and stream launches agree bit for bit
    on the paper's 4032 x 400 mesh (hundreds of CTAs per pass, several per SM, so a
    pass that read its predecessor's output early would differ)."""
    case = W.c3(20, variant, passes=3)
    out = []
    for env in ({}, {"STS_NO_PDL": "1"}):
        saved = os.environ.pop("STS_NO_PDL", None)
        os.environ.update(env)
        try:
            out.append(_run(S, case, 3, graph=True))
        finally:
            os.environ.pop("STS_NO_PDL", None)
            if saved is not None:
                os.environ["STS_NO_PDL"] = saved
    out.append(_run(S, case, 3, graph=False))
    _same(out[0], out[1])
    _same(out[0], out[2])


def test_fixed_pass_graph_bad_state_step(S):
    """A bad state in step 3 of a 4-step call made of graph launches: reported with
    its cumulative pass index (2 steps x 2 passes + its pass within step 3)."""
    case = W.c1_small("implicit_upwind", passes=2)
    g = S.Solver(case)
    g.advance(2)                                   # a healthy start: passes_done = 4
    T = g.get_field("T")
    T[5, 3] = -1.0
    g.set_field("T", T)
    st, stats = g.advance(3, check=False)
    assert st == S.STS_E_STATE
    assert stats["bad_pass"] == 4, stats


@pytest.mark.parametrize("variant", ["explicit_upwind", "explicit_tvd"])
@pytest.mark.parametrize("graph", [True, False])
def test_planes_in_first_pass_match_conv_kernel(S, variant, graph):
    """N2: the explicit planes computed inside the first pass of each step (the
    default on one context) against the separate conv kernel (STS_NO_FUSE=1, as the
    paper launches it): planes and fields bit for bit, C1 (square, walls,
    inlet / outlet) and a periodic channel (wrapped ghost planes), graph and stream
    drivers."""
    for case in (W.c1(variant, passes=3), W.c2(small=True, variant=variant, passes=3)):
        out = []
        for fuse in (True, False):
            saved = {k: os.environ.pop(k, None) for k in ("STS_NO_FUSE", "STS_NO_GRAPH")}
            if not fuse:
                os.environ["STS_NO_FUSE"] = "1"
            if not graph:
                os.environ["STS_NO_GRAPH"] = "1"
            try:
                g = S.Solver(case)
                st = W.perturbed_state({f: g.get_field(f) for f in ("u", "v", "p", "T")},
                                       W.perturbation(case, 13), vscale=0.01)
                for f in ("p", "T", "u", "v"):
                    g.set_field(f, st[f])
                g.advance(3)
                out.append({f: g.get_field(f) for f in FIELDS + ("uexp", "vexp", "Texp")})
            finally:
                for k in ("STS_NO_FUSE", "STS_NO_GRAPH"):
                    os.environ.pop(k, None)
                    if saved[k] is not None:
                        os.environ[k] = saved[k]
        for f in out[0]:
            assert np.array_equal(out[0][f], out[1][f]), (case["name"], f, np.abs(out[0][f] - out[1][f]).max())


@pytest.mark.parametrize("variant", ["explicit_upwind", "explicit_tvd"])
def test_graph_loop_vs_oracle_explicit(S, oracle_mod, variant):
    """Tolerance mode for the explicit schemes: the conditional-WHILE graph with the
    planes computed in the first pass (N2) takes the oracle's pass count (the oracle
    computes the planes separately, before loop 2) and matches its fields."""
    case = W.c1_small(variant, passes=300)
    case["tol"] = 1e-9
    g, o = seeded_pair(S, oracle_mod, case, seed=14)
    done = 0
    for _ in range(2):
        st, stats = g.advance(1)
        ost, ores, opasses = o.advance(1)
        assert st == 0 and ost == 0 and stats["converged"] == 1
        assert stats["passes_done"] - done == opasses, (stats["passes_done"] - done, opasses)
        done = stats["passes_done"]
    err = rel_errors({k: g.get_field(k) for k in FIELDS + ("uexp", "vexp", "Texp")},
                     {**o.fields(), **{k: o.get(k) for k in ("uexp", "vexp", "Texp")}}, o.get_map(0) == 0)
    assert max(err.values()) <= TOL, err
