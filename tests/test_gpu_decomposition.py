"""Decomposition invariance on one GPU.

* x-slabs: k in-process slab contexts (the multi-GPU halo pack / unpack path,
  with device copies in place of NCCL send/recv) must reproduce the one-slab
  result BIT FOR BIT -- every cell is computed by the same formula in the same
  order whichever slab owns it;
* y-segments of the marching kernel (forced short with STS_SEG) likewise.
"""
import os

import numpy as np
import pytest

from paper_1802_04243_b200 import workloads as W

pytestmark = pytest.mark.gpu
FIELDS = ("u", "v", "p", "T")


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    import __graft_entry__
    __graft_entry__.build()
    from paper_1802_04243_b200 import simplets
    return simplets


def _slabs(S, case, k, steps, seed=3):
    """Run `case` as k slabs; return the global fields assembled from the slabs."""
    ref = S.Solver(case)
    noise = W.perturbation(case, seed)
    st = W.perturbed_state({f: ref.get_field(f) for f in FIELDS}, noise, vscale=0.05)
    for f in ("p", "T", "u", "v"):
        ref.set_field(f, st[f])
    group = [S.Solver(case, rank=r, world=k) for r in range(k)]
    for g in group:
        for f in ("p", "T", "u", "v"):
            g.set_field(f, st[f])
    ranges = group[0].get_map(3).reshape(-1, 2)
    ref.advance(steps)
    S.advance_group(group, steps)
    out = {}
    for f in FIELDS:
        parts = [g.get_field(f) for g in group]
        out[f] = np.concatenate(parts, axis=1)
    return ref, out, ranges


@pytest.mark.parametrize("variant", list(W.VARIANTS))
@pytest.mark.parametrize("k", [2, 3])
def test_slabs_bitwise(S, variant, k):
    case = W.c1(variant, passes=4)
    ref, got, ranges = _slabs(S, case, k, steps=3)
    assert ranges[0, 0] == 0 and ranges[-1, 1] == case["nx"]
    for f in FIELDS:
        a = ref.get_field(f)
        assert a.shape == got[f].shape, f
        assert np.array_equal(a, got[f]), (f, np.abs(a - got[f]).max())


@pytest.mark.parametrize("variant", ["implicit_upwind", "explicit_tvd"])
@pytest.mark.parametrize("nx", [754, 1002])
def test_slabs_split_launch_bitwise(S, variant, nx):
    """Slabs wide enough for >= 3 strips of 125 columns: each pass launches the
    edge-strip CTAs and the interior CTAs separately (the multi-GPU overlap
    split).  nx = 754 gives slabs of 377 = 3 x 125 + 2 columns, whose last strip
    owns 2 columns, so the strip before it also reads ghost columns and must be
    an edge strip.  Still bit-identical to one slab."""
    case = W.channel(nx, 24, spacing=0.25, variant=variant, passes=3,
                     squares=[(5, 8, 4, 4), (370, 10, 6, 5), (nx - 9, 2, 4, 4)])
    ref, got, _ = _slabs(S, case, 2, steps=2)
    for f in FIELDS:
        assert np.array_equal(ref.get_field(f), got[f]), f


@pytest.mark.parametrize("variant", list(W.VARIANTS))
@pytest.mark.parametrize("nx", [377, 500])
def test_nccl_self_ring_overlap_bitwise(S, variant, nx):
    """Periodic single rank with an NCCL communicator and >= 3 strips: the edge
    strips and the halo (pack -> ncclSend/Recv -> unpack) run on the high-
    priority halo stream while the interior strips of the next pass run on the
    pass stream.  Bit-identical to the in-kernel wrap, in fixed-pass and in
    tolerance mode (which joins the halo stream before every residual check)."""
    case = W.periodic_box(nx, 20, 0.1, variant=variant, passes=4, dt=0.02, Kn=0.02,
                          squares=[(3, 6, 4, 4), (nx - 6, 9, 4, 5)])
    for tol in (0.0, 1e-3):
        case = dict(case, tol=tol, min_passes=2)
        a = S.Solver(case)
        b = S.Solver(case, nccl_id=S.nccl_unique_id())
        noise = W.perturbation(case, 11)
        st = W.perturbed_state({f: a.get_field(f) for f in FIELDS}, noise, vscale=0.2)
        for g in (a, b):
            for f in ("p", "T", "u", "v"):
                g.set_field(f, st[f])
        sa = a.advance(3, check=False)[1]
        sb = b.advance(3, check=False)[1]
        for f in FIELDS:
            assert np.array_equal(a.get_field(f), b.get_field(f)), (tol, f)
        assert sa["res"] == sb["res"] and sa["passes_done"] == sb["passes_done"]


def test_slabs_periodic_bitwise(S):
    """Periodic x with slabs: ring neighbours (rank 0 <-> rank k-1)."""
    case = W.c2(small=True, variant="implicit_tvd", passes=4)
    ref, got, _ = _slabs(S, case, 4, steps=3)
    for f in FIELDS:
        a = ref.get_field(f)
        if f == "u":          # periodic: the slab view has nx faces (face nx == face 0)
            a = a[:, : got[f].shape[1]]
        assert np.array_equal(a, got[f]), f


@pytest.mark.parametrize("variant", ["implicit_tvd", "explicit_tvd"])
def test_nccl_transport_self_ring(S, variant):
    """The real NCCL path on one GPU: a periodic single rank given an NCCL id
    exchanges its wrapped halo with itself through halo_pack -> ncclSend/ncclRecv
    (right strip first, left ghosts first) -> halo_unpack, and reduces the residual
    with ncclAllReduce(MAX), instead of writing the wrapped ghosts in-kernel.  The
    result must equal the in-kernel path bit for bit."""
    case = W.c2(small=True, variant=variant, passes=4)
    a = S.Solver(case)
    b = S.Solver(case, nccl_id=S.nccl_unique_id())
    noise = W.perturbation(case, 9)
    st = W.perturbed_state({f: a.get_field(f) for f in FIELDS}, noise, vscale=0.01)
    for g in (a, b):
        for f in ("p", "T", "u", "v"):
            g.set_field(f, st[f])
    _, sa = a.advance(3)
    _, sb = b.advance(3)
    for f in FIELDS:
        assert np.array_equal(a.get_field(f), b.get_field(f)), f
    assert sa["res"] == sb["res"]


@pytest.mark.parametrize("variant", list(W.VARIANTS))
@pytest.mark.parametrize("seg", ["1", "3", "5", "17"])
def test_segments_bitwise(S, seg, variant):
    """The y-march segmentation (warm-up rows) does not change a single bit."""
    case = W.c1(variant, passes=4)
    base = S.Solver(case)
    base.advance(3)
    ref = {f: base.get_field(f) for f in FIELDS}
    old = os.environ.get("STS_SEG")
    os.environ["STS_SEG"] = seg
    try:
        g = S.Solver(case)
    finally:
        if old is None:
            del os.environ["STS_SEG"]
        else:
            os.environ["STS_SEG"] = old
    g.advance(3)
    for f in FIELDS:
        assert np.array_equal(ref[f], g.get_field(f)), f


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_allreg_loop_bitwise(S, variant):
    """CTAs whose every point is regular run the regular-only copy of the row
    loop (launch-order bit 30) and skip the kind rows; forcing every CTA onto the
    general loop (STS_NO_ALLREG) must not change a single bit.  A 520 x 96
    channel with one square and 16-row segments has many all-regular CTAs."""
    case = W.channel(520, 96, spacing=0.25, variant=variant, passes=4, squares=[(200, 40, 10, 10)])
    out = []
    for env in ({"STS_SEG": "16"}, {"STS_SEG": "16", "STS_NO_ALLREG": "1"}, {"STS_SEG": "40"}):
        old = {k: os.environ.get(k) for k in ("STS_SEG", "STS_NO_ALLREG")}
        os.environ.pop("STS_NO_ALLREG", None)
        os.environ.update(env)
        try:
            g = S.Solver(case)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        base = {k: g.get_field(k) for k in ("u", "v", "p", "T")}
        st = W.perturbed_state(base, W.perturbation(case, seed=9), vscale=0.05)
        for k in ("p", "T", "u", "v"):
            g.set_field(k, st[k])
        g.advance(3)
        out.append({f: g.get_field(f) for f in FIELDS})
    for f in FIELDS:
        assert np.array_equal(out[0][f], out[1][f]), f
        assert np.array_equal(out[0][f], out[2][f]), f


def _peer_group(S, case, k, steps, seed=3):
    """k in-process slabs with the fused halo transport (N1): global fields."""
    ref = S.Solver(case)
    st = W.perturbed_state({f: ref.get_field(f) for f in FIELDS}, W.perturbation(case, seed), vscale=0.05)
    group = [S.Solver(case, rank=r, world=k) for r in range(k)]
    S.peer_connect_group(group)
    for g in [ref] + group:
        for f in ("p", "T", "u", "v"):
            g.set_field(f, st[f])
    ref.advance(steps)
    S.advance_group(group, steps)
    return ref, {f: np.concatenate([g.get_field(f) for g in group], axis=1) for f in FIELDS}, group


@pytest.mark.parametrize("variant", list(W.VARIANTS))
@pytest.mark.parametrize("k", [2, 3])
def test_peer_group_bitwise(S, variant, k):
    """Fused halo: the pass and explicit-plane epilogues store the
    edge columns straight into the neighbours' ghost columns (in-process slabs on
    one device: plain device pointers, the same stream-ordered flags as across
    processes).  Bit-identical to one slab, with no pack / copy / unpack launch."""
    case = W.c1(variant, passes=4)
    ref, got, group = _peer_group(S, case, k, steps=3)
    for f in FIELDS:
        assert np.array_equal(ref.get_field(f), got[f]), (f, np.abs(ref.get_field(f) - got[f]).max())


@pytest.mark.parametrize("k", [2, 3])
def test_peer_group_periodic_bitwise(S, k):
    """The same on a periodic channel (ring neighbours; k = 2: both neighbours are
    the same rank)."""
    case = W.c2(small=True, variant="explicit_tvd", passes=4)
    ref, got, _ = _peer_group(S, case, k, steps=3)
    for f in FIELDS:
        assert np.array_equal(ref.get_field(f), got[f]), f


def test_peer_group_no_halo_launches(S):
    """The fused transport adds no kernel launch per pass: the launches of a peer
    group equal the march launches alone (edge + interior sets per slab)."""
    case = W.c1("implicit_upwind", passes=4)
    group = [S.Solver(case, rank=r, world=2) for r in range(2)]
    S.peer_connect_group(group)
    for g in group:
        g.profile(True)
        g.profile_read(reset=True)
    S.advance_group(group, 2)
    for g in group:
        prof = g.profile_read(reset=True)
        assert prof["launches"] <= 3 * prof["pass_launches"], prof     # edge + general + regular sets only


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_general_instance_same_bits(S, variant):
    """The march kernel picks the regular or the general stage instances per warp
    (a warp with any general point runs the general ones). That is only
    decomposition-invariant because the general instance gives a regular point the
    regular instance's bits: every point of the general kernel forced general
    (STS_FORCE_GENERAL) must reproduce the default run bit for bit -- C1 and a
    channel of squares touching each other and the walls."""
    cases = [W.c1(variant, passes=3),
             W.channel(75, 37, spacing=0.25, variant=variant, passes=3,
                       squares=[(30, 14, 5, 4), (35, 18, 3, 3), (60, 0, 4, 6), (10, 31, 6, 6)])]
    for case in cases:
        out = []
        for force in (False, True):
            old = os.environ.pop("STS_FORCE_GENERAL", None)
            old2 = os.environ.pop("STS_NO_ALLREG", None)
            os.environ["STS_NO_ALLREG"] = "1"               # every CTA through the general kernel
            if force:
                os.environ["STS_FORCE_GENERAL"] = "1"
            try:
                g = S.Solver(case)
                st = W.perturbed_state({f: g.get_field(f) for f in FIELDS}, W.perturbation(case, 9), vscale=0.05)
                for f in ("p", "T", "u", "v"):
                    g.set_field(f, st[f])
                g.advance(3)
                out.append({f: g.get_field(f) for f in FIELDS})
            finally:
                os.environ.pop("STS_FORCE_GENERAL", None)
                os.environ.pop("STS_NO_ALLREG", None)
                if old is not None:
                    os.environ["STS_FORCE_GENERAL"] = old
                if old2 is not None:
                    os.environ["STS_NO_ALLREG"] = old2
        for f in FIELDS:
            assert np.array_equal(out[0][f], out[1][f]), (case["name"], f, np.abs(out[0][f] - out[1][f]).max())


@pytest.mark.parametrize("variant", list(W.VARIANTS))
def test_regk_same_bits(S, variant):
    """The all-regular CTAs run regk_body (sts_regk.cuh: the regular stage
    instances restated with register-resident operands) inside the one-launch
    march_fused_kernel; the two-kernel launch with regk_kernel for every variant
    (STS_NO_FUSED, STS_OLD_REGK=0), the round-2 kernel (march_kernel<..., REGK>,
    STS_OLD_REGK=1) and every CTA through the general kernel (STS_NO_ALLREG)
    must give the same bits (fixed-pass step graphs)."""
    case = W.channel(520, 96, spacing=0.25, variant=variant, passes=4, squares=[(200, 40, 10, 10)])
    out = []
    for env in ({"STS_SEG": "16"}, {"STS_SEG": "16", "STS_OLD_REGK": "0", "STS_NO_FUSED": "1"},
                {"STS_SEG": "16", "STS_OLD_REGK": "1"}, {"STS_SEG": "16", "STS_NO_ALLREG": "1"}):
        keys = ("STS_SEG", "STS_NO_ALLREG", "STS_OLD_REGK", "STS_NO_FUSED")
        old = {k: os.environ.get(k) for k in keys}
        for k in keys:
            os.environ.pop(k, None)
        os.environ.update(env)
        try:
            g = S.Solver(case)
            base = {k: g.get_field(k) for k in ("u", "v", "p", "T")}
            st = W.perturbed_state(base, W.perturbation(case, seed=9), vscale=0.05)
            for k in ("p", "T", "u", "v"):
                g.set_field(k, st[k])
            g.advance(3)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        out.append({f: g.get_field(f) for f in FIELDS})
    for f in FIELDS:
        for q in range(1, len(out)):
            assert np.array_equal(out[0][f], out[q][f]), (q, f, np.abs(out[0][f] - out[q][f]).max())
