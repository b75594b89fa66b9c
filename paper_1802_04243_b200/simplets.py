"""ctypes binding of libsimplets.so (include/simplets.h) -- argument marshalling only.

Every step of the SIMPLE-TS sweep runs in the sm_100a kernels of
``csrc/``; this module converts Python/numpy arguments to the C ABI and back.
There is no CPU fallback: if the shared library is missing or no CUDA device
is usable, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsimplets.so")
if os.environ.get("STS_LIB"):          # kernel A/B experiments (tools/ab.sh): another in-tree build
    LIB_PATH = os.path.abspath(os.environ["STS_LIB"])

STS_OK, STS_E_ARG, STS_E_CONFIG, STS_E_NONCONVERGED, STS_E_STATE, STS_E_CUDA, STS_E_COMM, STS_E_OOM = range(8)
STATUS_NAMES = {0: "STS_OK", 1: "STS_E_ARG", 2: "STS_E_CONFIG", 3: "STS_E_NONCONVERGED", 4: "STS_E_STATE",
                5: "STS_E_CUDA", 6: "STS_E_COMM", 7: "STS_E_OOM"}
STS_EXPLICIT, STS_IMPLICIT = 0, 1
STS_UPWIND, STS_TVD_VANLEER = 0, 1
STS_X_INFLOW_OUTFLOW, STS_X_PERIODIC = 0, 1
FIELDS = {"u": 0, "v": 1, "p": 2, "T": 3, "rho": 4, "uexp": 6, "vexp": 7, "Texp": 8}

EXPORTS = ["sts_create", "sts_destroy", "sts_last_error", "sts_set_stream", "sts_init_freestream",
           "sts_set_field", "sts_set_field_device", "sts_advance", "sts_advance_group", "sts_get_field", "sts_get_field_device",
           "sts_get_map", "sts_shape", "sts_constants", "sts_profile", "sts_profile_read", "sts_nccl_unique_id",
           "sts_plan", "sts_set_mesh", "sts_peer_export", "sts_peer_connect", "sts_peer_connect_group",
           "sts_stage_field", "sts_set_staged", "sts_fetch_field", "sts_io_sync"]


class StsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class sts_grid(ctypes.Structure):
    _fields_ = [("length_x", ctypes.c_double), ("length_y", ctypes.c_double), ("spacing", ctypes.c_double)]


class sts_square(ctypes.Structure):
    _fields_ = [("i0", ctypes.c_int32), ("j0", ctypes.c_int32), ("ni", ctypes.c_int32), ("nj", ctypes.c_int32)]


class sts_gas(ctypes.Structure):
    _fields_ = [("Kn", ctypes.c_double), ("mach", ctypes.c_double), ("gamma", ctypes.c_double),
                ("p_in", ctypes.c_double), ("T_in", ctypes.c_double),
                ("u_wall_bottom", ctypes.c_double), ("u_wall_top", ctypes.c_double),
                ("T_wall", ctypes.c_double), ("T_square", ctypes.c_double),
                ("g_x", ctypes.c_double), ("g_y", ctypes.c_double),
                ("pw_form", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("particle_frame", ctypes.c_int32), ("xbc", ctypes.c_int32)]


class sts_scheme(ctypes.Structure):
    _fields_ = [("time", ctypes.c_int32), ("space", ctypes.c_int32), ("dt", ctypes.c_double),
                ("min_passes", ctypes.c_int32), ("max_passes", ctypes.c_int32), ("tol", ctypes.c_double),
                ("loop3", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class sts_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p)]


class sts_plan_info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("nx", "ny", "i0", "i1", "pitch", "ghost", "left", "right")] + \
               [(n, ctypes.c_int32 * 2) for n in ("send_left", "send_right", "recv_left", "recv_right")]


class sts_stats(ctypes.Structure):
    _fields_ = [("steps_done", ctypes.c_int64), ("passes_done", ctypes.c_int64), ("res", ctypes.c_double * 4),
                ("converged", ctypes.c_int32), ("bad_field", ctypes.c_int32), ("bad_cell", ctypes.c_int64),
                ("bad_pass", ctypes.c_int64)]


_lib = None


def lib():
    """Load libsimplets.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, dp, ip, i64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
        st = ctypes.c_int
        L.sts_create.restype = st
        L.sts_create.argtypes = [ctypes.POINTER(sts_grid), ctypes.POINTER(sts_square), ctypes.c_int32,
                                 ctypes.POINTER(sts_gas), ctypes.POINTER(sts_scheme), ctypes.POINTER(sts_dist),
                                 ctypes.POINTER(vp)]
        L.sts_destroy.restype = None
        L.sts_destroy.argtypes = [vp]
        L.sts_last_error.restype = ctypes.c_char_p
        L.sts_last_error.argtypes = [vp]
        L.sts_set_stream.restype = st
        L.sts_set_stream.argtypes = [vp, vp]
        L.sts_init_freestream.restype = st
        L.sts_init_freestream.argtypes = [vp]
        for f in ("sts_set_field", "sts_get_field"):
            getattr(L, f).restype = st
            getattr(L, f).argtypes = [vp, ctypes.c_int32, dp, ctypes.c_int64]
        for f in ("sts_set_field_device", "sts_get_field_device"):
            getattr(L, f).restype = st
            getattr(L, f).argtypes = [vp, ctypes.c_int32, vp, ctypes.c_int64]
        for f in ("sts_stage_field", "sts_fetch_field"):
            getattr(L, f).restype = st
            getattr(L, f).argtypes = [vp, ctypes.c_int32, vp, ctypes.c_int64]
        L.sts_set_staged.restype = st
        L.sts_set_staged.argtypes = [vp, ctypes.c_int32]
        L.sts_io_sync.restype = st
        L.sts_io_sync.argtypes = [vp]
        L.sts_advance.restype = st
        L.sts_advance.argtypes = [vp, ctypes.c_int32, ctypes.POINTER(sts_stats)]
        L.sts_advance_group.restype = st
        L.sts_advance_group.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(sts_stats)]
        L.sts_get_map.restype = st
        L.sts_get_map.argtypes = [vp, ctypes.c_int32, ip, ctypes.c_int64]
        L.sts_shape.restype = st
        L.sts_shape.argtypes = [vp, ctypes.c_int32, i64p, i64p, i64p, i64p]
        L.sts_constants.restype = st
        L.sts_constants.argtypes = [vp, dp]
        L.sts_profile.restype = st
        L.sts_profile.argtypes = [vp, ctypes.c_int32]
        L.sts_profile_read.restype = st
        L.sts_profile_read.argtypes = [vp, dp, ctypes.c_int32]
        L.sts_nccl_unique_id.restype = st
        L.sts_nccl_unique_id.argtypes = [vp]
        L.sts_set_mesh.restype = st
        L.sts_set_mesh.argtypes = [vp, dp, ctypes.c_int64, dp, ctypes.c_int64]
        L.sts_peer_export.restype = st
        L.sts_peer_export.argtypes = [vp, vp, i64p]
        L.sts_peer_connect.restype = st
        L.sts_peer_connect.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
        L.sts_peer_connect_group.restype = st
        L.sts_peer_connect_group.argtypes = [ctypes.POINTER(vp), ctypes.c_int32]
        L.sts_plan.restype = st
        L.sts_plan.argtypes = [ctypes.POINTER(sts_grid), ctypes.POINTER(sts_square), ctypes.c_int32,
                               ctypes.POINTER(sts_gas), ctypes.c_int32, ctypes.c_int32,
                               ctypes.POINTER(sts_plan_info), ctypes.c_void_p]
        _lib = L
    return _lib


def _check(status, handle=None):
    if status != STS_OK:
        msg = lib().sts_last_error(handle)
        raise StsError(status, msg.decode() if msg else "")


def advance_group(solvers, n_steps):
    """Advance in-process slab solvers (ranks 0..n-1, nccl_id=None) in lockstep."""
    n = len(solvers)
    arr = (ctypes.c_void_p * n)(*[s._h.value for s in solvers])
    st = sts_stats()
    _check(lib().sts_advance_group(arr, n, int(n_steps), ctypes.byref(st)), solvers[0]._h)
    return {"steps_done": st.steps_done, "passes_done": st.passes_done, "res": list(st.res), "converged": st.converged}


def peer_connect_group(solvers):
    """Fused halo (N1) for in-process slab contexts: the pass epilogues store the
    edge columns straight into the neighbours' ghost columns (same device)."""
    arr = (ctypes.c_void_p * len(solvers))(*[s._h for s in solvers])
    _check(lib().sts_peer_connect_group(arr, len(solvers)), solvers[0]._h)


def _structs(case: dict):
    sp = float(case["spacing"])
    grid = sts_grid(case["nx"] * sp, case["ny"] * sp, sp)
    sq = list(case.get("squares", []))
    arr = (sts_square * max(1, len(sq)))(*[sts_square(*map(int, s)) for s in sq])
    gas = sts_gas(case["Kn"], case["mach"], case["gamma"], case.get("p_in", 1.0), case.get("T_in", 1.0),
                  case.get("u_wall_bottom", 0.0), case.get("u_wall_top", 0.0),
                  case.get("T_wall", 1.0), case.get("T_square", 1.0),
                  case.get("g_x", 0.0), case.get("g_y", 0.0), int(case.get("pw_form", 0)), 0,
                  int(case.get("particle_frame", 0)), int(case.get("xbc", 0)))
    return grid, arr, len(sq), gas


def plan(case: dict, world: int, rank: int, with_kinds: bool = True):
    """Host-only decomposition plan of `rank` (sts_plan): a dict of the plan
    fields and, optionally, the (3, ny+1, pitch) uint8 kind maps of its stored
    columns.  Needs no GPU."""
    grid, arr, nsq, gas = _structs(case)
    info = sts_plan_info()
    # first call for the pitch, second for the maps
    _check(lib().sts_plan(ctypes.byref(grid), arr, nsq, ctypes.byref(gas), world, rank, ctypes.byref(info), None))
    out = {n: getattr(info, n) for n in ("nx", "ny", "i0", "i1", "pitch", "ghost", "left", "right")}
    for n in ("send_left", "send_right", "recv_left", "recv_right"):
        out[n] = tuple(getattr(info, n))
    if with_kinds:
        kinds = np.zeros((3, out["ny"] + 1, out["pitch"]), dtype=np.uint8)
        ptr = kinds.ctypes.data_as(ctypes.c_void_p)
        _check(lib().sts_plan(ctypes.byref(grid), arr, nsq, ctypes.byref(gas), world, rank, ctypes.byref(info), ptr))
        out["kinds"] = kinds
    return out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().sts_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


class Solver:
    """One SIMPLE-TS case on one GPU (or one rank's slab).

    ``case`` is a dict as made by ``paper_1802_04243_b200.workloads``.
    """

    def __init__(self, case: dict, rank: int = 0, world: int = 1, device: int = 0,
                 nccl_id: bytes | None = None, stream: int | None = None):
        L = lib()
        self.case = dict(case)
        grid, arr, nsq, gas = _structs(case)
        sch = sts_scheme(int(case["time"]), int(case["space"]), float(case["dt"]),
                         int(case.get("min_passes", 1)), int(case["max_passes"]), float(case.get("tol", 0.0)),
                         int(case.get("loop3", 1)), 0)
        self._idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        dist = sts_dist(rank, world, device, ctypes.cast(self._idbuf, ctypes.c_void_p) if self._idbuf else None)
        h = ctypes.c_void_p()
        _check(L.sts_create(ctypes.byref(grid), arr, nsq, ctypes.byref(gas), ctypes.byref(sch),
                            ctypes.byref(dist), ctypes.byref(h)))
        self._h = h
        self.nx, self.ny = int(case["nx"]), int(case["ny"])
        self.rank, self.world = rank, world
        if stream is not None:
            self.set_stream(stream)
        if case.get("dxs") is not None or case.get("dys") is not None:
            self.set_mesh(case.get("dxs"), case.get("dys"))

    # --- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().sts_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- ABI calls (same names without the prefix)
    def set_stream(self, stream_ptr: int):
        _check(lib().sts_set_stream(self._h, ctypes.c_void_p(stream_ptr)), self._h)

    def set_mesh(self, dxs=None, dys=None):
        """Non-uniform mesh steps (global dx[nx], dy[ny]; None = uniform spacing)."""
        self._dxs = None if dxs is None else np.ascontiguousarray(dxs, dtype=np.float64)
        self._dys = None if dys is None else np.ascontiguousarray(dys, dtype=np.float64)
        dptr = lambda a: None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        _check(lib().sts_set_mesh(self._h, dptr(self._dxs), 0 if self._dxs is None else self._dxs.size,
                                  dptr(self._dys), 0 if self._dys is None else self._dys.size), self._h)

    def peer_export(self) -> bytes:
        """This rank's description for the fused halo transport (CUDA IPC handles)."""
        n = ctypes.c_int64(0)
        _check(lib().sts_peer_export(self._h, None, ctypes.byref(n)), self._h)
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().sts_peer_export(self._h, buf, ctypes.byref(n)), self._h)
        return buf.raw[:n.value]

    def peer_connect(self, blobs):
        """Attach to the other ranks (blobs of ranks 0..world-1 from peer_export)."""
        size = len(blobs[0])
        _check(lib().sts_peer_connect(self._h, b"".join(blobs), size), self._h)

    def init_freestream(self):
        _check(lib().sts_init_freestream(self._h), self._h)

    def global_shape(self, name):
        if name in ("u", "uexp"):
            return (self.ny, self.nx + 1)
        if name in ("v", "vexp"):
            return (self.ny + 1, self.nx)
        return (self.ny, self.nx)

    def shape(self, name):
        nx, ny, i0, ni = (ctypes.c_int64() for _ in range(4))
        _check(lib().sts_shape(self._h, FIELDS[name], ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(i0),
                               ctypes.byref(ni)), self._h)
        return (ny.value, nx.value), i0.value, ni.value

    def set_field(self, name, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        assert a.shape == self.global_shape(name), (name, a.shape)
        _check(lib().sts_set_field(self._h, FIELDS[name], a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), a.size),
               self._h)

    def set_field_device(self, name, dev_ptr: int, n: int):
        _check(lib().sts_set_field_device(self._h, FIELDS[name], ctypes.c_void_p(dev_ptr), n), self._h)

    def get_field(self, name):
        shp, _, _ = self.shape(name)
        a = np.empty(shp, dtype=np.float64)
        _check(lib().sts_get_field(self._h, FIELDS[name], a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), a.size),
               self._h)
        return a

    def get_field_device(self, name, dev_ptr: int, n: int):
        _check(lib().sts_get_field_device(self._h, FIELDS[name], ctypes.c_void_p(dev_ptr), n), self._h)

    # asynchronous host I/O (include/simplets.h): host_ptr is the address of a
    # (pinned) host buffer of n doubles that the caller keeps alive
    def stage_field(self, name, host_ptr: int, n: int):
        _check(lib().sts_stage_field(self._h, FIELDS[name], ctypes.c_void_p(host_ptr), n), self._h)

    def set_staged(self, name):
        _check(lib().sts_set_staged(self._h, FIELDS[name]), self._h)

    def fetch_field(self, name, host_ptr: int, n: int):
        _check(lib().sts_fetch_field(self._h, FIELDS[name], ctypes.c_void_p(host_ptr), n), self._h)

    def io_sync(self):
        _check(lib().sts_io_sync(self._h), self._h)

    def get_map(self, which):
        if which == 3:
            a = np.empty(2 * self.world, dtype=np.int32)
        else:
            name = {0: "p", 1: "u", 2: "v"}[which]
            shp, _, _ = self.shape(name)
            a = np.empty(shp, dtype=np.int32)
        _check(lib().sts_get_map(self._h, which, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), a.size), self._h)
        return a

    def advance(self, n_steps, check=True):
        s = sts_stats()
        st = lib().sts_advance(self._h, int(n_steps), ctypes.byref(s))
        if check:
            _check(st, self._h)
        return st, {"steps_done": s.steps_done, "passes_done": s.passes_done, "res": list(s.res),
                    "converged": s.converged, "bad_cell": s.bad_cell, "bad_field": s.bad_field,
                    "bad_pass": s.bad_pass}

    def constants(self):
        out = (ctypes.c_double * 7)()
        _check(lib().sts_constants(self._h, out), self._h)
        return dict(zip(("A", "B", "CT1", "CT2", "CT3", "u_in", "dt"), list(out)))

    def profile(self, enable=True):
        _check(lib().sts_profile(self._h, int(enable)), self._h)

    def profile_read(self, reset=False):
        out = (ctypes.c_double * 5)()
        _check(lib().sts_profile_read(self._h, out, int(reset)), self._h)
        return {"pass_launches": out[0], "pass_ms": out[1], "conv_launches": out[2], "conv_ms": out[3],
                "launches": out[4]}

    def fields(self):
        return {k: self.get_field(k) for k in ("u", "v", "p", "T", "rho")}
