"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the SIMPLE-TS parity oracle.

The oracle (``simplets_oracle.c``) is a plain single-threaded fp64 C
transcription of arXiv:1802.04243's SIMPLE-TS step.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_1802_04243_b200``) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "simplets_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Compiler flags of the oracle: no FMA contraction, no fast-math (DESIGN.md 3.6 R30).
CFLAGS = ["-std=c99", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-Wall"]

X_INOUT, X_PERIODIC = 0, 1
EXPLICIT, IMPLICIT = 0, 1
UPWIND, TVD = 0, 1
# pressure-work forms of S^T_c (reading R9)
PW_DPDT, PW_PRINTED, PW_NEG, PW_GAMMA = 0, 1, 2, 3
FIELDS = {"u": 0, "v": 1, "p": 2, "T": 3, "rho": 4, "gamma": 5, "uexp": 6, "vexp": 7, "Texp": 8}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (the checker, not the product)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "simplets_oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Params(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
        ("dx", ctypes.c_double), ("dy", ctypes.c_double),
        ("xbc", ctypes.c_int32),
        ("Kn", ctypes.c_double), ("mach", ctypes.c_double), ("gamma", ctypes.c_double),
        ("p_in", ctypes.c_double), ("T_in", ctypes.c_double),
        ("u_wall_bottom", ctypes.c_double), ("u_wall_top", ctypes.c_double),
        ("T_wall", ctypes.c_double), ("T_square", ctypes.c_double),
        ("g_x", ctypes.c_double), ("g_y", ctypes.c_double),
        ("particle_frame", ctypes.c_int32),
        ("pw_form", ctypes.c_int32), ("r37_off", ctypes.c_int32),
        ("time_scheme", ctypes.c_int32), ("space_scheme", ctypes.c_int32),
        ("dt", ctypes.c_double),
        ("min_passes", ctypes.c_int32), ("max_passes", ctypes.c_int32),
        ("tol", ctypes.c_double),
        ("loop3", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        L.orc_create.restype = ctypes.c_void_p
        L.orc_create.argtypes = [ctypes.POINTER(Params), ip, ctypes.c_int32]
        L.orc_destroy.argtypes = [ctypes.c_void_p]
        L.orc_init_freestream.argtypes = [ctypes.c_void_p]
        L.orc_set_field.argtypes = [ctypes.c_void_p, ctypes.c_int32, dp, ctypes.c_int64]
        L.orc_get_field.argtypes = [ctypes.c_void_p, ctypes.c_int32, dp, ctypes.c_int64]
        L.orc_get_map.argtypes = [ctypes.c_void_p, ctypes.c_int32, ip, ctypes.c_int64]
        L.orc_advance.argtypes = [ctypes.c_void_p, ctypes.c_int32, dp, ip]
        L.orc_poison_solids.argtypes = [ctypes.c_void_p]
        L.orc_set_mesh.argtypes = [ctypes.c_void_p, dp, dp]
        L.orc_constants.argtypes = [ctypes.c_void_p, dp]
        for f in ("orc_vanleer",):
            getattr(L, f).restype = ctypes.c_double
            getattr(L, f).argtypes = [ctypes.c_double]
        L.orc_upwind.restype = ctypes.c_double
        L.orc_upwind.argtypes = [ctypes.c_double] * 3
        L.orc_psi_s.restype = ctypes.c_double
        L.orc_psi_s.argtypes = [ctypes.c_double] * 9
        L.orc_psi_c.restype = ctypes.c_double
        L.orc_psi_c.argtypes = [ctypes.c_double] * 8
    return _lib


def vanleer(r):
    return lib().orc_vanleer(float(r))


def psi_s(f1, f2, f3, f4, d1, d2, d3, d4, w):
    return lib().orc_psi_s(*(float(x) for x in (f1, f2, f3, f4, d1, d2, d3, d4, w)))


def psi_c(f1, f2, f3, f4, d1, d2, d3, w):
    return lib().orc_psi_c(*(float(x) for x in (f1, f2, f3, f4, d1, d2, d3, w)))


def upwind(f1, f2, w):
    return lib().orc_upwind(float(f1), float(f2), float(w))


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class Case:
    """One oracle simulation.  ``case`` is a dict as produced by
    ``paper_1802_04243_b200.workloads`` (geometry, gas, scheme)."""

    def __init__(self, case: dict):
        self.case = dict(case)
        p = Params()
        p.nx, p.ny = case["nx"], case["ny"]
        p.dx = p.dy = case["spacing"]
        p.xbc = case.get("xbc", X_INOUT)
        p.Kn, p.mach, p.gamma = case["Kn"], case["mach"], case["gamma"]
        p.p_in, p.T_in = case.get("p_in", 1.0), case.get("T_in", 1.0)
        p.u_wall_bottom, p.u_wall_top = case.get("u_wall_bottom", 0.0), case.get("u_wall_top", 0.0)
        p.particle_frame = int(case.get("particle_frame", 0))
        p.pw_form = int(case.get("pw_form", PW_DPDT))
        p.r37_off = int(case.get("r37_off", 0))
        p.T_wall, p.T_square = case.get("T_wall", 1.0), case.get("T_square", 1.0)
        p.g_x, p.g_y = case.get("g_x", 0.0), case.get("g_y", 0.0)
        p.time_scheme, p.space_scheme = case["time"], case["space"]
        p.dt = case["dt"]
        p.min_passes, p.max_passes = case.get("min_passes", 1), case["max_passes"]
        p.tol = case.get("tol", 0.0)
        p.loop3 = int(case.get("loop3", 1))
        self.nx, self.ny = p.nx, p.ny
        sq = np.ascontiguousarray(np.asarray(case.get("squares", []), dtype=np.int32).reshape(-1, 4))
        self._sq = sq
        self._h = lib().orc_create(ctypes.byref(p), sq.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(sq))
        if not self._h:
            raise ValueError("oracle rejected the case configuration")
        # non-uniform mesh (N4): per-column / per-row steps, else uniform `spacing`
        dxs, dys = case.get("dxs"), case.get("dys")
        if dxs is not None or dys is not None:
            self._dxs = None if dxs is None else np.ascontiguousarray(dxs, dtype=np.float64)
            self._dys = None if dys is None else np.ascontiguousarray(dys, dtype=np.float64)
            assert self._dxs is None or self._dxs.shape == (self.nx,)
            assert self._dys is None or self._dys.shape == (self.ny,)
            if lib().orc_set_mesh(self._h, None if self._dxs is None else _dptr(self._dxs),
                                  None if self._dys is None else _dptr(self._dys)):
                raise ValueError("oracle rejected the mesh steps")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_destroy(h)
            self._h = None

    def shape(self, name):
        nx, ny = self.nx, self.ny
        if name in ("u", "uexp"):
            return (ny, nx + 1)
        if name in ("v", "vexp"):
            return (ny + 1, nx)
        return (ny, nx)

    def set(self, name, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        assert a.shape == self.shape(name), (name, a.shape)
        if lib().orc_set_field(self._h, FIELDS[name], _dptr(a), a.size):
            raise ValueError(name)

    def get(self, name):
        a = np.empty(self.shape(name), dtype=np.float64)
        if lib().orc_get_field(self._h, FIELDS[name], _dptr(a), a.size):
            raise ValueError(name)
        return a

    def get_map(self, which):
        shp = {0: (self.ny, self.nx), 1: (self.ny, self.nx + 1), 2: (self.ny + 1, self.nx)}[which]
        a = np.empty(shp, dtype=np.int32)
        if lib().orc_get_map(self._h, which, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), a.size):
            raise ValueError(which)
        return a

    def advance(self, n_steps):
        res = np.zeros(4)
        passes = ctypes.c_int32(0)
        st = lib().orc_advance(self._h, int(n_steps), _dptr(res), ctypes.byref(passes))
        return st, res, passes.value

    def poison_solids(self):
        lib().orc_poison_solids(self._h)

    def constants(self):
        out = np.zeros(7)
        lib().orc_constants(self._h, _dptr(out))
        return dict(A=out[0], B=out[1], CT1=out[2], CT2=out[3], CT3=out[4], u_in=out[5])

    def fields(self):
        return {k: self.get(k) for k in ("u", "v", "p", "T", "rho")}
