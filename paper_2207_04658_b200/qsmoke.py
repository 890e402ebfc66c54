"""ctypes binding of the quantized smoke step (include/qsmoke.h): argument marshalling only.

Array arguments are torch tensors (device; host tensors/numpy arrays only for
set_state / get_state).  There is no CPU fallback: the calls go to libqmpm.so.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import qmpm
from .qmpm import CScheme, _check, ptr, stream_handle

EXPORTS = ["qsmoke_create", "qsmoke_destroy", "qsmoke_layout", "qsmoke_advect_velocity", "qsmoke_divergence",
           "qsmoke_jacobi", "qsmoke_project", "qsmoke_advect_density", "qsmoke_set_state", "qsmoke_get_state",
           "qsmoke_step", "qsmoke_launch_count"]

JACOBI_ITERS = 64


class Params(ctypes.Structure):
    _fields_ = [("res", ctypes.c_int32 * 3), ("dx", ctypes.c_float), ("dt", ctypes.c_float),
                ("buoyancy", ctypes.c_float), ("source_lo", ctypes.c_int32 * 3), ("source_hi", ctypes.c_int32 * 3),
                ("jacobi_iters", ctypes.c_int32), ("pad", ctypes.c_int32)]


_ready = False


def lib():
    global _ready
    L = qmpm.lib()
    if not _ready:
        P, u32p, u64, f32 = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_float
        sig = {
            "qsmoke_create": [P, P, P, P, P],
            "qsmoke_destroy": [P],
            "qsmoke_layout": [P, P, P, P],
            "qsmoke_advect_velocity": [P, u32p, u32p, P, f32, f32, u64, u32p, P],
            "qsmoke_divergence": [P, u32p, P],
            "qsmoke_jacobi": [P, u32p, P, u64, u32p, P],
            "qsmoke_project": [P, u32p, u32p, u64, u32p, P],
            "qsmoke_advect_density": [P, P, u32p, f32, P],
            "qsmoke_set_state": [P, u32p, u32p, P, u64],
            "qsmoke_get_state": [P, u32p, u32p, P],
            "qsmoke_step": [P, u64],
            "qsmoke_launch_count": [P, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.restype = ctypes.c_int32
            fn.argtypes = args
        _ready = True
    return L


def make_params(p: dict) -> Params:
    c = Params()
    for a in range(3):
        c.res[a] = p["res"][a]
        c.source_lo[a] = p["source_lo"][a]
        c.source_hi[a] = p["source_hi"][a]
    c.dx, c.dt, c.buoyancy = p["dx"], p["dt"], p["buoyancy"]
    c.jacobi_iters = p.get("jacobi_iters", JACOBI_ITERS)
    return c


class Smoke:
    """One qsmoke_ctx: the specialised kernels for (u_scheme, p_scheme) + the state."""

    def __init__(self, params: dict, u_scheme: dict, p_scheme: dict, stream=None):
        self._cu, self._cp = CScheme(u_scheme), CScheme(p_scheme)
        self._params = make_params(params)
        self.stream = stream
        self.ctx = ctypes.c_void_p()
        _check(lib().qsmoke_create(ctypes.byref(self._params), self._cu.ref, self._cp.ref,
                                   stream_handle(stream), ctypes.byref(self.ctx)))
        wu, wp, n = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint64()
        _check(lib().qsmoke_layout(self.ctx, ctypes.byref(wu), ctypes.byref(wp), ctypes.byref(n)))
        self.Wu, self.Wp, self.n_records = wu.value, wp.value, n.value
        self.res = tuple(params["res"])

    def close(self):
        if self.ctx:
            lib().qsmoke_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # sub-steps (device tensors)
    def advect_velocity(self, u_vel, u_out, dt, u_refl=None, rho=None, bdt=0.0, dstep=0, dbg=None):
        _check(lib().qsmoke_advect_velocity(self.ctx, ptr(u_vel), ptr(u_refl), ptr(rho), dt, bdt, dstep, ptr(u_out),
                                            ptr(dbg)))

    def divergence(self, u, div):
        _check(lib().qsmoke_divergence(self.ctx, ptr(u), ptr(div)))

    def jacobi(self, p_in, div, p_out, dstep=0, dbg=None):
        _check(lib().qsmoke_jacobi(self.ctx, ptr(p_in), ptr(div), dstep, ptr(p_out), ptr(dbg)))

    def project(self, u_in, p, u_out, dstep=0, dbg=None):
        _check(lib().qsmoke_project(self.ctx, ptr(u_in), ptr(p), dstep, ptr(u_out), ptr(dbg)))

    def advect_density(self, rho_in, u, rho_out, dt):
        _check(lib().qsmoke_advect_density(self.ctx, ptr(rho_in), ptr(u), dt, ptr(rho_out)))

    # the ctx state
    def set_state(self, u_words, p_words, rho, step=0):
        _check(lib().qsmoke_set_state(self.ctx, ptr(u_words), ptr(p_words), ptr(rho), step))

    def get_state(self, u_words=None, p_words=None, rho=None):
        _check(lib().qsmoke_get_state(self.ctx, ptr(u_words), ptr(p_words), ptr(rho)))

    def get_state_numpy(self):
        nx, ny, nz = self.res
        u = np.zeros((self.n_records, self.Wu), np.uint32)
        p = np.zeros((self.n_records, self.Wp), np.uint32)
        rho = np.zeros((nx, ny, nz), np.float32)
        self.get_state(u, p, rho)
        return u, p, rho

    def step(self, n=1):
        _check(lib().qsmoke_step(self.ctx, n))

    def launch_count(self):
        v = ctypes.c_uint64()
        _check(lib().qsmoke_launch_count(self.ctx, ctypes.byref(v)))
        return v.value
