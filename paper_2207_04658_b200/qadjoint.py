"""ctypes binding of the gradient tallies (include/qadjoint.h): argument marshalling only.
There is no CPU fallback: the calls go to libqmpm.so."""
from __future__ import annotations

import ctypes

import numpy as np

from . import qmpm
from .qmpm import MATERIAL, _check, make_params, ptr, stream_handle

EXPORTS = ["qadj_create", "qadj_destroy", "qadj_forward", "qadj_adjoint_step", "qadj_gradient_tally",
           "qadj_launch_count"]


class Stats(ctypes.Structure):
    _fields_ = [("max_resident", ctypes.c_uint32), ("peak_buffers", ctypes.c_uint32), ("forward_steps", ctypes.c_uint64),
                ("adjoint_steps", ctypes.c_uint64)]


_ready = False


def lib():
    global _ready
    L = qmpm.lib()
    if not _ready:
        P = ctypes.c_void_p
        sig = {"qadj_create": [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, P, P],
               "qadj_destroy": [P],
               "qadj_forward": [P, P, P],
               "qadj_adjoint_step": [P, P, P, P, P],
               "qadj_gradient_tally": [P, P, ctypes.c_uint32, P, P, P, P],
               "qadj_launch_count": [P, P]}
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.restype = ctypes.c_int32
            fn.argtypes = args
        _ready = True
    return L


class Adjoint:
    """One qadj_ctx for n particles of a scene (sim dict as scenes.*; fluid or elastic)."""

    def __init__(self, sim: dict, n: int, stream=None):
        self._p = make_params(sim, n)
        self.dim = sim["dim"]
        self.n = n
        self.ns = 2 * self.dim + (1 if sim["material"] == "fluid" else self.dim ** 2) + self.dim ** 2
        self.ctx = ctypes.c_void_p()
        _check(lib().qadj_create(ctypes.byref(self._p), self.dim, MATERIAL[sim["material"]], n,
                                 stream_handle(stream), ctypes.byref(self.ctx)))

    def close(self):
        if self.ctx:
            lib().qadj_destroy(self.ctx)
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

    def forward(self, s_in, s_out):
        _check(lib().qadj_forward(self.ctx, ptr(s_in), ptr(s_out)))

    def adjoint_step(self, s_t, lam_next, lam_t, g=None):
        _check(lib().qadj_adjoint_step(self.ctx, ptr(s_t), ptr(lam_next), ptr(lam_t), ptr(g)))

    def gradient_tally(self, s0, T, lam0=None):
        """-> (g [ns] float64, z, stats dict)."""
        g = np.zeros(self.ns, np.float64)
        z = ctypes.c_double()
        st = Stats()
        _check(lib().qadj_gradient_tally(self.ctx, ptr(s0), T, g.ctypes.data, ctypes.byref(z), ptr(lam0),
                                         ctypes.byref(st)))
        return g, z.value, {"max_resident": st.max_resident, "peak_buffers": st.peak_buffers,
                            "forward_steps": st.forward_steps,
                            "adjoint_steps": st.adjoint_steps}

    def launch_count(self):
        v = ctypes.c_uint64()
        _check(lib().qadj_launch_count(self.ctx, ctypes.byref(v)))
        return v.value
