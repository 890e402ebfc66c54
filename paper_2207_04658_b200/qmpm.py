"""ctypes binding of libqmpm (include/qmpm.h): argument marshalling only.

Every entry point has the C name without the `qmpm_` prefix.  Array arguments may
be torch tensors (device or host) or numpy arrays (host); the library accepts host
or device pointers where the header says so.  There is no CPU fallback: if the
CUDA library is missing, `lib()` raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libqmpm.so")

MAX_FIELDS = 64
NUM_KERNELS = 9
ATTR = {"x": 0, "v": 1, "F": 2, "C": 3, "J": 4}
KIND = {"fixed": 0, "raw": 1, "shared_exp": 2}
MATERIAL = {"elastic": 0, "fluid": 1}
ROUNDING = {"rne": 0, "dither": 1}
TRACK_IDS, DEBUG_PREENCODE, NO_ROUND_COUNTERS, RECORD_RANGES = 1, 2, 4, 8
EDOMAIN = 7
STATUS = {0: "OK", 1: "EINVAL", 2: "ELAYOUT", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "ENONFINITE",
          7: "EDOMAIN", 8: "ECAPACITY", 9: "ESTATE"}


class QmpmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"qmpm {STATUS.get(code, code)}: {msg}")
        self.code = code


class Field(ctypes.Structure):
    _fields_ = [("attr", ctypes.c_uint8), ("comp", ctypes.c_uint8), ("kind", ctypes.c_uint8),
                ("frac_bits", ctypes.c_uint8), ("range", ctypes.c_float), ("offset", ctypes.c_float),
                ("exp_bits", ctypes.c_uint8), ("group", ctypes.c_uint8), ("pad", ctypes.c_uint8 * 2)]


class Scheme(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_uint32), ("material", ctypes.c_uint32), ("n_fields", ctypes.c_uint32),
                ("rounding", ctypes.c_uint32), ("fields", ctypes.POINTER(Field)),
                ("dither_seed", ctypes.c_uint64), ("layout_policy", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


class Params(ctypes.Structure):
    _fields_ = [("grid_res", ctypes.c_int32 * 3), ("dx", ctypes.c_float), ("dt", ctypes.c_float),
                ("gravity", ctypes.c_float * 3), ("p_rho", ctypes.c_float), ("p_vol", ctypes.c_float),
                ("E", ctypes.c_float), ("nu", ctypes.c_float), ("bound", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("max_particles", ctypes.c_uint64), ("pool_blocks", ctypes.c_uint64)]


class Slab(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("z0", ctypes.c_int32), ("z1", ctypes.c_int32),
                ("migrate_capacity", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [("step", ctypes.c_uint64), ("n_particles", ctypes.c_uint64),
                ("saturations", ctypes.c_uint64 * MAX_FIELDS), ("round_up", ctypes.c_uint64 * MAX_FIELDS),
                ("round_down", ctypes.c_uint64 * MAX_FIELDS), ("nonfinite", ctypes.c_uint64),
                ("out_of_domain", ctypes.c_uint64), ("active_blocks", ctypes.c_uint64),
                ("touched_blocks", ctypes.c_uint64), ("pool_overflow", ctypes.c_uint64)]


_lib = None
EXPORTS = ["qmpm_abi_version", "qmpm_last_error", "qmpm_layout", "qmpm_create", "qmpm_destroy",
           "qmpm_set_state", "qmpm_append_state", "qmpm_set_words", "qmpm_step", "qmpm_read_state",
           "qmpm_read_debug", "qmpm_stats", "qmpm_encode", "qmpm_decode", "qmpm_set_profiling",
           "qmpm_kernel_times", "qmpm_kernel_name", "qmpm_launch_count", "qmpm_create_slab",
           "qmpm_get_unique_id", "qmpm_connect_nccl", "qmpm_step_group", "qmpm_set_ids",
           "qmpm_read_ranges", "qmpm_predict_error", "qmpm_solve_error_bounded", "qmpm_solve_memory_bounded",
           "qmpm_codec_matmul3", "qmpm_create_dist"]


def lib():
    """Load libqmpm.so (in-tree).  Raises if it was not built: there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2207_04658_b200.build` "
                          "(the CUDA path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    sig = {
        "qmpm_abi_version": (ctypes.c_int, []),
        "qmpm_last_error": (ctypes.c_char_p, [P]),
        "qmpm_layout": (i32, [ctypes.POINTER(Scheme), P, P, P]),
        "qmpm_create": (i32, [ctypes.POINTER(Params), ctypes.POINTER(Scheme), P, ctypes.POINTER(P)]),
        "qmpm_destroy": (i32, [P]),
        "qmpm_set_state": (i32, [P, u64, P]),
        "qmpm_append_state": (i32, [P, u64, P]),
        "qmpm_set_words": (i32, [P, u64, P, u64]),
        "qmpm_step": (i32, [P, u32]),
        "qmpm_read_state": (i32, [P, P, P, P, u64, ctypes.POINTER(u64)]),
        "qmpm_read_debug": (i32, [P, P, u64, ctypes.POINTER(u64)]),
        "qmpm_stats": (i32, [P, ctypes.POINTER(Stats)]),
        "qmpm_encode": (i32, [ctypes.POINTER(Scheme), u64, P, P, u64, P, P, P]),
        "qmpm_decode": (i32, [ctypes.POINTER(Scheme), u64, P, P, P]),
        "qmpm_set_profiling": (i32, [P, ctypes.c_int]),
        "qmpm_kernel_times": (i32, [P, P, P]),
        "qmpm_kernel_name": (ctypes.c_char_p, [ctypes.c_int]),
        "qmpm_launch_count": (u64, [P]),
        "qmpm_create_slab": (i32, [ctypes.POINTER(Params), ctypes.POINTER(Scheme), P, ctypes.POINTER(Slab),
                                   ctypes.POINTER(P)]),
        "qmpm_create_dist": (i32, [ctypes.POINTER(Params), ctypes.POINTER(Scheme), P, ctypes.c_int, ctypes.c_int, P, P,
                                   ctypes.POINTER(ctypes.c_void_p)]),
        "qmpm_get_unique_id": (i32, [P]),
        "qmpm_connect_nccl": (i32, [P, P]),
        "qmpm_step_group": (i32, [P, ctypes.c_int, u32]),
        "qmpm_set_ids": (i32, [P, u64, P]),
        "qmpm_read_ranges": (i32, [P, P, ctypes.c_int]),
        "qmpm_codec_matmul3": (i32, [ctypes.POINTER(Scheme), u64, P, P, P, u64, P, P]),
        "qmpm_predict_error": (i32, [u32, P, P, P]),
        "qmpm_solve_error_bounded": (i32, [u32, P, P, P, ctypes.c_double, ctypes.c_double, i32, i32, P, P]),
        "qmpm_solve_memory_bounded": (i32, [u32, P, P, P, ctypes.c_double, i32, i32, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(rc, ctx=None):
    if rc != 0:
        msg = lib().qmpm_last_error(ctx)
        raise QmpmError(rc, msg.decode() if msg else "")


def ptr(a):
    """Raw address of a torch tensor or numpy array (None -> NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ------------------------------------------------------------ scheme / params marshalling
class CScheme:
    """Keeps the ctypes field array alive alongside the Scheme struct."""

    def __init__(self, scheme: dict):
        fields = scheme["fields"]
        self.fields = (Field * len(fields))()
        for i, f in enumerate(fields):
            F = self.fields[i]
            F.attr = ATTR.get(f.get("attr", "x"), 0)
            F.comp = f.get("comp", 0)
            F.kind = KIND[f["kind"]]
            F.frac_bits = f.get("frac_bits", 0)
            F.range = f.get("range", 1.0)
            F.offset = f.get("offset", 0.0)
            F.exp_bits = f.get("exp_bits", 0)
            F.group = f.get("group", 0)
        self.s = Scheme()
        self.s.dim = scheme.get("dim", 3) or 3
        self.s.material = MATERIAL[scheme.get("material", "elastic")]
        self.s.n_fields = len(fields)
        self.s.rounding = ROUNDING[scheme.get("rounding", "dither")]
        self.s.fields = ctypes.cast(self.fields, ctypes.POINTER(Field))
        self.s.dither_seed = scheme.get("seed", 0)
        self.s.layout_policy = {"pack": 0, "nostraddle": 1}[scheme.get("layout", "pack")]

    @property
    def ref(self):
        return ctypes.byref(self.s)


def make_params(sim: dict, max_particles: int, flags: int = 0, pool_blocks: int = 0) -> Params:
    p = Params()
    for a in range(3):
        p.grid_res[a] = sim["grid_res"][a]
        p.gravity[a] = sim["gravity"][a]
    p.dx, p.dt = sim["dx"], sim["dt"]
    p.p_rho, p.p_vol, p.E, p.nu = sim["p_rho"], sim["p_vol"], sim["E"], sim["nu"]
    p.bound = sim["bound"]
    p.flags = flags
    p.max_particles = max_particles
    p.pool_blocks = pool_blocks
    return p


def layout(scheme: dict):
    cs = CScheme(scheme)
    W = ctypes.c_uint32()
    bits = ctypes.c_uint32()
    offs = (ctypes.c_uint32 * len(scheme["fields"]))()
    _check(lib().qmpm_layout(cs.ref, ctypes.byref(W), ctypes.byref(bits), offs))
    return list(offs), W.value, bits.value


def encode(scheme: dict, vals, words, keys=None, step=0, counters=None, stream=None):
    """Standalone codec on device tensors: vals [n][n_fields] fp32 -> words [n][W] u32."""
    cs = CScheme(scheme)
    n = vals.shape[0]
    _check(lib().qmpm_encode(cs.ref, n, ptr(vals), ptr(keys), step, ptr(words), ptr(counters),
                             stream_handle(stream)))


def codec_matmul3(scheme: dict, words_in, a, words_out, keys=None, step=0, stream=None):
    """qmpm_codec_matmul3: records of a 3x3 matrix -> decode, times the constant a (3x3,
    host), re-encode (the paper's MatMul task)."""
    cs = CScheme(scheme)
    n = words_in.shape[0]
    am = np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(9))
    _check(lib().qmpm_codec_matmul3(cs.ref, n, ptr(words_in), am.ctypes.data, ptr(keys), step, ptr(words_out),
                                    stream_handle(stream)))


def decode(scheme: dict, words, vals, stream=None):
    cs = CScheme(scheme)
    _check(lib().qmpm_decode(cs.ref, words.shape[0], ptr(words), ptr(vals), stream_handle(stream)))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def predict_error(delta, g) -> float:
    """qmpm_predict_error: sigma_pred = sqrt(1/12 sum delta_h^2 g_h) (Eq. 8)."""
    d, gg = _f64(delta), _f64(g)
    out = ctypes.c_double()
    _check(lib().qmpm_predict_error(len(d), d.ctypes.data, gg.ctypes.data, ctypes.byref(out)))
    return out.value


def solve_error_bounded(P, g, R, z, eps, b_min=0, b_max=31, strict=True):
    """qmpm_solve_error_bounded (Eq. 9 + Algorithm 1): returns (delta_h, bits_h).  When the
    b_max clamp cannot meet the bound (QMPM_EDOMAIN) it raises, or with strict=False
    returns the clamped scheme."""
    P, g, R = _f64(P), _f64(g), _f64(R)
    d = np.zeros(len(P))
    b = np.zeros(len(P), np.int32)
    rc = lib().qmpm_solve_error_bounded(len(P), P.ctypes.data, g.ctypes.data, R.ctypes.data, float(z), float(eps),
                                        int(b_min), int(b_max), d.ctypes.data, b.ctypes.data)
    if not (rc == EDOMAIN and not strict):
        _check(rc)
    return d, b


def solve_memory_bounded(P, g, R, budget_bits, b_min=0, b_max=31):
    """qmpm_solve_memory_bounded (Eq. 7, closed form of SPEC.md:342): (delta_h, bits_h)."""
    P, g, R = _f64(P), _f64(g), _f64(R)
    d = np.zeros(len(P))
    b = np.zeros(len(P), np.int32)
    _check(lib().qmpm_solve_memory_bounded(len(P), P.ctypes.data, g.ctypes.data, R.ctypes.data, float(budget_bits),
                                           int(b_min), int(b_max), d.ctypes.data, b.ctypes.data))
    return d, b


def kernel_names():
    return [lib().qmpm_kernel_name(i).decode() for i in range(NUM_KERNELS)]


def get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().qmpm_get_unique_id(buf))
    return bytes(buf)


def step_group(sims, n_steps=1):
    """qmpm_step_group: advance the slabs of one decomposition living in this process."""
    arr = (ctypes.c_void_p * len(sims))(*[s.ctx.value for s in sims])
    _check(lib().qmpm_step_group(arr, len(sims), n_steps))


class Sim:
    """One qmpm context (qmpm_create .. qmpm_destroy); `slab=(nranks, rank, z0, z1)`
    creates the context of one slab of a z decomposition (qmpm_create_slab)."""

    def __init__(self, sim: dict, scheme: dict, max_particles: int, flags: int = 0, pool_blocks: int = 0,
                 stream=None, slab=None, migrate_capacity: int = 0):
        self.scheme = CScheme(scheme)
        self.params = make_params(sim, max_particles, flags, pool_blocks)
        self.dim = scheme["dim"]
        self.material = scheme["material"]
        d = self.dim
        self.n_scalars = 2 * d + (1 if self.material == "fluid" else d * d) + d * d
        _, self.W, self.bits = layout(scheme)
        self.stream = stream_handle(stream)
        h = ctypes.c_void_p()
        if slab is None:
            _check(lib().qmpm_create(ctypes.byref(self.params), self.scheme.ref, self.stream, ctypes.byref(h)))
        else:
            self.slab = Slab(slab[0], slab[1], slab[2], slab[3], migrate_capacity)
            _check(lib().qmpm_create_slab(ctypes.byref(self.params), self.scheme.ref, self.stream,
                                          ctypes.byref(self.slab), ctypes.byref(h)))
        self.ctx = h

    def close(self):
        if self.ctx:
            lib().qmpm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _c(self, rc):
        _check(rc, self.ctx)

    def set_state(self, vals):
        self._c(lib().qmpm_set_state(self.ctx, vals.shape[0], ptr(vals)))

    def append_state(self, vals):
        self._c(lib().qmpm_append_state(self.ctx, vals.shape[0], ptr(vals)))

    def set_words(self, words, step):
        self._c(lib().qmpm_set_words(self.ctx, words.shape[0], ptr(words), step))

    def set_ids(self, ids):
        self._c(lib().qmpm_set_ids(self.ctx, ids.shape[0], ptr(ids)))

    def step(self, n_steps=1):
        self._c(lib().qmpm_step(self.ctx, n_steps))

    def read_state(self, vals=None, words=None, ids=None, capacity=None):
        n = ctypes.c_uint64()
        cap = capacity
        if cap is None:
            for a in (vals, words, ids):
                if a is not None:
                    cap = a.shape[0]
                    break
        self._c(lib().qmpm_read_state(self.ctx, ptr(vals), ptr(words), ptr(ids), cap or 0, ctypes.byref(n)))
        return n.value

    def read_debug(self, pre):
        n = ctypes.c_uint64()
        self._c(lib().qmpm_read_debug(self.ctx, ptr(pre), pre.shape[0], ctypes.byref(n)))
        return n.value

    def read_ranges(self, reset=False):
        """qmpm_read_ranges: max |value| per state scalar since set_state / the last reset
        (needs flags |= RECORD_RANGES)."""
        out = np.zeros(self.n_scalars, np.float32)
        self._c(lib().qmpm_read_ranges(self.ctx, out.ctypes.data, 1 if reset else 0))
        return out

    def stats(self) -> Stats:
        st = Stats()
        self._c(lib().qmpm_stats(self.ctx, ctypes.byref(st)))
        return st

    def set_profiling(self, on=True):
        self._c(lib().qmpm_set_profiling(self.ctx, 1 if on else 0))

    def kernel_times(self):
        ms = (ctypes.c_double * NUM_KERNELS)()
        cnt = (ctypes.c_uint64 * NUM_KERNELS)()
        self._c(lib().qmpm_kernel_times(self.ctx, ms, cnt))
        return {name: (ms[i], cnt[i]) for i, name in enumerate(kernel_names())}

    def launch_count(self):
        return lib().qmpm_launch_count(self.ctx)

    def connect_nccl(self, uid: bytes):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self._c(lib().qmpm_connect_nccl(self.ctx, buf))
