"""CPU oracle for the quantized MLS-MPM hot path (arXiv 2207.04658) -- ctypes wrapper.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no code
with paper_2207_04658_b200/ (the CUDA path): it builds and loads its own plain-C
library (oracle/*.c, compiled with -ffp-contract=off) and reimplements the field
-> state-scalar mapping itself.

Every C function cites the paper passage it follows (see oracle/*.c headers).
Pins: tests/test_oracle_codec.py, tests/test_oracle_mpm.py.  "Parity unpinned":
the 100-step aggregates beyond the invariants, and the dither RNG's exact bits
(a self-defined generator, reading Q5; only statistical pins exist).
"""
from __future__ import annotations

import os as _os
_os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")  # see tests/conftest.py
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["codec.c", "mpm.c"]
_DEPS = _SOURCES + ["oracle.h", "mpm_impl.h"]

MAX_FIELDS = 64
NCOUNTERS = 194


def build(force=False):
    """Compile liboracle.so with plain gcc (no FMA contraction)."""
    srcs = [os.path.join(_HERE, s) for s in _SOURCES]
    deps = [os.path.join(_HERE, s) for s in _DEPS]
    if not force and os.path.exists(_LIB_PATH):
        t = os.path.getmtime(_LIB_PATH)
        if all(os.path.getmtime(d) <= t for d in deps):
            return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-fopenmp",
           "-shared", "-o", _LIB_PATH] + srcs + ["-lm"]
    subprocess.check_call(cmd, cwd=_HERE)
    return _LIB_PATH


class OracleScheme(ctypes.Structure):
    _fields_ = [("n_fields", ctypes.c_uint32),
                ("kind", ctypes.c_uint32 * MAX_FIELDS),
                ("frac_bits", ctypes.c_uint32 * MAX_FIELDS),
                ("range", ctypes.c_float * MAX_FIELDS),
                ("offset", ctypes.c_float * MAX_FIELDS),
                ("scalar", ctypes.c_uint32 * MAX_FIELDS),
                ("rounding", ctypes.c_uint32),
                ("layout_policy", ctypes.c_uint32),
                ("dither_seed", ctypes.c_uint64),
                ("exp_bits", ctypes.c_uint32 * MAX_FIELDS),
                ("group", ctypes.c_uint32 * MAX_FIELDS)]


class OracleSim(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("material", ctypes.c_int32),
                ("grid_res", ctypes.c_int32 * 3), ("bound", ctypes.c_int32),
                ("dx", ctypes.c_double), ("dt", ctypes.c_double),
                ("gravity", ctypes.c_double * 3),
                ("p_rho", ctypes.c_double), ("p_vol", ctypes.c_double),
                ("E", ctypes.c_double), ("nu", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        sig = {
            "oracle_mix32": (u32, [u32]),
            "oracle_pair_hash": (u32, [u64, u64, u32, u32]),
            "oracle_r16": (u32, [u64, u64, u32, u32]),
            "oracle_r16_batch": (None, [u64, u64, u64, P, u32, P]),
            "oracle_layout": (i32, [P, P, P, P]),
            "oracle_get_bits": (u32, [P, u32, u32]),
            "oracle_put_bits": (None, [P, u32, u32, u32]),
            "oracle_encode": (i32, [P, u64, P, P, u64, P, P]),
            "oracle_decode": (i32, [P, u64, P, P]),
            "oracle_particle_key": (u32, [P, i32, P]),
            "oracle_decode_state": (i32, [P, i32, i32, u64, P, P]),
            "oracle_encode_state": (i32, [P, i32, i32, u64, P, u64, P, P, P]),
            "oracle_p2g_f64": (None, [P, u64, P, P, P, P, P]),
            "oracle_grid_update_f64": (None, [P, P, P, P]),
            "oracle_g2p_f64": (None, [P, u64, P, P, P, P, P]),
            "oracle_polar_f64": (None, [i32, P, P]),
            "oracle_step_f64": (i32, [P, P, u64, P, u64, P, P, P]),
            "oracle_step_f32": (i32, [P, P, u64, P, u64, P, P, P]),
            "oracle_step_sampled_f64": (i32, [P, P, u64, P, u64, u64, P, P, P]),
            "oracle_run_f64": (i32, [P, P, u64, P, u64, u32, P]),
            "oracle_step_omp_f64": (i32, [P, P, u64, P, u64, P, P, P, i32]),
            "oracle_run_omp_f64": (i32, [P, P, u64, P, u64, u32, P, i32]),
            "oracle_num_threads": (i32, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------ scheme/state mapping
def n_scalars(dim, material):
    return 2 * dim + (1 if material == "fluid" else dim * dim) + dim * dim


def scalar_index(attr, comp, dim, material):
    """State scalar order: x[d], v[d], F[d*d] row-major | J, C[d*d] row-major."""
    d = dim
    if attr == "x":
        return comp
    if attr == "v":
        return d + comp
    if attr == "F":
        return 2 * d + comp
    if attr == "J":
        return 2 * d
    if attr == "C":
        return 2 * d + (1 if material == "fluid" else d * d) + comp
    raise ValueError(attr)


def make_scheme(scheme) -> OracleScheme:
    s = OracleScheme()
    fields = scheme["fields"]
    s.n_fields = len(fields)
    for i, f in enumerate(fields):
        s.kind[i] = {"fixed": 0, "raw": 1, "shared_exp": 2}[f["kind"]]
        s.exp_bits[i] = f.get("exp_bits", 0)
        s.group[i] = f.get("group", 0)
        s.frac_bits[i] = f.get("frac_bits", 0)
        s.range[i] = f.get("range", 1.0)
        s.offset[i] = f.get("offset", 0.0)
        if "attr" in f:
            s.scalar[i] = scalar_index(f["attr"], f["comp"], scheme["dim"], scheme["material"])
        else:
            s.scalar[i] = i
    s.rounding = 1 if scheme.get("rounding", "dither") == "dither" else 0
    s.layout_policy = {"pack": 0, "nostraddle": 1}[scheme.get("layout", "pack")]
    s.dither_seed = scheme.get("seed", 0)
    return s


def make_sim(sim) -> OracleSim:
    o = OracleSim()
    o.dim = sim["dim"]
    o.material = 1 if sim["material"] == "fluid" else 0
    for a in range(3):
        o.grid_res[a] = sim["grid_res"][a]
        o.gravity[a] = sim["gravity"][a]
    o.bound = sim["bound"]
    o.dx, o.dt = sim["dx"], sim["dt"]
    o.p_rho, o.p_vol, o.E, o.nu = sim["p_rho"], sim["p_vol"], sim["E"], sim["nu"]
    return o


def _mat(material):
    return 1 if material == "fluid" else 0


# ------------------------------------------------------------ codec
def mix32(x):
    return lib().oracle_mix32(x)


def r16(seed, step, key, field):
    """The 16-bit dither draw of reading Q5 (revision 3)."""
    return lib().oracle_r16(seed, step, key, field)


def r16_batch(seed, step, keys, field):
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    out = np.empty(keys.shape[0], dtype=np.uint32)
    lib().oracle_r16_batch(seed, step, keys.shape[0], _p(keys), field, _p(out))
    return out


def layout(scheme):
    s = make_scheme(scheme)
    offs = np.zeros(MAX_FIELDS, dtype=np.uint32)
    W = np.zeros(1, dtype=np.uint32)
    bits = np.zeros(1, dtype=np.uint32)
    rc = lib().oracle_layout(ctypes.byref(s), _p(offs), _p(W), _p(bits))
    if rc:
        raise ValueError("bad layout")
    return offs[: s.n_fields].copy(), int(W[0]), int(bits[0])


def encode(scheme, vals, keys=None, step=0):
    """vals [n][n_fields] float32 in packing order -> (words [n][W] u32, counters u64[194])."""
    s = make_scheme(scheme)
    _, W, _ = layout(scheme)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    n = vals.shape[0]
    words = np.zeros((n, W), dtype=np.uint32)
    cnt = np.zeros(NCOUNTERS, dtype=np.uint64)
    k = None if keys is None else np.ascontiguousarray(keys, dtype=np.uint32)
    rc = lib().oracle_encode(ctypes.byref(s), n, _p(vals), _p(k), step, _p(words), _p(cnt))
    assert rc == 0
    return words, cnt


def decode(scheme, words):
    s = make_scheme(scheme)
    words = np.ascontiguousarray(words, dtype=np.uint32)
    n = words.shape[0]
    vals = np.zeros((n, s.n_fields), dtype=np.float32)
    assert lib().oracle_decode(ctypes.byref(s), n, _p(words), _p(vals)) == 0
    return vals


def particle_key(scheme, rec):
    s = make_scheme(scheme)
    rec = np.ascontiguousarray(rec, dtype=np.uint32)
    return lib().oracle_particle_key(ctypes.byref(s), scheme["dim"], _p(rec))


def encode_state(scheme, state, step=0, keys=None):
    s = make_scheme(scheme)
    _, W, _ = layout(scheme)
    state = np.ascontiguousarray(state, dtype=np.float32)
    n = state.shape[0]
    words = np.zeros((n, W), dtype=np.uint32)
    cnt = np.zeros(NCOUNTERS, dtype=np.uint64)
    k = None if keys is None else np.ascontiguousarray(keys, dtype=np.uint32)
    rc = lib().oracle_encode_state(ctypes.byref(s), scheme["dim"], _mat(scheme["material"]), n,
                                   _p(state), step, _p(k), _p(words), _p(cnt))
    assert rc == 0, rc
    return words, cnt


def decode_state(scheme, words):
    s = make_scheme(scheme)
    words = np.ascontiguousarray(words, dtype=np.uint32)
    n = words.shape[0]
    st = np.zeros((n, n_scalars(scheme["dim"], scheme["material"])), dtype=np.float32)
    rc = lib().oracle_decode_state(ctypes.byref(s), scheme["dim"], _mat(scheme["material"]), n,
                                   _p(words), _p(st))
    assert rc == 0, rc
    return st


# ------------------------------------------------------------ MPM
def stencil_box(sim, state):
    """Bounding box (origin, gsize) of all particle stencils (plain numpy; fp64)."""
    d = sim["dim"]
    X = np.asarray(state, dtype=np.float64)[:, :d] / sim["dx"]
    base = np.floor(X - 0.5).astype(np.int64)
    for a in range(d):
        base[:, a] = np.clip(base[:, a], 0, sim["grid_res"][a] - 3)
    origin = np.zeros(3, dtype=np.int32)
    gsize = np.ones(3, dtype=np.int32)
    origin[:d] = base.min(axis=0)
    gsize[:d] = base.max(axis=0) + 3 - origin[:d]
    return origin, gsize


def p2g(sim, state, origin=None, gsize=None):
    """fp64 P2G -> (grid [gx][gy][gz][4] = (m, p), origin, gsize, oob)."""
    state = np.ascontiguousarray(state, dtype=np.float64)
    if origin is None:
        origin, gsize = stencil_box(sim, state)
    origin = np.ascontiguousarray(origin, dtype=np.int32)
    gsize = np.ascontiguousarray(gsize, dtype=np.int32)
    grid = np.zeros((int(gsize[0]), int(gsize[1]), int(gsize[2]), 4), dtype=np.float64)
    oob = np.zeros(1, dtype=np.uint64)
    so = make_sim(sim)
    lib().oracle_p2g_f64(ctypes.byref(so), state.shape[0], _p(state), _p(origin), _p(gsize),
                         _p(grid), _p(oob))
    return grid, origin, gsize, int(oob[0])


def grid_update(sim, grid, origin, gsize):
    grid = np.ascontiguousarray(grid, dtype=np.float64).copy()
    so = make_sim(sim)
    lib().oracle_grid_update_f64(ctypes.byref(so), _p(np.asarray(origin, dtype=np.int32)),
                                 _p(np.asarray(gsize, dtype=np.int32)), _p(grid))
    return grid


def g2p(sim, state, grid, origin, gsize):
    state = np.ascontiguousarray(state, dtype=np.float64)
    out = np.zeros_like(state)
    so = make_sim(sim)
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    lib().oracle_g2p_f64(ctypes.byref(so), state.shape[0], _p(state),
                         _p(np.asarray(origin, dtype=np.int32)), _p(np.asarray(gsize, dtype=np.int32)),
                         _p(grid), _p(out))
    return out


def polar(F):
    F = np.ascontiguousarray(F, dtype=np.float64)
    d = int(round(np.sqrt(F.size)))
    R = np.zeros(d * d, dtype=np.float64)
    lib().oracle_polar_f64(d, _p(F.reshape(-1)), _p(R))
    return R.reshape(d, d)


def num_threads():
    """OpenMP threads the parallel oracle uses by default (all host cores)."""
    return lib().oracle_num_threads()


def step(sim, scheme, words, step_index, precision="f64", threads=1):
    """One quantized step from packed words -> (pre_encode [n][ns], words_out, counters).
    threads != 1 (fp64 only): the OpenMP oracle (0 = all cores)."""
    s = make_scheme(scheme)
    so = make_sim(sim)
    words = np.ascontiguousarray(words, dtype=np.uint32)
    n = words.shape[0]
    ns = n_scalars(sim["dim"], sim["material"])
    dt = np.float64 if precision == "f64" else np.float32
    pre = np.zeros((n, ns), dtype=dt)
    out = np.zeros_like(words)
    cnt = np.zeros(NCOUNTERS, dtype=np.uint64)
    if threads != 1:
        assert precision == "f64"
        rc = lib().oracle_step_omp_f64(ctypes.byref(so), ctypes.byref(s), n, _p(words), step_index, _p(pre), _p(out),
                                       _p(cnt), int(threads))
        assert rc == 0, rc
        return pre, out, cnt
    fn = lib().oracle_step_f64 if precision == "f64" else lib().oracle_step_f32
    rc = fn(ctypes.byref(so), ctypes.byref(s), n, _p(words), step_index, _p(pre), _p(out), _p(cnt))
    assert rc == 0, rc
    return pre, out, cnt


def step_sampled(sim, scheme, words, step_index, sample):
    s = make_scheme(scheme)
    so = make_sim(sim)
    words = np.ascontiguousarray(words, dtype=np.uint32)
    sample = np.ascontiguousarray(sample, dtype=np.uint64)
    ns = n_scalars(sim["dim"], sim["material"])
    pre = np.zeros((sample.size, ns), dtype=np.float64)
    out = np.zeros((sample.size, words.shape[1]), dtype=np.uint32)
    rc = lib().oracle_step_sampled_f64(ctypes.byref(so), ctypes.byref(s), words.shape[0], _p(words),
                                       step_index, sample.size, _p(sample), _p(pre), _p(out))
    assert rc == 0, rc
    return pre, out


def run(sim, scheme, words, first_step, n_steps, threads=1):
    """n_steps fp64 steps; threads != 1: the OpenMP oracle (0 = all cores)."""
    s = make_scheme(scheme)
    so = make_sim(sim)
    w = np.ascontiguousarray(words, dtype=np.uint32).copy()
    cnt = np.zeros(NCOUNTERS, dtype=np.uint64)
    if threads != 1:
        rc = lib().oracle_run_omp_f64(ctypes.byref(so), ctypes.byref(s), w.shape[0], _p(w), first_step, n_steps,
                                      _p(cnt), int(threads))
        assert rc == 0, rc
        return w, cnt
    rc = lib().oracle_run_f64(ctypes.byref(so), ctypes.byref(s), w.shape[0], _p(w), first_step,
                              n_steps, _p(cnt))
    assert rc == 0, rc
    return w, cnt


def aggregates(sim, state):
    """KE = 1/2 sum m |v|^2 and COM = sum m x / sum m, fp64 (SURVEY §8(c) C-agg)."""
    d = sim["dim"]
    st = np.asarray(state, dtype=np.float64)
    m = sim["p_rho"] * sim["p_vol"]
    ke = 0.5 * m * float(np.sum(st[:, d:2 * d] ** 2))
    com = st[:, :d].mean(axis=0)
    return ke, com
