"""Stand-in quantization schemes {(b_h, R_h)} as plain data.

The paper's actual schemes live in an unavailable supplement,
so these are the stand-ins of SURVEY.md §8(c) Q1 / DESIGN.md "Readings": bit
widths follow the paper's compression figures (teaser P:85, T-large P:945-946),
ranges are powers of two (so Delta = R 2^-b is exact) chosen as 2x the recorded
magnitudes ("multiply the ranges by a factor (e.g., 2)").

A scheme is a dict:
  dim, material ("elastic" | "fluid"), rounding ("dither" | "rne"), seed,
  fields: list of {attr: x|v|F|J|C, comp, kind: fixed|raw, frac_bits, range, offset}
in PACKING order (bit pack).  Stored width of a fixed field is
frac_bits + 1 (two's complement, reading Q2).  This module holds data only.
"""

DITHER_SEED = 0x9E3779B97F4A7C15


def _fields(attr, n, kind, frac_bits=0, rng=1.0, offset=0.0):
    return [dict(attr=attr, comp=c, kind=kind, frac_bits=frac_bits, range=rng, offset=offset)
            for c in range(n)]


def fp32(dim, material="elastic"):
    """All fields RAW_F32: the uncompressed baseline (3D elastic W=24, fluid W=16, 2D W=12)."""
    d = dim
    f = _fields("x", d, "raw") + _fields("v", d, "raw")
    f += _fields("J", 1, "raw") if material == "fluid" else _fields("F", d * d, "raw")
    f += _fields("C", d * d, "raw")
    return dict(dim=dim, material=material, rounding="dither", seed=DITHER_SEED, fields=f)


def x16(v_range=8.0):
    """C1 (2D elastic): x, v 16-bit fixed (b=15); F, C raw fp32 -> 320 bits, W=10."""
    f = _fields("x", 2, "fixed", 15, 1.0) + _fields("v", 2, "fixed", 15, v_range)
    f += _fields("F", 4, "raw") + _fields("C", 4, "raw")
    return dict(dim=2, material="elastic", rounding="dither", seed=DITHER_SEED, fields=f)


def e01():
    """E0.1 (3D elastic, eps=0.1): x 3x19, v 3x15, F 9x14, C 9x13 = 345 bits, W=11."""
    f = _fields("x", 3, "fixed", 18, 1.0) + _fields("v", 3, "fixed", 14, 8.0)
    f += _fields("F", 9, "fixed", 13, 4.0) + _fields("C", 9, "fixed", 12, 256.0)
    return dict(dim=3, material="elastic", rounding="dither", seed=DITHER_SEED, fields=f)


def e001():
    """E0.01 (3D elastic, eps=0.01): x 3x20, v 3x16, F 9x14, C 9x13 = 351 bits, W=11."""
    f = _fields("x", 3, "fixed", 19, 1.0) + _fields("v", 3, "fixed", 15, 8.0)
    f += _fields("F", 9, "fixed", 13, 4.0) + _fields("C", 9, "fixed", 12, 256.0)
    return dict(dim=3, material="elastic", rounding="dither", seed=DITHER_SEED, fields=f)


def f2():
    """F2 (3D fluid): x 3x19, v 3x15, J 1x16 (offset 1), C 9x15 = 253 bits, W=8."""
    f = _fields("x", 3, "fixed", 18, 1.0) + _fields("v", 3, "fixed", 14, 8.0)
    f += _fields("J", 1, "fixed", 15, 0.25, 1.0) + _fields("C", 9, "fixed", 14, 256.0)
    return dict(dim=3, material="fluid", rounding="dither", seed=DITHER_SEED, fields=f)


def with_domain(sch, sim):
    """The scheme's position fields widened to the simulation domain: a FIXED x
    component whose range is below the domain's extent along its axis (grid_res * dx)
    gets range 2^ceil(log2 extent) and log2 of that many more fraction bits, so
    Delta = range 2^-b is unchanged (the integer next-step key and the grid stay
    aligned) and positions beyond 1 do not saturate.  The z-slab weak-scaling runs
    (bench.py --gpus N) extend C4's domain N times along z: F2's x_z goes from 19 to
    19 + log2 N bits (253 + 3 = 256 bits = 8 words at N = 8)."""
    import copy
    import math
    out = copy.deepcopy(sch)
    for f in out["fields"]:
        if f["attr"] != "x" or f["kind"] != "fixed" or f.get("offset", 0.0) != 0.0:
            continue
        ext = float(sim["grid_res"][f["comp"]]) * float(sim["dx"])
        if ext <= f["range"]:
            continue
        k = math.ceil(math.log2(ext / f["range"]))
        f["range"] = f["range"] * 2.0 ** k
        f["frac_bits"] = f["frac_bits"] + k
    return out


def ranges_from_record(max_abs, factor=2.0, pow2=True):
    """R_h from a recorded full-precision run ("record the ranges from the full
    precision simulation and multiply the ranges by a factor (e.g., 2)"); rounded up
    to a power of two so Delta = R 2^-b is exact (reading Q1).  Zero ranges become 1."""
    import math
    out = []
    for m in max_abs:
        r = factor * float(m)
        if not r > 0.0:
            r = 1.0
        if pow2:
            r = 2.0 ** math.ceil(math.log2(r))
        out.append(r)
    return out


def scalar_names(dim, material):
    """(attr, comp) of each state scalar, in the order of qmpm_set_state."""
    d = dim
    names = [("x", c) for c in range(d)] + [("v", c) for c in range(d)]
    names += [("J", 0)] if material == "fluid" else [("F", c) for c in range(d * d)]
    names += [("C", c) for c in range(d * d)]
    return names


def from_solution(dim, material, ranges, bits, rounding="dither"):
    """A scheme with every state scalar FIXED, in state-scalar order, from per-scalar
    ranges R_h and fraction bits b_h (Algorithm 1's output (b_h, R_h))."""
    f = [dict(attr=a, comp=c, kind="fixed", frac_bits=int(b), range=float(r), offset=0.0)
         for (a, c), r, b in zip(scalar_names(dim, material), ranges, bits)]
    return dict(dim=dim, material=material, rounding=rounding, seed=DITHER_SEED, fields=f)


def se2():
    """A SHARED_EXP stand-in (reading Q4) for the 3D fluid: x 3x19 fixed; v one group of
    3 mantissas (b = 11) sharing a 4-bit exponent from R_min = 2^-4; J 1x16 fixed
    (offset 1); C one group of 9 mantissas (b = 11) sharing a 5-bit exponent from
    R_min = 2^-3 -> 57 + 4 + 36 + 16 + 5 + 108 = 226 bits, W = 8."""
    f = _fields("x", 3, "fixed", 18, 1.0)
    f += [dict(attr="v", comp=c, kind="shared_exp", frac_bits=11, exp_bits=4, range=2.0 ** -4, offset=0.0,
               group=1) for c in range(3)]
    f += _fields("J", 1, "fixed", 15, 0.25, 1.0)
    f += [dict(attr="C", comp=c, kind="shared_exp", frac_bits=11, exp_bits=5, range=2.0 ** -3, offset=0.0,
               group=2) for c in range(9)]
    return dict(dim=3, material="fluid", rounding="dither", seed=DITHER_SEED, fields=f)


# ---------------------------------------------------------------- smoke (f4)
# Records of two cells (reading S2): velocity 6 fields (cell0 ux uy uz, cell1 ux uy uz),
# pressure 2 fields.  Fields carry no attr (the smoke path does not map MPM scalars).
def smoke_u(frac_bits=15, rng=2.0, rounding="dither"):
    """Velocity, 6 x (b+1)-bit fixed point; default 6 x 16 = 96 bits, W = 3 (48 bits per cell)."""
    f = [dict(kind="fixed", frac_bits=frac_bits, range=rng, offset=0.0) for _ in range(6)]
    return dict(dim=3, material="fluid", rounding=rounding, seed=DITHER_SEED ^ 0x5, fields=f)


def smoke_p(frac_bits=15, rng=1.0, rounding="dither"):
    """Pressure, 2 x (b+1)-bit fixed point; default 2 x 16 = 32 bits, W = 1 (16 bits per cell).
    With smoke_u: 64 bits per cell against 128 in fp32 -- 2.0x (the paper's smoke: 1.93x)."""
    f = [dict(kind="fixed", frac_bits=frac_bits, range=rng, offset=0.0) for _ in range(2)]
    return dict(dim=3, material="fluid", rounding=rounding, seed=DITHER_SEED ^ 0x6, fields=f)


def smoke_u_shared(frac_bits=13, exp_bits=4, r_min=2.0 ** -3):
    """Velocity as SHARED_EXP (reading Q4): each cell's 3 components share an exponent:
    2 x (4 + 3 x 14) = 92 bits, W = 3."""
    f = [dict(kind="shared_exp", frac_bits=frac_bits, exp_bits=exp_bits, range=r_min, offset=0.0, group=1 + c // 3)
         for c in range(6)]
    return dict(dim=3, material="fluid", rounding="dither", seed=DITHER_SEED ^ 0x7, fields=f)


def smoke_p_shared(frac_bits=11, exp_bits=4, r_min=2.0 ** -6):
    """Pressure as SHARED_EXP (reading Q4): the two cells of a record share an exponent:
    4 + 2 x 12 = 28 bits, W = 1."""
    f = [dict(kind="shared_exp", frac_bits=frac_bits, exp_bits=exp_bits, range=r_min, offset=0.0, group=1)
         for _ in range(2)]
    return dict(dim=3, material="fluid", rounding="dither", seed=DITHER_SEED ^ 0x8, fields=f)


def smoke_raw(n):
    """fp32 baseline records (n = 6 velocity or 2 pressure fields)."""
    return dict(dim=3, material="fluid", rounding="dither", seed=DITHER_SEED,
                fields=[dict(kind="raw") for _ in range(n)])


def with_layout(scheme, layout):
    """layout: "pack" (bit pack) or "nostraddle" (no field crosses a word: the
    bit struct's rule, P:540 -- the T-bitpack-perf analogue)."""
    s = dict(scheme)
    s["layout"] = layout
    return s


def with_rounding(scheme, rounding):
    s = dict(scheme)
    s["rounding"] = rounding
    return s


BY_NAME = {"x16": x16, "e0.1": e01, "e0.01": e001, "f2": f2, "se2": se2}
