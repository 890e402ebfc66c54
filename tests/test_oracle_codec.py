"""Pins for the oracle's codec, bit pack and dither (CPU only).

Each test pins the oracle to something other than itself: a worked example from
the paper/SPEC, a closed form, an invariant, brute force against an independent
Python big-integer bit vector, or a statistical property the paper states.
"""
import numpy as np
import pytest

import oracle


def fixed_scheme(widths_b, ranges, offsets=None, rounding="dither", seed=1234):
    offsets = offsets or [0.0] * len(widths_b)
    return dict(dim=0, material="elastic", rounding=rounding, seed=seed,
                fields=[dict(kind="fixed", frac_bits=b, range=r, offset=o)
                        for b, r, o in zip(widths_b, ranges, offsets)])


def raw_scheme(n):
    return dict(dim=0, material="elastic", rounding="dither", seed=0,
                fields=[dict(kind="raw") for _ in range(n)])


# --------------------------------------------------------------- Eq. 3 examples
def test_spec_worked_example_round_and_saturate():
    """b=2, R=1 (Delta=0.25): v=0.6 -> u=2, decodes to 0.5 (error 0.1);
    v=1.5 saturates at u=3 = 2^2-1 with one saturation counted; v=0 -> 0."""
    s = fixed_scheme([2], [1.0], rounding="rne")
    words, cnt = oracle.encode(s, np.array([[0.6]], np.float32))
    assert words[0, 0] == 2
    assert oracle.decode(s, words)[0, 0] == np.float32(0.5)
    words, cnt = oracle.encode(s, np.array([[1.5]], np.float32))
    assert words[0, 0] == 3 and cnt[0] == 1
    words, cnt = oracle.encode(s, np.array([[0.0]], np.float32))
    assert words[0, 0] == 0 and cnt[0] == 0


def test_negative_codes_two_complement():
    """Reading Q2: b+1-bit two's complement, range [-2^b, 2^b-1]."""
    s = fixed_scheme([2], [1.0], rounding="rne")
    words, cnt = oracle.encode(s, np.array([[-1.0], [-5.0], [-0.26]], np.float32))
    assert list(words[:, 0]) == [0b100, 0b100, 0b111]  # -4, -4 (saturated), -1
    assert cnt[0] == 1
    assert list(oracle.decode(s, words)[:, 0]) == [-1.0, -1.0, -0.25]


def test_round_half_even_ties():
    """Reading Q6: undithered ties round half to even."""
    s = fixed_scheme([4], [16.0], rounding="rne")  # Delta = 1
    v = np.array([[0.5], [1.5], [2.5], [-0.5], [-1.5]], np.float32)
    w, _ = oracle.encode(s, v)
    u = oracle.decode(s, w)[:, 0]
    assert list(u) == [0.0, 2.0, 2.0, 0.0, -2.0]


def test_roundtrip_half_ulp_power_of_two_range():
    """|decode(encode(v)) - v| <= Delta/2 for 1e5 random v in [-R+D, R-D]
    (exact bound: Delta is a power of two, so t = v/Delta is exact)."""
    rng = np.random.default_rng(0)
    for b, R in [(7, 1.0), (15, 8.0), (19, 1.0), (12, 256.0)]:
        D = R * 2.0 ** -b
        v = rng.uniform(-R + D, R - D, size=(100_000, 1)).astype(np.float32)
        s = fixed_scheme([b], [R], rounding="rne")
        w, cnt = oracle.encode(s, v)
        err = np.abs(oracle.decode(s, w).astype(np.float64) - v.astype(np.float64))
        assert err.max() <= D / 2
        assert cnt[0] == 0


def test_roundtrip_general_range_bound():
    """Non power-of-two R: error <= Delta/2 + 2^-23 |v| (one fp32 rounding of t)."""
    rng = np.random.default_rng(1)
    b, R = 13, 3.7
    D = float(np.float32(R * 2.0 ** -b))
    v = rng.uniform(-R + D, R - D, size=(50_000, 1)).astype(np.float32)
    s = fixed_scheme([b], [R], rounding="rne")
    w, _ = oracle.encode(s, v)
    err = np.abs(oracle.decode(s, w).astype(np.float64) - v.astype(np.float64))
    assert np.all(err[:, 0] <= D / 2 + 2.0 ** -23 * np.abs(v[:, 0]) * 2 + 1e-12)


@pytest.mark.parametrize("b", [0, 1, 5, 11, 15])
def test_exhaustive_idempotence(b):
    """re-encoding a decoded value is the identity, for every code (b <= 16)."""
    s = fixed_scheme([b], [2.0], rounding="rne")
    codes = np.arange(-(2 ** b), 2 ** b, dtype=np.int64)
    words = (codes & ((1 << (b + 1)) - 1)).astype(np.uint32).reshape(-1, 1)
    vals = oracle.decode(s, words)
    assert np.all(vals[:, 0] == codes * np.float32(2.0 * 2.0 ** -b))  # u * Delta exactly
    w2, cnt = oracle.encode(s, vals)
    assert np.array_equal(w2, words) and cnt[0] == 0
    # dithered re-encode of an on-grid value never moves it (y = 0)
    w3, cnt3 = oracle.encode(s, vals, keys=np.arange(len(vals), dtype=np.uint32), step=7)
    assert np.array_equal(w3, words) and cnt3[64] == 0 and cnt3[128] == 0


def test_offset_field():
    """Reading Q21: value = offset + u*Delta."""
    s = fixed_scheme([15], [0.25], offsets=[1.0], rounding="rne")
    v = np.array([[1.0], [1.1], [0.95]], np.float32)
    w, _ = oracle.encode(s, v)
    d = oracle.decode(s, w)[:, 0]
    assert d[0] == 1.0
    assert np.all(np.abs(d - v[:, 0]) <= 0.25 * 2 ** -15 / 2 + 1e-7)


def test_raw_f32_bitcast():
    s = raw_scheme(3)
    v = np.array([[1.5, -0.0, 3.4e38]], np.float32)
    w, _ = oracle.encode(s, v)
    assert np.array_equal(w.view(np.float32), v)
    assert np.array_equal(oracle.decode(s, w).view(np.uint32), v.view(np.uint32))


def test_nonfinite_counted():
    """non-finite input is flagged (code 0 for fixed fields)."""
    s = fixed_scheme([8, 8], [1.0, 1.0], rounding="rne")
    w, cnt = oracle.encode(s, np.array([[np.nan, np.inf]], np.float32))
    assert cnt[192] == 2 and w[0, 0] == 0


# --------------------------------------------------------------- bit pack layout
def test_layout_three_17bit_fields():
    """Fig. bit_struct: three 17-bit elements fit into two 32-bit words;
    S:119: offsets 0, 17, 34."""
    s = fixed_scheme([16, 16, 16], [1.0] * 3)
    offs, W, bits = oracle.layout(s)
    assert list(offs) == [0, 17, 34] and W == 2 and bits == 51


def test_cross_word_extraction_example():
    """field at offset 17, width 17, word0 = 0xFFFE0000, word1 = 0x3 -> 0x1FFFF."""
    rec = np.array([0xFFFE0000, 0x00000003], np.uint32)
    L = oracle.lib()
    assert L.oracle_get_bits(rec.ctypes.data, 17, 17) == 0x1FFFF


def test_layout_rejects_bad_widths():
    """width 0 or > 32 rejected."""
    with pytest.raises(ValueError):
        oracle.layout(fixed_scheme([32], [1.0]))  # width 33
    assert oracle.layout(fixed_scheme([31], [1.0]))[1] == 1


def _bigint_get(words, off, width):
    v = int.from_bytes(np.asarray(words, np.uint32).tobytes(), "little")
    return (v >> off) & ((1 << width) - 1)


def _bigint_put(words, off, width, value):
    v = int.from_bytes(np.asarray(words, np.uint32).tobytes(), "little")
    mask = ((1 << width) - 1) << off
    v = (v & ~mask) | ((value << off) & mask)
    return np.frombuffer(v.to_bytes(4 * len(words), "little"), np.uint32).copy()


def test_put_get_exhaustive_widths_offsets():
    """round trip for every width 1..32 at every offset 0..31, neighbours
    untouched; checked against an independent Python big-integer bit vector."""
    rng = np.random.default_rng(2)
    L = oracle.lib()
    for width in range(1, 33):
        for off in range(32):
            rec = rng.integers(0, 2 ** 32, size=3, dtype=np.uint64).astype(np.uint32)
            val = int(rng.integers(0, 2 ** width))
            expect = _bigint_put(rec, off, width, val)
            got = rec.copy()
            L.oracle_put_bits(got.ctypes.data, off, width, val)
            assert np.array_equal(got, expect), (width, off)
            assert L.oracle_get_bits(got.ctypes.data, off, width) == _bigint_get(got, off, width) == val


def test_sign_extension_boundaries():
    """boundary codes +-2^(w-1) -+ 1 decode exactly (Delta = 1)."""
    for b in range(1, 24):
        w = b + 1
        s = fixed_scheme([b], [float(2 ** b)], rounding="rne")
        codes = np.array([2 ** (w - 1) - 1, -(2 ** (w - 1)) + 1, -(2 ** (w - 1)), -1, 0])
        words = (codes & ((1 << w) - 1)).astype(np.uint32).reshape(-1, 1)
        assert np.array_equal(oracle.decode(s, words)[:, 0], codes.astype(np.float32))


def test_packed_record_matches_bigint_reference():
    """Random multi-field records: every field lands at its layout offset LSB-first."""
    rng = np.random.default_rng(3)
    b = [18, 14, 13, 12, 19, 7, 30, 0, 21]
    R = [1.0, 8.0, 4.0, 256.0, 2.0, 1.0, 16.0, 1.0, 0.5]
    s = fixed_scheme(b, R, rounding="rne")
    offs, W, bits = oracle.layout(s)
    vals = np.stack([rng.uniform(-r, r, 500) for r in R], axis=1).astype(np.float32)
    words, _ = oracle.encode(s, vals)
    dec = oracle.decode(s, words)
    for i in range(500):
        for f in range(len(b)):
            raw = _bigint_get(words[i], int(offs[f]), b[f] + 1)
            u = raw - (1 << (b[f] + 1)) if raw >> b[f] else raw
            assert dec[i, f] == np.float32(np.float32(u) * np.float32(R[f] * 2.0 ** -b[f]))


# --------------------------------------------------------------- dithering (Eq. 11)
def test_dither_round_up_probability_is_fraction():
    """P(round up) = Y = v/Delta - floor(v/Delta); binomial 3-sigma at n=1e5."""
    n = 100_000
    for Y in [0.1, 0.25, 0.4, 0.5, 0.9]:
        s = fixed_scheme([10], [1024.0])  # Delta = 1
        v = np.full((n, 1), 37.0 + Y, np.float32)
        w, cnt = oracle.encode(s, v, keys=np.arange(n, dtype=np.uint32), step=1)
        u = oracle.decode(s, w)[:, 0]
        assert set(np.unique(u)) <= {37.0, 38.0}
        p = float(np.mean(u == 38.0))
        yy = float(np.float32(37.0 + Y)) - 37.0
        assert abs(p - yy) <= 3 * np.sqrt(yy * (1 - yy) / n)
        assert cnt[64] == np.sum(u == 38.0) and cnt[128] == np.sum(u == 37.0)


def test_dither_unbiased_and_within_one_ulp():
    """bias < 4 Delta / sqrt(12 n) at n = 1e5 ("~3.6 standard errors"); |err| < Delta
    (1 ulp).  S:75's standard error takes the error variance as Delta^2 / 12; for a FIXED
    v the dithered error is Bernoulli, variance y (1 - y) Delta^2 (up to Delta^2 / 4 at
    y = 1/2), so the bound is applied as 4 of the actual standard errors when that is larger."""
    n = 100_000
    rng = np.random.default_rng(4)
    b, R = 12, 8.0
    D = R * 2.0 ** -b
    for v0 in rng.uniform(-R + D, R - D, 5):
        v = np.full((n, 1), v0, np.float32)
        s = fixed_scheme([b], [R])
        w, _ = oracle.encode(s, v, keys=rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32), step=3)
        err = oracle.decode(s, w)[:, 0].astype(np.float64) - float(v[0, 0])
        assert np.abs(err).max() < D
        t = float(v[0, 0]) / D
        y = t - np.floor(t)
        assert abs(err.mean()) < max(4 * D / np.sqrt(12 * n), 4 * D * np.sqrt(y * (1 - y) / n))


def test_drift_pathology():
    """Fig. dithering_illustration (reading Q7): adding 1.4 Delta ten
    times gives exactly 10 Delta with round-to-nearest, and 14 Delta +- 0.5 Delta on
    average over 2000 dithered trials (wide type b = 16)."""
    b, R = 16, 2.0 ** 16  # Delta = 1
    s_rne = fixed_scheme([b], [R], rounding="rne")
    s_dit = fixed_scheme([b], [R], rounding="dither")
    trials = 2000
    y_rne = np.zeros((1, 1), np.float32)
    y_dit = np.zeros((trials, 1), np.float32)
    keys = np.arange(trials, dtype=np.uint32)
    for t in range(1, 11):
        w, _ = oracle.encode(s_rne, y_rne + np.float32(1.4))
        y_rne = oracle.decode(s_rne, w)
        w, _ = oracle.encode(s_dit, y_dit + np.float32(1.4), keys=keys, step=t)
        y_dit = oracle.decode(s_dit, w)
    assert y_rne[0, 0] == 10.0
    assert abs(float(y_dit.mean()) - 14.0) < 0.5


def test_round_up_down_counts():
    """T-dither-eff reports round-up/round-down counts.  With dithering
    the expected ratio is sum(y)/sum(1-y) (P(up) = y), which is ~1 for
    uniformly distributed fractional parts; round-to-nearest counts follow
    numpy's round-half-even (np.rint)."""
    rng = np.random.default_rng(5)
    n = 200_000
    s_dit = fixed_scheme([10], [1024.0])
    s_rne = fixed_scheme([10], [1024.0], rounding="rne")
    for frac in (rng.uniform(0.0, 1.0, n), rng.uniform(0.0, 0.45, n) ** 0.5):
        v = (rng.integers(-100, 100, n) + frac).astype(np.float32).reshape(-1, 1)
        y = v[:, 0].astype(np.float64) - np.floor(v[:, 0].astype(np.float64))
        _, cd = oracle.encode(s_dit, v, keys=np.arange(n, dtype=np.uint32), step=1)
        _, cr = oracle.encode(s_rne, v)
        expect = y.sum() / (1 - y[y > 0]).sum()
        assert abs(cd[64] / cd[128] / expect - 1.0) < 0.02
        vv = v[:, 0].astype(np.float64)
        assert cr[64] == np.sum(np.rint(vv) > vv) and cr[128] == np.sum(np.rint(vv) < vv)
    # uniform fractional parts: dithered ratio ~ 1 (cf. 0.999976 in T-dither-eff)
    frac = rng.uniform(0.0, 1.0, n)
    v = (rng.integers(-100, 100, n) + frac).astype(np.float32).reshape(-1, 1)
    _, cd = oracle.encode(s_dit, v, keys=np.arange(n, dtype=np.uint32), step=2)
    assert abs(cd[64] / cd[128] - 1.0) < 0.02


# --------------------------------------------------------------- RNG (reading Q5, revision 3)
def _encode_value_fn():
    import ctypes
    L = oracle.lib()
    fn = L.oracle_encode_value
    fn.restype = ctypes.c_int64
    fn.argtypes = [ctypes.c_float, ctypes.c_uint32, ctypes.c_float, ctypes.c_float, ctypes.c_int, ctypes.c_uint32,
                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    return fn


def test_dither_rule_exact_probability_over_all_draws():
    """Eq. 11 with a 16-bit draw (reading Q5 rev. 3, Q6): u = floor(t) +
    [y >= 1 - r16 2^-16], so over all 2^16 draws exactly 2^16 - ceil((1 - y) 2^16) round
    up -- P(up) = y to within 2^-16 (closed form; a flipped comparison, an off-by-one in
    the threshold or a 24-bit scale all change the count)."""
    enc = _encode_value_fn()
    rng = np.random.default_rng(21)
    ys = [0.0, 2.0 ** -20, 0.25, 0.5, 1.0 - 2.0 ** -16, 1.0 - 2.0 ** -17, 0.7] + list(rng.uniform(0, 1, 6))
    for y in ys:
        v = np.float32(37.0 + y)  # Delta = 1: t = v, y = t - 37 exactly in fp32
        yy = float(v) - 37.0
        ups = sum(enc(float(v), 10, 1024.0, 0.0, 1, r, None, None, None, None) == 38 for r in range(0, 65536, 1))
        expect = 65536 - int(np.ceil((1.0 - yy) * 65536.0))
        assert ups == expect, (y, ups, expect)
        assert abs(ups / 65536.0 - yy) < 2.0 ** -16 + 1e-12


def test_r16_uniform_chi_square_and_step_decorrelation():
    """Self-defined RNG (the paper's, is unavailable): every r16 is uniform (chi^2
    over 256 bins, 2^18 keys), fields and steps are uncorrelated."""
    n = 1 << 18
    keys = np.arange(n, dtype=np.uint32)
    lim = 255 + 5 * np.sqrt(2 * 255)
    draws = {}
    for f in (0, 1, 2, 7, 23):
        r = oracle.r16_batch(7, 5, keys, f).astype(np.int64)
        assert r.max() < 2 ** 16
        hist = np.bincount(r >> 8, minlength=256)
        assert float(np.sum((hist - n / 256) ** 2 / (n / 256))) < lim, f
        draws[f] = r.astype(np.float64)
    assert abs(np.corrcoef(draws[0], draws[1])[0, 1]) < 0.01
    r_next = oracle.r16_batch(7, 6, keys, 0).astype(np.float64)
    assert abs(np.corrcoef(draws[0], r_next)[0, 1]) < 0.01


def test_r16_all_24_fields_pairwise_jointly_uniform():
    """All 24 fields of a 3D elastic record (C3 dithers 24 per particle): every pair of
    fields is jointly uniform (chi^2 over 32x32 bins of the top bits, 2^16 keys) and
    uncorrelated.  The pair (2p, 2p+1) shares one hash and is exactly jointly uniform by
    construction (disjoint bits of a bijection of h)."""
    n = 1 << 16
    keys = (np.arange(n, dtype=np.uint64) * 2654435761 % (1 << 32)).astype(np.uint32)
    r = np.stack([oracle.r16_batch(11, 3, keys, f) for f in range(24)], axis=1).astype(np.int64)
    e = n / 1024
    lim = 1023 + 5.5 * np.sqrt(2 * 1023)
    for f in range(24):
        hist = np.bincount(r[:, f] >> 6, minlength=1024)
        assert float(np.sum((hist - e) ** 2 / e)) < lim, f
        for g in range(f + 1, 24):
            joint = np.bincount((r[:, f] >> 11) * 32 + (r[:, g] >> 11), minlength=1024)
            assert float(np.sum((joint - e) ** 2 / e)) < lim, (f, g)
            assert abs(np.corrcoef(r[:, f], r[:, g])[0, 1]) < 0.02, (f, g)


def test_r16_pair_draws_partition_the_pair_hash():
    """The two draws of a pair are disjoint bit ranges that together cover the pair hash:
    even field = bits 7..22 of z, odd field = bits 23..31 and 0..6 (so (r_even, r_odd) is
    a bijection of z, the exact joint uniformity claimed in DESIGN.md reading Q5)."""
    L = oracle.lib()
    rng = np.random.default_rng(5)
    for key in rng.integers(0, 2 ** 32, 200, dtype=np.uint64):
        for p in range(12):
            z = L.oracle_pair_hash(3, 9, int(key), p)
            a, b = oracle.r16(3, 9, int(key), 2 * p), oracle.r16(3, 9, int(key), 2 * p + 1)
            assert a | (b << 16) == ((z >> 7) | (z << 25)) & 0xFFFFFFFF


def test_rng_golden_vector():
    """Regression pin of the definition (tests/golden/rng_rev3.json, tools/gen_rng_golden.py)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rng_rev3.json")))
    L = oracle.lib()
    for c in g["cases"]:
        assert [L.oracle_pair_hash(c["seed"], c["step"], c["key"], p) for p in range(4)] == c["pair_hash"]
        assert [oracle.r16(c["seed"], c["step"], c["key"], f) for f in range(8)] == c["r16"]
    from paper_2207_04658_b200 import schemes
    for c in g["particle_keys_f2"]:
        assert oracle.particle_key(schemes.f2(), np.array(c["record"], np.uint32)) == c["key"]


def test_particle_key_depends_on_x_words_only():
    """Reading Q5: the content key folds exactly the record words holding x bits (F2: words
    0 and 1, x = 3 x 19 bits); any other word leaves it unchanged, every x word changes it."""
    from paper_2207_04658_b200 import schemes
    sch = schemes.f2()
    rng = np.random.default_rng(3)
    for _ in range(50):
        r = rng.integers(0, 2 ** 32, 8, dtype=np.uint64).astype(np.uint32)
        k = oracle.particle_key(sch, r)
        for w in range(8):
            r2 = r.copy()
            r2[w] ^= np.uint32(1 << int(rng.integers(0, 32)))
            assert (oracle.particle_key(sch, r2) != k) == (w < 2), w


def test_mix32_is_a_bijection_on_a_sample():
    L = oracle.lib()
    xs = np.arange(0, 1 << 16, dtype=np.uint64) * 65537 + 12345
    hs = {L.oracle_mix32(int(x) & 0xFFFFFFFF) for x in xs}
    assert len(hs) == len(xs)
    assert L.oracle_mix32(0) == 0


# --------------------------------------------------------------- SHARED_EXP (reading Q4)
def shared_scheme(n, b, e, R, rounding="rne", groups=None):
    groups = groups or [0] * n
    return dict(dim=0, material="elastic", rounding=rounding, seed=11,
                fields=[dict(kind="shared_exp", frac_bits=b, exp_bits=e, range=R, offset=0.0, group=g)
                        for g in groups])


def test_shared_exp_worked_example():
    """Reading Q4 by hand: b = 3, e = 3, R_min = 1/4, v = (0.6, -0.1, 0.05): M = 0.6 ->
    smallest E with 0.6 < 2^E / 4 is E = 2 (range 1, Delta = 1/8); codes rne(4.8) = 5,
    rne(-0.8) = -1, rne(0.4) = 0 -> (0.625, -0.125, 0).  Layout: 3 + 4 + 4 + 4 bits."""
    s = shared_scheme(3, 3, 3, 0.25)
    offs, W, bits = oracle.layout(s)
    assert list(offs) == [0, 7, 11] and bits == 15
    w, cnt = oracle.encode(s, np.array([[0.6, -0.1, 0.05]], np.float32))
    L = oracle.lib()
    assert L.oracle_get_bits(w[0].ctypes.data, 0, 3) == 2
    assert L.oracle_get_bits(w[0].ctypes.data, 3, 4) == 5
    assert L.oracle_get_bits(w[0].ctypes.data, 7, 4) == 0b1111
    assert L.oracle_get_bits(w[0].ctypes.data, 11, 4) == 0
    assert list(oracle.decode(s, w)[0]) == [0.625, -0.125, 0.0]


def test_shared_exp_rounding_overflow_raises_the_exponent():
    """b = 3, R_min = 1: M = 0.97 < 1 gives E = 0, but rne(0.97 * 8) = 8 > 2^3 - 1, so
    E = 1 (Delta = 1/4) and the code is rne(3.88) = 4 -> 1.0, no saturation counted."""
    s = shared_scheme(2, 3, 2, 1.0)
    w, cnt = oracle.encode(s, np.array([[0.97, 0.1]], np.float32))
    assert oracle.lib().oracle_get_bits(w[0].ctypes.data, 0, 2) == 1
    assert list(oracle.decode(s, w)[0]) == [1.0, 0.0]
    assert cnt[0] == 0 and cnt[1] == 0


def test_shared_exp_zero_group_and_saturation():
    s = shared_scheme(3, 5, 2, 0.5)
    w, _ = oracle.encode(s, np.zeros((1, 3), np.float32))
    assert np.all(w == 0)
    # E_max = 3: range 0.5 * 8 = 4; 100 saturates at the largest code, counted
    w, cnt = oracle.encode(s, np.array([[100.0, -100.0, 1.0]], np.float32))
    d = oracle.decode(s, w)[0]
    assert oracle.lib().oracle_get_bits(w[0].ctypes.data, 0, 2) == 3
    assert d[0] == 4.0 * (31 / 32) and d[1] == -4.0 and d[2] == 1.0
    assert cnt[0] == 1 and cnt[1] == 1 and cnt[2] == 0


@pytest.mark.parametrize("rounding", ["rne", "dither"])
def test_shared_exp_error_bound_and_minimal_exponent(rounding):
    """Per group the stored E is the smallest that holds max |v| (or one more after a
    rounding overflow), and every member is within 1/2 Delta_E (RNE) or below Delta_E
    (dithered) of its value (Eq. 3 / Eq. 11 with the group's resolution)."""
    rng = np.random.default_rng(3)
    b, e, R = 9, 4, 2.0 ** -6
    s = shared_scheme(6, b, e, R, rounding=rounding, groups=[0, 0, 0, 1, 1, 1])
    n = 20000
    mag = 2.0 ** rng.uniform(-8, 7, (n, 2))
    v = (rng.uniform(-1, 1, (n, 6)) * np.repeat(mag, 3, axis=1)).astype(np.float32)
    keys = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32) if rounding == "dither" else None
    w, _ = oracle.encode(s, v, keys=keys, step=3)
    d = oracle.decode(s, w)
    offs, _, _ = oracle.layout(s)
    L = oracle.lib()
    for g, f0 in enumerate((0, 3)):
        E = np.array([L.oracle_get_bits(w[i].ctypes.data, int(offs[f0]), e) for i in range(n)])
        M = np.abs(v[:, f0:f0 + 3]).max(axis=1).astype(np.float64)
        delta = R * 2.0 ** (E - b)
        err = np.abs(d[:, f0:f0 + 3] - v[:, f0:f0 + 3]).max(axis=1)
        ok = E < 2 ** e - 1
        if rounding == "rne":
            assert np.all(err[ok] <= 0.5 * delta[ok] * (1 + 1e-7))
        else:
            assert np.all(err[ok] < delta[ok])
        minimal = (E == 0) | (M >= R * 2.0 ** (E - 1)) | (M >= R * 2.0 ** (E - 1) * (1 - 2.0 ** -b))
        assert np.all(minimal)
        assert np.all(M[ok] < R * 2.0 ** E[ok])
