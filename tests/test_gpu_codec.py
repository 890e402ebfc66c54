"""GPU parity of the codec (P1): the CUDA encode/decode must be BIT-EXACT to the
oracle on identical fp32 inputs and keys, dithered and not (Eq. 3, Eq. 11, bit
pack P:542-549).  Calls go through the C ABI (qmpm_encode / qmpm_decode /
qmpm_set_state / qmpm_read_state)."""
import numpy as np
import pytest

import oracle
from paper_2207_04658_b200 import qmpm, scenes, schemes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def random_vals(scheme, n, rng, oversat=0.02):
    cols = []
    for f in scheme["fields"]:
        R = f.get("range", 1.0)
        off = f.get("offset", 0.0)
        v = rng.uniform(-R, R, n) + off
        m = rng.random(n) < oversat
        v[m] *= 3.0  # saturating values
        if f["kind"] == "raw":
            v = rng.normal(0, 10, n)
        if f["kind"] == "shared_exp":  # magnitudes across the group's exponent range (and beyond)
            v = rng.uniform(-1, 1, n) * R * 2.0 ** rng.uniform(-3, 2 ** f["exp_bits"] + 1, n)
        cols.append(v)
    return np.stack(cols, 1).astype(np.float32)


def mixed_scheme(rng, nf=23):
    """Random widths 1..32 (some raw), arbitrary ranges/offsets: many straddles."""
    fields = []
    for i in range(nf):
        if rng.random() < 0.15:
            fields.append(dict(kind="raw"))
        else:
            b = int(rng.integers(0, 32))
            fields.append(dict(kind="fixed", frac_bits=b, range=float(2.0 ** rng.integers(-3, 9)),
                               offset=float(rng.choice([0.0, 1.0, -0.5]))))
    return dict(dim=3, material="elastic", rounding="dither", seed=int(rng.integers(0, 2 ** 63)), fields=fields)


def mixed_shared_scheme(rng, nf=24):
    """Fixed / raw fields interleaved with SHARED_EXP groups of 1..9 members (reading Q4),
    random mantissa widths and exponent widths, groups adjacent to each other too."""
    fields, g = [], 0
    while len(fields) < nf:
        r = rng.random()
        if r < 0.5:
            k, b, e = int(rng.integers(1, 10)), int(rng.integers(1, 20)), int(rng.integers(1, 7))
            R = float(2.0 ** rng.integers(-8, 4))
            g += 1
            fields += [dict(kind="shared_exp", frac_bits=b, exp_bits=e, range=R, offset=0.0, group=g)
                       for _ in range(k)]
        elif r < 0.6:
            fields.append(dict(kind="raw"))
        else:
            fields.append(dict(kind="fixed", frac_bits=int(rng.integers(0, 24)), range=float(2.0 ** rng.integers(-3, 9)),
                               offset=0.0))
    fields = fields[:nf]
    return dict(dim=3, material="elastic", rounding="dither", seed=int(rng.integers(0, 2 ** 63)), fields=fields)


SCHEMES = {"x16": schemes.x16(), "e0.1": schemes.e01(), "e0.01": schemes.e001(), "f2": schemes.f2(),
           "fp32": schemes.fp32(3), "se2": schemes.se2(),
           "e0.01_nostraddle": schemes.with_layout(schemes.e001(), "nostraddle"),
           "se2_nostraddle": schemes.with_layout(schemes.se2(), "nostraddle")}


@pytest.mark.parametrize("name", list(SCHEMES) + ["mixed0", "mixed1", "mixed2", "mixed_se0", "mixed_se1", "mixed_se2"])
@pytest.mark.parametrize("dithered", [False, True])
def test_encode_decode_bit_exact(name, dithered):
    rng = np.random.default_rng(sum(map(ord, name)) + dithered)
    if name in SCHEMES:
        sch = SCHEMES[name]
    elif name.startswith("mixed_se"):
        sch = mixed_shared_scheme(rng)
    else:
        sch = mixed_scheme(rng)
    n = 100_003  # ragged tail
    vals = random_vals(sch, n, rng)
    vals[rng.integers(0, n, 20), rng.integers(0, vals.shape[1], 20)] = np.nan
    keys = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32) if dithered else None
    step = 12345
    w_ref, c_ref = oracle.encode(sch, vals, keys=keys, step=step)
    _, W, _ = qmpm.layout(sch)
    words = torch.zeros((n, W), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(3 * 64, dtype=torch.int64, device="cuda")
    qmpm.encode(sch, dev(vals), words, keys=None if keys is None else dev(keys), step=step, counters=cnt)
    torch.cuda.synchronize()
    w_gpu = words.cpu().numpy().view(np.uint32)
    assert np.array_equal(w_gpu, w_ref)
    c = cnt.cpu().numpy().astype(np.uint64)
    nf = len(sch["fields"])
    assert np.array_equal(c[:nf], c_ref[:nf])              # saturations
    assert np.array_equal(c[64:64 + nf], c_ref[64:64 + nf])    # round-ups
    assert np.array_equal(c[128:128 + nf], c_ref[128:128 + nf])  # round-downs
    out = torch.zeros((n, nf), dtype=torch.float32, device="cuda")
    qmpm.decode(sch, words, out)
    torch.cuda.synchronize()
    d_ref = oracle.decode(sch, w_ref)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), d_ref.view(np.uint32))


@pytest.mark.parametrize("b", [0, 3, 11, 15])
def test_exhaustive_codes(b):
    sch = dict(dim=3, material="elastic", rounding="dither", seed=5,
               fields=[dict(kind="fixed", frac_bits=b, range=4.0), dict(kind="fixed", frac_bits=b, range=0.5,
                                                                      offset=1.0)])
    codes = np.arange(-(2 ** b), 2 ** b, dtype=np.int64)
    m = (1 << (b + 1)) - 1
    w = ((codes & m) | ((codes[::-1] & m) << (b + 1))).astype(np.uint64)
    W = (2 * (b + 1) + 31) // 32
    words = np.zeros((codes.size, W), np.uint32)
    words[:, 0] = (w & 0xFFFFFFFF).astype(np.uint32)
    if W > 1:
        words[:, 1] = (w >> 32).astype(np.uint32)
    ref = oracle.decode(sch, words)
    out = torch.zeros((codes.size, 2), dtype=torch.float32, device="cuda")
    qmpm.decode(sch, dev(words), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    # re-encode (dithered) of on-grid values is the identity
    w2 = torch.zeros((codes.size, W), dtype=torch.int32, device="cuda")
    qmpm.encode(sch, out, w2, keys=dev(np.arange(codes.size, dtype=np.uint32)), step=3)
    torch.cuda.synchronize()
    assert np.array_equal(w2.cpu().numpy().view(np.uint32), words)


@pytest.mark.parametrize("name", ["x16", "e0.1", "f2", "se2"])
def test_set_state_read_state_bit_exact(name):
    """qmpm_set_state encodes with RNE at step 0 (reading Q20), bit-exact to the oracle;
    qmpm_read_state returns the oracle's decode."""
    sch = SCHEMES[name]
    sc = scenes.c1() if sch["dim"] == 2 else (scenes.small_fluid_3d() if sch["material"] == "fluid"
                                              else scenes.small_elastic_3d())
    st = sc.state()
    w_ref, _ = oracle.encode_state(sch, st)
    sim = qmpm.Sim(sc.sim, sch, st.shape[0] + 17, flags=qmpm.TRACK_IDS)
    sim.set_state(dev(st))
    words = np.zeros_like(w_ref)
    vals = np.zeros(st.shape, np.float32)
    ids = np.zeros(st.shape[0], np.uint32)
    n = sim.read_state(vals=vals, words=words, ids=ids)
    assert n == st.shape[0]
    assert np.array_equal(ids, np.arange(n))
    assert np.array_equal(words, w_ref)
    assert np.array_equal(vals, oracle.decode_state(sch, w_ref))
    # host-pointer input gives the same words
    sim.set_state(st)
    words2 = np.zeros_like(w_ref)
    sim.read_state(words=words2)
    assert np.array_equal(words2, w_ref)
    sim.close()


def _matmul3_oracle(sch, words, a, keys, step):
    """Oracle of qmpm_codec_matmul3 (P:797 MatMul task): oracle decode -> fp32 product
    summed left to right without FMA (numpy float32 elementwise ops) -> oracle encode."""
    m = oracle.decode(sch, words).astype(np.float32).reshape(-1, 3, 3)
    A = np.asarray(a, np.float32).reshape(3, 3)
    out = np.zeros_like(m)
    for r in range(3):
        for c in range(3):
            out[:, r, c] = (m[:, r, 0] * A[0, c] + m[:, r, 1] * A[1, c]) + m[:, r, 2] * A[2, c]
    return oracle.encode(sch, out.reshape(-1, 9), keys=keys, step=step)[0]


@pytest.mark.parametrize("dithered", [False, True])
@pytest.mark.parametrize("bits", [15, 11])
def test_codec_matmul3_bit_exact(dithered, bits):
    rng = np.random.default_rng(bits)
    sch = dict(dim=3, material="elastic", rounding="dither" if dithered else "rne", seed=99,
               fields=[dict(kind="fixed", frac_bits=bits, range=2.0, offset=0.0) for _ in range(9)])
    n = 5000
    v = rng.uniform(-0.9, 0.9, (n, 9)).astype(np.float32)
    w_in, _ = oracle.encode(sch, v)
    a = rng.uniform(-1.2, 1.2, 9).astype(np.float32)
    keys = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32) if dithered else None
    out = torch.zeros((n, w_in.shape[1]), dtype=torch.int32, device="cuda")
    qmpm.codec_matmul3(sch, dev(w_in), a, out, keys=None if keys is None else dev(keys), step=7)
    torch.cuda.synchronize()
    ref = _matmul3_oracle(sch, w_in, a, keys, 7)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)


def test_codec_vector_paths_and_unaligned_pointers():
    """The specialised codec picks 16/8/4-byte vector accesses from the row sizes and the
    pointers' alignment: an offset (unaligned) view must give the same bits."""
    rng = np.random.default_rng(5)
    sch = dict(dim=3, material="elastic", rounding="dither", seed=3,
               fields=[dict(kind="fixed", frac_bits=15, range=1.0, offset=0.0) for _ in range(8)])
    n = 1000
    v = rng.uniform(-0.99, 0.99, (n + 1, 8)).astype(np.float32)
    keys = rng.integers(0, 2 ** 32, n + 1, dtype=np.uint64).astype(np.uint32)
    ref, _ = oracle.encode(sch, v[1:], keys=keys[1:], step=2)
    vt, kt = dev(v), dev(keys)
    out = torch.zeros((n + 1) * 4 + 1, dtype=torch.int32, device="cuda")  # W = 4
    qmpm.encode(sch, vt[1:], out[1:1 + n * 4].view(n, 4), keys=kt[1:], step=2)  # unaligned vals and words
    torch.cuda.synchronize()
    assert np.array_equal(out[1:1 + n * 4].cpu().numpy().view(np.uint32).reshape(n, 4), ref)
    back = torch.zeros((n, 8), dtype=torch.float32, device="cuda")
    qmpm.decode(sch, out[1:1 + n * 4].view(n, 4), back)
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), oracle.decode(sch, ref))
