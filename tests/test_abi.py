"""CPU checks of the C-ABI library: it loads, exports every symbol include/qmpm.h
declares, and its host-side layout function follows the bit-pack layout."""
import re
import sys
import subprocess
import os

import numpy as np
import pytest

from paper_2207_04658_b200 import qmpm, schemes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="qmpm.h", prefix="qmpm_"):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(" + prefix + r"[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    path = qmpm.LIB_PATH
    assert os.path.exists(path), "libqmpm.so not built"
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    decl = declared_symbols()
    assert len(decl) >= 15
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    L = qmpm.lib()
    for s in decl:
        assert hasattr(L, s)
    assert L.qmpm_abi_version() == 1


def test_binding_names_match_header():
    assert sorted(qmpm.EXPORTS) == declared_symbols()


def test_smoke_header_symbols_exported_and_bound():
    from paper_2207_04658_b200 import qsmoke
    decl = declared_symbols("qsmoke.h", "qsmoke_")
    assert len(decl) == 12
    out = subprocess.check_output(["nm", "-D", "--defined-only", qmpm.LIB_PATH], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    assert not [s for s in decl if s not in exported]
    assert sorted(qsmoke.EXPORTS) == decl
    L = qsmoke.lib()
    for s in decl:
        assert hasattr(L, s)


def test_smoke_create_rejects_bad_params_without_gpu():
    """Argument validation happens before any device work, so it runs here."""
    import ctypes
    from paper_2207_04658_b200 import qsmoke, scenes
    params, _, _, _ = scenes.smoke(res=(8, 8, 8))

    def create(p, su, sp):
        cu, cp, pp, ctx = qmpm.CScheme(su), qmpm.CScheme(sp), qsmoke.make_params(p), ctypes.c_void_p()
        return qsmoke.lib().qsmoke_create(ctypes.byref(pp), cu.ref, cp.ref, None, ctypes.byref(ctx))

    assert create(dict(params, res=(7, 8, 8)), schemes.smoke_u(), schemes.smoke_p()) == 1
    assert create(dict(params, jacobi_iters=99), schemes.smoke_u(), schemes.smoke_p()) == 1
    assert create(params, schemes.smoke_p(), schemes.smoke_p()) == 2
    assert create(params, schemes.smoke_u(), schemes.smoke_u()) == 2
    assert b"6 fields" in qmpm.lib().qmpm_last_error(None) or b"2 fields" in qmpm.lib().qmpm_last_error(None)


@pytest.mark.parametrize("name", ["x16", "e0.1", "e0.01", "f2"])
def test_layout_of_stand_in_schemes(name):
    sch = schemes.BY_NAME[name]()
    offs, W, bits = qmpm.layout(sch)
    widths = [32 if f["kind"] == "raw" else f["frac_bits"] + 1 for f in sch["fields"]]
    assert offs == list(np.cumsum([0] + widths[:-1]))
    assert bits == sum(widths) and W == (bits + 31) // 32
    assert {"x16": 10, "e0.1": 11, "e0.01": 11, "f2": 8}[name] == W


def test_layout_fig_bit_struct_and_errors():
    s = dict(dim=3, material="elastic", rounding="dither", seed=0,
             fields=[dict(kind="fixed", frac_bits=16, range=1.0) for _ in range(3)])
    offs, W, bits = qmpm.layout(s)
    assert offs == [0, 17, 34] and W == 2  # three 17-bit values in two words
    offs, W, bits = qmpm.layout(schemes.with_layout(s, "nostraddle"))
    assert offs == [0, 32, 64] and W == 3  # "the three 17-bit elements consume three bit structs"
    bad = dict(s, fields=[dict(kind="fixed", frac_bits=32, range=1.0)])
    with pytest.raises(qmpm.QmpmError) as e:
        qmpm.layout(bad)
    assert e.value.code == 2
    bad = dict(s, fields=[dict(kind="shared_exp", frac_bits=8, range=1.0)])
    with pytest.raises(qmpm.QmpmError):
        qmpm.layout(bad)


def test_create_without_gpu_fails_loudly_or_validates():
    """Argument validation happens before any device work."""
    from paper_2207_04658_b200 import scenes
    sc = scenes.c1()
    bad = dict(schemes.x16())
    bad["fields"] = bad["fields"][:-1]  # a state scalar missing
    cs = qmpm.CScheme(bad)
    p = qmpm.make_params(sc.sim, 100)
    import ctypes
    h = ctypes.c_void_p()
    rc = qmpm.lib().qmpm_create(ctypes.byref(p), cs.ref, None, ctypes.byref(h))
    assert rc == 2


def test_adjoint_header_symbols_exported_and_bound():
    from paper_2207_04658_b200 import qadjoint
    decl = declared_symbols("qadjoint.h", "qadj_")
    assert len(decl) == 6
    out = subprocess.check_output(["nm", "-D", "--defined-only", qmpm.LIB_PATH], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    assert not [s for s in decl if s not in exported]
    assert sorted(qadjoint.EXPORTS) == decl
    L = qadjoint.lib()
    for s in decl:
        assert hasattr(L, s)


def test_adjoint_create_rejects_bad_arguments_without_gpu():
    import ctypes
    from paper_2207_04658_b200 import qadjoint, scenes
    sim, s0 = scenes.adjoint_fluid(dim=2, side=4)
    p = qmpm.make_params(sim, s0.shape[0])
    ctx = ctypes.c_void_p()
    L = qadjoint.lib()
    assert L.qadj_create(ctypes.byref(p), 2, 7, s0.shape[0], None, ctypes.byref(ctx)) == 1  # material
    assert L.qadj_create(ctypes.byref(p), 4, 1, s0.shape[0], None, ctypes.byref(ctx)) == 1  # dim
    assert L.qadj_create(ctypes.byref(p), 2, 1, 0, None, ctypes.byref(ctx)) == 1            # n = 0


@pytest.mark.parametrize("seed", range(6))
def test_nostraddle_layout_matches_oracle_and_never_straddles(seed):
    """Layout policy 1 (the bit struct's rule): library == oracle offsets, no
    field crosses a word, bit pack never needs more words, fields keep their order."""
    import oracle
    from test_gpu_codec import mixed_scheme, mixed_shared_scheme
    rng = np.random.default_rng(seed)
    sch = (mixed_shared_scheme if seed % 2 else mixed_scheme)(rng)
    ns = schemes.with_layout(sch, "nostraddle")
    offs, W, bits = qmpm.layout(ns)
    o_offs, o_W, o_bits = oracle.layout(ns)
    assert offs == list(o_offs) and W == o_W and bits == o_bits
    _, W_pack, _ = qmpm.layout(sch)
    assert W >= W_pack
    widths = []
    for i, f in enumerate(ns["fields"]):
        w = 32 if f["kind"] == "raw" else f["frac_bits"] + 1
        lead = f["kind"] == "shared_exp" and (i == 0 or ns["fields"][i - 1]["kind"] != "shared_exp"
                                              or ns["fields"][i - 1].get("group", 0) != f.get("group", 0))
        widths.append(w + (f["exp_bits"] if lead else 0))
    for o, w in zip(offs, widths):
        assert o % 32 + w <= 32
    assert all(a < b for a, b in zip(offs, offs[1:]))


def test_create_dist_validates_cuts_without_gpu():
    import ctypes
    from paper_2207_04658_b200 import scenes
    sc = scenes.c4(n_target=1000, res=64)
    p = qmpm.make_params(sc.sim, 1000)
    cs = qmpm.CScheme(schemes.f2())
    ctx = ctypes.c_void_p()
    uid = (ctypes.c_uint8 * 128)()
    L = qmpm.lib()
    bad = (ctypes.c_int32 * 3)(0, 40, 32)      # not increasing
    assert L.qmpm_create_dist(ctypes.byref(p), cs.ref, None, 2, 0, uid, bad, ctypes.byref(ctx)) == 1
    short = (ctypes.c_int32 * 3)(0, 32, 60)    # does not reach grid_res[2] = 64
    assert L.qmpm_create_dist(ctypes.byref(p), cs.ref, None, 2, 0, uid, short, ctypes.byref(ctx)) == 1
    ok = (ctypes.c_int32 * 3)(0, 32, 64)
    assert L.qmpm_create_dist(ctypes.byref(p), cs.ref, None, 2, 2, uid, ok, ctypes.byref(ctx)) == 1  # rank


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with the library absent, every binding raises instead of
    computing (run in a subprocess with LIB_PATH pointed at a missing file)."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_2207_04658_b200 import qmpm, qsmoke, qadjoint\n"
        "qmpm.LIB_PATH = %r\n"
        "qmpm._lib = None\n"
        "for f in (qmpm.lib, qsmoke.lib, qadjoint.lib):\n"
        "    try:\n"
        "        f(); print('LOADED'); sys.exit(1)\n"
        "    except ImportError:\n"
        "        pass\n"
        "print('OK')\n" % (ROOT, str(tmp_path / "missing.so")))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr
