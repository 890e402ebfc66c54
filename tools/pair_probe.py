"""Probe: the packed-pair fast encode (senc_pair_fast) vs the scalar one (senc1_fast)
for every pair of a stand-in scheme, on random values -- run on the GPU box.
    python tools/pair_probe.py [f2|e0.01]"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_04658_b200 import build as B, schemes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "f2"
sch = schemes.BY_NAME[name]()
src = "#define QMPM_JIT 1\n" + B.sample_spec(sch) + r'''
#include "field_codec.cuh"
using namespace qmpm;
extern "C" __global__ void probe(const float* v, const unsigned* hs, int n, int* out_pair, int* out_one) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  constexpr int NS = Spec::NS, W = Spec::W;
  float o[NS];
  for (int i = 0; i < NS; ++i) o[i] = v[(size_t)t * NS + i];
  const unsigned h = hs[t];
  uint32_t w1[W + 1], w2[W + 1];
#pragma unroll
  for (int q = 0; q <= W; ++q) w1[q] = w2[q] = 0u;
  bool fl = false, z = false;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    int sb;
    if (fast_ok<Spec>(i)) sput_code<Spec>(w1, i, senc1_fast<Spec>(i, o[i], dither_s(h, Spec::idx(i)), sb, fl, z));
  }
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    if (pair_role<Spec>(i) == 0 && fast_ok<Spec>(i)) {
      int sb;
      sput_code<Spec>(w2, i, senc1_fast<Spec>(i, o[i], dither_s(h, Spec::idx(i)), sb, fl, z));
    }
    if (pair_role<Spec>(i) != 1) continue;
    int ui, uj, si, sj;
    senc_pair_fast<Spec>(i, i + 1, o[i], o[i + 1], dither_s(h, Spec::idx(i)), dither_s(h, Spec::idx(i + 1)), ui, uj, si, sj, fl, z);
    sput_code<Spec>(w2, i, ui);
    sput_code<Spec>(w2, i + 1, uj);
  }
#pragma unroll
  for (int q = 0; q < W; ++q) {
    out_one[(size_t)t * W + q] = w1[q];
    out_pair[(size_t)t * W + q] = w2[q];
  }
}
'''
os.makedirs("/tmp/probe", exist_ok=True)
open("/tmp/probe/p.cu", "w").write(src)
VAR = os.environ.get("VAR", "0")  # (historical: -DQMPM_SB_VARIANT, now unused)
subprocess.check_call([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin", "-I", B.CSRC,
                       f"-DQMPM_SB_VARIANT={VAR}", "/tmp/probe/p.cu", "-o", "/tmp/probe/p.cubin"])
if "--compile-only" in sys.argv:
    sys.exit(0)
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402

torch.cuda.init()
torch.zeros(1, device="cuda")
err, mod = cu.cuModuleLoad(b"/tmp/probe/p.cubin")
assert err == 0, err
err, fn = cu.cuModuleGetFunction(mod, b"probe")
ns = {"f2": 16}.get(name, 24)
n = 1 << 16
rng = np.random.default_rng(1)
v = torch.tensor(rng.uniform(-0.4, 0.4, (n, ns)).astype(np.float32), device="cuda")
v[:, 6] = torch.tensor(rng.uniform(0.9, 1.1, n).astype(np.float32), device="cuda") if name == "f2" else v[:, 6]
hs = torch.tensor(rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32).view(np.int32), device="cuda")
Wd = {"f2": 8}.get(name, 11)
op = torch.zeros((n, Wd), dtype=torch.int32, device="cuda")
o1 = torch.zeros((n, Wd), dtype=torch.int32, device="cuda")
import ctypes  # noqa: E402
args = [ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(hs.data_ptr()), ctypes.c_int(n),
        ctypes.c_void_p(op.data_ptr()), ctypes.c_void_p(o1.data_ptr())]
arr = (ctypes.c_void_p * len(args))(*[ctypes.cast(ctypes.pointer(a), ctypes.c_void_p) for a in args])
err, = cu.cuLaunchKernel(fn, (n + 127) // 128, 1, 1, 128, 1, 1, 0, 0, ctypes.addressof(arr), 0)
assert err == 0, err
torch.cuda.synchronize()
a, b = op.cpu().numpy(), o1.cpu().numpy()
bad = np.nonzero((a != b).any(axis=0))[0]
print("variant", VAR, "scheme", name, "mismatching words:", bad.tolist())
for i in bad[:6]:
    k = np.nonzero(a[:, i] != b[:, i])[0][:3]
    print(i, [(hex(int(a[j, i]) & 0xffffffff), hex(int(b[j, i]) & 0xffffffff)) for j in k])
