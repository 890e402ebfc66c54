"""Dump the SASS of the smoke kernels for the sample layout (static instruction counts)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_04658_b200 import build as B  # noqa: E402

su = B.sample_codec_spec(nf=6, bits=15).replace("struct Spec {", "struct SpecU {")
sp = B.sample_codec_spec(nf=2, bits=15).replace("struct Spec {", "struct SpecP {")
tmp = "/tmp/_smoke_sass.cu"
open(tmp, "w").write("#define QMPM_JIT 1\n" + su + sp + '#include "smoke_kernels.cuh"\n')
cub = "/tmp/_smoke_sass.cubin"
subprocess.check_call([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin", "-I", B.CSRC,
                       tmp, "-o", cub])
kern = sys.argv[1] if len(sys.argv) > 1 else "qsmoke_jacobi"
out = subprocess.check_output(["cuobjdump", "-sass", "-fun", kern, cub], text=True)
print(out)
