"""Dump the SASS of the NVRTC-specialised step kernels for a stand-in scheme, offline
(static instruction counts; build-time inspection only).

    python tools/step_sass.py [f2|e0.01|...] [qmpm_g2p|qmpm_p2g] [--hist] [--minb P2G,G2P]
"""
import collections
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_04658_b200 import build as B, schemes  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "f2"
kern = args[1] if len(args) > 1 else "qmpm_g2p"
sch = schemes.BY_NAME[name]()
mat_fluid = sch["material"] == "fluid"
minb = (5, 4) if mat_fluid else (6, 3)
for a in sys.argv[1:]:
    if a.startswith("--minb="):
        minb = tuple(int(x) for x in a[7:].split(","))
tmp = "/tmp/sass/_step.cu"
open(tmp, "w").write("#define QMPM_JIT 1\n" + B.sample_spec(sch, p2g_minb=minb[0], g2p_minb=minb[1]) +
                     '#include "step_kernels.cuh"\n')
cub = "/tmp/sass/_step.cubin"
res = subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin",
                      "-Xptxas", "-v", "-I", B.CSRC, tmp, "-o", cub], capture_output=True, text=True)
if res.returncode:
    print(res.stderr)
    sys.exit(1)
print("\n".join(l for l in res.stderr.splitlines() if kern in l or "registers" in l)[-2000:], file=sys.stderr)
out = subprocess.check_output(["cuobjdump", "-sass", "-fun", kern, cub], text=True)
if "--hist" in sys.argv:
    ops = collections.Counter()
    for line in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m:
            ops[m.group(2)] += 1
    tot = sum(ops.values())
    print(f"{kern} {name}: {tot} static instructions")
    for op, c in ops.most_common(40):
        print(f"  {op:10s} {c}")
else:
    print(out)
