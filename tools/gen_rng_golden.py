"""Write tests/golden/rng_rev3.json: the first outputs of the dither RNG (reading Q5,
revision 3) as the oracle computes them.  Calls only oracle/ (the RNG is self-defined:
the paper's generator, is in an unavailable supplement, so this golden vector is a
regression pin of the definition in DESIGN.md §2, not an external truth).

    python tools/gen_rng_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

SEED = 0x9E3779B97F4A7C15  # the bench's dither seed
cases = []
for step in (1, 2, 1000):
    for key in (0, 1, 0xDEADBEEF):
        cases.append({"seed": SEED, "step": step, "key": key,
                      "pair_hash": [oracle.lib().oracle_pair_hash(SEED, step, key, p) for p in range(4)],
                      "r16": [oracle.r16(SEED, step, key, f) for f in range(8)]})
# particle keys (content keys over the x words) of a few F2 records
import numpy as np  # noqa: E402
from paper_2207_04658_b200 import schemes  # noqa: E402
sch = schemes.f2()
recs = [[0] * 8, [1, 2, 3, 4, 5, 6, 7, 8], [0xFFFFFFFF] * 8, [0x12345678, 0x9ABCDEF0, 0, 0, 0, 0, 0, 0]]
keys = [{"record": r, "key": oracle.particle_key(sch, np.array(r, np.uint32))} for r in recs]
out = {"citation": "reading Q5 rev. 3 (DESIGN.md §2); P:421 (Eq. 11), P:811 (the paper's RNG, unavailable)",
       "generator": "tools/gen_rng_golden.py (oracle only)", "cases": cases,
       "particle_keys_f2": keys}
path = os.path.join(ROOT, "tests", "golden", "rng_rev3.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(path)
