"""Debug helper: run a small scene step by step with CUDA_LAUNCH_BLOCKING=1 and report errors."""
import os, sys
os.environ["CUDA_LAUNCH_BLOCKING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2207_04658_b200 import qmpm, scenes, schemes
sc = scenes.small_fluid_3d() if "fluid" in sys.argv else scenes.c1()
sch = schemes.f2() if "fluid" in sys.argv else schemes.x16()
st = sc.state()
sim = qmpm.Sim(sc.sim, sch, st.shape[0])
sim.set_state(torch.from_numpy(st).cuda())
for t in range(3):
    try:
        sim.step(1)
        s = sim.stats()
        print("step", t, "ok", s.active_blocks, s.touched_blocks)
    except Exception as e:
        print("step", t, "failed:", e)
        break
