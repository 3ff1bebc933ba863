"""Bitwise comparison of two library builds on C2 (init + 41 steps: two device rebuilds):
LJMD_LIB_A=... LJMD_LIB_B=... python tools/same_traj.py"""
import os, subprocess, sys, json
if len(sys.argv) > 1:   # worker: run one build, save positions and forces
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import ljinputs as li
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = li.CONFIGS["C2"].build()
    with LJMD(pos, vel, box) as md:
        md.step(41)
        np.savez(sys.argv[1], x=md.positions(), f=md.forces())
    sys.exit(0)
import numpy as np
outs = []
for k in ("A", "B"):
    fn = f"/tmp/same_{k}.npz"
    subprocess.run([sys.executable, __file__, fn], check=True, env=dict(os.environ, LJMD_LIB=os.environ[f"LJMD_LIB_{k}"]))
    outs.append(np.load(fn))
print("positions bitwise equal:", np.array_equal(outs[0]["x"], outs[1]["x"]),
      "forces bitwise equal:", np.array_equal(outs[0]["f"], outs[1]["f"]))
