"""Bitwise comparison of one build under two environment settings on a config:
python tools/same_env.py VAR a b [config] -- positions and forces after 41 steps (two rebuilds)."""
import os, subprocess, sys
if sys.argv[1] == "--worker":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import ljinputs as li
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = li.CONFIGS[sys.argv[3]].build()
    with LJMD(pos, vel, box) as md:
        md.step(41)
        np.savez(sys.argv[2], x=md.positions(), f=md.forces())
    sys.exit(0)
import numpy as np
var, va, vb = sys.argv[1:4]
cfg = sys.argv[4] if len(sys.argv) > 4 else "C1"
outs = []
for v in (va, vb):
    fn = f"/tmp/same_env_{v}.npz"
    subprocess.run([sys.executable, __file__, "--worker", fn, cfg], check=True, env=dict(os.environ, **{var: v}))
    outs.append(np.load(fn))
print(cfg, var, va, "vs", vb, "positions bitwise equal:", np.array_equal(outs[0]["x"], outs[1]["x"]),
      "forces bitwise equal:", np.array_equal(outs[0]["f"], outs[1]["f"]))
