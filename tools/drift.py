"""NVE energy drift on C2 with the continuous (shifted) potential, V(rc) = 0: the paper's fixed
Ns = 20 against the displacement-checked policy, 1000 MD steps, PE/KE sampled every 10 steps.
Prints the relative drift of E = PE + KE and its RMS fluctuation per policy.
usage: python tools/drift.py [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import ljinputs as li
from paper_1704_03329_b200 import LJMD

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
pos, vel, box = li.CONFIGS["C2"].build()
shift = (1.0 / li.RC) ** 6 - (1.0 / li.RC) ** 12   # V(rc) = 0
for check in (0, 1):
    with LJMD(pos, vel, box, rebuild_check=check, energy_shift=shift) as md:
        md.step(steps)
        pe, ke = md.energy_history()
        st = md.stats()
    e = pe + ke
    rel = (e - e[0]) / abs(e[0])
    t = np.arange(len(e)) * 10
    slope = np.polyfit(t, rel, 1)[0]
    print(f"policy={'safe' if check else 'fixed-20'} steps={steps} rebuilds={st['n_rebuilds']} "
          f"dangerous={st['dangerous_builds']} E0={e[0]:.6f} final_rel_drift={rel[-1]:.3e} "
          f"max_abs_rel={np.abs(rel).max():.3e} slope_per_step={slope:.3e}")
