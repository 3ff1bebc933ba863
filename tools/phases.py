"""Force-kernel phase timers (measurement build): LJMD_LIB=.../libljmd_phases.so python tools/phases.py [config]
Per CTA of the last force launch of a ljmd_step(19) call (a kKKD launch, no energy): time from
entry to the end of the halo staging, staging to the first / last warp's loop end, the
epilogue, the CTA lifetime; and per SM the idle time between consecutive CTAs."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import ljinputs as li
from paper_1704_03329_b200 import LJMD, ljmd

cfg = li.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
pos, vel, box = cfg.build()
with LJMD(pos, vel, box, graphs=0) as ctx:
    ctx.step(20)
    ctx.step(19)   # the last launch of this call is kKick: use step(19)'s ... all launches alike
    lib = ljmd.load()
    n = 16384
    buf = np.zeros(10 * n, dtype=np.uint64)
    assert lib.ljmd_debug_phases(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), n) == 0
b = buf.reshape(n, 10).astype(np.int64)
b = b[b[:, 0] > 0]
t0 = b[:, 0].min()
ent, stg, l1, l2, epi, end, sm, m, trow, twait = (b[:, k] for k in range(10))
total = sm >> 32
sm = sm & 0xffffffff
issue = m >> 32
m = m & 0xffffffff
life = end - ent
print(f"{len(b)} CTAs, launch span {(end.max() - t0) / 1e3:.1f} us")
print(f"  staged bytes per CTA mean {24 * total.mean() / 1e3:.1f} KB, particles per CTA {m.mean():.0f}")
for name, v in (("entry -> row tables loaded", trow), ("entry -> PDL wait done", twait),
                 ("entry -> copies issued", issue), ("copies issued -> staged", stg - ent - issue),
                ("entry -> staged", stg - ent), ("staged -> first warp loop end", l1 - stg),
                ("staged -> last warp loop end", l2 - stg), ("last loop end -> epilogue end", epi - l2),
                ("epilogue end -> CTA end", end - epi), ("CTA lifetime", life)):
    print(f"  {name:32s} mean {v.mean() / 1e3:6.2f} us  p10 {np.percentile(v, 10) / 1e3:6.2f}  p90 {np.percentile(v, 90) / 1e3:6.2f}")
# per SM: busy CTA-time vs 2 x span (2 CTA slots per SM)
busy = 0.0
for s in np.unique(sm):
    busy += life[sm == s].sum()
nsm = len(np.unique(sm))
span = end.max() - t0
print(f"  CTA slot occupancy {busy / (2 * nsm * span):.3f} (busy CTA-time / (2 slots x {nsm} SMs x span))")
frac_loop = ((l2 - stg).sum()) / busy
print(f"  share of CTA time: staging {(stg - ent).sum() / busy:.3f}, loop(to last warp) {frac_loop:.3f}, "
      f"epilogue+exit {((end - l2)).sum() / busy:.3f}")
print(f"  warp spread within a CTA (last - first loop end) mean {(l2 - l1).mean() / 1e3:.2f} us")
