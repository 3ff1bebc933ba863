"""Per-kernel GPU time (CUPTI via torch.profiler) of ljmd_step on C2 for the library in LJMD_LIB.
usage: LJMD_LIB=... python tools/kprof.py [cycles]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ljinputs as li
from paper_1704_03329_b200 import LJMD, ljmd

cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = li.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C2"]
pos, vel, box = cfg.build()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
split = int(os.environ.get("LJMD_SPLIT_SELF", "0"))
opts = ljmd.default_options(device=0, stream=s.cuda_stream, rebuild_check=cfg.rebuild_check,
                            graphs=int(os.environ.get("LJMD_GRAPHS", "1")),
                            list_order=int(os.environ.get("LJMD_LIST_ORDER", "1")), split_self=split)
if split:
    import ctypes
    _idb = ctypes.create_string_buffer(bytes(ljmd.nccl_unique_id()), 128)
    opts.nccl_id = ctypes.cast(_idb, ctypes.c_void_p)
ctx = LJMD(pos, vel, box, rc=li.RC, dt=li.DT, options=opts)
for _ in range(3):
    ctx.step(20)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(cycles):
        ctx.step(20)
    torch.cuda.synchronize()
tot = 0.0
rows = []
for e in prof.key_averages():
    if e.device_type.name != "CUDA" and getattr(e, "self_device_time_total", 0) == 0:
        continue
    t = getattr(e, "self_device_time_total", None) or getattr(e, "self_cuda_time_total", 0)
    if t <= 0:
        continue
    rows.append((t, e.count, e.key))
    tot += t
tag = os.path.basename(os.environ.get("LJMD_LIB", "libljmd.so"))
print(f"== {tag} {cfg.name}: {tot / cycles:.1f} us per 20-step cycle, rebuilds {ctx.stats()['n_rebuilds']}")
for t, c, k in sorted(rows, reverse=True)[:14]:
    print(f"  {t / cycles:8.1f} us/cycle  {t / c:8.1f} us/launch  x{c // cycles:<3d} {k[:70]}")
ctx.close()

# gaps between consecutive device activities (kernels + memcpy/memset) on the engine's stream
import json, tempfile
fn = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(fn)
ev = [e for e in json.load(open(fn))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
gaps = []
for a, b in zip(ev, ev[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    gaps.append((g, a["name"][:40], b["name"][:40]))
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
busy = sum(e["dur"] for e in ev)
print(f"  span {span / cycles:.1f} us/cycle, busy {busy / cycles:.1f}, idle {(span - busy) / cycles:.1f}")
from collections import defaultdict
agg = defaultdict(lambda: [0.0, 0])
for g, a, b in gaps:
    if g > 3:
        agg[(a, b)][0] += g
        agg[(a, b)][1] += 1
for (a, b), (g, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:12]:
    print(f"  gap {g / cycles:7.1f} us/cycle (x{c}) after {a} -> {b}")
