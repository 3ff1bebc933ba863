"""Timeline of bench.py's end-to-end loop (one rank, overlapped copies) under CUPTI: per
cycle set_staged_state (init sequence), step(20), positions_async, energy.  Prints the
kernel / copy time per cycle and the idle gaps on the compute stream.
usage: python tools/e2e_prof.py [cycles]"""
import os, sys, time, json, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ljinputs as li
from paper_1704_03329_b200 import LJMD, ljmd

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pos, vel, box = li.CONFIGS["C2"].build()
n = len(pos)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = LJMD(pos, vel, box, options=ljmd.default_options(device=0, stream=s.cuda_stream))
hp = [torch.from_numpy(pos.copy()).pin_memory() for _ in range(2)]
hv = [torch.from_numpy(vel.copy()).pin_memory() for _ in range(2)]
ho = [torch.empty((n, 3), dtype=torch.float64).pin_memory() for _ in range(2)]


def cycle(kk, k0):
    ctx.set_staged_state()
    if kk + 1 < k0:
        ctx.stage_state_ptr(hp[(kk + 1) % 2].data_ptr(), hv[(kk + 1) % 2].data_ptr())
    ctx.step(20)
    ctx.positions_async_ptr(ho[kk % 2].data_ptr())
    ctx.energy()


ctx.stage_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
for kk in range(3):
    cycle(kk, 3 + 1)
ctx.wait_transfers()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ctx.stage_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
    for kk in range(k):
        cycle(kk, k)
    ctx.wait_transfers()
    torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"wall {wall / k * 1e3:.3f} ms per cycle -> {n * 20 * k / wall / 1e9:.3f} e9 PTS/s (under the profiler)")
fn = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(fn)
ev = [e for e in json.load(open(fn))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
from collections import defaultdict
tot = defaultdict(float)
for e in ev:
    tot[e["name"][:60]] += e["dur"]
for name, t in sorted(tot.items(), key=lambda x: -x[1])[:16]:
    print(f"  {t / k:9.1f} us/cycle  {name}")
comp = [e for e in ev if e.get("cat") == "kernel"]
gaps = []
for a, b in zip(comp, comp[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 5:
        gaps.append((g, a["name"][:35], b["name"][:35]))
span = comp[-1]["ts"] + comp[-1]["dur"] - comp[0]["ts"]
print(f"  kernel span {span / k:.1f} us/cycle; gaps > 5 us: {sum(g for g, _, _ in gaps) / k:.1f} us/cycle")
agg = defaultdict(lambda: [0.0, 0])
for g, a, b in gaps:
    agg[(a, b)][0] += g
    agg[(a, b)][1] += 1
for (a, b), (g, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:12]:
    print(f"  gap {g / k:8.1f} us/cycle (x{c}) {a} -> {b}")
ctx.close()
