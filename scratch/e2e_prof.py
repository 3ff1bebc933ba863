"""Timeline of the overlapped e2e loop of bench.py on C2 (CUPTI via torch.profiler)."""
import os, sys, json, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ljinputs as li
from paper_1704_03329_b200 import LJMD, ljmd
pos, box = li.fcc(64, 64, 64)
vel = li.velocities(len(pos), 1.44)
n = len(pos)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = LJMD(pos, vel, box, rc=li.RC, dt=li.DT, options=ljmd.default_options(device=0, stream=s.cuda_stream))
hp = [torch.from_numpy(pos.copy()).pin_memory() for _ in range(2)]
hv = [torch.from_numpy(vel.copy()).pin_memory() for _ in range(2)]
ho = [torch.empty((n, 3), dtype=torch.float64).pin_memory() for _ in range(2)]
K = 6
def loop():
    ctx.stage_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
    for k in range(K):
        t = time.perf_counter(); ctx.set_staged_state(); t1 = time.perf_counter()
        if k + 1 < K: ctx.stage_state_ptr(hp[(k + 1) % 2].data_ptr(), hv[(k + 1) % 2].data_ptr())
        ctx.step(20); t2 = time.perf_counter()
        ctx.positions_async_ptr(ho[k % 2].data_ptr())
        ctx.energy(); t3 = time.perf_counter()
        print(f"host: set_state {1e3*(t1-t):.2f} ms, step {1e3*(t2-t1):.2f}, out+energy {1e3*(t3-t2):.2f}")
    ctx.wait_transfers()
loop(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    loop(); torch.cuda.synchronize()
print("wall per state", 1e3 * (time.perf_counter() - t0) / K, "ms")
fn = tempfile.mktemp(suffix=".json"); prof.export_chrome_trace(fn)
ev = [e for e in json.load(open(fn))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t00 = ev[0]["ts"]
cs = [e for e in ev if e["args"].get("stream") != ev[-1]["args"].get("stream") or "Memcpy" in e["name"]]
for e in ev:
    if "Memcpy" in e["name"] and e["dur"] > 50 or "k_load_rows" in e["name"] or "k_kick_drift" in e["name"]:
        print(f"{(e['ts'] - t00) / 1e3:9.3f} ms  dur {e['dur'] / 1e3:7.3f}  stream {e['args'].get('stream')}  {e['name'][:50]}")
comp = [e for e in ev if e["args"].get("stream") == s.cuda_stream or True]
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
busy = {}
for e in ev:
    busy.setdefault(e["args"].get("stream"), 0.0)
    busy[e["args"].get("stream")] += e["dur"]
print("span per state", span / 1e3 / K, "busy per stream per state", {k: round(v / 1e3 / K, 3) for k, v in busy.items()})
ctx.close()
