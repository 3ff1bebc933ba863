#!/usr/bin/env python
"""bench.py -- LJ particle-timesteps/s of the B200-native PairLoop engine (arXiv 1704.03329).

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE JSON line on
rank 0.  One bench "step" = one rebuild cycle of the paper's benchmark: Ns = 20 MD steps of
velocity Verlet, i.e. one cell binning + neighbour-list build, 20 force
evaluations (2 of them with PE, energy_every = 10) and the Verlet updates --
every row of SURVEY.md §8(a).

N = 1 workload: BASELINE.json configs[1] (C2: FCC 64^3 cells, N = 1,048,576, rho = 0.8442,
rc = 2.5, rbar_c = 2.75, dt = 0.005, T0 = 1.44).  N > 1: weak scaling at 1,048,576 particles
per GPU (64 x 64 x 64N cells, z-slabs).

--impl reference: the CPU oracle (oracle/, the only other place this script executes it)
timed on the box's host cores on the same config; each of its steps is one MD step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ljinputs as li  # noqa: E402

MD_PER_STEP = li.NS           # one rebuild cycle
# Listing lst:LJ-kernel, a user kernel for the DSL timing below
LJ_LISTING = """
const double dr0 = r.i[0] - r.j[0];
const double dr1 = r.i[1] - r.j[1];
const double dr2 = r.i[2] - r.j[2];
double dr_sq = dr0*dr0+dr1*dr1+dr2*dr2;
const double r_m2 = sigma2/dr_sq;
const double r_m4 = r_m2*r_m2;
const double r_m6 = r_m4*r_m2;
const double r_m8 = r_m4*r_m4;
u[0]+= (dr_sq<rc_sq) ? CV*((r_m6-1.0)*r_m6+0.25) : 0.0;
const double f_tmp=CF*(r_m6-0.5)*r_m8;
F.i[0]+= (dr_sq<rc_sq)?f_tmp*dr0:0.0;
F.i[1]+= (dr_sq<rc_sq)?f_tmp*dr1:0.0;
F.i[2]+= (dr_sq<rc_sq)?f_tmp*dr2:0.0;
"""
METRIC = "LJ particle-timesteps/s"
UNIT = "particle-timesteps/s"
FLOPS_PER_CAND = 21.0         # Listing lst:LJ-kernel, force only
FLOPS_PER_CAND_E = 26.0       # + potential energy
# nominal FP64 FMA peak of one B200: 148 SMs x 64 FP64 lanes x 2 flops x 1.965 GHz
PEAK_FP64_NOMINAL = 148 * 64 * 2 * 1.965e9 / 1e12


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def workload(n_gpus: int, name: str | None):
    if name:
        cfg = li.CONFIGS[name]
    elif n_gpus == 1:
        cfg = li.CONFIGS["C2"]
    else:
        cfg = li.weak_config(n_gpus)
    return cfg


def clocks_start(path):
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        f = open(path, "w")
        p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "50"],
                             stdout=f, stderr=subprocess.DEVNULL)
        return p, f
    except Exception:
        return None, None


def clocks_stop(h, path, gpu_index):
    p, f = h
    if p is None:
        return None
    p.terminate()
    try:
        p.wait(timeout=5)
    except Exception:
        p.kill()
    f.close()
    sm, smax, reasons = [], 0.0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in open(path):
        parts = [x.strip() for x in line.split(",")]
        if len(parts) < 9:
            continue
        try:
            if int(parts[0]) != gpu_index:
                continue
            sm.append(float(parts[1]))
            smax = max(smax, float(parts[2]))
        except ValueError:
            continue
        for k, v in zip(names, parts[5:9]):
            if v.lower() == "active":
                reasons.add(k)
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
            "samples": len(sm)}


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


# ---------------------------------------------------------------------------------- oracle legs

def oracle_cycle_rate(pos, vel, box, n_steps=2, omp=False):
    """Bounded oracle sample: init (wrap + cell/neighbour list + F) and n_steps list-mode VV
    steps (plain build: one host core; OpenMP build: all cores, identical results);
    extrapolated to one rebuild cycle (1 build + 20 steps)."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    oracle.run(pos, vel, box, 0, mode="list", energy_every=0, omp=omp)
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.run(pos, vel, box, n_steps, mode="list", energy_every=10, omp=omp)
    t_run = time.perf_counter() - t0
    t_step = max(t_run - t_init, 1e-9) / n_steps
    cycle = t_init + MD_PER_STEP * t_step
    return len(pos) * MD_PER_STEP / cycle, t_init, t_step


def oracle_brute_rate(n_steps=40):
    """C1 (N = 4000) with the O(N^2) brute-force force (the physics truth, no list) on one
    host core: n_steps VV steps; particle-timesteps/s."""
    import oracle
    c1 = li.CONFIGS["C1"]
    pos, vel, box = c1.build()
    t0 = time.perf_counter()
    oracle.run(pos, vel, box, n_steps, mode="brute", energy_every=10)
    t = time.perf_counter() - t0
    return len(pos) * n_steps / t, t


def run_reference(args, cfg):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    full = cfg
    if args.gpus > 1 and args.config is None:
        # bounded sample: the oracle's cost per particle-step does not depend on N, so the
        # weak-scaling workload (1,048,576 x N particles) is timed on one GPU's share (C2)
        cfg = workload(1, None)
    pos, vel, box = cfg.build()
    n = len(pos)
    cores, model = cpu_info()
    threads = oracle.threads()   # the OpenMP build of the oracle on every host core
    # warm-up: W MD steps (includes one init build)
    oracle.run(pos, vel, box, max(args.warmup, 0), mode="list", energy_every=10, omp=True)
    t0 = time.perf_counter()
    r = oracle.run(pos, vel, box, args.steps, mode="list", energy_every=10, omp=True)
    t = time.perf_counter() - t0
    value = n * args.steps / t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "md_steps_per_step": 1, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic FCC (ljinputs, seeded)",
        "config": {"workload": full.name, "n_particles": full.n, "rho": li.RHO,
                   "rc": li.RC, "rbar_c": li.RC + li.DELTA, "rebuild_every": li.NS, "dt": li.DT, "t0": cfg.t0},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{cfg.name} (N={n}"
                                   + (f", one GPU's share of {full.name}" if full is not cfg else "")
                                   + f"): oracle list-mode VV (OpenMP build, {threads} threads), "
                                   f"{args.steps} MD steps in one call (init build + rebuilds every {li.NS}), "
                                   f"{model}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "rebuilds": int(len(r.rebuild_steps)),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------- our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="C1..C5 (default: C2 at N=1, weak C2 per GPU at N>1)")
    ap.add_argument("--check", type=int, default=0, help="1: displacement-checked rebuild (safe policy)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-boa", action="store_true")
    ap.add_argument("--no-dsl", action="store_true")
    ap.add_argument("--no-policy", action="store_true", help="skip the other rebuild policy's timing")
    ap.add_argument("--no-validation", action="store_true", help="skip the missed-pair validation leg")
    ap.add_argument("--split-self", action="store_true",
                    help="one GPU through the full z-slab exchange path (halo planes sent to itself over NCCL)")
    ap.add_argument("--newton3", action="store_true",
                    help="NEXT-1 half-list force with reaction reductions (single GPU; slower)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    cfg = workload(args.gpus, args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if os.environ.get("LJMD_BENCH_DEVICE") is not None:   # debugging: all ranks on one GPU
        local = env_int("LJMD_BENCH_DEVICE", 0)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    from paper_1704_03329_b200 import LJMD, ljmd

    dist = None
    id_buf = None
    one_device = os.environ.get("LJMD_BENCH_DEVICE") is not None
    if world > 1 and one_device:
        # every rank on ONE GPU (NCCL refuses two ranks per device): gloo for the host-side
        # plumbing and the engine's host-staged multi-process transport (LJMDSHM); the same
        # rank logic, barriers and max-over-ranks timing as the NCCL run, for testing it
        import ctypes
        import uuid
        import torch.distributed as dist
        dist.init_process_group("gloo")
        key = [uuid.uuid4().hex if rank == 0 else None]
        dist.broadcast_object_list(key, 0)
        id_buf = ctypes.create_string_buffer(ljmd.shm_group_id(key[0]), 128)
    elif world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # the engine's own NCCL communicator: rank 0 creates the id, torch broadcasts it
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(ljmd.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        import ctypes
        id_buf = ctypes.create_string_buffer(bytes(idt.cpu().numpy().tobytes()), 128)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if one_device else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    pos, vel, box = cfg.build()
    n = len(pos)
    # a dedicated (non-default) stream: the engine launches on it and every CUDA event below is
    # recorded on it (torch's default stream has handle 0, which the ABI reads as "create one")
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    check = 1 if (args.check or cfg.rebuild_check) else 0
    opts = ljmd.default_options(device=local, stream=stream.cuda_stream, profile=0,
                                rebuild_check=check, rank=rank, nranks=world,
                                newton3=1 if args.newton3 else 0, split_self=1 if args.split_self else 0)
    if id_buf is None and args.split_self and world == 1:
        import ctypes
        id_buf = ctypes.create_string_buffer(bytes(ljmd.nccl_unique_id()), 128)
    if id_buf is not None:
        import ctypes
        opts.nccl_id = ctypes.cast(id_buf, ctypes.c_void_p)
    ctx = LJMD(pos, vel, box, rc=li.RC, dt=li.DT, options=opts)
    for _ in range(args.warmup):
        ctx.step(MD_PER_STEP)
    barrier()
    st0 = ctx.stats()
    clk_path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else f"/tmp/ljmd_clocks_{os.getpid()}.csv"
    clk = (None, None) if args.no_clocks else clocks_start(clk_path)
    time.sleep(0.3 if clk[0] is not None else 0.0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # also the spread over 5 equal parts of the timed region (events between
    # ljmd_step calls, which end with a host synchronisation anyway)
    n_rep = 5 if args.steps >= 5 else 1
    cuts = sorted({round(i * args.steps / n_rep) for i in range(1, n_rep)})
    evs = {k: torch.cuda.Event(enable_timing=True) for k in cuts}
    barrier()
    ev0.record(stream)
    for k in range(args.steps):
        if k in evs:
            evs[k].record(stream)
        ctx.step(MD_PER_STEP)
    ev1.record(stream)
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    marks = [(0, ev0)] + [(k, evs[k]) for k in cuts] + [(args.steps, ev1)]
    part_rates = [n * MD_PER_STEP * (k1 - k0) / (a.elapsed_time(b) * 1e-3)
                  for (k0, a), (k1, b) in zip(marks, marks[1:]) if k1 > k0]
    clocks = clocks_stop(clk, clk_path, local) if clk[0] is not None else None
    st1 = ctx.stats()
    md_steps = args.steps * MD_PER_STEP
    value = n * md_steps / (ms * 1e-3)

    # dominant kernel: the force kernel, timed in a second region of the same workload with
    # CUDA events around every force launch on the engine's stream (the events add a few us
    # per step, so the headline region above runs without them)
    k_prof = max(3, min(args.steps, 10))
    ctx.set_profile(True)
    barrier()
    sp0 = ctx.stats()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(k_prof):
        ctx.step(MD_PER_STEP)
    p1.record(stream)
    barrier()
    ms_prof = p0.elapsed_time(p1)
    sp1 = ctx.stats()
    ctx.set_profile(False)
    launches = sp1["force_launches"] - sp0["force_launches"]
    # per-rank force figures (rank 0's slab; the slabs are equal by construction)
    f_ms = (sp1["force_ms"] - sp0["force_ms"]) / max(launches, 1)
    cand = st1["total_neighbours"]
    e_frac = 1.0 / 10.0
    # the half list holds each pair once: half the candidates per launch
    flops = (cand / 2 if args.newton3 else cand) * (FLOPS_PER_CAND * (1 - e_frac) + FLOPS_PER_CAND_E * e_frac)
    achieved = flops / (f_ms * 1e-3) / 1e12
    # DRAM bytes per force launch from the committed ncu --set full capture of this config
    traffic, traffic_src = None, None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "force_traffic.json")))
        if tj.get("workload") == cfg.name and not args.newton3:
            traffic = tj["dram_bytes_per_launch"]
            traffic_src = tj["source"]
    except (OSError, ValueError, KeyError):
        pass
    # roofline denominator: MEASURED_PEAKS.json has no FP64 entry and the profiling guide no
    # FP64 fallback, so the peak is derived from the unit counts and clocks;
    # the achievable DFMA throughput measured by a probe kernel is reported beside it
    peak = PEAK_FP64_NOMINAL
    peak_src = "derived: 148 SMs x 64 FP64 FMA lanes x 2 flops x 1.965 GHz (sm max clock)"
    try:
        peak_probe = ljmd.measure_fp64_peak(local)
    except Exception:
        peak_probe = None

    # end to end through the public API with host buffers (pinned), per bench step: a new
    # state from the host (H2D pos+vel, the init sequence), step(20), positions (D2H) and
    # energy readback.  One rank: the copies run on the library's copy stream, overlapped
    # with the previous / next state's compute (ljmd_stage_state, ljmd_get_positions_async);
    # every copy is inside the timed region.  Several ranks: synchronous set_state.
    e2e = None
    if not args.no_e2e:
        hp = [torch.from_numpy(pos.copy()).pin_memory() for _ in range(2)]
        hv = [torch.from_numpy(vel.copy()).pin_memory() for _ in range(2)]
        ho = [torch.empty((n, 3), dtype=torch.float64).pin_memory() for _ in range(2)]
        k_e2e = max(2, min(args.steps, 10))
        overlapped = world == 1 and not args.split_self
        if overlapped:   # warm-up (allocates the copy stream and staging buffers)
            ctx.stage_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
            ctx.set_staged_state()
            ctx.step(MD_PER_STEP)
            ctx.positions_async_ptr(ho[0].data_ptr())
            ctx.wait_transfers()
        else:
            ctx.set_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
            ctx.step(MD_PER_STEP)
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if overlapped:
            ctx.stage_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
            for k in range(k_e2e):
                ctx.set_staged_state()
                if k + 1 < k_e2e:
                    ctx.stage_state_ptr(hp[(k + 1) % 2].data_ptr(), hv[(k + 1) % 2].data_ptr())
                ctx.step(MD_PER_STEP)
                ctx.positions_async_ptr(ho[k % 2].data_ptr())
                ctx.energy()
            ctx.wait_transfers()
        else:
            for _ in range(k_e2e):
                ctx.set_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
                ctx.step(MD_PER_STEP)
                ctx.positions_into_ptr(ho[0].data_ptr())
                ctx.energy()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms_e2e = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3))
        e2e = {"value": n * MD_PER_STEP * k_e2e / (ms_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(2 * 24 * n), "d2h_bytes_per_step": int(24 * n + 16),
               "steps": k_e2e, "transfers": "overlapped (copy stream)" if overlapped else "synchronous"}

    # the other rebuild policy on the same workload (reading R7) -- the
    # displacement-checked one when the headline ran the paper's fixed Ns = 20, and vice versa;
    # a fresh context, W warm-up cycles, 10 timed cycles (not the headline number)
    policy = None
    if not args.no_policy and world == 1:
        other = 0 if check else 1
        o2 = ljmd.default_options(device=local, stream=stream.cuda_stream, rebuild_check=other)
        with LJMD(pos, vel, box, rc=li.RC, dt=li.DT, options=o2) as c2:
            for _ in range(args.warmup):
                c2.step(MD_PER_STEP)
            r0 = c2.stats()["n_rebuilds"]
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            kq = 10
            q0.record(stream)
            for _ in range(kq):
                c2.step(MD_PER_STEP)
            q1.record(stream)
            torch.cuda.synchronize()
            ms_q = q0.elapsed_time(q1)
            sq = c2.stats()
            policy = {"rebuild_policy": "safe" if other else "paper-fixed-20",
                      "value": n * MD_PER_STEP * kq / (ms_q * 1e-3), "unit": UNIT,
                      "rebuilds_per_20_steps": (sq["n_rebuilds"] - r0) / kq, "cycles": kq,
                      "dangerous_builds": sq["dangerous_builds"]}

    # Validation leg (ljmd_options.validate, reading R7): the headline's rebuild policy on the
    # same workload with the missed-pair count on every step -- what the paper's fixed Ns = 20
    # costs in interactions it does not see (pairs inside rc that the list does not serve).
    # Fresh context from the same state, W + 2 cycles; not timed.
    validation = None
    if not args.no_validation and world == 1 and not args.split_self and not args.newton3:
        o3 = ljmd.default_options(device=local, stream=stream.cuda_stream, rebuild_check=check, validate=1)
        kv = args.warmup + 2
        with LJMD(pos, vel, box, rc=li.RC, dt=li.DT, options=o3) as c3:
            for _ in range(kv):
                c3.step(MD_PER_STEP)
            sv = c3.stats()
            vrows = c3.validation()
        last = vrows[-MD_PER_STEP:]
        validation = {"rebuild_policy": "safe" if check else "paper-fixed-20", "md_steps": int(len(vrows)),
                      "missed_pairs": int(sv["missed_pairs"]), "missed_particle_steps": int(sv["missed_particle_steps"]),
                      "max_missed_particles_per_step": int(sv["max_missed_particles"]),
                      "steps_with_missed_pairs": int((vrows[:, 1] > 0).sum()),
                      "last_cycle_missed_particle_steps": int(last[:, 1].sum()),
                      "dangerous_builds": int(sv["dangerous_builds"]), "rebuilds": int(sv["n_rebuilds"]),
                      "max_build_disp": sv["max_build_disp"], "delta": li.DELTA,
                      "note": "missed pair = r < rc at a step's positions but not in the list in use "
                              "(ljmd validate mode: fresh cell search minus in-range list entries)"}

    # what the rebuild policy costs in energy conservation: 1000 NVE steps of the same workload
    # with the continuous potential (V(rc) = 0, so that only a missed pair breaks conservation),
    # relative drift of PE + KE under each policy (fresh contexts, not timed)
    nve_drift = None
    if not args.no_validation and world == 1 and not args.split_self and not args.newton3:
        shift = (1.0 / li.RC) ** 6 - (1.0 / li.RC) ** 12
        nve_drift = {"md_steps": 1000, "potential": "LJ shifted to V(rc) = 0", "energy_every": 10}
        for name, chk in (("paper-fixed-20", 0), ("safe", 1)):
            od = ljmd.default_options(device=local, stream=stream.cuda_stream, rebuild_check=chk,
                                      energy_shift=shift)
            with LJMD(pos, vel, box, rc=li.RC, dt=li.DT, options=od) as cd:
                cd.step(1000)
                pe_h, ke_h = cd.energy_history()
                sd = cd.stats()
            e_h = pe_h + ke_h
            nve_drift[name] = {"rel_drift": float((e_h[-1] - e_h[0]) / abs(e_h[0])),
                               "rebuilds": int(sd["n_rebuilds"]), "dangerous_builds": int(sd["dangerous_builds"])}

    # §8(f) NEXT-2 bond-order analysis on the same state (not part of the headline metric):
    # Q_6 with the first-shell cutoff 1.5 sigma, CUDA events around the call (kernel +
    # D2H of Q and |N(i)| + host scatter into caller order)
    boa = None
    if not args.no_boa:
        ctx.boa(6, 1.5)
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        nb = 3
        for _ in range(nb):
            Qb, _nn = ctx.boa(6, 1.5)
        b1.record(stream)
        torch.cuda.synchronize()
        boa = {"ell": 6, "rcut": 1.5, "ms_per_call_incl_readback": b0.elapsed_time(b1) / nb,
               "mean_Q6": float(np.mean(Qb))}

    # §8(f) NEXT-3: the paper's LJ kernel (Listing lst:LJ-kernel) as a user PairLoop compiled
    # at run time (NVRTC), timed on the same state against the hand-written force kernel
    dsl_info = None
    if not args.no_dsl and world == 1:
        from paper_1704_03329_b200 import dsl
        consts = (dsl.Constant("sigma2", 1.0), dsl.Constant("rc_sq", li.RC * li.RC), dsl.Constant("CV", 4.0),
                  dsl.Constant("CF", 48.0))
        Fd, ud = dsl.ParticleDat(ctx, ncomp=3), dsl.ScalarArray(ctx)
        dsl_info = {"kernel": "Listing lst:LJ-kernel as a PairLoop (shell_cutoff = rc), NVRTC sm_100a",
                    "handwritten_force_ms": f_ms}
        for fmad in (False, True):
            loop = dsl.PairLoop(dsl.Kernel("lj", LJ_LISTING, consts),
                                {"r": dsl.PositionDat(ctx)(dsl.READ), "F": Fd(dsl.INC_ZERO), "u": ud(dsl.INC_ZERO)},
                                shell_cutoff=li.RC, fmad=fmad)
            loop.execute()
            torch.cuda.synchronize()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            for _ in range(5):
                loop.execute()
            d1.record(stream)
            torch.cuda.synchronize()
            dsl_info["ms_per_execute_fmad" if fmad else "ms_per_execute_exact"] = d0.elapsed_time(d1) / 5
            loop.free()

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        import oracle
        cores, model = cpu_info()
        threads = oracle.threads()
        rate, t_init, t_step = oracle_cycle_rate(pos, vel, box, n_steps=2, omp=True)
        rate1, t_init1, t_step1 = oracle_cycle_rate(pos, vel, box, n_steps=1, omp=False)
        rate_b, t_b = oracle_brute_rate(40)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{cfg.name} (N={n}): oracle (OpenMP build, {threads} threads of {cores}, {model}) "
                         f"init build ({t_init:.2f} s) + 2 list-mode VV steps ({t_step:.3f} s/step); "
                         f"rate = N*20/(build+20*step)",
               "one_core": {"value": rate1, "unit": UNIT, "cores": 1,
                            "sample": f"{cfg.name}: plain build, init {t_init1:.1f} s + 1 step {t_step1:.2f} s, "
                                      "extrapolated to one 20-step cycle"},
               "c1_brute_force_one_core": {"value": rate_b, "unit": UNIT, "cores": 1,
                                           "sample": f"C1 (N=4000): 40 VV steps with the O(N^2) brute-force "
                                                     f"force (no list) in {t_b:.1f} s"}}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "md_steps_per_step": MD_PER_STEP,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic FCC crystal (ljinputs: rho 0.8442, PCG64 seeds 87287/1704)",
        "config": {"workload": cfg.name, "n_particles": n, "rho": li.RHO, "rc": li.RC,
                   "rbar_c": li.RC + li.DELTA, "rebuild_every": li.NS, "energy_every": 10, "dt": li.DT,
                   "t0": cfg.t0, "rebuild_policy": "safe" if check else "paper-fixed-20",
                   "parallelism": f"z-slab x{world}" + (" (slab exchange through NCCL to itself)" if args.split_self else ""),
                   "force_path": "newton3 half list + reductions (NEXT-1)" if args.newton3 else
                   "full list, fused velocity Verlet",
                   "l2": "working set > L2 (16-bit list %.0f MB + positions %.0f MB + v, F %.0f MB)" % (
                       2 * cand / 1e6, 56 * (n + st1["n_ghost"]) / 1e6, 48 * n / 1e6)},
        "gpu_launches": int(st1["kernel_launches"] - st0["kernel_launches"]),
        "transport": ("shm (all ranks on one GPU)" if one_device and world > 1 else "nccl")
        if (world > 1 or args.split_self) else "none",
        "roofline": {"bound": "alu",
                     "kernel": "k_force_half (fp64 LJ pair loop)" if args.newton3 else "k_force (fp64 LJ pair loop)", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_probe": peak_probe, "frac_probe": achieved / peak_probe if peak_probe else None,
                     "traffic_source": traffic_src,
                     "flops_per_launch": flops, "avg_launch_ms": f_ms, "peak_source": peak_src,
                     "flop_count": "Listing 9: 21 flops per list candidate (+5 with PE every 10th step)"},
        "repeats": {"parts": len(part_rates), "median": statistics.median(part_rates), "min": min(part_rates),
                    "max": max(part_rates), "unit": UNIT, "note": "rank-0 rates of equal parts of the timed region"},
        "force_share": (sp1["force_ms"] - sp0["force_ms"]) / ms_prof,
        "force_timing": {"region_steps": k_prof, "ms_per_step_with_events": ms_prof / k_prof},
        "neighbours_per_particle": cand / n,
        "e2e": e2e,
        "other_rebuild_policy": policy,
        "validation": validation,
        "nve_drift": nve_drift,
        "dangerous_builds": int(st1["dangerous_builds"] - st0["dangerous_builds"]),
        "rebuilds": int(st1["n_rebuilds"] - st0["n_rebuilds"]),
        "cpu_baseline": cpu,
        "boa": boa,
        "dsl": dsl_info,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
