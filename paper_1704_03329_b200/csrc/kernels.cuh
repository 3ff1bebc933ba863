// kernels.cuh -- sm_100a kernels of the LJ PairLoop hot path (arXiv 1704.03329).
//
// Data layout in HBM:
//   slot space  : every particle image a list can reference -- owned particles and ghosts
//                 (periodic images / halo copies) -- sorted by EXTENDED cell (x fastest
//                 over ncx+2, then y over ncy+2, then z over nzl+2), within a cell by
//                 (x, gid): a 3-cell x-row of the 27-cell stencil is one contiguous,
//                 x-sorted slot range.  Positions double4 {x,y,z,0} (x[2], double-buffered),
//                 a packed 24-byte copy xp[2] (the force kernel's bulk-copy source) and an
//                 fp32 float4 mirror for the list build.
//   owned space : owned particles t = 0..n_own-1, tile-major (one force CTA's particles
//                 are contiguous); v, F SoA fp64, gid, own_slot[t], e_i, ghost-image CSR.
//   tile halo   : per force tile the (ty+2)(tz+2) halo x-rows as slot ranges with padded
//                 offsets into the tile's shared-memory staging buffer (tr_begin/off/len).
//   list        : 16-bit local indices into that staging buffer, blocks of 8 entries,
//                 nbr8[b * n_pad + t] (one 16-byte load per 8 neighbours), ncount[t];
//                 a short last block is padded with the tile's sentinel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// 1: nranks > 1, the boundary force tiles wait in-kernel on a flag the halo stream releases
// (one launch over every tile); hangs with NCCL on one GPU, so off
#ifndef LJMD_HALO_GATE
#define LJMD_HALO_GATE 0
#endif

namespace ljmd {

struct DevFlags {
    int max_nbr;                 // longest list at the last build
    int slots_needed;            // slot count required by the last binning
    int nonfinite_gid;           // smallest gid with a non-finite coordinate (INT_MAX: none)
    int val_error;               // validation: a listed in-range pair the fresh search missed
    int rr_ovf;                  // list build: a bank-aware overflow run exceeded kRrRun
    int halo_timeout;            // a boundary force tile waited too long for the halo
    int pad2;
    int max_staged;              // largest tile staging count at the last build
    int migrate_gid;             // a particle that moved further than one cell plane (INT_MAX: none)
    int overflow;     // analysis capacity exceeded (ljmd_cna)
    int n_gflat;                 // ghost slots listed by the build-time refresh
    int n_grecv;                 // of those, images of received halo planes (nranks > 1)
    unsigned long long maxdisp2; // bits of max |x - x_build|^2 (non-negative double)
    unsigned long long total_nbr;
    unsigned long long overlap_pair;   // min over coincident pairs of (gid_i << 32 | gid_j),
                                       // gid_i < gid_j (~0: none) -- one atomic names both
};

// --------------------------------------------------------------------------- helpers
// Small device->host results (flags, counts, energies) are written by a kernel into mapped
// page-locked memory instead of a copy-engine transfer, so they never queue behind a bulk
// host transfer of the copy stream (ljmd_get_positions_async / ljmd_stage_state).
// device memory cleared by a kernel, not cudaMemsetAsync: a memset can queue behind bulk host
// transfers on the copy engine (measured: tens of microseconds of compute-stream idle while
// ljmd_stage_state / ljmd_get_positions_async copies run)
__global__ void k_zero_words(unsigned* __restrict__ p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0u;
}

__global__ void k_copy_words(const unsigned* __restrict__ src, unsigned* dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// keep_errors: the error fields (non-finite / migration gids, coincident pair, validation)
// survive, so a failure in one rebuild of a captured step sequence is still seen when the
// host reads the flags at the end of the call
__global__ void k_reset_flags(DevFlags* fl, int keep_errors) {
    DevFlags f;
    memset(&f, 0, sizeof f);
    f.migrate_gid = keep_errors ? fl->migrate_gid : INT_MAX;
    f.nonfinite_gid = keep_errors ? fl->nonfinite_gid : INT_MAX;
    f.overlap_pair = keep_errors ? fl->overlap_pair : ~0ull;
    f.val_error = keep_errors ? fl->val_error : 0;
    *fl = f;
}

// ------------------------------------------------------------------------ graph-mode control
// Step control of a captured step sequence (ljmd_step on one rank): the
// rebuild decision of reading R7 is taken on the device and gates the rebuild through a
// conditional graph node, so no step waits for the host.  Capacities are checked on the
// device as well; a shortfall aborts the rest of the sequence (every later kernel of it
// returns at once) and the host resumes at that step with regrown buffers.
struct DevCtl {
    int abort;        // 0 running; 1 slots short (nothing mutated); 2 staging / list width short
                      // (new layout in place, list incomplete)
    int abort_step;   // step of the call (1-based) whose rebuild aborted
    int nreb;         // rebuilds in this call (steps in rstep[])
    int nsamp;        // energy samples written in this call
    int step;         // step of the last decision
    int since;        // steps since the last rebuild (persists across calls; set by the host)
};

// One step's decision: since += 1; due = forced || since >= Ns || (check && 4 max|dx|^2 >
// delta^2), the last from the previous step's epilogue (non-negative doubles compare as
// their bit patterns); the maximum is cleared for this step's epilogue.
// step_now: the step of the call (1-based) this decision belongs to
// has_cond = 0 (a forced rebuild of the fixed schedule, captured without a conditional node:
// its kernels check the abort flag themselves): the decision is only recorded
__global__ void k_decide(DevCtl* ctl, DevFlags* fl, int ns, int check, int forced, double delta2, int* rstep,
                         int step_now, cudaGraphConditionalHandle h, int has_cond) {
    if (ctl->abort) {
        if (has_cond) cudaGraphSetConditional(h, 0u);
        return;
    }
    ctl->step = step_now;
    ctl->since += 1;
    bool due = forced || ctl->since >= ns;
    if (!due && check) due = 4.0 * __longlong_as_double((long long)fl->maxdisp2) > delta2;
    fl->maxdisp2 = 0ull;
    if (due) {
        ctl->since = 0;
        rstep[ctl->nreb++] = ctl->step;
    }
    if (has_cond) cudaGraphSetConditional(h, due ? 1u : 0u);
}

__global__ void k_set_since(DevCtl* ctl, int since) { ctl->since = since; }

// First node of a captured call: clears the per-call control -- unless an earlier call queued
// on the stream aborted (deferred settlement): then the abort record stays and
// every kernel of this call returns at once, so the host can resume the aborted call first.
__global__ void k_call_begin(DevCtl* ctl) {
    if (ctl->abort) return;
    ctl->abort_step = 0;
    ctl->nreb = 0;
    ctl->nsamp = 0;
    ctl->step = 0;
}

// Last node after a captured call: the call's control, flags, slot count, rebuild steps and
// energy samples into mapped page-locked memory (one of two buffers, alternating per call),
// so the host can read them after the NEXT call is queued.
struct CallOut {
    DevCtl ctl;
    int slots;
    int pad;
    DevFlags fl;
};

__global__ void k_call_out(const DevCtl* __restrict__ ctl, const DevFlags* __restrict__ fl,
                           const int* __restrict__ slots, const int* __restrict__ rstep,
                           const double* __restrict__ hist, CallOut* out, int* out_rstep, double* out_hist) {
    const DevCtl cc = *ctl;
    if (threadIdx.x == 0) {
        out->ctl = cc;
        out->slots = *slots;
        out->fl = *fl;
    }
    for (int i = threadIdx.x; i < cc.nreb; i += blockDim.x) out_rstep[i] = rstep[i];
    for (int i = threadIdx.x; i < 2 * cc.nsamp; i += blockDim.x) out_hist[i] = hist[i];
}

// capacity checks inside a captured rebuild: stage 1 (before anything is permuted) the slot
// count, stage 2 (after the tile tables) the staging size, stage 3 the list width
// (the kernels after a failed check return at entry: cctl() in the launches)
__global__ void k_check_caps(DevCtl* ctl, const DevFlags* fl, const int* need_slots, int slot_cap, int stage_cap,
                             int K, int stage) {
    bool ok = !ctl->abort;
    if (ok && stage == 1 && *need_slots > slot_cap) { ctl->abort = 1; ok = false; }
    if (ok && stage == 2 && fl->max_staged > stage_cap) { ctl->abort = 2; ok = false; }
    if (ok && stage == 3 && fl->max_nbr > K) { ctl->abort = 2; ok = false; }
    if (!ok && ctl->abort_step == 0) ctl->abort_step = ctl->step;
}

__device__ __forceinline__ double4 ld256(const double4* p) {
    double4 r;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void st256(double4* p, double4 v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}
// packed positions (24 B per slot): what the force kernel's bulk copies stage
__device__ __forceinline__ void st_packed(double* xp, int slot, double4 v) {
    double* q = xp + 3 * (size_t)slot;
    q[0] = v.x;
    q[1] = v.y;
    q[2] = v.z;
}

// Wrap into [0,L) -- reading R10; same operation sequence as the oracle's O1 (the
// two are written independently).  IEEE division / explicit roundings, no FMA.
__device__ __forceinline__ double wrap_coord(double x, double L) {
    double k = floor(__ddiv_rn(x, L));
    double t = __dsub_rn(x, __dmul_rn(L, k));
    if (t < 0.0) t = __dadd_rn(t, L);
    if (t >= L) t = __dsub_rn(t, L);
    return t;
}

// canonical r^2 = (dx*dx + dy*dy) + dz*dz with explicit roundings (reading R9): the
// cutoff decisions (r^2 < rbar_c^2 in the list, r^2 < rc^2 in the force) are taken on
// exactly the value the oracle computes.
__device__ __forceinline__ double r2_canon(double dx, double dy, double dz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// 1/a: MUFU.RCP64H seed (~2^-22) + one cubic Newton correction y(1 + e + e^2),
// e = 1 - a y  (3 DFMA, error ~2^-64 before rounding).  LJMD_RCP_QUAD: one quadratic
// correction y(1 + e) (2 DFMA, relative error ~2^-44: ~1e-13 in F_i, inside the 1e-10 bar).
#ifndef LJMD_RCP_QUAD
#define LJMD_RCP_QUAD 1
#endif
__device__ __forceinline__ double rcp64(double a) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
#if LJMD_RCP_QUAD
    return fma(y, e, y);
#else
    return fma(y, fma(e, e, e), y);
#endif
}

// max of a non-negative u64 over the block, one atomicMax per block (a per-warp atomic on
// one address serialises in L2: ~30 us for a million particles)
__device__ __forceinline__ void block_atomic_max(unsigned long long v, unsigned long long* out) {
    __shared__ unsigned long long sm[32];
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_down_sync(0xffffffffu, v, o);
        v = ob > v ? ob : v;
    }
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0ull;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_down_sync(0xffffffffu, v, o);
            v = ob > v ? ob : v;
        }
        if (threadIdx.x == 0 && v) atomicMax(out, v);
    }
}

// --------------------------------------------------------------------------- scan
// exclusive scan of int32 counts (3 phases).  Tile = 2048 elements per block.
constexpr int kScanThreads = 512;
constexpr int kScanTile = 2048;

__device__ __forceinline__ int block_excl_scan(int v, int* sh, int& total) {
    // sh has blockDim.x/32 + 1 ints
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        int s = lane < nw ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) sh[lane] = s;
    }
    __syncthreads();
    int pre = (w > 0 ? sh[w - 1] : 0) + x - v;
    total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return pre;
}

__global__ void k_scan_reduce(const int* __restrict__ in, int n, int* __restrict__ bsum) {
    __shared__ int sh[33];
    int base = blockIdx.x * kScanTile;
    int s = 0;
    for (int i = threadIdx.x; i < kScanTile; i += blockDim.x) {
        int g = base + i;
        if (g < n) s += in[g];
    }
    int tot;
    block_excl_scan(s, sh, tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void k_scan_top(int* __restrict__ bsum, int nb, int* __restrict__ total_out) {
    __shared__ int sh[33];
    int carry = 0;
    for (int base = 0; base < nb; base += blockDim.x) {
        int i = base + threadIdx.x;
        int v = i < nb ? bsum[i] : 0;
        int tot;
        int pre = block_excl_scan(v, sh, tot);
        if (i < nb) bsum[i] = carry + pre;
        carry += tot;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

// Small arrays (n <= kScanSingle): the whole exclusive scan and its total in one CTA -- one
// launch instead of three (the per-rebuild scans of small systems are launch-latency-bound).
constexpr int kScanSingle = 8192;
__device__ __forceinline__ void scan_single_block(const int* __restrict__ in, int n, int* __restrict__ out, int* sh) {
    const int per = (n + 1023) / 1024;
    const int b0 = min(n, (int)threadIdx.x * per), b1 = min(n, b0 + per);
    int s = 0;
    for (int i = b0; i < b1; ++i) s += in[i];
    int tot;
    int pre = block_excl_scan(s, sh, tot);
    for (int i = b0; i < b1; ++i) {
        const int v = in[i];
        out[i] = pre;
        pre += v;
    }
    if (threadIdx.x == 0) out[n] = tot;
}

// Small systems (both cell counts <= kScanSingle): the owned-cell offsets, the extended-cell
// counts (as k_ext_counts) and their offsets in one CTA -- one launch instead of three.
__global__ void __launch_bounds__(1024) k_bin_offsets_single(const int* __restrict__ ocount, int n_ocell,
                                                            int* __restrict__ obegin, int n_ecell,
                                                            const int* __restrict__ ecell_src,
                                                            const int* __restrict__ recv_cnt,
                                                            int* __restrict__ ecount, int* __restrict__ ebegin,
                                                            DevCtl* ctl, int slot_cap) {
    __shared__ int sh[33];
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    scan_single_block(ocount, n_ocell, obegin, sh);
    for (int ec = threadIdx.x; ec < n_ecell; ec += blockDim.x) {
        const int src = ecell_src[ec];
        ecount[ec] = src >= 0 ? ocount[src] : recv_cnt[-src - 1];
    }
    __syncthreads();   // the block's ecount writes are visible to the whole block
    scan_single_block(ecount, n_ecell, ebegin, sh);
    // device-checked rebuilds: k_check_caps' stage 1 (the slot count) folded in
    if (ctl && threadIdx.x == 0 && ebegin[n_ecell] > slot_cap) {
        ctl->abort = 1;
        if (ctl->abort_step == 0) ctl->abort_step = ctl->step;
    }
}

__global__ void __launch_bounds__(1024) k_scan_single(const int* __restrict__ in, int n, int* __restrict__ out) {
    __shared__ int sh[33];
    const int per = (n + 1023) / 1024;
    const int b0 = min(n, (int)threadIdx.x * per), b1 = min(n, b0 + per);
    int s = 0;
    for (int i = b0; i < b1; ++i) s += in[i];
    int tot;
    int pre = block_excl_scan(s, sh, tot);
    for (int i = b0; i < b1; ++i) {
        const int v = in[i];
        out[i] = pre;
        pre += v;
    }
    if (threadIdx.x == 0) out[n] = tot;
}

// out[i] = exclusive prefix of in[0..i) (the total is written by k_scan_top)
__global__ void k_scan_down(const int* __restrict__ in, int n, const int* __restrict__ bsum,
                            int* __restrict__ out, int /*unused*/) {
    __shared__ int sh[33];
    constexpr int kPer = kScanTile / kScanThreads;  // 4 consecutive per thread
    int base = blockIdx.x * kScanTile + threadIdx.x * kPer;
    int v[kPer];
    int s = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        v[q] = (base + q < n) ? in[base + q] : 0;
        s += v[q];
    }
    int tot;
    int pre = block_excl_scan(s, sh, tot) + bsum[blockIdx.x];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        if (base + q < n) out[base + q] = pre;
        pre += v[q];
    }
}

// --------------------------------------------------------------------------- init / binning
// Load caller rows [n][3] (pos, vel) into owned space with identity order (t = gid).
// gid_in: caller row of each loaded particle (nullptr: identity, single rank)
__global__ void k_load_rows(int n, const double* __restrict__ pos, const double* __restrict__ vel,
                            double4* __restrict__ x, double* __restrict__ vx, double* __restrict__ vy,
                            double* __restrict__ vz, int* __restrict__ gid, int* __restrict__ own_slot,
                            const int* __restrict__ gid_in, DevFlags* fl) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double a = pos[3 * t], b = pos[3 * t + 1], c = pos[3 * t + 2];
    double p = vel[3 * t], q = vel[3 * t + 1], r = vel[3 * t + 2];
    const int gi = gid_in ? gid_in[t] : t;
    if (!(isfinite(a) && isfinite(b) && isfinite(c) && isfinite(p) && isfinite(q) && isfinite(r)))
        atomicMin(&fl->nonfinite_gid, gi);
    x[t] = make_double4(a, b, c, 0.0);
    vx[t] = p;
    vy[t] = q;
    vz[t] = r;
    gid[t] = gi;
    own_slot[t] = t;
}

// Force tiles: blocks of kTX x kTY x kTZ owned cells.  Owned cells (and hence owned
// particles t) are numbered tile-major -- tile (z, y, x), then cell (z, y, x) inside the
// tile -- so one CTA's particles are contiguous; its stencil halo is (ty+2)(tz+2) x-rows.
// 4 x 3 x 2 cells (~444 particles at rho = 0.8442): the halo is 6 x 5 x 4 cells, 5x the
// owned ones (4 x 2 x 2: 6x); measured on C2 with 480-thread CTAs: force 159.3 -> 157.5 us
// per launch, list build 564 -> 528 us, 20-step cycle 4128 -> 4039 us
#ifndef LJMD_TX
#define LJMD_TX 4
#define LJMD_TY 3
#define LJMD_TZ 2
#endif
constexpr int kTX = LJMD_TX, kTY = LJMD_TY, kTZ = LJMD_TZ;
constexpr int kRowsMax = (kTY + 2) * (kTZ + 2);

struct Geo {
    double L[3];
    double w[3];        // cell widths
    double inv_w[3];
    int nc[3];          // global cell grid
    int z0, nzl;        // this rank's slab [z0, z0+nzl)
    int ex, ey, ez;     // extended grid dims = ncx+2, ncy+2, nzl+2
    int ntx, nty, ntz;  // tile grid over the owned cells
    const int* oc_of_lex;   // lexicographic owned cell (x fastest) -> tile-major index
    const int* lex_of_oc;   // inverse
};

__device__ __forceinline__ void lex_xyz(const Geo& g, int lex, int& cx, int& cy, int& cz) {
    cx = lex % g.nc[0];
    cy = (lex / g.nc[0]) % g.nc[1];
    cz = lex / (g.nc[0] * g.nc[1]);
}
__device__ __forceinline__ int tile_of_cell(const Geo& g, int cx, int cy, int cz) {
    return ((cz / kTZ) * g.nty + cy / kTY) * g.ntx + cx / kTX;
}
// tile extents and its halo-row geometry
struct TileGeo {
    int x0, y0, z0, tx, ty, tz, R;
};
__device__ __forceinline__ TileGeo tile_geo(const Geo& g, int tile) {
    TileGeo T;
    const int a = tile % g.ntx, b = (tile / g.ntx) % g.nty, c = tile / (g.ntx * g.nty);
    T.x0 = a * kTX; T.y0 = b * kTY; T.z0 = c * kTZ;
    T.tx = min(kTX, g.nc[0] - T.x0);
    T.ty = min(kTY, g.nc[1] - T.y0);
    T.tz = min(kTZ, g.nzl - T.z0);
    T.R = (T.ty + 2) * (T.tz + 2);
    return T;
}

// Wrap owned positions (R10) and bin them: cell_of[t] = owned-cell index, rank_in[t] = slot
// inside the cell from the atomic counter (order fixed later by the gid sort).
// vcopy / gcopy (single rank): the velocities and gids are copied aside here, so that the cell
// sort can permute them in place (v[0], gid[0] are the only live copies: the rebuild flips no
// buffer, and a captured step sequence keeps fixed pointers whether or not it rebuilds).
__global__ void k_wrap_bin(int n_own, const double4* __restrict__ x, const int* __restrict__ own_slot,
                           Geo g, double4* __restrict__ xw, int* __restrict__ ocount,
                           int* __restrict__ cell_of, int* __restrict__ rank_in,
                           const int* __restrict__ gid, DevFlags* fl, const double* __restrict__ v,
                           double* __restrict__ vcopy, int* __restrict__ gcopy, int cap, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    if (vcopy) {
        vcopy[t] = v[t];
        vcopy[t + cap] = v[t + cap];
        vcopy[t + 2 * (size_t)cap] = v[t + 2 * (size_t)cap];
        gcopy[t] = gid[t];
    }
    double4 p = x[own_slot[t]];
    if (!(isfinite(p.x) && isfinite(p.y) && isfinite(p.z))) {
        atomicMin(&fl->nonfinite_gid, gid[t]);
        p = make_double4(0.0, 0.0, 0.0, 0.0);
    }
    p.x = wrap_coord(p.x, g.L[0]);
    p.y = wrap_coord(p.y, g.L[1]);
    p.z = wrap_coord(p.z, g.L[2]);
    p.w = 0.0;
    int c[3];
    const double q[3] = {p.x, p.y, p.z};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        int k = (int)floor(__ddiv_rn(q[d], g.w[d]));
        k = k < 0 ? 0 : (k > g.nc[d] - 1 ? g.nc[d] - 1 : k);
        c[d] = k;
    }
    int cz = c[2] - g.z0;   // slab-local plane (0..nzl-1 for owned particles)
    if (cz < 0) cz = 0;
    if (cz > g.nzl - 1) cz = g.nzl - 1;
    int oc = g.oc_of_lex[(cz * g.nc[1] + c[1]) * g.nc[0] + c[0]];
    xw[t] = p;
    cell_of[t] = oc;
    rank_in[t] = atomicAdd(&ocount[oc], 1);
}

// Extended-cell counts: owned cells take their own count, ghost cells the count of
// their source cell (ghost table built on the host at init).
// ecell_src[ec] >= 0: owned cell whose particles (or periodic images) fill ec;
// ecell_src[ec] < 0: cell -(src+1) of the planes received from the z neighbours (nranks > 1).
__global__ void k_ext_counts(int n_ecell, const int* __restrict__ ocount, Geo g,
                             const int* __restrict__ ecell_src, const int* __restrict__ recv_cnt,
                             int* __restrict__ ecount) {
    int ec = blockIdx.x * blockDim.x + threadIdx.x;
    if (ec >= n_ecell) return;
    int src = ecell_src[ec];
    ecount[ec] = src >= 0 ? ocount[src] : recv_cnt[-src - 1];
}

__global__ void k_scatter(int n_own, const int* __restrict__ cell_of, const int* __restrict__ rank_in,
                          const int* __restrict__ obegin, int* __restrict__ perm, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    perm[obegin[cell_of[t]] + rank_in[t]] = t;
}

// One warp per owned cell: order members by (x, gid) -- deterministic (reading R15), and
// every 3-cell stencil row of the extended layout is then sorted by x, so the list build
// can binary-search each particle's x-window -- and write the new owned-space arrays and
// the owned slots of the new slot space.
__global__ void k_cell_sort(int n_ocell, Geo g, const int* __restrict__ obegin,
                            const int* __restrict__ ocount, const int* __restrict__ ebegin,
                            const int* __restrict__ perm, const int* __restrict__ gid_old,
                            const double4* __restrict__ xw, const double* __restrict__ vx_o,
                            const double* __restrict__ vy_o, const double* __restrict__ vz_o,
                            double4* __restrict__ x_new, float4* __restrict__ xf,
                            double* __restrict__ vx_n, double* __restrict__ vy_n,
                            double* __restrict__ vz_n, int* __restrict__ gid_new,
                            int* __restrict__ own_slot, int* __restrict__ ocell_of,
                            int* __restrict__ slot_gid, double4* __restrict__ xbuild,
                            double* __restrict__ xp_new, DevFlags* fl, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= n_ocell) return;
    int oc = warp;
    int m = ocount[oc];
    int b = obegin[oc];
    int cx, cy, cz;
    lex_xyz(g, g.lex_of_oc[oc], cx, cy, cz);
    int ec = ((cz + 1) * g.ey + (cy + 1)) * g.ex + (cx + 1);
    int sb = ebegin[ec];
    for (int k = lane; k < m + (m <= 32 ? 32 - m : 0); k += 32) {
        // rank of member k by (x, gid); cells of <= 32 particles (all of them at liquid
        // densities) exchange the keys by shuffles instead of re-reading them per member
        const bool mine = k < m;
        const int t_old = mine ? perm[b + k] : 0;
        const int gk = mine ? gid_old[t_old] : 0;
        const double xk = mine ? xw[t_old].x : 0.0;
        int r = 0;
        bool samex = false;   // another member with the same x: candidate for coincidence
        if (m <= 32) {
            for (int s = 0; s < m; ++s) {
                const double xs = __shfl_sync(0xffffffffu, xk, s);
                const int gs = __shfl_sync(0xffffffffu, gk, s);
                r += (xs < xk) || (xs == xk && gs < gk);
                samex |= xs == xk && gs != gk;
            }
        } else {
            for (int s = 0; s < m; ++s) {
                const int ts = perm[b + s];
                const double xs = xw[ts].x;
                const int gs = gid_old[ts];
                r += (xs < xk) || (xs == xk && gs < gk);
                samex |= xs == xk && gs != gk;
            }
        }
        if (mine && samex) {   // rare: coincident particles (r^2 == 0) are an error
            const double4 pk = xw[t_old];
            for (int s = 0; s < m; ++s) {
                const int ts = perm[b + s];
                const double4 ps = xw[ts];
                if (ts != t_old && ps.x == pk.x && ps.y == pk.y && ps.z == pk.z && gk < gid_old[ts])
                    atomicMin(&fl->overlap_pair,
                              ((unsigned long long)(unsigned)gk << 32) | (unsigned)gid_old[ts]);
            }
        }
        if (!mine) continue;
        int t = b + r;
        int slot = sb + r;
        double4 p = xw[t_old];
        x_new[slot] = p;
        st_packed(xp_new, slot, p);
        xf[slot] = make_float4((float)p.x, (float)p.y, (float)p.z, 0.f);
        if (xbuild) xbuild[t] = p;
        vx_n[t] = vx_o[t_old];
        vy_n[t] = vy_o[t_old];
        vz_n[t] = vz_o[t_old];
        gid_new[t] = gk;
        own_slot[t] = slot;
        ocell_of[t] = oc;
        slot_gid[slot] = gk;
    }
}

// Ghost refresh: one warp per ghost cell copies its source cell's slot range with the
// periodic shift s*L (one rounding: x_src + s*L, exactly the oracle's image position).
// at_build: also write the fp32 mirror and the slot -> gid map.
struct GhostCells {
    const int* dst;    // extended cell id
    const int* src;    // extended cell id of the (owned) source cell
    const int* shift;  // packed (sx+1) | (sy+1)<<2 | (sz+1)<<4
    int n;
};

// Sources: gc.src >= 0 -> extended cell (local owned slots); gc.src < 0 -> received plane
// cell -(src+1), stored after the slot range at n_slots + recv_off[cell] (nranks > 1).
// at_build also lists every ghost slot as {dst slot, src slot, shift code} (gflat, order
// immaterial) for the per-step refresh k_ghost_flat.
template <bool AT_BUILD>
__global__ void k_ghost_refresh(GhostCells gc, const int* __restrict__ ebegin,
                                const int* __restrict__ ecount, Geo g, double4* __restrict__ x,
                                float4* __restrict__ xf, int* __restrict__ slot_gid,
                                const int* __restrict__ recv_cnt, const int* __restrict__ recv_off,
                                int n_slots, int4* __restrict__ gflat, double* __restrict__ xp, DevFlags* fl,
                                const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= gc.n) return;
    int d = gc.dst[warp], s = gc.src[warp], code = gc.shift[warp];
    int db = ebegin[d];
    int sb, m;
    if (s >= 0) {
        sb = ebegin[s];
        m = ecount[s];
    } else {
        sb = n_slots + recv_off[-s - 1];
        m = recv_cnt[-s - 1];
    }
    double sx = (double)((code & 3) - 1), sy = (double)(((code >> 2) & 3) - 1),
           sz = (double)(((code >> 4) & 3) - 1);
    double Lx = sx * g.L[0], Ly = sy * g.L[1], Lz = sz * g.L[2];   // exact
    int base = 0;
    if (AT_BUILD) {
        if (lane == 0) base = atomicAdd(&fl->n_gflat, m);
        base = __shfl_sync(0xffffffffu, base, 0);
    }
    for (int k = lane; k < m; k += 32) {
        double4 p = ld256(x + sb + k);
        double4 q = make_double4(__dadd_rn(p.x, Lx), __dadd_rn(p.y, Ly), __dadd_rn(p.z, Lz), 0.0);
        st256(x + db + k, q);
        st_packed(xp, db + k, q);
        if (AT_BUILD) {
            xf[db + k] = make_float4((float)q.x, (float)q.y, (float)q.z, 0.f);
            slot_gid[db + k] = slot_gid[sb + k];
            gflat[base + k] = make_int4(db + k, sb + k, code, 0);
        }
    }
}

// Per-step ghost refresh: thread per ghost slot from the build-time list (one 16-byte
// descriptor, one 32-byte read, one 32-byte write; every lane busy).
__global__ void __launch_bounds__(256) k_ghost_flat(int n, const int4* __restrict__ gflat, Geo g,
                                                    double4* __restrict__ x, double* __restrict__ xp) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 e = gflat[i];
    const double sx = (double)((e.z & 3) - 1), sy = (double)(((e.z >> 2) & 3) - 1),
                 sz = (double)(((e.z >> 4) & 3) - 1);
    const double4 p = ld256(x + e.y);
    const double4 q = make_double4(__dadd_rn(p.x, sx * g.L[0]), __dadd_rn(p.y, sy * g.L[1]),
                                   __dadd_rn(p.z, sz * g.L[2]), 0.0);
    st256(x + e.x, q);
    st_packed(xp, e.x, q);
}

// Ghost images per owned particle (CSR, built at the rebuild from the ghost list): the
// kernels that move a particle -- the fused force epilogue and the opening kick-drift --
// also write its periodic images x + s L (one rounding, as k_ghost_refresh), so the ghost
// slots never need a separate per-step refresh.  Images of received halo planes
// (nranks > 1) are listed apart (grecv) and refreshed after each exchange.
struct Images {
    const int* off;    // [n_own + 1]; null: the kernel writes no images
    const int2* e;     // {dst slot, shift code}; code bit 7: a send-area entry (nranks > 1),
                       // written as double4 only
};

__device__ __forceinline__ void write_images(const Images& im, int t, const Geo& g, double4* __restrict__ x,
                                             double* __restrict__ xp, double4 p) {
    if (!im.off) return;
    const int b = im.off[t], e = im.off[t + 1];
    for (int i = b; i < e; ++i) {
        const int2 d = im.e[i];
        const double4 q = make_double4(__dadd_rn(p.x, (double)((d.y & 3) - 1) * g.L[0]),
                                       __dadd_rn(p.y, (double)(((d.y >> 2) & 3) - 1) * g.L[1]),
                                       __dadd_rn(p.z, (double)(((d.y >> 4) & 3) - 1) * g.L[2]), 0.0);
        st256(x + d.x, q);
        if (!(d.y & 0x80)) st_packed(xp, d.x, q);
    }
}

// release of a step's halo to the gated boundary tiles of the force launch
__global__ void k_set_flag(unsigned* flag, unsigned seq) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(flag), "r"(seq) : "memory");
}

// ghost planes arrive as double4 (32-byte records: every slot is aligned for the transfer);
// the force kernel stages packed positions, written here for the two planes
__global__ void k_xp_from_x(int b0, int n0, int b1, int n1, const double4* __restrict__ x, double* __restrict__ xp) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n0 + n1) return;
    const int sl = k < n0 ? b0 + k : b1 + (k - n0);
    st_packed(xp, sl, ld256(x + sl));
}

// also clears the image counts of k_img_build (one memset node fewer)
__global__ void k_slot2t(int n_own, const int* __restrict__ own_slot, int* __restrict__ slot2t, int* __restrict__ img_cnt,
                         const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_own) {
        slot2t[own_slot[t]] = t;
        img_cnt[t] = 0;
    }
}

// FILL = false: count the images of each owned source (and move received-plane images to
// grecv); FILL = true: place them (the counts return to zero)
// n_dev != null: the ghost count is read on the device (captured rebuilds: grid over a cap)
template <bool FILL>
__global__ void k_img_build(int n, const int4* __restrict__ gflat, int n_slots, const int* __restrict__ slot2t,
                            int* __restrict__ cnt, const int* __restrict__ off, int2* __restrict__ img,
                            int4* __restrict__ grecv, DevFlags* fl, const int* n_dev, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (n_dev) n = *n_dev;
    if (i >= n) return;
    const int4 e = gflat[i];
    if (e.y < n_slots) {
        const int t = slot2t[e.y];
        if (FILL) img[off[t] + atomicSub(&cnt[t], 1) - 1] = make_int2(e.x, e.z);
        else atomicAdd(&cnt[t], 1);
    } else if (!FILL) {
        grecv[atomicAdd(&fl->n_grecv, 1)] = e;
    }
}

// --------------------------------------------------------------------------- z-slab decomposition
// (spatial decomposition, halo cells, particle migration every n steps)
struct MigRec {           // one migrating particle: wrapped position, velocity, gid (64 B)
    double x, y, z, vx, vy, vz;
    long long gid;
    long long pad;
};

// Wrap every owned particle (R10), find its owner slab by global cell plane; stayers are
// copied to the compact arrays (atomic slot, order fixed later by the cell sort), leavers
// to the send buffer of the lower / upper neighbour.
__global__ void k_migrate_mark(int n_own, const double4* __restrict__ x, const int* __restrict__ own_slot,
                               const double* __restrict__ vx, const double* __restrict__ vy,
                               const double* __restrict__ vz, const int* __restrict__ gid, Geo g,
                               double4* __restrict__ xs, double* __restrict__ vxs, double* __restrict__ vys,
                               double* __restrict__ vzs, int* __restrict__ gids, MigRec* __restrict__ lo,
                               MigRec* __restrict__ hi, int cap_mig, int* __restrict__ counters,
                               DevFlags* fl, int* __restrict__ stay_t) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    double4 p = x[own_slot[t]];
    if (!(isfinite(p.x) && isfinite(p.y) && isfinite(p.z))) {
        atomicMin(&fl->nonfinite_gid, gid[t]);
        p = make_double4(0.0, 0.0, 0.0, 0.0);
    }
    p.x = wrap_coord(p.x, g.L[0]);
    p.y = wrap_coord(p.y, g.L[1]);
    p.z = wrap_coord(p.z, g.L[2]);
    p.w = 0.0;
    int cz = (int)floor(__ddiv_rn(p.z, g.w[2]));
    cz = cz < 0 ? 0 : (cz > g.nc[2] - 1 ? g.nc[2] - 1 : cz);
    int dir = 0;
    if (cz < g.z0 || cz >= g.z0 + g.nzl) {
        // only the adjacent planes are reachable between rebuilds (displacement < w)
        if (cz == (g.z0 - 1 + g.nc[2]) % g.nc[2]) dir = -1;
        else if (cz == (g.z0 + g.nzl) % g.nc[2]) dir = 1;
        else {
            atomicMin(&fl->migrate_gid, gid[t]);
            dir = -1;
        }
    }
    if (dir == 0) {
        const int k = atomicAdd(&counters[0], 1);
        xs[k] = p;
        vxs[k] = vx[t];
        vys[k] = vy[t];
        vzs[k] = vz[t];
        gids[k] = gid[t];
        stay_t[k] = t;   // the compaction order, for particle data that travels along (DSL)
    } else {
        const int k = atomicAdd(&counters[dir < 0 ? 1 : 2], 1);
        if (k < cap_mig) {
            MigRec r;
            r.x = p.x; r.y = p.y; r.z = p.z;
            r.vx = vx[t]; r.vy = vy[t]; r.vz = vz[t];
            r.gid = gid[t];
            r.pad = t;       // source row of the particle's other data (DSL)
            (dir < 0 ? lo : hi)[k] = r;
        }
    }
}

// append the received migrants after the n_stay stayers
__global__ void k_migrate_append(int n_in, int base, const MigRec* __restrict__ in, double4* __restrict__ xs,
                                 double* __restrict__ vxs, double* __restrict__ vys, double* __restrict__ vzs,
                                 int* __restrict__ gids) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_in) return;
    const MigRec r = in[k];
    xs[base + k] = make_double4(r.x, r.y, r.z, 0.0);
    vxs[base + k] = r.vx;
    vys[base + k] = r.vy;
    vzs[base + k] = r.vz;
    gids[base + k] = (int)r.gid;
}

__global__ void k_iota(int n, int* __restrict__ out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = k;
}

// per-cell counts of the bottom (side 0) and top (side 1) owned planes, lex (cy, cx) order
__global__ void k_plane_counts(Geo g, const int* __restrict__ ocount, int* __restrict__ send_cnt) {
    const int npc = g.nc[0] * g.nc[1];
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 2 * npc) return;
    const int side = k / npc, c = k % npc;
    const int cz = side == 0 ? 0 : g.nzl - 1;
    send_cnt[k] = ocount[g.oc_of_lex[cz * npc + c]];
}

// slot index of every particle of the two boundary planes, in (cy, cx, cell order)
__global__ void k_plane_index(Geo g, const int* __restrict__ send_cnt, const int* __restrict__ send_off,
                              const int* __restrict__ ebegin, int* __restrict__ send_idx) {
    const int npc = g.nc[0] * g.nc[1];
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= 2 * npc) return;
    const int side = warp / npc, c = warp % npc;
    const int cx = c % g.nc[0], cy = c / g.nc[0];
    const int iz = side == 0 ? 1 : g.nzl;
    const int ec = (iz * g.ey + (cy + 1)) * g.ex + (cx + 1);
    const int b = ebegin[ec], m = send_cnt[warp], o = send_off[warp];
    for (int k = lane; k < m; k += 32) send_idx[o + k] = b + k;
}

// gather the boundary-plane positions (w = gid) into the send buffer
__global__ void k_pack(int n, const int* __restrict__ idx, const double4* __restrict__ x,
                       const int* __restrict__ slot_gid, double4* __restrict__ out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = idx[k];
    double4 p = ld256(x + s);
    p.w = (double)slot_gid[s];
    st256(out + k, p);
}

// ------------------------------------------------------------- direct-landing halo (nranks > 1)
// The boundary planes travel every step in the RECEIVER's ghost-plane layout: the whole
// extended z-plane (the owned plane plus its periodic x/y images, cells in (iy, ix) order,
// particles in slot order) with the z shift of the periodic seam already added, so the
// receive lands straight in the receiver's ghost slots (positions and packed positions) and
// no unpack or image pass runs.  The sender's copy lives in a send area after the slot range
// of the position buffers and is written by the kernels that move the particles (force
// epilogue, opening kick-drift), through the same per-particle image lists as the periodic
// images: one entry {send-area index, source slot, shift code} per boundary particle image.

// counts per extended plane cell: side 0 = bottom owned plane (-> lower neighbour), 1 = top
__global__ void k_plane_ext_counts(Geo g, const int* __restrict__ ecount, int* __restrict__ cnt) {
    const int np = g.ex * g.ey;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 2 * np) return;
    const int side = k / np, c = k % np, ix = c % g.ex, iy = c / g.ex;
    const int ox = (ix - 1 + g.nc[0]) % g.nc[0], oy = (iy - 1 + g.nc[1]) % g.nc[1];
    const int iz = side == 0 ? 1 : g.nzl;
    cnt[k] = ecount[(iz * g.ey + (oy + 1)) * g.ex + (ox + 1)];
}

// one warp per extended plane cell: image entries {base + offset, source slot, shift code}
// appended to the ghost-image list (gflat) from which the per-particle image lists are built.
// zs[side]: z shift of the plane as the receiver sees it (-1, 0, +1 in units of Lz).
__global__ void k_send_map(Geo g, const int* __restrict__ ebegin, const int* __restrict__ ecount,
                           const int* __restrict__ off, int base, int zs0, int zs1, int4* __restrict__ gflat,
                           int cap, DevFlags* fl) {
    const int np = g.ex * g.ey;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= 2 * np) return;
    const int side = warp / np, c = warp % np, ix = c % g.ex, iy = c / g.ex;
    const int ox = (ix - 1 + g.nc[0]) % g.nc[0], oy = (iy - 1 + g.nc[1]) % g.nc[1];
    const int sx = ix == 0 ? -1 : (ix == g.nc[0] + 1 ? 1 : 0);
    const int sy = iy == 0 ? -1 : (iy == g.nc[1] + 1 ? 1 : 0);
    const int sz = side == 0 ? zs0 : zs1;
    const int iz = side == 0 ? 1 : g.nzl;
    const int ec = (iz * g.ey + (oy + 1)) * g.ex + (ox + 1);
    const int sb = ebegin[ec], m = ecount[ec];
    int at = 0;
    if (lane == 0 && m) at = atomicAdd(&fl->n_gflat, m);
    at = __shfl_sync(0xffffffffu, at, 0);
    const int code = (sx + 1) | ((sy + 1) << 2) | ((sz + 1) << 4) | 0x80;   // bit 7: send area
    for (int k = lane; k < m; k += 32)   // past cap: the host regrows and rebuilds again
        if (at + k < cap) gflat[at + k] = make_int4(base + off[warp] + k, sb + k, code, 0);
}

// received plane particles: gid from the w component (at build)
__global__ void k_unpack_gid(int n, const double4* __restrict__ xr, int* __restrict__ gid_out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) gid_out[k] = (int)xr[k].w;
}

// --------------------------------------------------------------------------- tile rows
// Per tile: the (ty+2)(tz+2) halo x-rows that hold every stencil cell of its particles, as
// slot ranges [begin, begin + len) of the extended-cell layout, and their offsets in the
// tile's shared-memory staging buffer.  One warp per tile; rebuilt with the cells.
struct TileRows {
    int* begin;   // [n_tiles][kRowsMax]
    int* off;     // [n_tiles][kRowsMax + 1]
    int* len;     // [n_tiles][kRowsMax] true row lengths (rows are padded in the layout)
};

__global__ void k_tile_rows(int n_tiles, Geo g, const int* __restrict__ ebegin,
                            const int* __restrict__ ecount, TileRows tr, DevFlags* fl, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    const int tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (tile >= n_tiles) return;
    const TileGeo T = tile_geo(g, tile);
    int len = 0, beg = 0;
    if (lane < T.R) {
        const int ry = lane % (T.ty + 2), rz = lane / (T.ty + 2);
        const int iy = T.y0 + ry, iz = T.z0 + rz;          // extended coordinates
        const int e0 = (iz * g.ey + iy) * g.ex + T.x0;      // ext x = x0 .. x0 + tx + 1
        const int e1 = e0 + T.tx + 1;
        beg = ebegin[e0];
        len = ebegin[e1] + ecount[e1] - beg;
    }
    // padded rows: each starts at an offset of the same parity as its first slot (24-byte
    // records then start 16-byte aligned in the packed positions and in shared memory up to
    // the same 8-byte shift, as the bulk copy needs) and is followed by a spare record
    const int plen = lane < T.R ? len + 2 : 0;
    int x = plen;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane < T.R) {
        int o0 = x - plen;
        o0 += (o0 ^ beg) & 1;
        tr.len[tile * kRowsMax + lane] = len;
        tr.begin[tile * kRowsMax + lane] = beg;
        tr.off[tile * (kRowsMax + 1) + lane] = o0;
    }
    const int total = __shfl_sync(0xffffffffu, x, 31);
    if (lane == 0) {
        tr.off[tile * (kRowsMax + 1) + T.R] = total;
        atomicMax(&fl->max_staged, total);
    }
}

// --------------------------------------------------------------------------- neighbour list
// Cell method (Sec. 3.4) on the force tiles: one CTA per tile stages the
// fp32 mirror of the tile's halo rows; thread per particle i walks its 9 stencil rows (each
// a contiguous, x-sorted run of 3 cells) inside a binary-searched x-window.  Decision
// r^2 < rbar_c^2 (strict, R4): an fp32 distance decides every candidate outside a provably
// conservative band around rbar_c^2; candidates inside the band take the canonical fp64
// test, which is the oracle's decision (coincident particles are caught by the cell sort).
// Each list is emitted in (stencil row, slot) order as 16-bit indices into the tile's
// shared-memory staging buffer, in blocks of 8 (nbr8[b * n_pad + t], one 16-byte load per 8
// neighbours in the force kernel; the last block is padded with the tile's sentinel).
struct NlistArgs {
    Geo g;
    const double4* x;
    const float4* xf;
    const int* obegin;
    const int* ocount;
    const int* ebegin;
    const int* ecount;
    const int* own_slot;
    const int* ocell_of;
    const int* tile_oc0;
    TileRows tr;
    uint4* nbr8;         // blocks of 8 16-bit local indices, nbr8[b * n_pad + t] (force layout)
    int* ncount;
    const float* ylo_f;  // fp32 faces of the owned cells along y: ylo_f[cy] = cy * w_y, cy = 0..ncy
    const float* zlo_f;  // along z, slab-local: zlo_f[cz] = (z0 + cz) * w_z, cz = 0..nzl
    float slop_f;        // fp32 margin for the row / x-window pruning (conservative)
    int n_own, n_pad, K, n_groups, ngx;
    double rn2;          // rbar_c^2 (fp64, canonical)
    float thr_lo;        // r2f <  thr_lo  =>  r^2 < rbar_c^2 for sure
    float thr_hi;        // r2f >= thr_hi  =>  r^2 >= rbar_c^2 for sure
    DevFlags* fl;
    const int* slot_gid;
    int stage_cap;       // staged records per tile the dynamic shared memory is sized for
    int parts;           // CTAs per tile (small systems)
    int* own_li;         // out: each owned particle's index in its tile's staged halo
    const DevCtl* ctl;   // captured rebuild: skip after a failed capacity check
};

// One CTA per force tile (the same halo rows and local numbering as k_force).
//   Prologue: the fp32 mirror of the tile's halo rows is staged in shared memory (cp.async),
//   and three tables are built there: the tile's owned cells (first particle), per halo row
//   and cell the local index where that cell's run starts (a particle's 3-cell stencil
//   segment of row R is [seg[R][lx], seg[R][lx + 3])), and per cell kSub x sub-bins.
//   Thread per particle: per stencil row, the x-window of the x-sorted segment comes from two
//   sub-bin lookups (one sub-bin of margin each side: conservative against the fp32 rounding)
//   instead of two binary searches; candidates outside a provably conservative band around
//   rbar_c^2 are decided by their fp32 distance, those inside it by the canonical fp64 test
//   (the oracle's decision).  Accepted entries are shifted into four registers and leave as
//   one 16-byte store per 8 entries, in (stencil row, slot) order; the last block is padded
//   with the tile's sentinel.
#ifndef LJMD_BUILD_THREADS
#define LJMD_BUILD_THREADS 480
#endif
constexpr int kBuildThreads = LJMD_BUILD_THREADS;
// Flattened candidate loop (round 2): each thread walks the concatenation of its non-empty
// x-windows (one loop, the window switch predicated) instead of one loop per stencil row, so a
// warp runs max_lanes(sum of windows) iterations instead of sum_rows(max_lanes(window)): the
// lanes idle only at the end of the warp's longest list (55 % of lanes active before).  The
// windows wait in shared memory (9 words per thread), the next candidate's position is loaded
// one iteration ahead.  Same candidates, same order, same decisions: the list is unchanged.
#ifndef LJMD_BUILD_FLAT
#define LJMD_BUILD_FLAT 0
#endif
#ifndef LJMD_BUILD_MINB
#define LJMD_BUILD_MINB (LJMD_BUILD_FLAT ? 3 : 4)
#endif
constexpr int kBuildWinWords = LJMD_BUILD_FLAT ? 9 * LJMD_BUILD_THREADS : 0;   // per-thread windows
constexpr int kTileCells = kTX * kTY * kTZ;
constexpr int kSegW = kTX + 3;            // cell boundaries per halo row (ext x = 0 .. tx + 2)
#ifndef LJMD_KSUB
#define LJMD_KSUB 16
#endif
constexpr int kSub = LJMD_KSUB;           // x sub-bins per cell for the window lookup

struct BuildSmem {
    int cell_t0[kTileCells + 1];          // first particle (tile-relative) of each owned cell
    int seg[kRowsMax][kSegW];             // local index where ext-x cell ex of row R starts
    int delta[kRowsMax];                  // slot = local index + delta[R]
    // sub[R][c][k]: first local index of cell c of row R whose fp32 x >= the sub-bin boundary
    // b(c, k) = x0 + (kSub c + k) w_sub (k = 1 .. kSub - 1); k = 0 / kSub: the cell's bounds
    unsigned short sub[kRowsMax][kTX + 2][kSub + 1];
};

// SMALL (small systems, a.parts > 1 CTAs per tile, each with a few dozen particles): a WARP per
// particle instead of a thread -- lanes test 32 consecutive candidates of a window at a time,
// a ballot compacts the accepted ones into the list -- so a CTA's latency chain is a few
// chunks per particle instead of one thread's ~270 candidates.  Same windows, same (row,
// slot) order, same decisions: the list is identical to the thread-per-particle build's.
template <bool SMALL>
__global__ void __launch_bounds__(kBuildThreads, LJMD_BUILD_MINB) k_build_nlist(NlistArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ BuildSmem S;
    if (a.ctl && a.ctl->abort) return;
    // a.parts CTAs per tile on small systems (each stages the whole halo, takes a share of
    // the particles): enough CTAs for the chip where tiles are few
    const int tile = blockIdx.x / a.parts, part = blockIdx.x % a.parts;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Geo& g = a.g;
    const TileGeo T = tile_geo(g, tile);
    const int oc0 = a.tile_oc0[tile];
    const int t0 = a.obegin[oc0];
    const int m = a.obegin[a.tile_oc0[tile + 1]] - t0;
    const int ncell = T.tx * T.ty * T.tz;
    float4* sF = reinterpret_cast<float4*>(smem);
#if LJMD_BUILD_FLAT
    unsigned* sWin = reinterpret_cast<unsigned*>(smem + 16 * ((size_t)a.stage_cap + 1));
#endif
    // (1) staging of the halo rows (fp32 mirror, 16 B per particle)
    for (int r = warp; r < T.R; r += kBuildThreads / 32) {
        const int b0 = a.tr.begin[tile * kRowsMax + r];
        const int o0 = a.tr.off[tile * (kRowsMax + 1) + r];
        const int len = a.tr.len[tile * kRowsMax + r];
        for (int k = lane; k < len; k += 32) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(sF + o0 + k);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" :: "r"(d), "l"(a.xf + b0 + k) : "memory");
        }
    }
    // (2) tables
    for (int k = threadIdx.x; k <= ncell; k += kBuildThreads) S.cell_t0[k] = a.obegin[oc0 + k] - t0;
    for (int k = threadIdx.x; k < T.R * (T.tx + 3); k += kBuildThreads) {
        const int R = k / (T.tx + 3), ex = k % (T.tx + 3);
        const int ry = R % (T.ty + 2), rz = R / (T.ty + 2);
        const int rbeg = a.tr.begin[tile * kRowsMax + R];
        const int roff = a.tr.off[tile * (kRowsMax + 1) + R];
        const int ec = ((T.z0 + rz) * g.ey + (T.y0 + ry)) * g.ex + T.x0 + ex;
        // ex = tx + 2 is the end of the row: begin of the last cell + its count
        const int sb = ex < T.tx + 2 ? a.ebegin[ec] : a.ebegin[ec - 1] + a.ecount[ec - 1];
        S.seg[R][ex] = roff + (sb - rbeg);
        if (ex == 0) S.delta[R] = rbeg - roff;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const float x0f = (float)((double)(T.x0 - 1) * g.w[0]);
    const float wsub = (float)(g.w[0] / kSub), inv_wsub = 1.f / wsub;
    for (int k = threadIdx.x; k < T.R * (T.tx + 2); k += kBuildThreads) {
        const int R = k / (T.tx + 2), c = k % (T.tx + 2);
        const int end = S.seg[R][c + 1];
        int i = S.seg[R][c];
        S.sub[R][c][0] = (unsigned short)i;
        for (int q = 1; q < kSub; ++q) {
            const float b = x0f + (float)(kSub * c + q) * wsub;
            while (i < end && sF[i].x < b) ++i;
            S.sub[R][c][q] = (unsigned short)i;
        }
        S.sub[R][c][kSub] = (unsigned short)end;
    }
    __syncthreads();

    const size_t stride = (size_t)a.n_pad;
    const float thr_lo = a.thr_lo, thr_hi = a.thr_hi, slop = a.slop_f;
    const int K = a.K;
    unsigned long long kk = 0ull;
    int kmax = 0;
    const int per = (m + a.parts - 1) / a.parts;
    const int q_end = min(m, (part + 1) * per);
    if (SMALL) {
        unsigned short* nbr16 = reinterpret_cast<unsigned short*>(a.nbr8);
        for (int q = part * per + warp; q < q_end; q += kBuildThreads / 32) {   // warp-uniform
            int ci = 0;
            while (ci + 1 < ncell && S.cell_t0[ci + 1] <= q) ++ci;
            const int lx = ci % T.tx, ly = (ci / T.tx) % T.ty, lz = ci / (T.tx * T.ty);
            const int R0 = (lz + 1) * (T.ty + 2) + (ly + 1);
            const int li = S.seg[R0][lx + 1] + (q - S.cell_t0[ci]);
            const int t = t0 + q;
            if (lane == 0) a.own_li[t] = li;
            const float4 fi = sF[li];
            const int cy = T.y0 + ly, cz = T.z0 + lz;
            const float ylo = a.ylo_f[cy], yhi = a.ylo_f[cy + 1];
            const float zlo = a.zlo_f[cz], zhi = a.zlo_f[cz + 1];
            int k = 0;
            for (int rz = 0; rz < 3; ++rz) {
                const float ddz = rz == 0 ? fi.z - zlo : (rz == 2 ? zhi - fi.z : 0.f);
                const float dz2 = fmaxf(ddz - slop, 0.f) * fmaxf(ddz - slop, 0.f);
                for (int ry = 0; ry < 3; ++ry) {
                    const float ddy = ry == 0 ? fi.y - ylo : (ry == 2 ? yhi - fi.y : 0.f);
                    const float dyz2 = fmaf(fmaxf(ddy - slop, 0.f), fmaxf(ddy - slop, 0.f), dz2);
                    if (dyz2 >= thr_hi) continue;
                    const float xw = sqrtf(thr_hi - dyz2) + slop;
                    const int R = (lz + rz) * (T.ty + 2) + (ly + ry);
                    const float xl = fi.x - xw, xh = fi.x + xw;
                    const int g0 = kSub * lx, g1 = kSub * (lx + 3);
                    int gl = (int)floorf((xl - x0f) * inv_wsub) - 1;
                    int gh = (int)floorf((xh - x0f) * inv_wsub) + 2;
                    gl = min(max(gl, g0), g1);
                    gh = min(max(gh, g0), g1);
                    const int cl = min(gl / kSub, lx + 2), ch = min(gh / kSub, lx + 2);
                    const int lo = S.sub[R][cl][gl - kSub * cl];
                    const int hi = S.sub[R][ch][gh - kSub * ch];
                    for (int base = lo; base < hi; base += 32) {   // 32 candidates per step
                        const int jl = base + lane;
                        bool take = false;
                        if (jl < hi && jl != li) {   // R4 self exclusion
                            const float4 fj = sF[jl];
                            const float fx = fi.x - fj.x, fy = fi.y - fj.y, fz = fi.z - fj.z;
                            const float r2f = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
                            if (r2f < thr_hi) {
                                take = r2f < thr_lo;
                                if (!take) {   // the canonical fp64 test in the band
                                    const double4 xi = a.x[li + S.delta[R0]];
                                    const double4 xj = a.x[jl + S.delta[R]];
                                    take = r2_canon(xi.x - xj.x, xi.y - xj.y, xi.z - xj.z) < a.rn2;
                                }
                            }
                        }
                        const unsigned mk = __ballot_sync(0xffffffffu, take);
                        if (take) {
                            const int pos = k + __popc(mk & ((1u << lane) - 1u));
                            if (pos < K) nbr16[(((size_t)(pos >> 3) * stride + t) << 3) + (pos & 7)] = (unsigned short)jl;
                        }
                        k += __popc(mk);
                    }
                }
            }
            if ((k & 7) && k < K && lane < 8 - (k & 7)) {   // the last block: the tile's sentinel
                const int pos = k + lane;
                nbr16[(((size_t)(pos >> 3) * stride + t) << 3) + (pos & 7)] =
                    (unsigned short)a.tr.off[tile * (kRowsMax + 1) + T.R];
            }
            if (lane == 0) {
                a.ncount[t] = k;
                kk += (unsigned long long)k;
            }
            kmax = max(kmax, k);
        }
    }
    for (int q = part * per + (int)threadIdx.x; !SMALL && q < q_end; q += kBuildThreads) {
        int ci = 0;
        while (ci + 1 < ncell && S.cell_t0[ci + 1] <= q) ++ci;
        const int lx = ci % T.tx, ly = (ci / T.tx) % T.ty, lz = ci / (T.tx * T.ty);
        const int R0 = (lz + 1) * (T.ty + 2) + (ly + 1);
        const int li = S.seg[R0][lx + 1] + (q - S.cell_t0[ci]);   // own local index
        a.own_li[t0 + q] = li;
        const float4 fi = sF[li];
        const int cy = T.y0 + ly, cz = T.z0 + lz;
        const float ylo = a.ylo_f[cy], yhi = a.ylo_f[cy + 1];
        const float zlo = a.zlo_f[cz], zhi = a.zlo_f[cz + 1];
        const int t = t0 + q;
        uint4* outb = a.nbr8 + t;
        unsigned w0 = 0u, w1 = 0u, w2 = 0u, w3 = 0u;
        int k = 0;
#if LJMD_BUILD_FLAT
        // accepted entries shift into four registers and leave as one 16-byte store per 8
        auto emit = [&](int jl) {
            w0 = __funnelshift_r(w0, w1, 16);
            w1 = __funnelshift_r(w1, w2, 16);
            w2 = __funnelshift_r(w2, w3, 16);
            w3 = __funnelshift_r(w3, (unsigned)jl, 16);
            if ((k & 7) == 7) {
                if (k < K) *outb = make_uint4(w0, w1, w2, w3);
                outb += stride;
            }
            ++k;
        };
        // (a) the x-windows of the non-empty stencil rows, in stencil order
        int nr = 0, tot = 0;
        unsigned long long sid = 0ull;   // stencil row rz * 3 + ry of window j, 4 bits each
        for (int rz = 0; rz < 3; ++rz) {
            const float ddz = rz == 0 ? fi.z - zlo : (rz == 2 ? zhi - fi.z : 0.f);
            const float dz2 = fmaxf(ddz - slop, 0.f) * fmaxf(ddz - slop, 0.f);
            for (int ry = 0; ry < 3; ++ry) {
                const float ddy = ry == 0 ? fi.y - ylo : (ry == 2 ? yhi - fi.y : 0.f);
                const float dyz2 = fmaf(fmaxf(ddy - slop, 0.f), fmaxf(ddy - slop, 0.f), dz2);
                if (dyz2 >= thr_hi) continue;
                const float xw = sqrtf(thr_hi - dyz2) + slop;
                const int R = (lz + rz) * (T.ty + 2) + (ly + ry);
                const float xl = fi.x - xw, xh = fi.x + xw;
                const int g0 = kSub * lx, g1 = kSub * (lx + 3);
                int gl = (int)floorf((xl - x0f) * inv_wsub) - 1;
                int gh = (int)floorf((xh - x0f) * inv_wsub) + 2;
                gl = min(max(gl, g0), g1);
                gh = min(max(gh, g0), g1);
                const int cl = min(gl / kSub, lx + 2), ch = min(gh / kSub, lx + 2);
                const int lo = S.sub[R][cl][gl - kSub * cl];
                const int hi = S.sub[R][ch][gh - kSub * ch];
                if (hi > lo) {
                    sWin[nr * kBuildThreads + threadIdx.x] = (unsigned)lo | ((unsigned)hi << 16);
                    sid |= (unsigned long long)(rz * 3 + ry) << (4 * nr);
                    ++nr;
                    tot += hi - lo;
                }
            }
        }
        // (b) one loop over the concatenated windows (the own index is skipped: R4 self
        // exclusion); candidate it + 1 is read while candidate it is decided
        int j = 0;
        unsigned wv = nr ? sWin[threadIdx.x] : 0u;
        int jl = (int)(wv & 0xffffu), jend = (int)(wv >> 16);
        float4 fj = sF[jl];
        for (int it = 0; it < tot; ++it) {
            const int jc = jl, jrow = j;
            const float4 fc = fj;
            if (++jl == jend) {
                ++j;
                wv = j < nr ? sWin[j * kBuildThreads + threadIdx.x] : 0u;
                jl = (int)(wv & 0xffffu);
                jend = (int)(wv >> 16);
            }
            fj = sF[jl];
            const float fx = fi.x - fc.x, fy = fi.y - fc.y, fz = fi.z - fc.z;
            const float r2f = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
            if (r2f >= thr_hi || jc == li) continue;
            bool take = r2f < thr_lo;
            if (!take) {   // rare: decide in fp64 on the canonical r^2 (the oracle's test)
                const int sr = (int)(sid >> (4 * jrow)) & 15;
                const int R = (lz + sr / 3) * (T.ty + 2) + (ly + sr % 3);
                const double4 xi = a.x[li + S.delta[R0]];
                const double4 xj = a.x[jc + S.delta[R]];
                take = r2_canon(xi.x - xj.x, xi.y - xj.y, xi.z - xj.z) < a.rn2;
            }
            if (take) emit(jc);
        }
#else
        for (int rz = 0; rz < 3; ++rz) {
            const float ddz = rz == 0 ? fi.z - zlo : (rz == 2 ? zhi - fi.z : 0.f);
            const float dz2 = fmaxf(ddz - slop, 0.f) * fmaxf(ddz - slop, 0.f);
            for (int ry = 0; ry < 3; ++ry) {
                const float ddy = ry == 0 ? fi.y - ylo : (ry == 2 ? yhi - fi.y : 0.f);
                const float dyz2 = fmaf(fmaxf(ddy - slop, 0.f), fmaxf(ddy - slop, 0.f), dz2);
                if (dyz2 >= thr_hi) continue;
                const float xw = sqrtf(thr_hi - dyz2) + slop;
                const int R = (lz + rz) * (T.ty + 2) + (ly + ry);
                const float xl = fi.x - xw, xh = fi.x + xw;
                const int g0 = kSub * lx, g1 = kSub * (lx + 3);
                int gl = (int)floorf((xl - x0f) * inv_wsub) - 1;
                int gh = (int)floorf((xh - x0f) * inv_wsub) + 2;
                gl = min(max(gl, g0), g1);
                gh = min(max(gh, g0), g1);
                const int cl = min(gl / kSub, lx + 2), ch = min(gh / kSub, lx + 2);
                const int lo = S.sub[R][cl][gl - kSub * cl];
                const int hi = S.sub[R][ch][gh - kSub * ch];
                // self exclusion by splitting the window around the own local index
                for (int part = 0; part < 2; ++part) {
                    const int j0 = part ? max(lo, li + 1) : lo;
                    const int j1 = part ? hi : min(hi, li);
                    for (int jl = j0; jl < j1; ++jl) {
                        const float4 fj = sF[jl];
                        const float fx = fi.x - fj.x, fy = fi.y - fj.y, fz = fi.z - fj.z;
                        const float r2f = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
                        if (r2f >= thr_hi) continue;
                        bool take = r2f < thr_lo;
                        if (!take) {   // rare: decide in fp64 on the canonical r^2 (the oracle's test)
                            const double4 xi = a.x[li + S.delta[R0]];
                            const double4 xj = a.x[jl + S.delta[R]];
                            take = r2_canon(xi.x - xj.x, xi.y - xj.y, xi.z - xj.z) < a.rn2;
                        }
                        if (take) {
                            w0 = __funnelshift_r(w0, w1, 16);
                            w1 = __funnelshift_r(w1, w2, 16);
                            w2 = __funnelshift_r(w2, w3, 16);
                            w3 = __funnelshift_r(w3, (unsigned)jl, 16);
                            if ((k & 7) == 7) {
                                if (k < K) *outb = make_uint4(w0, w1, w2, w3);
                                outb += stride;
                            }
                            ++k;
                        }
                    }
                }
            }
        }
#endif
        if ((k & 7) && k < K) {   // pad the last block with the tile's sentinel index
            const unsigned sen = (unsigned)a.tr.off[tile * (kRowsMax + 1) + T.R];
            for (int e = k & 7; e < 8; ++e) {
                w0 = __funnelshift_r(w0, w1, 16);
                w1 = __funnelshift_r(w1, w2, 16);
                w2 = __funnelshift_r(w2, w3, 16);
                w3 = __funnelshift_r(w3, sen, 16);
            }
            *outb = make_uint4(w0, w1, w2, w3);
        }
        a.ncount[t] = k;
        kmax = max(kmax, k);
        kk += (unsigned long long)k;
    }
    for (int o = 16; o > 0; o >>= 1) {
        kk += __shfl_down_sync(0xffffffffu, kk, o);
        kmax = max(kmax, __shfl_down_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0 && kk) {
        atomicAdd(&a.fl->total_nbr, kk);
        atomicMax(&a.fl->max_nbr, kmax);
    }
}

// --------------------------------------------------------------------------- bank-aware list order
// The force CTA's thread q reads neighbour l from shared memory at byte 24 l: the bank pair
// of an 8-byte load is 3 l mod 16, so two lanes of a half-warp conflict when their local
// indices differ by a multiple of 16.  Re-sequencing each list so that entry k targets
// residue (q + k) mod 16 (the next non-empty residue, cyclically, when that one is used
// up) spreads the 16 lanes of a phase over distinct banks most of the time; measured on C2
// the force kernel drops from ~199 to ~170 us.  Only the order of a particle's sum
// changes, not its terms.  Thread per particle; buckets of kRrCap entries per residue in
// bank-padded shared memory (288 B, stride 73 words per thread); the per-residue fill and
// remaining counts live in registers as 16 nibbles each, so the output walk reads a bucket
// entry at (filled - remaining); the availability mask is kept twice (bits r and r + 16) so
// the cyclic search for the next available residue is one shift and one find-first-set
// (225 us per C2 rebuild against 300 us with count and head arrays in shared memory).  A particle with a fuller
// residue keeps the build order.
// Round 2 (LJMD_RR_LEAN): the per-residue fill and take counters live as bytes in the
// thread's shared-memory record instead of 64-bit nibble registers (whose variable 64-bit
// shifts made the pass issue-bound: ~70 instructions per list entry, 232 us per C2 rebuild);
// the same buckets, the same greedy walk, the same output.
#ifndef LJMD_RR_LEAN
#define LJMD_RR_LEAN 1
#endif
constexpr int kRrThreads = 128;
constexpr int kRrCap = 8;                        // per-residue capacity (mean ~4.6)
constexpr int kRrOvf = 16;                       // entries beyond a full bucket, emitted last
#if LJMD_RR_LEAN
// per thread: buckets u16[16][kRrCap], overflow u16[kRrOvf], fill counts u8[16], taken u8[16];
// odd word stride (no bank aliasing between the threads' records)
constexpr int kRrStrideW = (16 * kRrCap + kRrOvf) / 2 + 8 + 1;
constexpr size_t kRrSmem = sizeof(unsigned) * (size_t)kRrThreads * kRrStrideW;

__global__ void __launch_bounds__(kRrThreads) k_list_rr(int n_own, int n_pad, int K, Geo g,
                                                       const uint4* in,
                                                       const int* __restrict__ ncount,
                                                       const int* __restrict__ ocell_of,
                                                       const int* __restrict__ obegin,
                                                       const int* __restrict__ tile_oc0,
                                                       uint4* out, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    extern __shared__ unsigned rr_smem[];
    const int tid = threadIdx.x;
    const int t = blockIdx.x * kRrThreads + tid;
    unsigned* rec = rr_smem + (size_t)tid * kRrStrideW;
    unsigned short* bkt = reinterpret_cast<unsigned short*>(rec);
    unsigned short* ovf = bkt + 16 * kRrCap;
    constexpr int kCw = (16 * kRrCap + kRrOvf) / 2;   // first counter word
    unsigned char* C = reinterpret_cast<unsigned char*>(rec + kCw);
    unsigned char* U = C + 16;
    if (t >= n_own) return;
#pragma unroll
    for (int w = 0; w < 8; ++w) rec[kCw + w] = 0u;
    const int n = min(ncount[t], K);
    const int nb = (n + 7) >> 3;
    const size_t stride = (size_t)n_pad;
    int cx, cy, cz;
    lex_xyz(g, g.lex_of_oc[ocell_of[t]], cx, cy, cz);
    const int tile = tile_of_cell(g, cx, cy, cz);
    const int off = (t - obegin[tile_oc0[tile]]) & 15;
    int novf = 0;
    bool overflow = false;
    unsigned short pad = 0;
    // filing, branch-free per entry: a bucket slot while the residue has room, else the
    // next overflow slot (clamped; a full overflow area makes the particle keep build order)
    auto file = [&](unsigned short l) {
        const int r = l & 15;
        const int c = C[r];
        const bool ok = c < kRrCap;
        unsigned short* dst = ok ? bkt + r * kRrCap + c : ovf + min(novf, kRrOvf - 1);
        *dst = l;
        C[r] = (unsigned char)(c + (ok ? 1 : 0));
        overflow |= !ok && novf >= kRrOvf;
        novf += ok ? 0 : 1;
    };
    const int nfull = n >> 3;
    uint4 vn = nb > 0 ? in[t] : make_uint4(0u, 0u, 0u, 0u);
    for (int b = 0; b < nb; ++b) {
        const uint4 v = vn;
        if (b + 1 < nb) vn = in[(size_t)(b + 1) * stride + t];   // next block in flight
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
        if (b < nfull) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                file((unsigned short)((e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xffffu)));
        } else {   // the last, padded block
            for (int e = 0; e < 8; ++e) {
                const unsigned short l = (unsigned short)((w[e >> 1] >> (16 * (e & 1))) & 0xffffu);
                if (b * 8 + e < n) file(l);
                else pad = l;   // the tile's sentinel
            }
        }
    }
    if (overflow) {
        for (int b = 0; b < nb; ++b) out[(size_t)b * stride + t] = in[(size_t)b * stride + t];
        return;
    }
    unsigned avail = 0u;
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if (C[r]) avail |= 1u << r;
    const int nin = n - novf;
    unsigned w0 = 0u, w1 = 0u, w2 = 0u, w3 = 0u;   // 8 pending entries, shifted in from the top
    uint4* o = out + t;
    int k = 0;
    auto emit = [&](unsigned l) {
        w0 = __funnelshift_r(w0, w1, 16);
        w1 = __funnelshift_r(w1, w2, 16);
        w2 = __funnelshift_r(w2, w3, 16);
        w3 = __funnelshift_r(w3, l, 16);
        if ((k & 7) == 7) {
            *o = make_uint4(w0, w1, w2, w3);
            o += stride;
        }
        ++k;
    };
    unsigned av2 = avail | (avail << 16);   // bit r and r + 16: a rotation is one shift
    int tgt = off;                          // (off + k) mod 16
    for (int q = 0; q < nin; ++q) {         // the greedy walk over the residues
        const int rr = (tgt + __ffs(av2 >> tgt) - 1) & 15;
        tgt = (tgt + 1) & 15;
        const int u = U[rr];
        const unsigned l = bkt[rr * kRrCap + u];
        U[rr] = (unsigned char)(u + 1);
        av2 &= u + 1 == (int)C[rr] ? ~(0x10001u << rr) : 0xffffffffu;
        emit(l);
    }
    for (int q = 0; q < novf; ++q) emit(ovf[q]);   // overflow entries, build order
    while (k < nb * 8) emit(pad);                  // the last block's sentinel padding
}
#else
constexpr int kRrStrideW = (16 * kRrCap + kRrOvf) / 2 + 1;   // words per thread (odd: no bank aliasing)
constexpr size_t kRrSmem = sizeof(unsigned) * (size_t)kRrThreads * kRrStrideW;

__device__ __forceinline__ unsigned nib(unsigned long long w, int r) { return (unsigned)(w >> (4 * r)) & 15u; }

__global__ void __launch_bounds__(kRrThreads) k_list_rr(int n_own, int n_pad, int K, Geo g,
                                                       const uint4* in,
                                                       const int* __restrict__ ncount,
                                                       const int* __restrict__ ocell_of,
                                                       const int* __restrict__ obegin,
                                                       const int* __restrict__ tile_oc0,
                                                       uint4* out, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    extern __shared__ unsigned rr_smem[];
    const int tid = threadIdx.x;
    const int t = blockIdx.x * kRrThreads + tid;
    unsigned short* bkt = reinterpret_cast<unsigned short*>(rr_smem + (size_t)tid * kRrStrideW);
    if (t >= n_own) return;
    const int n = min(ncount[t], K);
    const int nb = (n + 7) >> 3;
    const size_t stride = (size_t)n_pad;
    int cx, cy, cz;
    lex_xyz(g, g.lex_of_oc[ocell_of[t]], cx, cy, cz);
    const int tile = tile_of_cell(g, cx, cy, cz);
    const int off = (t - obegin[tile_oc0[tile]]) & 15;
    unsigned long long cnt = 0ull;   // entries filed per residue (nibbles)
    bool overflow = false;
    int novf = 0;
    unsigned short pad = 0;
    uint4 vn = nb > 0 ? in[t] : make_uint4(0u, 0u, 0u, 0u);
    for (int b = 0; b < nb; ++b) {
        const uint4 v = vn;
        if (b + 1 < nb) vn = in[(size_t)(b + 1) * stride + t];   // next block in flight
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const unsigned short l = (unsigned short)((e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xffffu));
            if (b * 8 + e < n) {
                const int r = l & 15;
                const unsigned c = nib(cnt, r);
                if (c < (unsigned)kRrCap) {
                    bkt[r * kRrCap + c] = l;
                    cnt += 1ull << (4 * r);
                } else if (novf < kRrOvf) {
                    bkt[16 * kRrCap + novf++] = l;
                } else {
                    overflow = true;
                }
            } else {
                pad = l;   // the tile's sentinel
            }
        }
    }
    if (overflow) {
        for (int b = 0; b < nb; ++b) out[(size_t)b * stride + t] = in[(size_t)b * stride + t];
        return;
    }
    unsigned avail = 0u;
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if (nib(cnt, r)) avail |= 1u << r;
    unsigned long long rem = cnt;   // entries not yet emitted per residue
    const int nin = n - novf;
    unsigned w0 = 0u, w1 = 0u, w2 = 0u, w3 = 0u;   // 8 pending entries, shifted in from the top
    uint4* o = out + t;
    unsigned av2 = avail | (avail << 16);   // bit r and r + 16: a rotation is one shift
    int tgt = off;                          // (off + k) mod 16
    for (int k = 0; k < nb * 8; ++k) {
        unsigned l = pad;
        if (k < nin) {
            const int rr = (tgt + __ffs(av2 >> tgt) - 1) & 15;
            tgt = (tgt + 1) & 15;
            const int sh = 4 * rr;
            const unsigned m = (unsigned)(rem >> sh) & 15u;
            l = bkt[rr * kRrCap + (((unsigned)(cnt >> sh) & 15u) - m)];
            rem -= 1ull << sh;
            if (m == 1u) av2 &= ~(0x10001u << rr);
        } else if (k < n) {
            l = bkt[16 * kRrCap + (k - nin)];
        }
        w0 = __funnelshift_r(w0, w1, 16);
        w1 = __funnelshift_r(w1, w2, 16);
        w2 = __funnelshift_r(w2, w3, 16);
        w3 = __funnelshift_r(w3, l, 16);
        if ((k & 7) == 7) {
            *o = make_uint4(w0, w1, w2, w3);
            o += stride;
        }
    }
}

#endif

// --------------------------------------------------------------------------- force
// LJ force over the full (both-orders) list, written only to i: no atomics.
// Eq. eqn:LJforce with u = 1/r^2:
//   g = 48 eps sigma^6 u^4 [sigma^6 u^3 - 1/2] = u^4 (c12 u^3 - c6),
//   c12 = 48 eps sigma^12, c6 = 24 eps sigma^6;  F_i += g (r_i - r_j)     (reading R1)
//   V = 4 eps [sigma^12 u^6 - sigma^6 u^3 + s] = (a12 u^3 - a6) u^3 + a0;  e_i = V/2 (R2)
// Epilogue modes (velocity Verlet fused around the force, Alg. alg:VelocityVerlet):
//   kStore : F_i stored (init / readback)
//   kKick  : v += h F (line 8), F stored          -- last step of ljmd_step
//   kKKD   : v += h F (line 8) ; [KE sample] ; v += h F ; x' = x + dt v (line 6 of the
//            next step) written to the other position buffer
//   | kThermo : Andersen collisions after line 8, a separate instantiation so the
//            default kernels keep their register allocation
enum { kStore = 0, kKick = 1, kKKD = 2, kThermo = 4 };

struct ForceArgs {
    Geo g;
    const double4* x;        // current positions (slot space)
    double4* x_next;         // kKKD output buffer (slot space)
    const double* xp;        // packed {x, y, z} per slot (24 B) of the current positions
    double* xp_next;         // kKKD: packed x(n+1)
    const int* own_slot;
    const int* own_li;       // owned particle -> its index in the tile's staged halo
    const uint4* nbr;        // blocks of 8 16-bit local indices: nbr[b * n_pad + t]
    const int* ncount;
    const int* obegin;
    const int* tile_oc0;     // first owned cell of each tile (tile-major), [n_tiles + 1]
    TileRows tr;
    double* fx; double* fy; double* fz;
    double* vx; double* vy; double* vz;
    double* e;               // per-particle e_i (ENERGY)
    double* pe_part;         // per-block partial sums (ENERGY)
    double* ke_part;
    const double4* xbuild;   // displacement check (may be null)
    Images im;               // ghost images written with x(n+1) (kKKD)
    int tile_base;           // first tile of this launch
    int seg0, gap;           // tiles seg0.. of the launch are shifted by gap (two ranges, one launch)
    // gated halo (nranks > 1): one launch over every tile, interior tiles first; the two
    // boundary tile layers (whose halos hold received planes) wait in-kernel for the halo
    const unsigned* halo_flag;   // null: no gating
    unsigned halo_seq;           // the value the flag reaches once this step's halo has landed
    int nint, layer;             // interior tiles, tiles per z layer
    // boundary-first launch (nranks > 1): the two boundary tile layers go first (launch
    // indices [0, 2 layer)), each of their CTAs adds 1 to *bdone when its epilogue (which
    // writes the outgoing halo) is done, so the next halo exchange starts during the interior
    int bfirst;
    unsigned* bdone;
    DevFlags* fl;
    int n_own, n_pad;
    double rc2, c12, nc6, a12, na6, a0;   // nc6 = -c6, na6 = -a6 (fold into DFMA operands)
    double h, dt, half_m;
    // Andersen thermostat (reading R19): nu_dt = 0 disables
    const int* gid;
    double nu_dt, sd;                     // collision probability per step, sqrt(T/m)
    unsigned long long seed;
    long long step;                       // 1-based index of the step this launch completes
    const DevCtl* ctl;                    // captured steps: skip everything after an abort
    int parts;                            // CTAs per tile (small systems: more CTAs than tiles)
};

// Philox4x32-10 (Salmon et al., SC'11): counter-based, so the draws of (gid, step) do not
// depend on the decomposition or the launch order.
__device__ __forceinline__ uint4 philox4x32(uint4 c, unsigned k0, unsigned k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ double uniform53(unsigned a, unsigned b) {
    return __dmul_rn(__dadd_rn(__dmul_rn((double)(a >> 5), 67108864.0), (double)(b >> 6)),
                     1.0 / 9007199254740992.0);
}

// Andersen collision of one particle at the end of step a.step: with probability nu_dt the
// velocity is replaced by a Maxwell-Boltzmann draw (Box-Muller on Philox uniforms).
__device__ __forceinline__ void andersen(unsigned long long seed, long long step, double nu_dt, double sd, int g,
                                         double& vx, double& vy, double& vz) {
    const unsigned k0 = (unsigned)seed, k1 = (unsigned)(seed >> 32);
    uint4 c = make_uint4((unsigned)g, (unsigned)step, (unsigned)((unsigned long long)step >> 32), 0u);
    const uint4 w = philox4x32(c, k0, k1);
    if (!(uniform53(w.x, w.y) < nu_dt)) return;
    c.w = 1u;
    const uint4 w1 = philox4x32(c, k0, k1);
    c.w = 2u;
    const uint4 w2 = philox4x32(c, k0, k1);
    const double U1 = uniform53(w.z, w.w), U2 = uniform53(w1.x, w1.y);
    const double U3 = uniform53(w1.z, w1.w), U4 = uniform53(w2.x, w2.y);
    const double two_pi = 6.283185307179586;
    const double R1 = sqrt(__dmul_rn(-2.0, log(__dadd_rn(1.0, -U1))));
    const double R2 = sqrt(__dmul_rn(-2.0, log(__dadd_rn(1.0, -U3))));
    vx = __dmul_rn(sd, __dmul_rn(R1, cos(__dmul_rn(two_pi, U2))));
    vy = __dmul_rn(sd, __dmul_rn(R1, sin(__dmul_rn(two_pi, U2))));
    vz = __dmul_rn(sd, __dmul_rn(R2, cos(__dmul_rn(two_pi, U4))));
}

#ifndef LJMD_FORCE_THREADS
#define LJMD_FORCE_THREADS 480   // ~24 cells x 18.5 particles per tile at rho = 0.8442
#endif
constexpr int kForceThreads = LJMD_FORCE_THREADS;
// 2 CTAs of 480 threads (3 of 320 with 4 x 2 x 2 tiles) per SM with up to 64 registers:
// measured on C2 (320-thread tiles) 160 us per launch against 167 us at 4 CTAs / 48
// registers and 170 us at 2 CTAs / 96 registers (more in-flight neighbours per warp beats
// more warps)
#ifndef LJMD_FORCE_MINB
#define LJMD_FORCE_MINB 2
#endif
// programmatic dependent launch of consecutive force launches (C2: -46 us per 20 steps)
#ifndef LJMD_PDL
#define LJMD_PDL 1
#endif
// L2 prefetch of the epilogue's velocities right after the PDL wait (-0.5 us per launch)
#ifndef LJMD_VPREF2
#define LJMD_VPREF2 1
#endif
// halo copies issued by warp 0 right after the PDL wait, ahead of the per-particle loads; x_i
// read from the staged halo (own_li, written by the list build)
#ifndef LJMD_EARLY_TMA
#define LJMD_EARLY_TMA 1
#endif
#if LJMD_EARLY_TMA && LJMD_HALO_GATE
#error "LJMD_HALO_GATE gates the halo copies, which LJMD_EARLY_TMA issues first"
#endif

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    // deterministic fixed-shape tree (warp shuffles, then warp 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < NT / 32 ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;
}

// r^2 < rc^2 decided on the canonical r^2 (the oracle's decision) while the force uses the
// FMA-contracted r^2: the two differ by a few ulps, so only candidates within 16 ulps of
// rc^2 (integer distance of the bit patterns of two positive doubles) recompute the
// canonical value -- a warp-rare branch that keeps 2 FP64 instructions off the hot loop.
__device__ __forceinline__ bool inside_rc(double r2f, double dx, double dy, double dz, double rc2) {
    const long long b = __double_as_longlong(r2f), c = __double_as_longlong(rc2);
    const long long d = b - c;
    if (d > 16 || d < -16) return d < 0;
    return r2_canon(dx, dy, dz) < rc2;
}

// L1 prefetch (no register): the list blocks stream from DRAM, and the compiler sinks the
// register "prefetch" of the next block to the end of the loop under register pressure.
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" :: "l"(p) : "memory");   // pinned: no sinking
}


// Per-particle state loaded before the tile is staged (hides the list/position latency).
struct FPart {
    int t, si, cnt;
    double4 xi;
    uint4 nb0;
};

__device__ __forceinline__ FPart fpart_load(const ForceArgs& a, int t) {
    FPart P;
    P.t = t;
    P.si = a.own_slot[t];
    P.cnt = a.ncount[t];
    P.xi = ld256(a.x + P.si);
    P.nb0 = P.cnt > 0 ? a.nbr[t] : make_uint4(0u, 0u, 0u, 0u);
    return P;
}

// List blocks 1.. of a particle stream into a per-thread ring of kRing 16-byte slots in
// shared memory with cp.async (no registers held, kRing - 1 blocks of look-ahead): the
// register prefetch of one block ahead left the loop head waiting on the list load (the top
// long_scoreboard stall of the kernel).  Slot d of thread q: ring + (d * kForceThreads + q)
// * 16, so a warp's 32 slots are one contiguous 512-byte run (conflict-free LDS.128).
#ifndef LJMD_PF_L2
#define LJMD_PF_L2 0       // > 0: also an L2 prefetch this many blocks ahead
#endif
#ifndef LJMD_PF_DIST
#define LJMD_PF_DIST 2     // list block prefetched into L1 this many blocks ahead
#endif
#ifndef LJMD_RING
#define LJMD_RING 0        // 0: register prefetch of one block + L1 prefetch of the next (default)
#endif
constexpr int kRing = LJMD_RING;
// the cutoff test r^2 < rc^2 on the integer bit patterns of the two positive doubles (the
// same decision as DSETP, on the ALU pipe instead of the FP64 pipe)
#ifndef LJMD_INT_CUT
#define LJMD_INT_CUT 0
#endif

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ uint4 lds128(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// blocks 1 .. kRing - 1 of particle P into the ring (one commit group per block)
__device__ __forceinline__ void ring_start(const ForceArgs& a, const FPart& P, unsigned ring) {
    if (kRing == 0) {
        if (P.cnt > 8) prefetch_l1(a.nbr + (size_t)a.n_pad + P.t);
        return;
    }
    const int nblk = (P.cnt + 7) >> 3;
#pragma unroll
    for (int d = 1; d < kRing; ++d) {
        if (d < nblk) cp_async16(ring + (unsigned)(d * kForceThreads * 16), a.nbr + (size_t)d * a.n_pad + P.t);
        cp_commit();
    }
}

// Phase timers of the force kernel (measurement build only, LJMD_PHASES=1): per CTA the
// globaltimer at entry, after the halo staging, the first and last warp's loop end, the
// last warp's epilogue end, the CTA's end, and the SM id -- tools/phases.py.
#ifndef LJMD_PHASES
#define LJMD_PHASES 0
#endif
#if LJMD_PHASES
__device__ unsigned long long ljmd_phase_buf[16384 * 10];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

template <bool ENERGY, int MODE, bool CHECK>
__device__ __forceinline__ void force_particle(const ForceArgs& a, const FPart& P, const char* sPb,
                                               double& epart, double& ke, unsigned long long& dbits,
                                               unsigned ring, unsigned long long* ph = nullptr) {
    const int t = P.t;
    const double4 xi = P.xi;
    const uint4* nb = a.nbr + t;
    const size_t stride = (size_t)a.n_pad;
    double fx = 0.0, fy = 0.0, fz = 0.0, u = 0.0;
    const int nblk = (P.cnt + 7) >> 3;
    uint4 cur = P.nb0;
#if LJMD_INT_CUT
    const long long rc2b = __double_as_longlong(a.rc2);
#endif
    for (int b = 0; b < nblk; ++b) {
        // a short block is padded with the sentinel, so every entry is evaluated unpredicated
        uint4 nxt = make_uint4(0u, 0u, 0u, 0u);
        if (kRing == 0) {   // block b+2 into L1 now, block b+1 into registers
            if (b + LJMD_PF_DIST < nblk) prefetch_l1(nb + (size_t)(b + LJMD_PF_DIST) * stride);
#if LJMD_PF_L2
            if (b + LJMD_PF_L2 < nblk)
                asm volatile("prefetch.global.L2 [%0];" :: "l"(nb + (size_t)(b + LJMD_PF_L2) * stride));
#endif
            if (b + 1 < nblk) nxt = nb[(size_t)(b + 1) * stride];
#if LJMD_LOADFENCE
            __syncwarp(__activemask());   // keeps ptxas from sinking the load to the loop end
#endif
        } else if (b > 0) {
            cp_wait<(kRing > 0 ? kRing - 1 : 0)>();   // the group of block b has landed
            cur = lds128(ring + (unsigned)((b % (kRing > 0 ? kRing : 1)) * kForceThreads * 16));
        }
        const unsigned w4[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const unsigned l = (e & 1) ? (w4[e >> 1] >> 16) : (w4[e >> 1] & 0xffffu);
            const double* pj = reinterpret_cast<const double*>(sPb + 24u * l);
            const double dx = xi.x - pj[0], dy = xi.y - pj[1], dz = xi.z - pj[2];
            const double r2 = r2_canon(dx, dy, dz);          // the oracle's r^2
            const double ir2 = rcp64(r2);
            const double ir4 = ir2 * ir2;
            const double ir6 = ir4 * ir2;
            const double ir8 = ir4 * ir4;
            double gg = ir8 * fma(a.c12, ir6, a.nc6);
#if LJMD_INT_CUT
            const bool in = __double_as_longlong(r2) < rc2b;
#else
            const bool in = r2 < a.rc2;
#endif
            gg = in ? gg : 0.0;
            fx = fma(gg, dx, fx);
            fy = fma(gg, dy, fy);
            fz = fma(gg, dz, fz);
            if (ENERGY) {
                const double v = fma(fma(a.a12, ir6, a.na6), ir6, a.a0);
                u += in ? v : 0.0;
            }
        }

        // block b + kRing into the slot of block b (just consumed): blocks b + 1 .. b + kRing - 1
        // stay in flight; block j >= 1 is commit group j - 1 of this particle
        if (kRing == 0) {
            cur = nxt;
        } else {
            const int bn = b + kRing;
            if (bn < nblk)
                cp_async16(ring + (unsigned)((bn % (kRing > 0 ? kRing : 1)) * kForceThreads * 16), nb + (size_t)bn * stride);
            cp_commit();
        }
    }
#if LJMD_PHASES
    if (ph) {   // this warp's loop end (lanes reconverge here)
        __syncwarp(__activemask());
        if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) {
            const unsigned long long now = gtimer();
            atomicMin(&ph[2], now);
            atomicMax(&ph[3], now);
        }
    }
#else
    (void)ph;
#endif
    if ((MODE & 3) == kStore) {
        a.fx[t] = fx; a.fy[t] = fy; a.fz[t] = fz;
        if (ENERGY) {
            const double vx = a.vx[t], vy = a.vy[t], vz = a.vz[t];
            ke += a.half_m * __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
        }
    } else {
        double vx = a.vx[t], vy = a.vy[t], vz = a.vz[t];
        // line 8: v += dt/(2m) F  (two roundings, as Listing lst:velocity_update)
        vx = __dadd_rn(vx, __dmul_rn(a.h, fx));
        vy = __dadd_rn(vy, __dmul_rn(a.h, fy));
        vz = __dadd_rn(vz, __dmul_rn(a.h, fz));
        if (MODE & kThermo) andersen(a.seed, a.step, a.nu_dt, a.sd, a.gid[t], vx, vy, vz);
        if (ENERGY)
            ke += a.half_m * __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
        if ((MODE & 3) == kKick) {
            a.fx[t] = fx; a.fy[t] = fy; a.fz[t] = fz;
        } else {
            // line 6 of the next step: v += dt/(2m) F ; r += dt v (Listing lst:position_update)
            vx = __dadd_rn(vx, __dmul_rn(a.h, fx));
            vy = __dadd_rn(vy, __dmul_rn(a.h, fy));
            vz = __dadd_rn(vz, __dmul_rn(a.h, fz));
            const double4 xn = make_double4(__dadd_rn(xi.x, __dmul_rn(a.dt, vx)),
                                            __dadd_rn(xi.y, __dmul_rn(a.dt, vy)),
                                            __dadd_rn(xi.z, __dmul_rn(a.dt, vz)), 0.0);
            st256(a.x_next + P.si, xn);
            st_packed(a.xp_next, P.si, xn);
            write_images(a.im, t, a.g, a.x_next, a.xp_next, xn);
            if (CHECK) {
                const double4 bb = a.xbuild[t];
                // non-negative doubles order like their bit patterns
                const unsigned long long d2 =
                    __double_as_longlong(r2_canon(xn.x - bb.x, xn.y - bb.y, xn.z - bb.z));
                dbits = d2 > dbits ? d2 : dbits;
            }
        }
        a.vx[t] = vx; a.vy[t] = vy; a.vz[t] = vz;
    }
    if (ENERGY) {
        a.e[t] = 0.5 * u;
        epart += 0.5 * u;
    }
}

// One TMA bulk copy per halo row of the tile (warp 0; lane r copies row r), completion on
// the mbarrier with the total byte count (expect_tx by lane 0).
__device__ __forceinline__ void issue_halo(const ForceArgs& a, const TileGeo& T, int rb, int ro, int rl,
                                           double* sP, unsigned mb, int lane) {
        unsigned sz = 0u;
        unsigned long long src = 0ull;
        unsigned dst = 0u;
        if (lane < T.R) {
            const unsigned d = (unsigned)(rb & 1) * 8u;
            src = reinterpret_cast<unsigned long long>(a.xp + 3 * (size_t)rb) - d;
            dst = (unsigned)__cvta_generic_to_shared(sP + 3 * ro) - d;
            sz = (24u * (unsigned)rl + d + 15u) & ~15u;
        }
        unsigned tot = sz;
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(tot) : "memory");
        __syncwarp();
        if (sz)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(dst), "l"(src), "r"(sz), "r"(mb) : "memory");
}

// One CTA per tile.  (1) Each thread issues the global loads of its particle (slot, count,
// first index block, position); (2) warp 0 copies the tile's halo rows -- x, y, z of every
// particle any of its particles can list -- into shared memory with one TMA bulk copy per
// row from the packed positions (24 B per particle), plus a far-away sentinel for list
// padding;
// (3) thread per particle over its list of 16-bit local indices: each neighbour is three
// LDS.64 from one address (bank group = 3 l mod 16, spread across a half-warp by the
// bank-aware list order) instead of a scattered 32 B global gather.
template <bool ENERGY, int MODE, bool CHECK>
__global__ void __launch_bounds__(kForceThreads, LJMD_FORCE_MINB) k_force(ForceArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double sh[kForceThreads / 32];
#if LJMD_PHASES
    __shared__ unsigned long long ph[8];
    if (threadIdx.x == 0) {
        ph[0] = gtimer();
        ph[2] = ~0ull;
        ph[3] = 0ull;
        ph[4] = 0ull;
    }
    unsigned long long* php = ph;
#else
    unsigned long long* php = nullptr;
#endif
    // a launch covers a range of tiles, a.parts CTAs per tile (each stages the whole tile
    // halo and takes a share of its particles: small systems get enough CTAs for the chip)
#if LJMD_FPARTS_OFF
    const int part = 0;
    const int ti = blockIdx.x;
#else
    const int part = blockIdx.x % a.parts;
    const int ti = blockIdx.x / a.parts;
#endif
#if LJMD_SEG_OFF
    int tile = a.tile_base + ti;
    const bool gated = false;
#else
    int tile = a.tile_base + ti + (ti >= a.seg0 ? a.gap : 0);
    const bool gated = a.halo_flag && ti >= a.nint;
#endif
    // gated order: interior tiles [L, T - L) first, then the lower layer [0, L), then the upper
    // layer [T - L, T) -- whose launch index is its own tile index
#if !LJMD_SEG_OFF
    if (a.halo_flag) tile = ti < a.nint ? a.layer + ti : (ti - a.nint < a.layer ? ti - a.nint : ti);
    // boundary-first order: lower layer [0, L), upper layer [T - L, T), then the interior
    if (a.bfirst) tile = ti < a.layer ? ti : (ti < 2 * a.layer ? a.nint + ti : ti - a.layer);
#endif
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // one bulk copy per halo row (TMA engine), issued by warp 0, completion on an mbarrier
    __shared__ __align__(8) unsigned long long mbar;
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
#if LJMD_EARLY_TMA
    if (threadIdx.x == 0) {   // at entry, before any load: the fence then waits for nothing
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) __syncwarp();   // the lanes that issue the copies see the initialised barrier
#endif
    // captured steps: skip everything after an aborted rebuild, before any table of it is
    // read (the flag is written only by rebuild kernels, never by a force launch)
    if (a.ctl && a.ctl->abort) return;
    const TileGeo T = tile_geo(a.g, tile);
    const int tt0 = a.obegin[a.tile_oc0[tile]];
    const int mt = a.obegin[a.tile_oc0[tile + 1]] - tt0;
    // shares in multiples of 16 particles: a particle's thread keeps its residue mod 16 (the
    // bank-aware list order is relative to it)
    const int per = ((mt + a.parts - 1) / a.parts + 15) & ~15;
    const int qb = min(part * per, mt);
    const int t0 = tt0 + qb;
    const int m = min(qb + per, mt) - qb;
    const bool has = (int)threadIdx.x < m;
    FPart P;
    // halo rows of this tile: lane r holds (begin, offset, length) of row r -- tables of the
    // rebuild, read before waiting for the previous launch
    const int rb = lane < T.R ? a.tr.begin[tile * kRowsMax + lane] : 0;
    const int ro = lane <= T.R ? a.tr.off[tile * (kRowsMax + 1) + lane] : 0;
    const int rl = lane < T.R ? a.tr.len[tile * kRowsMax + lane] : 0;
    const int total = __shfl_sync(0xffffffffu, ro, T.R);
    double* sP = reinterpret_cast<double*>(smem);   // packed {x, y, z} per staged particle
    // list ring after the staging buffer (16-byte aligned)
    const unsigned ring = ((unsigned)__cvta_generic_to_shared(smem) + 24u * (unsigned)(total + 1) + 15u) & ~15u;
    const unsigned myring = ring + 16u * threadIdx.x;
    if (threadIdx.x == 0) {
#if !LJMD_EARLY_TMA
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
        sP[3 * total] = 1e30;   // sentinel (list padding): far away, contributes exactly 0
        sP[3 * total + 1] = 1e30;
        sP[3 * total + 2] = 1e30;
    }
#if LJMD_PDL
    // programmatic dependent launch: the next force launch may start its CTAs on SMs this
    // one frees, loading the list indices (not written by this kernel) before it waits for
    // the positions and velocities
    asm volatile("griddepcontrol.launch_dependents;");
#if LJMD_EARLY_TMA
    // the halo copies first: they need only the row tables, so warp 0 waits for the previous
    // launch and issues them before any per-particle load (measured: the per-particle load
    // chain -- tile tables, slot / count / first list block -- held the copies back ~4 us)
    if (warp == 0) {
#if LJMD_PHASES
        if (lane == 0) ph[6] = gtimer() + 0ull * (unsigned long long)(rb + rl + ro);   // row tables in
#endif
        asm volatile("griddepcontrol.wait;" ::: "memory");
#if LJMD_PHASES
        if (lane == 0) ph[7] = gtimer();   // the previous launch is complete
#endif
        issue_halo(a, T, rb, ro, rl, sP, mb, lane);
#if LJMD_PHASES
        if (lane == 0) ph[5] = gtimer();   // the copies are issued
#endif
    }
#endif
    int li = 0;
    if (has) {
        const int t = t0 + threadIdx.x;
        P.t = t;
        P.si = a.own_slot[t];
        P.cnt = a.ncount[t];
#if LJMD_EARLY_TMA
        P.nb0 = a.nbr[t];       // unconditional (a count of 0 never reads it)
        li = a.own_li[t];       // x_i from the staged halo (no dependent global load)
#else
        P.nb0 = P.cnt > 0 ? a.nbr[t] : make_uint4(0u, 0u, 0u, 0u);
#endif
        ring_start(a, P, myring);   // the list is not written by the force kernel
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
#if LJMD_HALO_GATE
    if (warp == 0 && gated) {   // boundary tile: wait until this step's halo has landed
        if (lane == 0) {
            unsigned v = 0u;
            long long spins = 0;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.halo_flag) : "memory");
                if ((int)(v - a.halo_seq) >= 0) break;
                if (++spins > (1ll << 26)) {   // ~10 s: report instead of hanging the device
                    atomicOr(&a.fl->halo_timeout, 1);
                    break;
                }
                __nanosleep(128);
            }
            // the staging below reads the received planes through the async (TMA) proxy
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
    }
#else
    (void)gated;
#endif
#if !(LJMD_PDL && LJMD_EARLY_TMA)
    if (warp == 0) issue_halo(a, T, rb, ro, rl, sP, mb, lane);   // as soon as positions may be read
#endif
#if LJMD_PDL && !LJMD_EARLY_TMA
    if (has) P.xi = ld256(a.x + P.si);
#if LJMD_VPREF2
    if (has && (MODE & 3) != kStore) {   // the epilogue's velocities, into L2 ahead of time
        asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(a.vx + P.t) : "memory");
        asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(a.vy + P.t) : "memory");
        asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(a.vz + P.t) : "memory");
    }
#endif
#elif !LJMD_PDL
    if (has) {
        P = fpart_load(a, t0 + threadIdx.x);
        ring_start(a, P, myring);
    }
#endif
    __syncthreads();   // the barrier's initialisation and the sentinel are visible
    {
        unsigned done = 0u;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(mb) : "memory");
    }
#if LJMD_PHASES
    if (threadIdx.x == 0) ph[1] = gtimer();
#endif
#if LJMD_PDL && LJMD_EARLY_TMA
    if (has) {   // the owned particle's staged position (the same value as x[si])
        const double* q = sP + 3 * li;
        P.xi = make_double4(q[0], q[1], q[2], 0.0);
    }
#endif

    const char* sPb = reinterpret_cast<const char*>(sP);
    double epart = 0.0, ke = 0.0;
    unsigned long long dbits = 0ull;
    if (has) force_particle<ENERGY, MODE, CHECK>(a, P, sPb, epart, ke, dbits, myring, php);
    for (int q = threadIdx.x + kForceThreads; q < m; q += kForceThreads) {   // dense tiles only
        const FPart Q = fpart_load(a, t0 + q);
        ring_start(a, Q, myring);
        force_particle<ENERGY, MODE, CHECK>(a, Q, sPb, epart, ke, dbits, myring, php);
    }
#if LJMD_PHASES
    __syncwarp();
    if ((threadIdx.x & 31) == 0) atomicMax(&ph[4], gtimer());
#endif
    if (CHECK) block_atomic_max(dbits, &a.fl->maxdisp2);
    if (ENERGY) {
        const double pe = block_sum<kForceThreads>(epart, sh);
        const double k2 = block_sum<kForceThreads>(ke, sh);
        if (threadIdx.x == 0) {
            a.pe_part[tile * a.parts + part] = pe;
            a.ke_part[tile * a.parts + part] = k2;
        }
    }
#if LJMD_PHASES
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < 16384) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        unsigned long long* o = ljmd_phase_buf + 10 * (size_t)blockIdx.x;
        o[8] = ph[6] - ph[0];
        o[9] = ph[7] - ph[0];
        o[0] = ph[0]; o[1] = ph[1]; o[2] = ph[2]; o[3] = ph[3]; o[4] = ph[4]; o[5] = gtimer();
        o[6] = smid | ((unsigned long long)total << 32); o[7] = (unsigned long long)m | ((ph[5] - ph[0]) << 32);
    }
#endif
#if !LJMD_SEG_OFF
    if (a.bfirst && ti < 2 * a.layer) {   // this CTA's outgoing halo copies are written
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(a.bdone, 1u);
    }
#endif
}


// opening half of a step() call: v += h F ; x += dt v  (in place, owned slots)
// The pre-drift position is also written to the other buffer's owned slot (xprev), so that
// at the top of every step the other buffer holds x(s-1) (the fused force epilogue keeps
// that invariant on the following steps): the dangerous-build test of the next rebuild
// reads it.
template <bool CHECK>
__global__ void k_kick_drift(int n_own, double4* __restrict__ x, const int* __restrict__ own_slot,
                             double* __restrict__ vx, double* __restrict__ vy, double* __restrict__ vz,
                             const double* __restrict__ fx, const double* __restrict__ fy,
                             const double* __restrict__ fz, double h, double dt,
                             const double4* __restrict__ xbuild, DevFlags* fl, Images im, Geo g,
                             double* __restrict__ xp, double4* __restrict__ xprev, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured call behind an aborted one (k_call_begin)
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long bits = 0ull;
    if (t < n_own) {
        int si = own_slot[t];
        double4 p = x[si];
        xprev[si] = p;
        double a = __dadd_rn(vx[t], __dmul_rn(h, fx[t]));
        double b = __dadd_rn(vy[t], __dmul_rn(h, fy[t]));
        double c = __dadd_rn(vz[t], __dmul_rn(h, fz[t]));
        p.x = __dadd_rn(p.x, __dmul_rn(dt, a));
        p.y = __dadd_rn(p.y, __dmul_rn(dt, b));
        p.z = __dadd_rn(p.z, __dmul_rn(dt, c));
        x[si] = p;
        st_packed(xp, si, p);
        write_images(im, t, g, x, xp, p);
        vx[t] = a; vy[t] = b; vz[t] = c;
        if (CHECK) {
            double4 q = xbuild[t];
            bits = __double_as_longlong(r2_canon(p.x - q.x, p.y - q.y, p.z - q.z));
        }
    }
    if (CHECK) block_atomic_max(bits, &fl->maxdisp2);
}

// ---------------------------------------------------------------- rebuild certification
// Dangerous builds (Eq. eqn:extended_cutoff; reading R7): the skin
// argument certifies a list built at x_build for positions x as long as
// 2 max_i |x_i - x_i(build)| <= delta (no pair can then have closed in from beyond rbar_c to
// inside rc).  At each rebuild the displacement of the LAST step the old list served,
// x(s-1) (the other position buffer, owned slots in the old layout), is reduced here; a
// rebuild whose 4 max|dx|^2 > delta^2 is counted as dangerous (the fixed-Ns policy of the
// paper's benchmark may have served uncertified steps; the displacement-checked policy
// never does).
__global__ void k_maxdisp(int n_own, const double4* __restrict__ xprev, const int* __restrict__ own_slot,
                          const double4* __restrict__ xbuild, unsigned long long* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long bits = 0ull;
    if (t < n_own) {
        const double4 p = xprev[own_slot[t]];
        const double4 q = xbuild[t];
        bits = __double_as_longlong(r2_canon(p.x - q.x, p.y - q.y, p.z - q.z));
    }
    block_atomic_max(bits, out);
}

struct DevStats {                  // persistent device counters (not reset by k_reset_flags)
    unsigned long long dangerous;  // rebuilds with 4 max|x(s-1) - x_build|^2 > delta^2
    unsigned long long disp_bits;  // scratch: max |x(s-1) - x_build|^2 of the current rebuild
    double max_disp2;              // largest such value seen since init / set_state
};

// captured rebuilds: k_maxdisp also clears the owned-cell counts for the binning (one
// memset node fewer)
// record_step > 0 (the fixed schedule's captured rebuild): also k_decide's record of the
// rebuild step (one node fewer)
__global__ void k_maxdisp_z(int n_own, const double4* __restrict__ xprev, const int* __restrict__ own_slot,
                            const double4* __restrict__ xbuild, unsigned long long* __restrict__ out,
                            int* __restrict__ ocount, int n_ocell, DevCtl* ctl, DevFlags* fl, int* rstep,
                            int record_step) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (record_step > 0 && t == 0) {
        ctl->step = record_step;
        ctl->since = 0;
        fl->maxdisp2 = 0ull;
        rstep[ctl->nreb++] = record_step;
    }
    for (int i = t; i < n_ocell; i += gridDim.x * blockDim.x) ocount[i] = 0;
    unsigned long long bits = 0ull;
    if (t < n_own) {
        const double4 p = xprev[own_slot[t]];
        const double4 q = xbuild[t];
        bits = __double_as_longlong(r2_canon(p.x - q.x, p.y - q.y, p.z - q.z));
    }
    block_atomic_max(bits, out);
}

__global__ void k_dangerous(DevStats* st, double delta2) {
    const double m2 = __longlong_as_double((long long)st->disp_bits);
    if (4.0 * m2 > delta2) st->dangerous += 1ull;
    if (m2 > st->max_disp2) st->max_disp2 = m2;
    st->disp_bits = 0ull;
}

// captured rebuilds: k_dangerous and k_reset_flags(keep_errors = 1) in one launch
__global__ void k_dangerous_reset(DevStats* st, double delta2, DevFlags* fl, const DevCtl* ctl) {
    if (ctl && ctl->abort) return;   // captured rebuild after a failed capacity check
    const double m2 = __longlong_as_double((long long)st->disp_bits);
    if (4.0 * m2 > delta2) st->dangerous += 1ull;
    if (m2 > st->max_disp2) st->max_disp2 = m2;
    st->disp_bits = 0ull;
    DevFlags f;
    memset(&f, 0, sizeof f);
    f.migrate_gid = fl->migrate_gid;
    f.nonfinite_gid = fl->nonfinite_gid;
    f.overlap_pair = fl->overlap_pair;
    f.val_error = fl->val_error;
    *fl = f;
}

// Validation mode (ljmd_options.validate; single rank): for every step, the number of
// ordered pairs the list misses -- pairs with canonical r^2 < rc^2 at the step's positions
// (minimum image, reading R9) that are not served by the Verlet list -- counted per particle
// as  #{j : r_ij^2 < rc^2} (fresh cell search) - #{list entries with r^2 < rc^2}.  An
// independent cell binning of the current positions (cells of the engine's grid, width >=
// rbar_c >= rc) provides the search; it never touches the engine's own layout.
__global__ void k_val_bin(int n_own, const double4* __restrict__ x, const int* __restrict__ own_slot, Geo g,
                          int* __restrict__ vcount, int* __restrict__ vcell, int* __restrict__ vrank) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    const double4 p = x[own_slot[t]];
    const double q[3] = {wrap_coord(p.x, g.L[0]), wrap_coord(p.y, g.L[1]), wrap_coord(p.z, g.L[2])};
    int c[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        int k = (int)floor(__ddiv_rn(q[d], g.w[d]));
        c[d] = k < 0 ? 0 : (k > g.nc[d] - 1 ? g.nc[d] - 1 : k);
    }
    const int cell = (c[2] * g.nc[1] + c[1]) * g.nc[0] + c[0];
    vcell[t] = cell;
    vrank[t] = atomicAdd(&vcount[cell], 1);
}

__global__ void k_val_scatter(int n_own, const double4* __restrict__ x, const int* __restrict__ own_slot,
                              const int* __restrict__ vcell, const int* __restrict__ vrank,
                              const int* __restrict__ vbegin, double4* __restrict__ vpos) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    double4 p = x[own_slot[t]];
    p.w = __longlong_as_double((long long)t);
    vpos[vbegin[vcell[t]] + vrank[t]] = p;
}

// minimum-image displacement x_i - (x_j + s L) with s from d0 = x_i - x_j (reading R9, the
// oracle's O2); the list side uses the stored image x_j + s L, the same rounding
__device__ __forceinline__ double mi_d(double xi, double xj, double L) {
    const double d0 = xi - xj;
    const double s = d0 > 0.5 * L ? 1.0 : (d0 < -0.5 * L ? -1.0 : 0.0);
    return __dsub_rn(xi, __dadd_rn(xj, __dmul_rn(s, L)));
}

struct ValArgs {
    Geo g;
    const double4* x;        // current positions (slot space)
    const int* own_slot;
    const int* vcell;
    const int* vbegin;
    const double4* vpos;     // positions sorted by validation cell, w = owned index
    const unsigned short* nbr;   // blocked-8 list (build or bank-aware order: a set)
    const int* ncount;
    const int* ocell_of;
    TileRows tr;
    int n_own, n_pad;
    double rc2;
    int* vhist;              // [step][2]: particles with missed pairs, missed ordered pairs
    int vslot;               // row of vhist for this step
    DevFlags* fl;
};

__global__ void __launch_bounds__(256) k_val_count(ValArgs a) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    int miss = 0;
    if (t < a.n_own) {
        const Geo& g = a.g;
        const double4 xi = a.x[a.own_slot[t]];
        const int cell = a.vcell[t];
        const int cx = cell % g.nc[0], cy = (cell / g.nc[0]) % g.nc[1], cz = cell / (g.nc[0] * g.nc[1]);
        int truth = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int ex = (cx + dx + g.nc[0]) % g.nc[0], ey = (cy + dy + g.nc[1]) % g.nc[1],
                              ez = (cz + dz + g.nc[2]) % g.nc[2];
                    const int c2 = (ez * g.nc[1] + ey) * g.nc[0] + ex;
                    for (int k = a.vbegin[c2]; k < a.vbegin[c2 + 1]; ++k) {
                        const double4 xj = a.vpos[k];
                        if ((int)__double_as_longlong(xj.w) == t) continue;
                        const double r2 = r2_canon(mi_d(xi.x, xj.x, g.L[0]), mi_d(xi.y, xj.y, g.L[1]),
                                                   mi_d(xi.z, xj.z, g.L[2]));
                        truth += r2 < a.rc2;
                    }
                }
        // the list side: entries resolved to slots through the tile's halo rows
        int cx2, cy2, cz2;
        lex_xyz(g, g.lex_of_oc[a.ocell_of[t]], cx2, cy2, cz2);
        const int tile = tile_of_cell(g, cx2, cy2, cz2);
        const int* rbeg = a.tr.begin + tile * kRowsMax;
        const int* roff = a.tr.off + tile * (kRowsMax + 1);
        const int n = a.ncount[t];
        int listed = 0;
        for (int k = 0; k < n; ++k) {
            const int l = a.nbr[((size_t)(k >> 3) * a.n_pad + t) * 8 + (k & 7)];
            int r = 0;
            while (l >= roff[r + 1]) ++r;
            const double4 xj = a.x[rbeg[r] + (l - roff[r])];
            listed += r2_canon(xi.x - xj.x, xi.y - xj.y, xi.z - xj.z) < a.rc2;
        }
        miss = truth - listed;
        if (miss < 0) atomicOr(&a.fl->val_error, 1);   // impossible: a listed pair the search missed
    }
    const int vs = a.vslot;
    int np = miss > 0 ? 1 : 0, nm = miss > 0 ? miss : 0;
    for (int o = 16; o > 0; o >>= 1) {
        np += __shfl_down_sync(0xffffffffu, np, o);
        nm += __shfl_down_sync(0xffffffffu, nm, o);
    }
    if ((threadIdx.x & 31) == 0 && (np || nm)) {
        atomicAdd(&a.vhist[2 * vs], np);
        atomicAdd(&a.vhist[2 * vs + 1], nm);
    }
}

// fixed-order final reduction of the per-block partials -> out[0] = PE, out[1] = KE
// ctl != null (captured steps): out is the history base, the sample index comes from ctl
__global__ void k_finalize_energy(const double* __restrict__ pe_part, const double* __restrict__ ke_part,
                                  int nb, double* __restrict__ out, DevCtl* ctl) {
    __shared__ double sh[32];
    if (ctl) {
        if (ctl->abort) return;
        out += 2 * ctl->nsamp;
    }
    double p = 0.0, k = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        p += pe_part[i];
        k += ke_part[i];
    }
    // blockDim = 1024 fixed
    double ps = block_sum<1024>(p, sh);
    double ks = block_sum<1024>(k, sh);
    if (threadIdx.x == 0) {
        out[0] = ps;
        out[1] = ks;
        if (ctl) ctl->nsamp += 1;
    }
}

// readback: owned-order rows of `width` doubles into caller (gid) order
__global__ void k_rows_to_gid(int n, int width, const int* __restrict__ gid, const double* __restrict__ src,
                              double* __restrict__ dst) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)n * width) return;
    const int t = (int)(idx / width), k = (int)(idx % width);
    dst[(size_t)gid[t] * width + k] = src[idx];
}

// readback helpers: compact owned-space copies
__global__ void k_gather_pos(int n_own, const double4* __restrict__ x, const int* __restrict__ own_slot,
                             double* __restrict__ out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    double4 p = x[own_slot[t]];
    out[3 * t] = p.x;
    out[3 * t + 1] = p.y;
    out[3 * t + 2] = p.z;
}

__global__ void k_gather_soa(int n_own, const double* __restrict__ a, const double* __restrict__ b,
                             const double* __restrict__ c, double* __restrict__ out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    out[3 * t] = a[t];
    out[3 * t + 1] = b[t];
    out[3 * t + 2] = c[t];
}

__global__ void k_list_gids(int n_own, int n_pad, Geo g, const unsigned short* __restrict__ nbr,   // blocked-8
                            const int* __restrict__ ncount, const int* __restrict__ ocell_of, TileRows tr,
                            const int* __restrict__ slot_gid, const long long* __restrict__ off,
                            long long* __restrict__ out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    int cx, cy, cz;
    lex_xyz(g, g.lex_of_oc[ocell_of[t]], cx, cy, cz);
    const int tile = tile_of_cell(g, cx, cy, cz);
    const int* rbeg = tr.begin + tile * kRowsMax;
    const int* roff = tr.off + tile * (kRowsMax + 1);
    int c = ncount[t];
    long long o = off[t];
    for (int k = 0; k < c; ++k) {
        const int l = nbr[((size_t)(k >> 3) * n_pad + t) * 8 + (k & 7)];
        int r = 0;
        while (l >= roff[r + 1]) ++r;
        out[o + k] = slot_gid[rbeg[r] + (l - roff[r])];
    }
}

}  // namespace ljmd

namespace ljmd {
// FP64 pipe peak probe (roofline denominator for the ALU-bound force kernel): 8 independent
// DFMA chains per thread, enough warps to saturate every SMSP's FP64 unit.
__global__ void __launch_bounds__(256) k_fp64_peak(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
    double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[blockIdx.x] = s;   // keep the chains alive
}
}  // namespace ljmd

namespace ljmd {
// ----------------------------------------------------------------------------- bond order
// Steinhardt bond-order parameters (Sec. 4.1, Eqs. eqn:qellm / eqn:Qell)
// as a second Local Particle Pair Loop over the engine's lists (Alg. alg:sph_I), then the
// particle loop Q_l = sqrt(4 pi/(2l+1) sum_m |q_lm|^2) (Alg. alg:sph_II).  Neighbours: the
// list entries with canonical r^2 < rcut^2 (rcut <= rc keeps the Verlet list complete).
// Y_l^m(r_hat) = K_lm Pbar_l^m(z) (x + i y)^m with Pbar_l^m = P_l^m / (1 - z^2)^{m/2}
// (three-term recurrence in l), m >= 0 only: |q_{l,-m}| = |q_{l,m}|; the Condon-Shortley
// sign is dropped (Q_l depends on |q_lm| only).
constexpr int kBoaMaxL = 12;
constexpr int kBoaMaxSel = 160;   // > K: every list entry fits

struct BoaArgs {
    Geo g;
    const double4* x;
    const int* own_slot;
    const uint4* nbr;
    const int* ncount;
    const int* obegin;
    const int* tile_oc0;
    TileRows tr;
    double* Q;        // [n_own]
    double* nnb;      // [n_own]
    int n_own, n_pad;
    double rcut2;
    double K[kBoaMaxL + 1];   // K_lm = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!)
};

template <int L>
__global__ void __launch_bounds__(kForceThreads) k_boa(BoaArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const TileGeo T = tile_geo(a.g, tile);
    const int t0 = a.obegin[a.tile_oc0[tile]];
    const int m_own = a.obegin[a.tile_oc0[tile + 1]] - t0;
    const int rb = lane < T.R ? a.tr.begin[tile * kRowsMax + lane] : 0;
    const int ro = lane <= T.R ? a.tr.off[tile * (kRowsMax + 1) + lane] : 0;
    const int total = __shfl_sync(0xffffffffu, ro, T.R);
    double* sP = reinterpret_cast<double*>(smem);
    for (int r = warp; r < T.R; r += kForceThreads / 32) {
        const int b0 = __shfl_sync(0xffffffffu, rb, r);
        const int o0 = __shfl_sync(0xffffffffu, ro, r);
        const int len = a.tr.len[tile * kRowsMax + r];
        for (int k = lane; k < len; k += 32) {
            const double4 p = ld256(a.x + b0 + k);
            sP[3 * (o0 + k)] = p.x;
            sP[3 * (o0 + k) + 1] = p.y;
            sP[3 * (o0 + k) + 2] = p.z;
        }
    }
    if (threadIdx.x == 0) {
        sP[3 * total] = 1e30;
        sP[3 * total + 1] = 1e30;
        sP[3 * total + 2] = 1e30;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m_own; q += kForceThreads) {
        const int t = t0 + q;
        const double4 xi = a.x[a.own_slot[t]];
        const int cnt = a.ncount[t];
        double re[L + 1], im[L + 1];
#pragma unroll
        for (int m = 0; m <= L; ++m) re[m] = im[m] = 0.0;
        // pass 1: the list entries inside rcut (compacted, so the spherical-harmonic work
        // below is not executed by the whole warp for every list entry)
        unsigned short sel[kBoaMaxSel];
        int nu = 0;
        for (int k = 0; k < cnt; ++k) {
            const uint4 w = a.nbr[(size_t)(k >> 3) * a.n_pad + t];
            const unsigned ww = (k & 7) < 2 ? w.x : (k & 7) < 4 ? w.y : (k & 7) < 6 ? w.z : w.w;
            const unsigned l = (k & 1) ? (ww >> 16) : (ww & 0xffffu);
            const double* pj = sP + 3 * l;
            const double r2 = r2_canon(xi.x - pj[0], xi.y - pj[1], xi.z - pj[2]);
            if (r2 < a.rcut2 && nu < kBoaMaxSel) sel[nu++] = (unsigned short)l;
        }
        for (int s = 0; s < nu; ++s) {
            const double* pj = sP + 3 * sel[s];
            const double dx = xi.x - pj[0], dy = xi.y - pj[1], dz = xi.z - pj[2];
            const double r2 = r2_canon(dx, dy, dz);
            const double ir = rsqrt(r2);
            const double ux = dx * ir, uy = dy * ir, z = dz * ir;       // r_hat_ij
            double cr = 1.0, ci = 0.0;                                   // (x + i y)^m
            double pmm = 1.0;                                            // Pbar_m^m = (2m-1)!!
#pragma unroll
            for (int m = 0; m <= L; ++m) {
                double p0 = pmm, p1 = 0.0;
                if (m < L) {
                    p1 = (2 * m + 1) * z * pmm;                           // Pbar_{m+1}^m
                    double a0 = p0, a1 = p1;
#pragma unroll
                    for (int ll = m + 2; ll <= L; ++ll) {
                        // (ll - m) is a compile-time constant: multiply by its reciprocal
                        const double an = ((2 * ll - 1) * z * a1 - (ll + m - 1) * a0) * (1.0 / (ll - m));
                        a0 = a1;
                        a1 = an;
                    }
                    p0 = a1;                                              // Pbar_L^m
                }
                const double y = a.K[m] * p0;
                re[m] += y * cr;
                im[m] += y * ci;
                const double nr = cr * ux - ci * uy, ni = cr * uy + ci * ux;
                cr = nr;
                ci = ni;
                pmm *= (2 * m + 1);
            }
        }
        double acc = 0.0;
        if (nu > 0) {
            const double inv = 1.0 / nu;
#pragma unroll
            for (int m = 0; m <= L; ++m) {
                const double qr = re[m] * inv, qi = im[m] * inv;
                acc += (m == 0 ? 1.0 : 2.0) * (qr * qr + qi * qi);
            }
        }
        a.Q[t] = sqrt(4.0 * 3.14159265358979323846 / (2 * L + 1) * acc);
        a.nnb[t] = (double)nu;
    }
}
}  // namespace ljmd

namespace ljmd {
// ----------------------------------------------------------------------------- common neighbours
// Common-neighbour analysis (Sec. 4.2, Algs. alg:cna_I-III and alg:max_cluster_size,
// PAPER.md:522-653, 1151-1174) on the engine's lists, single rank.  Pass 1 (alg:cna_I):
// the bonded neighbours of every particle (canonical r^2 < rcut^2) as a gid-sorted table.
// Pass 2 (alg:cna_II/III): for each bond (i, j) the common neighbours C = N(i) & N(j), the
// bonds among them (the indirect bonds of alg:cna_II restricted to C), and the edges of the
// largest connected component (alg:max_cluster_size) via bitmask adjacency.
constexpr int kCnaMax = 24;   // bonded neighbours per particle (12 fcc/hcp, 14 bcc)

struct CnaArgs {
    Geo g;
    const double4* x;
    const int* own_slot;
    const uint4* nbr;
    const int* ncount;
    const int* ocell_of;
    const int* slot_gid;
    const int* gid;      // owned t -> gid
    TileRows tr;
    int* tab;            // [n_own][kCnaMax] sorted neighbour gids
    int* tcnt;           // [n_own]
    const int* tmap;     // gid -> owned t
    int* trip;           // [n_own][kCnaMax] packed n_nb | n_b << 8 | n_lcb << 16
    int* cls;            // [n_own] 0 other, 1 fcc, 2 hcp, 3 bcc
    DevFlags* fl;
    int n_own, n_pad;
    double rcut2;
};

__global__ void k_cna_bonds(CnaArgs a) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n_own) return;
    int cx, cy, cz;
    lex_xyz(a.g, a.g.lex_of_oc[a.ocell_of[t]], cx, cy, cz);
    const int tile = tile_of_cell(a.g, cx, cy, cz);
    const int* rbeg = a.tr.begin + tile * kRowsMax;
    const int* roff = a.tr.off + tile * (kRowsMax + 1);
    const double4 xi = a.x[a.own_slot[t]];
    int nb[kCnaMax];
    int n = 0;
    const int cnt = a.ncount[t];
    const unsigned short* lst = reinterpret_cast<const unsigned short*>(a.nbr);
    for (int k = 0; k < cnt; ++k) {
        const int l = lst[((size_t)(k >> 3) * a.n_pad + t) * 8 + (k & 7)];
        int r = 0;
        while (l >= roff[r + 1]) ++r;
        const int s = rbeg[r] + (l - roff[r]);
        const double4 xj = a.x[s];
        if (!(r2_canon(xi.x - xj.x, xi.y - xj.y, xi.z - xj.z) < a.rcut2)) continue;   // alg:cna_I
        const int gj = a.slot_gid[s];
        if (n == kCnaMax) {
            a.fl->overflow = 1;
            break;
        }
        int p = n++;
        while (p > 0 && nb[p - 1] > gj) {   // insertion: ascending gid
            nb[p] = nb[p - 1];
            --p;
        }
        nb[p] = gj;
    }
    for (int k = 0; k < n; ++k) a.tab[(size_t)t * kCnaMax + k] = nb[k];
    a.tcnt[t] = n;
}

__device__ __forceinline__ bool cna_has(const int* row, int n, int g) {
    for (int k = 0; k < n; ++k)
        if (row[k] == g) return true;
    return false;
}

__global__ void k_cna_triplets(CnaArgs a) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n_own) return;
    const int* Ni = a.tab + (size_t)t * kCnaMax;
    const int ni = a.tcnt[t];
    int c421 = 0, c422 = 0, c666 = 0, c444 = 0;
    for (int k = 0; k < ni; ++k) {
        const int tj = a.tmap[Ni[k]];
        const int* Nj = a.tab + (size_t)tj * kCnaMax;
        const int nj = a.tcnt[tj];
        // common neighbours (both rows ascending): two-pointer intersection
        int C[kCnaMax];
        int nc = 0;
        for (int p = 0, q = 0; p < ni && q < nj;) {
            if (Ni[p] < Nj[q]) ++p;
            else if (Ni[p] > Nj[q]) ++q;
            else { C[nc++] = Ni[p]; ++p; ++q; }
        }
        // bonds among the common neighbours (alg:cna_II / III), adjacency as bitmasks
        unsigned adj[kCnaMax];
        int nb = 0;
        for (int u = 0; u < nc; ++u) adj[u] = 0u;
        for (int u = 0; u < nc; ++u) {
            const int tu = a.tmap[C[u]];
            const int* Nu = a.tab + (size_t)tu * kCnaMax;
            const int nu = a.tcnt[tu];
            for (int w = u + 1; w < nc; ++w)
                if (cna_has(Nu, nu, C[w])) {
                    adj[u] |= 1u << w;
                    adj[w] |= 1u << u;
                    ++nb;
                }
        }
        // largest cluster, counted in edges (alg:max_cluster_size)
        unsigned left = nc >= 32 ? 0xffffffffu : ((1u << nc) - 1u);
        int lcb = 0;
        while (left) {
            const int v = __ffs(left) - 1;
            unsigned comp = 1u << v, frontier = comp;
            while (frontier) {
                const int u = __ffs(frontier) - 1;
                frontier &= frontier - 1;
                const unsigned nw = adj[u] & ~comp;
                comp |= nw;
                frontier |= nw;
            }
            int e = 0;
            for (unsigned m = comp; m; m &= m - 1) e += __popc(adj[__ffs(m) - 1] & comp);
            lcb = max(lcb, e / 2);
            left &= ~comp;
        }
        a.trip[(size_t)t * kCnaMax + k] = nc | (nb << 8) | (lcb << 16);
        c421 += (nc == 4 && nb == 2 && lcb == 1);
        c422 += (nc == 4 && nb == 2 && lcb == 2);
        c666 += (nc == 6 && nb == 6 && lcb == 6);
        c444 += (nc == 4 && nb == 4 && lcb == 4);
    }
    int cl = 0;
    if (ni == 12 && c421 == 12) cl = 1;
    else if (ni == 12 && c421 == 6 && c422 == 6) cl = 2;
    else if (ni == 14 && c666 == 8 && c444 == 6) cl = 3;
    a.cls[t] = cl;
}

__global__ void k_cna_tmap(int n_own, const int* __restrict__ gid, int* __restrict__ tmap) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_own) tmap[gid[t]] = t;
}
}  // namespace ljmd

namespace ljmd {
// ----------------------------------------------------------------------------- Newton-3 half list
// SURVEY §8(f) NEXT-1 ("a factor of two" from Newton's third law, which the paper
// does not use).  Each unordered pair is kept once, at the particle with the smaller gid (a
// periodic image carries its source's gid, so the pair with an image is also kept once); the
// force kernel adds f_ij to i in registers and the reaction -f_ij to j's owner with fp64
// global reductions (RED.ADD.F64 in L2), then a separate velocity-Verlet kernel runs on the
// completed F.  Single rank only (a reverse halo for the ghosts of other ranks is not built).

// slot -> owned index of its particle (ghost slots: the source particle), single rank
__global__ void k_slot_owner(int n_slots, const int* __restrict__ slot_gid, const int* __restrict__ tmap,
                             int* __restrict__ slot_t) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n_slots) slot_t[s] = tmap[slot_gid[s]];
}

// half list: the entries of the full build-order list whose gid is larger than the particle's
__global__ void k_list_half(int n_own, int n_pad, Geo g, const uint4* __restrict__ in, const int* __restrict__ ncount,
                            const int* __restrict__ ocell_of, TileRows tr, const int* __restrict__ slot_gid,
                            const int* __restrict__ gid, uint4* __restrict__ out, int* __restrict__ ncount_h) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    int cx, cy, cz;
    lex_xyz(g, g.lex_of_oc[ocell_of[t]], cx, cy, cz);
    const int tile = tile_of_cell(g, cx, cy, cz);
    const int* rbeg = tr.begin + tile * kRowsMax;
    const int* roff = tr.off + tile * (kRowsMax + 1);
    const int gi = gid[t];
    const int n = ncount[t];
    const unsigned short* lst = reinterpret_cast<const unsigned short*>(in);
    uint4* outb = out + t;
    unsigned w0 = 0u, w1 = 0u, w2 = 0u, w3 = 0u;
    int k = 0;
    for (int e = 0; e < n; ++e) {
        const int l = lst[((size_t)(e >> 3) * n_pad + t) * 8 + (e & 7)];
        int r = 0;
        while (l >= roff[r + 1]) ++r;
        if (slot_gid[rbeg[r] + (l - roff[r])] <= gi) continue;
        w0 = __funnelshift_r(w0, w1, 16);
        w1 = __funnelshift_r(w1, w2, 16);
        w2 = __funnelshift_r(w2, w3, 16);
        w3 = __funnelshift_r(w3, (unsigned)l, 16);
        if ((k & 7) == 7) {
            *outb = make_uint4(w0, w1, w2, w3);
            outb += n_pad;
        }
        ++k;
    }
    if (k & 7) {
        const unsigned sen = (unsigned)roff[tile_geo(g, tile).R];
        for (int e = k & 7; e < 8; ++e) {
            w0 = __funnelshift_r(w0, w1, 16);
            w1 = __funnelshift_r(w1, w2, 16);
            w2 = __funnelshift_r(w2, w3, 16);
            w3 = __funnelshift_r(w3, sen, 16);
        }
        *outb = make_uint4(w0, w1, w2, w3);
    }
    ncount_h[t] = k;
}

struct HalfArgs {
    Geo g;
    const double4* x;
    const int* own_slot;
    const uint4* nbr;       // half list, blocked like the full one
    const int* ncount;
    const int* obegin;
    const int* tile_oc0;
    const int* slot_t;
    TileRows tr;
    double* fx; double* fy; double* fz;
    double* e;
    double* pe_part;
    int n_own, n_pad;
    double rc2, c12, nc6, a12, na6, a0;
};

// F and e must be zero before the launch (they are accumulated from both ends of a pair).
template <bool ENERGY>
__global__ void __launch_bounds__(kForceThreads, 3) k_force_half(HalfArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double sh[kForceThreads / 32];
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const TileGeo T = tile_geo(a.g, tile);
    const int t0 = a.obegin[a.tile_oc0[tile]];
    const int m = a.obegin[a.tile_oc0[tile + 1]] - t0;
    const int rb = lane < T.R ? a.tr.begin[tile * kRowsMax + lane] : 0;
    const int ro = lane <= T.R ? a.tr.off[tile * (kRowsMax + 1) + lane] : 0;
    const int total = __shfl_sync(0xffffffffu, ro, T.R);
    double* sP = reinterpret_cast<double*>(smem);                 // packed {x, y, z}
    int* sO = reinterpret_cast<int*>(sP + 3 * (total + 1));         // owner of each staged particle
    for (int r = warp; r < T.R; r += kForceThreads / 32) {
        const int b0 = __shfl_sync(0xffffffffu, rb, r);
        const int o0 = __shfl_sync(0xffffffffu, ro, r);
        const int len = a.tr.len[tile * kRowsMax + r];
        for (int k = lane; k < len; k += 32) {
            const double4 p = a.x[b0 + k];
            sP[3 * (o0 + k)] = p.x;
            sP[3 * (o0 + k) + 1] = p.y;
            sP[3 * (o0 + k) + 2] = p.z;
            sO[o0 + k] = a.slot_t[b0 + k];
        }
    }
    if (threadIdx.x == 0) {
        sP[3 * total] = 1e30;
        sP[3 * total + 1] = 1e30;
        sP[3 * total + 2] = 1e30;
        sO[total] = -1;
    }
    __syncthreads();
    double epart = 0.0;
    for (int q = threadIdx.x; q < m; q += kForceThreads) {
        const int t = t0 + q;
        const double4 xi = a.x[a.own_slot[t]];
        const int cnt = a.ncount[t];
        double fx = 0.0, fy = 0.0, fz = 0.0, u = 0.0;
        for (int b = 0; b < ((cnt + 7) >> 3); ++b) {
            const uint4 blk = a.nbr[(size_t)b * a.n_pad + t];
            const unsigned w4[4] = {blk.x, blk.y, blk.z, blk.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const unsigned l = (e & 1) ? (w4[e >> 1] >> 16) : (w4[e >> 1] & 0xffffu);
                const double* pj = sP + 3 * l;
                const double dx = xi.x - pj[0], dy = xi.y - pj[1], dz = xi.z - pj[2];
                const double r2 = r2_canon(dx, dy, dz);
                if (r2 < a.rc2) {
                    const double ir2 = rcp64(r2);
                    const double ir4 = ir2 * ir2;
                    const double ir6 = ir4 * ir2;
                    const double ir8 = ir4 * ir4;
                    const double gg = ir8 * fma(a.c12, ir6, a.nc6);
                    const double gx = gg * dx, gy = gg * dy, gz = gg * dz;
                    fx += gx; fy += gy; fz += gz;
                    const int tj = sO[l];
                    atomicAdd(a.fx + tj, -gx);
                    atomicAdd(a.fy + tj, -gy);
                    atomicAdd(a.fz + tj, -gz);
                    if (ENERGY) {
                        const double v = fma(fma(a.a12, ir6, a.na6), ir6, a.a0);
                        u += v;
                        atomicAdd(a.e + tj, 0.5 * v);
                    }
                }
            }
        }
        atomicAdd(a.fx + t, fx);
        atomicAdd(a.fy + t, fy);
        atomicAdd(a.fz + t, fz);
        if (ENERGY) {
            atomicAdd(a.e + t, 0.5 * u);
            epart += u;
        }
    }
    if (ENERGY) {
        const double pe = block_sum<kForceThreads>(epart, sh);
        if (threadIdx.x == 0) a.pe_part[blockIdx.x] = pe;
    }
}

// velocity Verlet on the completed F (Newton-3 path): [line 8: v += h F] [Andersen]
// [KE sample] [line 6 of the next step: v += h F; x' = x + dt v, displacement check].
// Grid = n_tiles blocks (grid-stride) so the KE partials line up with the PE partials.
struct VvArgs {
    int n_own;
    const double4* x;
    double4* x_next;
    const int* own_slot;
    double* vx; double* vy; double* vz;
    const double* fx; const double* fy; const double* fz;
    double* ke_part;
    const double4* xbuild;
    DevFlags* fl;
    const int* gid;
    double h, dt, half_m, nu_dt, sd;
    unsigned long long seed;
    long long step;
};

template <bool KICK2, bool ENERGY, bool KD, bool CHECK, bool THERMO>
__global__ void __launch_bounds__(256) k_vv(VvArgs a) {
    __shared__ double sh[8];
    double ke = 0.0;
    unsigned long long dbits = 0ull;
    for (int t = blockIdx.x * 256 + threadIdx.x; t < a.n_own; t += gridDim.x * 256) {
        double vx = a.vx[t], vy = a.vy[t], vz = a.vz[t];
        const double fx = a.fx[t], fy = a.fy[t], fz = a.fz[t];
        if (KICK2) {
            vx = __dadd_rn(vx, __dmul_rn(a.h, fx));
            vy = __dadd_rn(vy, __dmul_rn(a.h, fy));
            vz = __dadd_rn(vz, __dmul_rn(a.h, fz));
            if (THERMO) andersen(a.seed, a.step, a.nu_dt, a.sd, a.gid[t], vx, vy, vz);
        }
        if (ENERGY) ke += a.half_m * __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
        if (KD) {
            vx = __dadd_rn(vx, __dmul_rn(a.h, fx));
            vy = __dadd_rn(vy, __dmul_rn(a.h, fy));
            vz = __dadd_rn(vz, __dmul_rn(a.h, fz));
            const int si = a.own_slot[t];
            const double4 xi = a.x[si];
            const double4 xn = make_double4(__dadd_rn(xi.x, __dmul_rn(a.dt, vx)), __dadd_rn(xi.y, __dmul_rn(a.dt, vy)),
                                            __dadd_rn(xi.z, __dmul_rn(a.dt, vz)), 0.0);
            a.x_next[si] = xn;
            if (CHECK) {
                const double4 bb = a.xbuild[t];
                const unsigned long long d2 =
                    __double_as_longlong(r2_canon(xn.x - bb.x, xn.y - bb.y, xn.z - bb.z));
                dbits = d2 > dbits ? d2 : dbits;
            }
        }
        if (KICK2 || KD) {
            a.vx[t] = vx; a.vy[t] = vy; a.vz[t] = vz;
        }
    }
    if (CHECK) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_down_sync(0xffffffffu, dbits, o);
            dbits = ob > dbits ? ob : dbits;
        }
        if ((threadIdx.x & 31) == 0 && dbits) atomicMax(&a.fl->maxdisp2, dbits);
    }
    if (ENERGY) {
        const double k2 = block_sum<256>(ke, sh);
        if (threadIdx.x == 0) a.ke_part[blockIdx.x] = k2;
    }
}
}  // namespace ljmd
