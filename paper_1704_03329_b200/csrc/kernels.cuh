// kernels.cuh -- sm_100a kernels of the LJ PairLoop hot path (arXiv 1704.03329).
//
// Data layout in HBM:
//   slot space  : every particle image the list can reference -- owned particles and
//                 ghosts (periodic images / halo copies) -- sorted by EXTENDED cell
//                 (x fastest over ncx+2, then y over ncy+2, then z over nzl+2), within a
//                 cell by gid.  A 3-cell x-row of the 27-cell stencil is therefore one
//                 contiguous slot range.  Positions: double4 {x,y,z,0} (32 B, one sector,
//                 one 256-bit LDG per neighbour); fp32 mirror float4 for the list build.
//   owned space : owned particles t = 0..n_own-1 in owned-cell order (same order as their
//                 slots); v (SoA), F (SoA), gid, own_slot[t], e_i.
//   list        : ELL, column-major nbr[k * n_pad + t] (int32 slot), ncount[t].
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ljmd {

struct DevFlags {
    int max_nbr;                 // longest list at the last build
    int slots_needed;            // slot count required by the last binning
    int nonfinite_gid;           // smallest gid with a non-finite coordinate (INT_MAX: none)
    int overlap_gid;             // smallest gid i with a partner at r^2 == 0 (INT_MAX: none)
    int overlap_gid_j;
    int pad0;
    unsigned long long maxdisp2; // bits of max |x - x_build|^2 (non-negative double)
    unsigned long long total_nbr;
};

// --------------------------------------------------------------------------- helpers
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
// e = 1 - a y  (3 DFMA, error ~2^-64 before rounding).
__device__ __forceinline__ double rcp64(double a) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
    return fma(y, fma(e, e, e), y);
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
__global__ void k_load_rows(int n, const double* __restrict__ pos, const double* __restrict__ vel,
                            double4* __restrict__ x, double* __restrict__ vx, double* __restrict__ vy,
                            double* __restrict__ vz, int* __restrict__ gid, int* __restrict__ own_slot,
                            DevFlags* fl) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double a = pos[3 * t], b = pos[3 * t + 1], c = pos[3 * t + 2];
    double p = vel[3 * t], q = vel[3 * t + 1], r = vel[3 * t + 2];
    if (!(isfinite(a) && isfinite(b) && isfinite(c) && isfinite(p) && isfinite(q) && isfinite(r)))
        atomicMin(&fl->nonfinite_gid, t);
    x[t] = make_double4(a, b, c, 0.0);
    vx[t] = p;
    vy[t] = q;
    vz[t] = r;
    gid[t] = t;
    own_slot[t] = t;
}

struct Geo {
    double L[3];
    double w[3];        // cell widths
    double inv_w[3];
    int nc[3];          // global cell grid
    int z0, nzl;        // this rank's slab [z0, z0+nzl)
    int ex, ey, ez;     // extended grid dims = ncx+2, ncy+2, nzl+2
};

// Wrap owned positions (R10) and bin them: cell_of[t] = owned-cell index, rank_in[t] = slot
// inside the cell from the atomic counter (order fixed later by the gid sort).
__global__ void k_wrap_bin(int n_own, const double4* __restrict__ x, const int* __restrict__ own_slot,
                           Geo g, double4* __restrict__ xw, int* __restrict__ ocount,
                           int* __restrict__ cell_of, int* __restrict__ rank_in,
                           const int* __restrict__ gid, DevFlags* fl) {
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
    int oc = (cz * g.nc[1] + c[1]) * g.nc[0] + c[0];
    xw[t] = p;
    cell_of[t] = oc;
    rank_in[t] = atomicAdd(&ocount[oc], 1);
}

// Extended-cell counts: owned cells take their own count, ghost cells the count of
// their source cell (ghost table built on the host at init).
__global__ void k_ext_counts(int n_ecell, const int* __restrict__ ocount, Geo g,
                             const int* __restrict__ ecell_src, int* __restrict__ ecount) {
    int ec = blockIdx.x * blockDim.x + threadIdx.x;
    if (ec >= n_ecell) return;
    int src = ecell_src[ec];   // owned-cell index whose particles fill this cell
    ecount[ec] = ocount[src];
}

__global__ void k_scatter(int n_own, const int* __restrict__ cell_of, const int* __restrict__ rank_in,
                          const int* __restrict__ obegin, int* __restrict__ perm) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    perm[obegin[cell_of[t]] + rank_in[t]] = t;
}

// One warp per owned cell: order members by gid (deterministic layout, reading R15),
// write the new owned-space arrays and the owned slots of the new slot space.
__global__ void k_cell_sort(int n_ocell, Geo g, const int* __restrict__ obegin,
                            const int* __restrict__ ocount, const int* __restrict__ ebegin,
                            const int* __restrict__ perm, const int* __restrict__ gid_old,
                            const double4* __restrict__ xw, const double* __restrict__ vx_o,
                            const double* __restrict__ vy_o, const double* __restrict__ vz_o,
                            double4* __restrict__ x_new, float4* __restrict__ xf,
                            double* __restrict__ vx_n, double* __restrict__ vy_n,
                            double* __restrict__ vz_n, int* __restrict__ gid_new,
                            int* __restrict__ own_slot, int* __restrict__ ocell_of,
                            int* __restrict__ slot_gid, double4* __restrict__ xbuild) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= n_ocell) return;
    int oc = warp;
    int m = ocount[oc];
    int b = obegin[oc];
    int cx = oc % g.nc[0];
    int cy = (oc / g.nc[0]) % g.nc[1];
    int cz = oc / (g.nc[0] * g.nc[1]);
    int ec = ((cz + 1) * g.ey + (cy + 1)) * g.ex + (cx + 1);
    int sb = ebegin[ec];
    for (int k = lane; k < m; k += 32) {
        int t_old = perm[b + k];
        int gk = gid_old[t_old];
        int r = 0;
        for (int s = 0; s < m; ++s) r += (gid_old[perm[b + s]] < gk);
        int t = b + r;
        int slot = sb + r;
        double4 p = xw[t_old];
        x_new[slot] = p;
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

template <bool AT_BUILD>
__global__ void k_ghost_refresh(GhostCells gc, const int* __restrict__ ebegin,
                                const int* __restrict__ ecount, Geo g, double4* __restrict__ x,
                                float4* __restrict__ xf, int* __restrict__ slot_gid) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= gc.n) return;
    int d = gc.dst[warp], s = gc.src[warp], code = gc.shift[warp];
    int db = ebegin[d], sb = ebegin[s], m = ecount[s];
    double sx = (double)((code & 3) - 1), sy = (double)(((code >> 2) & 3) - 1),
           sz = (double)(((code >> 4) & 3) - 1);
    double Lx = sx * g.L[0], Ly = sy * g.L[1], Lz = sz * g.L[2];   // exact
    for (int k = lane; k < m; k += 32) {
        double4 p = ld256(x + sb + k);
        double4 q = make_double4(__dadd_rn(p.x, Lx), __dadd_rn(p.y, Ly), __dadd_rn(p.z, Lz), 0.0);
        st256(x + db + k, q);
        if (AT_BUILD) {
            xf[db + k] = make_float4((float)q.x, (float)q.y, (float)q.z, 0.f);
            slot_gid[db + k] = slot_gid[sb + k];
        }
    }
}

// --------------------------------------------------------------------------- neighbour list
// Thread per owned particle.  Candidates: the 9 contiguous x-rows of the 27-cell stencil
// (Sec. 3.4), rows/cells pruned by their distance to x_i; an fp32
// prefilter with a provably conservative threshold, then the canonical fp64 test
// r^2 < rbar_c^2 (strict, R4).  Emitted in (row, slot) = (stencil offset, gid) order.
struct NlistArgs {
    Geo g;
    const double4* x;
    const float4* xf;
    const int* own_slot;
    const int* ocell_of;
    const int* ebegin;
    const int* ecount;
    int* nbr;
    int* ncount;
    int n_own, n_pad, K;
    double rn2;          // rbar_c^2 (fp64, canonical)
    float thr_f;         // conservative fp32 threshold
    double prune2;       // (rbar_c + slop)^2 for row / cell pruning
    DevFlags* fl;
    const int* slot_gid;
};

__global__ void __launch_bounds__(128) k_build_nlist(NlistArgs a) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n_own) return;
    const Geo& g = a.g;
    int si = a.own_slot[t];
    double4 xi = a.x[si];
    float4 fi = a.xf[si];
    int oc = a.ocell_of[t];
    int cx = oc % g.nc[0];
    int cy = (oc / g.nc[0]) % g.nc[1];
    int cz = oc / (g.nc[0] * g.nc[1]);
    // cell bounds along each axis in the coordinates the particles live in (global cells;
    // ghost layer cells -1 and n lie just outside [0,L))
    double lo_x = cx * g.w[0];
    double lo_y = cy * g.w[1];
    double lo_z = (cz + g.z0) * g.w[2];
    double rx0 = xi.x - lo_x;                 // distance into own cell from the low face
    double rx1 = lo_x + g.w[0] - xi.x;        // to the high face
    double ry0 = xi.y - lo_y, ry1 = lo_y + g.w[1] - xi.y;
    double rz0 = xi.z - lo_z, rz1 = lo_z + g.w[2] - xi.z;
    int k = 0;
    int* out = a.nbr + t;
    const size_t stride = (size_t)a.n_pad;
    for (int dz = -1; dz <= 1; ++dz) {
        double ddz = dz < 0 ? rz0 : (dz > 0 ? rz1 : 0.0);
        double ddz2 = ddz > 0.0 ? ddz * ddz : 0.0;
        for (int dy = -1; dy <= 1; ++dy) {
            double ddy = dy < 0 ? ry0 : (dy > 0 ? ry1 : 0.0);
            double dyz2 = ddz2 + (ddy > 0.0 ? ddy * ddy : 0.0);
            if (dyz2 >= a.prune2) continue;
            int xs = (rx0 > 0.0 && dyz2 + rx0 * rx0 >= a.prune2) ? 0 : -1;
            int xe = (rx1 > 0.0 && dyz2 + rx1 * rx1 >= a.prune2) ? 0 : 1;
            int erow = ((cz + 1 + dz) * g.ey + (cy + 1 + dy)) * g.ex + (cx + 1);
            int jb = a.ebegin[erow + xs];
            int je = a.ebegin[erow + xe] + a.ecount[erow + xe];
            for (int j = jb; j < je; ++j) {
                float4 fj = a.xf[j];
                float fx = fi.x - fj.x, fy = fi.y - fj.y, fz = fi.z - fj.z;
                float r2f = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
                if (r2f >= a.thr_f || j == si) continue;
                double4 xj = a.x[j];
                double r2 = r2_canon(xi.x - xj.x, xi.y - xj.y, xi.z - xj.z);
                if (r2 < a.rn2) {
                    if (r2 == 0.0) {
                        atomicMin(&a.fl->overlap_gid, a.slot_gid[si]);
                        a.fl->overlap_gid_j = a.slot_gid[j];
                    }
                    if (k < a.K) out[(size_t)k * stride] = j;
                    ++k;
                }
            }
        }
    }
    a.ncount[t] = k;
    atomicMax(&a.fl->max_nbr, k);
    // warp-aggregated total (for stats)
    unsigned long long kk = (unsigned long long)k;
    for (int o = 16; o > 0; o >>= 1) kk += __shfl_down_sync(__activemask(), kk, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&a.fl->total_nbr, kk);
}

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
enum { kStore = 0, kKick = 1, kKKD = 2 };

struct ForceArgs {
    const double4* x;        // current positions (slot space)
    double4* x_next;         // kKKD output buffer (slot space)
    const int* own_slot;
    const int* nbr;
    const int* ncount;
    double* fx; double* fy; double* fz;
    double* vx; double* vy; double* vz;
    double* e;               // per-particle e_i (ENERGY)
    double* pe_part;         // per-block partial sums (ENERGY)
    double* ke_part;
    const double4* xbuild;   // displacement check (may be null)
    DevFlags* fl;
    int n_own, n_pad;
    double rc2, c12, c6, a12, a6, a0;
    double h, dt, half_m;
};

constexpr int kForceThreads = 128;

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

template <bool ENERGY, int MODE, bool CHECK>
__global__ void __launch_bounds__(kForceThreads) k_force(ForceArgs a) {
    __shared__ double sh[kForceThreads / 32];
    const int t = blockIdx.x * kForceThreads + threadIdx.x;
    double fx = 0.0, fy = 0.0, fz = 0.0, u = 0.0, ke = 0.0;
    if (t < a.n_own) {
        const int si = a.own_slot[t];
        const double4 xi = ld256(a.x + si);
        const int cnt = a.ncount[t];
        const int* nb = a.nbr + t;
        const size_t stride = (size_t)a.n_pad;
#pragma unroll 4
        for (int k = 0; k < cnt; ++k) {
            const int j = __ldg(nb + (size_t)k * stride);
            const double4 xj = ld256(a.x + j);
            const double dx = xi.x - xj.x, dy = xi.y - xj.y, dz = xi.z - xj.z;
            const double r2 = r2_canon(dx, dy, dz);
            const double ir2 = rcp64(r2);
            const double ir4 = ir2 * ir2;
            const double ir6 = ir4 * ir2;
            const double ir8 = ir4 * ir4;
            double gg = ir8 * fma(a.c12, ir6, -a.c6);
            const bool in = r2 < a.rc2;
            gg = in ? gg : 0.0;
            fx = fma(gg, dx, fx);
            fy = fma(gg, dy, fy);
            fz = fma(gg, dz, fz);
            if (ENERGY) {
                double v = fma(fma(a.a12, ir6, -a.a6), ir6, a.a0);
                u += in ? v : 0.0;
            }
        }
        if (MODE == kStore) {
            a.fx[t] = fx; a.fy[t] = fy; a.fz[t] = fz;
            if (ENERGY) {
                double vx = a.vx[t], vy = a.vy[t], vz = a.vz[t];
                ke = a.half_m * __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
            }
        } else {
            double vx = a.vx[t], vy = a.vy[t], vz = a.vz[t];
            // line 8: v += dt/(2m) F  (two roundings, as Listing lst:velocity_update)
            vx = __dadd_rn(vx, __dmul_rn(a.h, fx));
            vy = __dadd_rn(vy, __dmul_rn(a.h, fy));
            vz = __dadd_rn(vz, __dmul_rn(a.h, fz));
            if (ENERGY)
                ke = a.half_m * __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
            if (MODE == kKick) {
                a.fx[t] = fx; a.fy[t] = fy; a.fz[t] = fz;
            } else {
                // line 6 of the next step: v += dt/(2m) F ; r += dt v (Listing lst:position_update)
                vx = __dadd_rn(vx, __dmul_rn(a.h, fx));
                vy = __dadd_rn(vy, __dmul_rn(a.h, fy));
                vz = __dadd_rn(vz, __dmul_rn(a.h, fz));
                double4 xn = make_double4(__dadd_rn(xi.x, __dmul_rn(a.dt, vx)),
                                          __dadd_rn(xi.y, __dmul_rn(a.dt, vy)),
                                          __dadd_rn(xi.z, __dmul_rn(a.dt, vz)), 0.0);
                st256(a.x_next + si, xn);
                if (CHECK) {
                    double4 b = a.xbuild[t];
                    double d2 = r2_canon(xn.x - b.x, xn.y - b.y, xn.z - b.z);
                    // non-negative doubles order like their bit patterns
                    unsigned long long bits = __double_as_longlong(d2);
                    for (int o = 16; o > 0; o >>= 1) {
                        unsigned long long ob = __shfl_down_sync(__activemask(), bits, o);
                        bits = ob > bits ? ob : bits;
                    }
                    if ((threadIdx.x & 31) == 0) atomicMax(&a.fl->maxdisp2, bits);
                }
            }
            a.vx[t] = vx; a.vy[t] = vy; a.vz[t] = vz;
        }
        if (ENERGY) a.e[t] = 0.5 * u;
    }
    if (ENERGY) {
        double pe = block_sum<kForceThreads>(t < a.n_own ? 0.5 * u : 0.0, sh);
        double k2 = block_sum<kForceThreads>(ke, sh);
        if (threadIdx.x == 0) {
            a.pe_part[blockIdx.x] = pe;
            a.ke_part[blockIdx.x] = k2;
        }
    }
}

// opening half of a step() call: v += h F ; x += dt v  (in place, owned slots)
template <bool CHECK>
__global__ void k_kick_drift(int n_own, double4* __restrict__ x, const int* __restrict__ own_slot,
                             double* __restrict__ vx, double* __restrict__ vy, double* __restrict__ vz,
                             const double* __restrict__ fx, const double* __restrict__ fy,
                             const double* __restrict__ fz, double h, double dt,
                             const double4* __restrict__ xbuild, DevFlags* fl) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long bits = 0ull;
    if (t < n_own) {
        int si = own_slot[t];
        double4 p = x[si];
        double a = __dadd_rn(vx[t], __dmul_rn(h, fx[t]));
        double b = __dadd_rn(vy[t], __dmul_rn(h, fy[t]));
        double c = __dadd_rn(vz[t], __dmul_rn(h, fz[t]));
        p.x = __dadd_rn(p.x, __dmul_rn(dt, a));
        p.y = __dadd_rn(p.y, __dmul_rn(dt, b));
        p.z = __dadd_rn(p.z, __dmul_rn(dt, c));
        x[si] = p;
        vx[t] = a; vy[t] = b; vz[t] = c;
        if (CHECK) {
            double4 q = xbuild[t];
            bits = __double_as_longlong(r2_canon(p.x - q.x, p.y - q.y, p.z - q.z));
        }
    }
    if (CHECK) {
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long ob = __shfl_down_sync(0xffffffffu, bits, o);
            bits = ob > bits ? ob : bits;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&fl->maxdisp2, bits);
    }
}

// fixed-order final reduction of the per-block partials -> out[0] = PE, out[1] = KE
__global__ void k_finalize_energy(const double* __restrict__ pe_part, const double* __restrict__ ke_part,
                                  int nb, double* __restrict__ out) {
    __shared__ double sh[32];
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
    }
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

__global__ void k_list_gids(int n_own, int n_pad, const int* __restrict__ nbr, const int* __restrict__ ncount,
                            const int* __restrict__ slot_gid, const long long* __restrict__ off,
                            long long* __restrict__ out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_own) return;
    int c = ncount[t];
    long long o = off[t];
    for (int k = 0; k < c; ++k) out[o + k] = slot_gid[nbr[(size_t)k * n_pad + t]];
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
