// ljmd.cu -- host side of libljmd.so: the C ABI declared in include/ljmd.h.
// Owns device memory, the stream, the rebuild policy (IntegratorRange)
// and the velocity-Verlet step loop (Alg. alg:VelocityVerlet).
#include "../../include/ljmd.h"
#include "kernels.cuh"
#include "dsl.h"
#include "transport.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

using namespace ljmd;

static constexpr size_t kMaxStageSmem = 200 * 1024;   // dynamic smem cap for the tile staging
#ifndef LJMD_STAGE_MARGIN
#define LJMD_STAGE_MARGIN 8   // stage_cap = max_staged (1 + 1/MARGIN) + 16 when it grows
#endif

namespace {

thread_local std::string g_init_error;

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
};

}  // namespace

struct ljmd_ctx {
    // ---- parameters
    int64_t n_global = 0;
    int n_own = 0;
    double rc = 0, eps = 0, sigma = 0, dt = 0, rn = 0;
    ljmd_options opt{};
    Geo geo{};
    int n_ocell = 0, n_ecell = 0, n_gcell = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // nranks > 1: the per-step halo exchange runs on aux_stream while the interior tiles'
    // force launch runs on `stream`; the boundary tile layers wait for ev_halo
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    // ---- status
    ljmd_status err = LJMD_OK;
    std::string msg;
    // ---- capacities
    int own_cap = 0, slot_cap = 0, K = 0, n_pad = 0;
    int n_tiles = 0;
    int max_staged = 0;               // largest tile halo (particles) at the last build
    int n_slots = 0;
    // ---- slot space
    double4* x[2] = {nullptr, nullptr};
    int xc = 0;                       // current position buffer
    double nu_dt = 0.0, thermo_sd = 0.0;   // Andersen thermostat (ljmd_set_thermostat)
    unsigned long long thermo_seed = 0;
    float4* xf = nullptr;
    int* slot_gid = nullptr;
    // ---- owned space (double-buffered across rebuilds)
    double* v[2] = {nullptr, nullptr};  // [3][own_cap]
    int* gid[2] = {nullptr, nullptr};
    int oc_cur = 0;
    int* own_slot = nullptr;
    int* own_li = nullptr;            // the owned particle's index in its tile's staged halo (list build)
    int* ocell_of = nullptr;
    double* F = nullptr;                // [3][own_cap]
    double* e = nullptr;
    double4* xbuild = nullptr;
    double4* xw = nullptr;
    int* cell_of = nullptr;
    int* rank_in = nullptr;
    int* perm = nullptr;
    // ---- cells
    int* ocount = nullptr;
    int* obegin = nullptr;   // n_ocell + 1
    int* ecount = nullptr;
    int* ebegin = nullptr;   // n_ecell + 1
    int* ecell_src = nullptr;
    int4* gflat = nullptr;            // ghost slots {dst, src, shift code} (k_ghost_flat)
    int n_gflat = 0;
    int* slot2t = nullptr;            // owned slot -> owned index (image build)
    int* img_cnt = nullptr;           // [own_cap] images per owned particle (scratch)
    int* img_off = nullptr;           // [own_cap + 1] CSR offsets of the ghost images
    int2* img = nullptr;              // {dst slot, shift code}
    int4* grecv = nullptr;            // images of received halo planes (nranks > 1)
    int n_grecv = 0;
    int* gc_dst = nullptr;
    int* gc_src = nullptr;
    int* gc_shift = nullptr;
    int* oc_of_lex = nullptr;         // tile-major owned-cell numbering
    int* lex_of_oc = nullptr;
    int* tile_oc0 = nullptr;          // [n_tiles + 1]
    int* tr_begin = nullptr;          // tile halo rows
    float* ylo_f = nullptr;           // fp32 cell faces (list-build pruning)
    float* zlo_f = nullptr;
    int* tr_off = nullptr;
    int* tr_len = nullptr;
    double* xp[2] = {nullptr, nullptr};   // packed {x, y, z} per slot, kept with x[2] (force staging)
    int* scan_tmp = nullptr;
    int scan_tmp_n = 0;
    // ---- list
    uint4* nbr8 = nullptr;            // 16-bit tile-local indices in blocks of 8: [K/8][n_pad]
    int bank_order = 1;               // 0: the force kernel walks the build order
    bool use_rr = false;              // the current list is in the bank-aware order
    double interval_ema = 0.0;        // steps a list has served, running estimate
    int64_t ncalls = 0;               // ljmd_step calls so far
    double ema_after[4] = {0, 0, 0, 0};   // interval_ema after call k (k mod 4): list order lags 2 calls
    bool dev_since_ok = false;        // the device's step control holds the current since (graph calls)
    int64_t last_build_step = -1;     // steps_done at the last rebuild (-1: none yet)
    bool newton3 = false;             // half list + reaction reductions (NEXT-1)
    uint4* nbr8h = nullptr;           // half list (newton3), blocked like nbr8
    int* ncount_h = nullptr;
    int* slot_t = nullptr;            // slot -> owned index (newton3)
    int* tmap = nullptr;              // gid -> owned index (newton3, DSL)
    // ---- DSL front end (dsl.cuh): particle data and compiled loops
    std::vector<ljmd::DslDat> dats;
    std::vector<ljmd::DslLoop*> loops;
    bool dsl_on = false;
    bool slot_t_valid = false;
    int* tile_R = nullptr;
    double* ld_pos = nullptr;         // load_state staging
    double* ld_vel = nullptr;
    int* ld_gid = nullptr;
    int* ncount = nullptr;
    // ---- energies
    double* pe_part = nullptr;
    double* ke_part = nullptr;
    int n_fblocks = 0;
    int fparts = 1;                   // force CTAs per tile
    double* hist = nullptr;   // [hist_cap][2]
    double* h_histm = nullptr;   // mapped page-locked readback of hist
    int64_t h_histm_cap = 0;
    int64_t hist_cap = 0, hist_count = 0;
    std::vector<double> h_hist;
    // ---- flags / staging
    DevFlags* d_fl = nullptr;
    DevFlags* h_fl = nullptr;      // pinned
    DevStats* d_st = nullptr;      // persistent device counters (dangerous builds)
    DevStats* h_st = nullptr;      // mapped page-locked readback of d_st
    bool pdl_ok = false;           // the previous force launch may overlap the next (PDL): false
                                   // right after a rebuild (the list was just written)
    // ---- validation mode (ljmd_options.validate): missed pairs per step
    int* vcount = nullptr;         // [n_cells + 1] (count, then exclusive begin)
    int* vbegin = nullptr;
    int* vcell = nullptr;
    int* vrank = nullptr;
    double4* vpos = nullptr;
    int* vhist = nullptr;          // [vhist_cap][2]
    int64_t vhist_cap = 0;
    std::vector<int64_t> h_val;    // (step, particles with missed pairs, missed ordered pairs)
    // energies of the current state are in hist/e (the last step of the previous ljmd_step
    // call was a sample step, or the init sequence): ljmd_get_energy need not recompute
    bool energy_current = false;
    double cur_pe = 0.0, cur_ke = 0.0;
    // the init sequence's PE/KE travel to mapped memory without a host wait; read at the next
    // synchronisation (end of ljmd_step) or on demand (settle_init)
    double* h_init = nullptr;
    bool init_pending = false, init_current = false;
    // ---- graph mode (single rank): ljmd_step captured into CUDA graphs, rebuild decided and
    // capacity-checked on the device
    DevCtl* d_ctl = nullptr;
    int* d_rstep = nullptr;           // rebuild steps of the current call (1-based within it)
    int64_t rstep_cap = 0;
    int stage_cap = 0;                // staged particles per tile the force/build launches are sized for
    struct GraphEntry {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ex = nullptr;
        int64_t launches = 0;         // kernels outside the conditional rebuild bodies
        int64_t body_k = 0;           // kernels of one conditional rebuild body
    };
    std::map<std::string, GraphEntry> graphs;
    bool capturing = false;           // launches go into a graph being captured
    bool spec = false;                // eager rebuild with device-side capacity checks (one host wait)
    DevCtl* h_sctl = nullptr;         // mapped: its control
    int64_t spec_aborts = 0;
    cudaStream_t cap_stream[3] = {nullptr, nullptr, nullptr};   // capture of nested rebuild bodies
    int64_t graph_calls = 0, graph_aborts = 0;
    int64_t call_nsamp = 0;           // energy samples of the current ljmd_step call
    // deferred settlement (graph mode, fixed rebuild schedule): ljmd_step returns once its
    // graph is queued; the host reads the call's control (k_call_out, two alternating mapped
    // buffers) after queueing the next call, or at the next API call
    struct Pending {
        bool on = false;
        bool deferred = false;        // the host state was advanced at launch
        int64_t step0 = 0, nsteps = 0, launches = 0, body_k = 0, call = 0;
        int64_t sim_since = 0;        // fixed schedule: steps since the last rebuild at the end
        int xc0 = 0, buf = 0;
    };
    Pending pend;
    CallOut* h_out[2] = {nullptr, nullptr};     // mapped
    int* h_orstep[2] = {nullptr, nullptr};      // mapped [out_cap]
    double* h_ohist[2] = {nullptr, nullptr};    // mapped [2 out_cap]
    int64_t out_cap = 0;
    int out_next = 0;
    cudaEvent_t ev_call[2] = {nullptr, nullptr};
    int* h_slots = nullptr;        // pinned
    double* d_stage = nullptr;     // [3][own_cap] readback staging
    // overlapped host transfers (ljmd_stage_state / ljmd_get_positions_async)
    cudaStream_t copy_stream = nullptr;
    double* stg[2] = {nullptr, nullptr};      // [pos 3n | vel 3n] staged states
    cudaEvent_t stg_ev[2] = {nullptr, nullptr}, stg_used[2] = {nullptr, nullptr};
    int stg_next = 0, stg_queued = 0;         // next buffer to fill, states queued
    double* rb[2] = {nullptr, nullptr};       // [3n] positions in caller order
    cudaEvent_t rb_ev[2] = {nullptr, nullptr}, rb_done[2] = {nullptr, nullptr};
    int rb_next = 0;
    // ---- policy / stats
    int64_t since = 0, steps_done = 0, n_rebuilds = 0, regrows = 0;
    std::vector<int64_t> rebuild_steps;
    int max_nbr = 0;
    unsigned long long total_nbr = 0;
    // ---- profiling
    std::vector<cudaEvent_t> ev;
    int64_t force_launches = 0;
    double force_ms = 0.0;
    int64_t kernel_launches = 0;   // launches of this library's kernels (CKL after each)
    // ---- z-slab decomposition (nranks > 1)
    Transport* tr = nullptr;
    int rank = 0, nranks = 1, lo_rank = 0, hi_rank = 0, npc = 0;
    bool split = false;           // run the slab-exchange path (nranks > 1, or split_self)
    int* send_cnt = nullptr;      // [2 * npc] bottom / top plane cell counts
    int* send_off = nullptr;      // [2 * npc + 1]
    int* recv_cnt = nullptr;      // [2 * npc] lower / upper ghost plane cell counts
    int* recv_off = nullptr;      // [2 * npc + 1]
    int* send_idx = nullptr;      // slot of every boundary-plane particle
    double4* send_buf = nullptr;
    int send_cap = 0;
    int n_send[2] = {0, 0}, n_recv[2] = {0, 0};
    MigRec* mig_send[2] = {nullptr, nullptr};
    MigRec* mig_recv[2] = {nullptr, nullptr};
    int mig_cap = 0;
    int* mig_cnt = nullptr;       // device [3]: stay, lo, hi ; [3..5]: received counts
    int* h_mig = nullptr;         // pinned mirror
    double4* xs = nullptr;        // compacted (post-migration) positions / velocities / gids
    double* vs = nullptr;
    int* gs = nullptr;
    int* iota = nullptr;
    int* stay_t = nullptr;        // compaction order of the stayers (migrate)
    int* h_tot = nullptr;         // pinned: send/recv plane totals
    // direct-landing halo (per step): send area after the slot range of x / xp, in the
    // receiver's ghost-plane layout; receives land in the ghost planes
    int send_extra = 0;           // entries of x / xp / gflat / img beyond slot_cap
    int* pl_cnt = nullptr;        // [2 ex ey] extended-plane cell counts (bottom, top)
    int* pl_off = nullptr;        // [2 ex ey + 1]
    int* h_pl = nullptr;          // mapped: {send total, bottom part, lower ghost begin, lower
                                  //          ghost end, upper ghost begin, upper ghost end}
    int area[2] = {0, 0};         // send-area entries for the lower / upper neighbour
    int gbeg[2] = {0, 0}, glen[2] = {0, 0};   // my lower / upper ghost plane: slots
    unsigned* halo_flag = nullptr;    // gated boundary tiles: released per step by the halo stream
    unsigned halo_seq = 0;
    // boundary-first force launches (nranks > 1): the boundary CTAs count themselves done in
    // *bdone; the next step's halo exchange waits for that count on aux_stream (a stream
    // memory wait) and overlaps the interior tiles of the same launch
    unsigned* bdone = nullptr;
    unsigned bdone_issued = 0;        // the count every boundary CTA issued so far reaches
    bool halo_queued = false;         // the next step's halo is in flight on aux_stream (ev_halo)
};

ljmd_status dsl_before_sort(ljmd_ctx* c, const int* gid_old);
ljmd_status dsl_after_sort(ljmd_ctx* c);
ljmd_status dsl_to_gid_order(ljmd_ctx* c);
ljmd_status dsl_migrate(ljmd_ctx* c, int stay, int out_lo, int out_hi, int in_lo, int in_hi);
void dsl_destroy(ljmd_ctx* c);

namespace {

ljmd_status set_err(ljmd_ctx* c, ljmd_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) {
        if (c->err == LJMD_OK) {
            c->err = s;
            c->msg = buf;
        }
    } else {
        g_init_error = buf;
    }
    return s;
}

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return set_err(c, LJMD_E_CUDA, "%s failed: %s (%s:%d)", #call,                 \
                           cudaGetErrorString(e_), __FILE__, __LINE__);                     \
    } while (0)

#define CKL()                                                                               \
    do {                                                                                    \
        ++c->kernel_launches;                                                               \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess)                                                              \
            return set_err(c, LJMD_E_CUDA, "kernel launch failed: %s (%s:%d)",             \
                           cudaGetErrorString(e_), __FILE__, __LINE__);                     \
    } while (0)

#define TRY(expr)                       \
    do {                                \
        ljmd_status s_ = (expr);        \
        if (s_ != LJMD_OK) return s_;   \
    } while (0)

void drop_graphs(ljmd_ctx* c) {
    for (auto& kv : c->graphs) {
        if (kv.second.ex) cudaGraphExecDestroy(kv.second.ex);
        if (kv.second.g) cudaGraphDestroy(kv.second.g);
    }
    c->graphs.clear();
}

template <class T>
ljmd_status dalloc(ljmd_ctx* c, T** p, size_t n) {
    if (c) drop_graphs(c);   // captured step graphs hold raw pointers
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return set_err(c, LJMD_E_CAPACITY, "cudaMalloc of %zu bytes failed: %s", n * sizeof(T),
                       cudaGetErrorString(e));
    }
    return LJMD_OK;
}

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// the control a captured rebuild's kernels check (skip after a failed capacity check)
inline const DevCtl* cctl(const ljmd_ctx* c) { return (c->capturing || c->spec) ? c->d_ctl : nullptr; }
// the rebuild's capacities are checked on the device (captured, or speculative eager)
inline bool dev_caps(const ljmd_ctx* c) { return c->capturing || c->spec; }

// exclusive scan of n ints: out[0..n) prefixes, out[n] = total
ljmd_status scan(ljmd_ctx* c, const int* in, int n, int* out) {
    if (n <= kScanSingle) {
        k_scan_single<<<1, 1024, 0, c->stream>>>(in, n, out);
        CKL();
        return LJMD_OK;
    }
    int nb = std::max(1, nblk(n, kScanTile));
    if (nb > c->scan_tmp_n) {
        TRY(dalloc(c, &c->scan_tmp, nb));
        c->scan_tmp_n = nb;
    }
    k_scan_reduce<<<nb, kScanThreads, 0, c->stream>>>(in, n, c->scan_tmp);
    k_scan_top<<<1, 1024, 0, c->stream>>>(c->scan_tmp, nb, out + n);
    k_scan_down<<<nb, kScanThreads, 0, c->stream>>>(in, n, c->scan_tmp, out, 0);
    c->kernel_launches += 2;
    CKL();
    return LJMD_OK;
}

// the binning's cell offsets: owned-cell begin (scan of ocount), extended-cell counts and begin
ljmd_status bin_offsets(ljmd_ctx* c) {
    if (c->n_ocell <= kScanSingle && c->n_ecell <= kScanSingle) {   // small systems: one launch
        k_bin_offsets_single<<<1, 1024, 0, c->stream>>>(c->ocount, c->n_ocell, c->obegin, c->n_ecell, c->ecell_src,
                                                       c->recv_cnt, c->ecount, c->ebegin,
                                                       const_cast<DevCtl*>(cctl(c)), c->slot_cap);
        CKL();
        return LJMD_OK;
    }
    TRY(scan(c, c->ocount, c->n_ocell, c->obegin));
    k_ext_counts<<<nblk(c->n_ecell, 256), 256, 0, c->stream>>>(c->n_ecell, c->ocount, c->geo, c->ecell_src,
                                                              c->recv_cnt, c->ecount);
    CKL();
    return scan(c, c->ecount, c->n_ecell, c->ebegin);
}

// zero `bytes` (a multiple of 4) of device memory on the engine's stream (k_zero_words)
ljmd_status zero_async(ljmd_ctx* c, void* p, size_t bytes) {
    const size_t n = bytes / 4;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 1184);
    k_zero_words<<<std::max(blocks, 1), 256, 0, c->stream>>>(static_cast<unsigned*>(p), n);
    CKL();
    return LJMD_OK;
}

// device -> mapped host memory by a kernel (no copy engine); complete after a stream sync
ljmd_status to_host(ljmd_ctx* c, void* hmapped, const void* dsrc, size_t bytes) {
    k_copy_words<<<1, 256, 0, c->stream>>>(static_cast<const unsigned*>(dsrc), static_cast<unsigned*>(hmapped),
                                          (int)(bytes / 4));
    CKL();
    return LJMD_OK;
}

ljmd_status sync_flags(ljmd_ctx* c) {
    TRY(to_host(c, c->h_fl, c->d_fl, sizeof(DevFlags)));
    CK(cudaStreamSynchronize(c->stream));
    return LJMD_OK;
}

ljmd_status reset_flags(ljmd_ctx* c) {
    k_reset_flags<<<1, 1, 0, c->stream>>>(c->d_fl, 1);
    CKL();
    return LJMD_OK;
}

// ------------------------------------------------------------------ geometry / tables
ljmd_status plan_geometry(ljmd_ctx* c, const double box[3]) {
    int64_t nc[3];
    if (ljmd_plan_cells(box, c->rn, nc) != LJMD_OK)
        return set_err(c, LJMD_E_BOX,
                       "box (%g, %g, %g) too small: need >= 3 cells of width >= rbar_c = %g per dimension",
                       box[0], box[1], box[2], c->rn);
    int64_t z0 = 0, z1 = nc[2];
    if (ljmd_plan_slab(nc[2], c->opt.nranks, c->opt.rank, &z0, &z1) != LJMD_OK)
        return set_err(c, LJMD_E_BOX, "cannot split %lld z-planes over %lld ranks", (long long)nc[2],
                       (long long)c->opt.nranks);
    Geo& g = c->geo;
    for (int d = 0; d < 3; ++d) {
        g.L[d] = box[d];
        g.nc[d] = (int)nc[d];
        g.w[d] = box[d] / (double)nc[d];
        g.inv_w[d] = 1.0 / g.w[d];
    }
    g.z0 = (int)z0;
    g.nzl = (int)(z1 - z0);
    g.ex = g.nc[0] + 2;
    g.ey = g.nc[1] + 2;
    g.ez = g.nzl + 2;
    c->n_ocell = g.nc[0] * g.nc[1] * g.nzl;
    c->n_ecell = g.ex * g.ey * g.ez;
    c->n_gcell = c->n_ecell - c->n_ocell;
    if ((int64_t)c->n_ecell > (int64_t)INT_MAX / 2)
        return set_err(c, LJMD_E_ARG, "cell grid too large");
    // tile-major numbering of the owned cells (force tiles of kTX x kTY x kTZ cells)
    g.ntx = (g.nc[0] + kTX - 1) / kTX;
    g.nty = (g.nc[1] + kTY - 1) / kTY;
    g.ntz = (g.nzl + kTZ - 1) / kTZ;
    c->n_tiles = g.ntx * g.nty * g.ntz;
    std::vector<int> oc_of_lex(c->n_ocell), lex_of_oc(c->n_ocell), tile_oc0(c->n_tiles + 1);
    {
        int oc = 0, tile = 0;
        for (int tz = 0; tz < g.ntz; ++tz)
            for (int ty = 0; ty < g.nty; ++ty)
                for (int tx = 0; tx < g.ntx; ++tx, ++tile) {
                    tile_oc0[tile] = oc;
                    for (int cz = tz * kTZ; cz < std::min(g.nzl, (tz + 1) * kTZ); ++cz)
                        for (int cy = ty * kTY; cy < std::min(g.nc[1], (ty + 1) * kTY); ++cy)
                            for (int cx = tx * kTX; cx < std::min(g.nc[0], (tx + 1) * kTX); ++cx) {
                                const int lex = (cz * g.nc[1] + cy) * g.nc[0] + cx;
                                oc_of_lex[lex] = oc;
                                lex_of_oc[oc] = lex;
                                ++oc;
                            }
                }
        tile_oc0[c->n_tiles] = oc;
    }
    TRY(dalloc(c, &c->oc_of_lex, c->n_ocell));
    TRY(dalloc(c, &c->lex_of_oc, c->n_ocell));
    TRY(dalloc(c, &c->tile_oc0, c->n_tiles + 1));
    TRY(dalloc(c, &c->tr_begin, (size_t)c->n_tiles * kRowsMax));
    TRY(dalloc(c, &c->tr_off, (size_t)c->n_tiles * (kRowsMax + 1)));
    TRY(dalloc(c, &c->tr_len, (size_t)c->n_tiles * kRowsMax));
    CK(cudaMemcpy(c->oc_of_lex, oc_of_lex.data(), sizeof(int) * c->n_ocell, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->lex_of_oc, lex_of_oc.data(), sizeof(int) * c->n_ocell, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->tile_oc0, tile_oc0.data(), sizeof(int) * (c->n_tiles + 1), cudaMemcpyHostToDevice));
    g.oc_of_lex = c->oc_of_lex;
    g.lex_of_oc = c->lex_of_oc;
    {
        std::vector<float> yf(g.nc[1] + 1), zf(g.nzl + 1);
        for (int k = 0; k <= g.nc[1]; ++k) yf[k] = (float)(k * g.w[1]);
        for (int k = 0; k <= g.nzl; ++k) zf[k] = (float)((g.z0 + k) * g.w[2]);
        TRY(dalloc(c, &c->ylo_f, yf.size()));
        TRY(dalloc(c, &c->zlo_f, zf.size()));
        CK(cudaMemcpy(c->ylo_f, yf.data(), sizeof(float) * yf.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->zlo_f, zf.data(), sizeof(float) * zf.size(), cudaMemcpyHostToDevice));
    }

    // ghost-cell table.  Single rank: every ghost cell is a periodic image of an owned cell.
    // nranks > 1: the two z-ghost planes hold the neighbours' boundary planes (received each
    // step, source index -(cell + 1) into the receive region; images in x/y of those cells
    // too); the periodic z shift applies on the ranks at z = 0 and z = Lz.
    std::vector<int> src(c->n_ecell), gd, gs, gsh;
    gd.reserve(c->n_gcell);
    const int npc = g.nc[0] * g.nc[1];
    const bool split = c->opt.nranks > 1 || c->opt.split_self;
    for (int iz = 0; iz < g.ez; ++iz)
        for (int iy = 0; iy < g.ey; ++iy)
            for (int ix = 0; ix < g.ex; ++ix) {
                int ec = (iz * g.ey + iy) * g.ex + ix;
                int cx = ix - 1, cy = iy - 1, cz = iz - 1;
                int sx = cx < 0 ? -1 : (cx >= g.nc[0] ? 1 : 0);
                int sy = cy < 0 ? -1 : (cy >= g.nc[1] ? 1 : 0);
                int sz = cz < 0 ? -1 : (cz >= g.nzl ? 1 : 0);
                int ox = cx - sx * g.nc[0], oy = cy - sy * g.nc[1], oz = cz - sz * g.nzl;
                if (split && sz != 0) {
                    const int rc = (sz < 0 ? 0 : npc) + oy * g.nc[0] + ox;
                    const int zs = (sz < 0 && g.z0 == 0) ? -1 : ((sz > 0 && g.z0 + g.nzl == g.nc[2]) ? 1 : 0);
                    src[ec] = -(rc + 1);
                    gd.push_back(ec);
                    gs.push_back(-(rc + 1));
                    gsh.push_back((sx + 1) | ((sy + 1) << 2) | ((zs + 1) << 4));
                    continue;
                }
                int oc = oc_of_lex[(oz * g.nc[1] + oy) * g.nc[0] + ox];
                src[ec] = oc;
                if (sx || sy || sz) {
                    gd.push_back(ec);
                    gs.push_back(((oz + 1) * g.ey + (oy + 1)) * g.ex + (ox + 1));
                    gsh.push_back((sx + 1) | ((sy + 1) << 2) | ((sz + 1) << 4));
                }
            }
    c->npc = npc;
    if (split) {
        TRY(dalloc(c, &c->send_cnt, 2 * npc));
        TRY(dalloc(c, &c->send_off, 2 * npc + 1));
        TRY(dalloc(c, &c->recv_cnt, 2 * npc));
        TRY(dalloc(c, &c->recv_off, 2 * npc + 1));
    }
    TRY(dalloc(c, &c->ecell_src, c->n_ecell));
    TRY(dalloc(c, &c->gc_dst, c->n_gcell));
    TRY(dalloc(c, &c->gc_src, c->n_gcell));
    TRY(dalloc(c, &c->gc_shift, c->n_gcell));
    CK(cudaMemcpy(c->ecell_src, src.data(), sizeof(int) * src.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->gc_dst, gd.data(), sizeof(int) * gd.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->gc_src, gs.data(), sizeof(int) * gs.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->gc_shift, gsh.data(), sizeof(int) * gsh.size(), cudaMemcpyHostToDevice));
    TRY(dalloc(c, &c->ocount, c->n_ocell));
    TRY(dalloc(c, &c->obegin, c->n_ocell + 1));
    TRY(dalloc(c, &c->ecount, c->n_ecell));
    TRY(dalloc(c, &c->ebegin, c->n_ecell + 1));
    return LJMD_OK;
}

ljmd_status alloc_owned(ljmd_ctx* c, int cap) {
    c->own_cap = cap;
    c->n_pad = (cap + 31) / 32 * 32;
    for (int b = 0; b < 2; ++b) {
        TRY(dalloc(c, &c->v[b], (size_t)3 * cap));
        TRY(dalloc(c, &c->gid[b], cap));
    }
    TRY(dalloc(c, &c->own_slot, cap));
    TRY(dalloc(c, &c->own_li, cap));
    TRY(dalloc(c, &c->ocell_of, cap));
    TRY(dalloc(c, &c->F, (size_t)3 * cap));
    TRY(dalloc(c, &c->e, cap));
    TRY(dalloc(c, &c->xw, cap));
    TRY(dalloc(c, &c->cell_of, cap));
    TRY(dalloc(c, &c->rank_in, cap));
    TRY(dalloc(c, &c->perm, cap));
    TRY(dalloc(c, &c->ncount, cap));
    TRY(dalloc(c, &c->img_cnt, cap));
    TRY(dalloc(c, &c->img_off, (size_t)cap + 1));
    TRY(dalloc(c, &c->d_stage, (size_t)3 * cap));
    TRY(dalloc(c, &c->xbuild, cap));   // dangerous-build test (and the safe policy's check)
    // force CTAs per tile: enough CTAs for two per SM on small systems (C1: 14 tiles -> 8 parts)
    c->fparts = c->newton3 ? 1 : std::max(1, std::min(8, (2 * 148 + c->n_tiles - 1) / c->n_tiles));
    c->n_fblocks = c->n_tiles * c->fparts;
    TRY(dalloc(c, &c->pe_part, c->n_fblocks));
    TRY(dalloc(c, &c->ke_part, c->n_fblocks));
    if (c->newton3) {
        TRY(dalloc(c, &c->ncount_h, cap));
        TRY(dalloc(c, &c->tmap, (size_t)c->n_global));
    }
    return LJMD_OK;
}

ljmd_status alloc_slots(ljmd_ctx* c, int cap, bool keep_current) {
    double4* nx[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b) {
        cudaError_t e = cudaMalloc(&nx[b], sizeof(double4) * ((size_t)cap + c->send_extra));
        if (e != cudaSuccess) {
            cudaGetLastError();
            if (nx[0]) cudaFree(nx[0]);
            return set_err(c, LJMD_E_CAPACITY, "cudaMalloc of %zu position slots failed", (size_t)cap);
        }
    }
    if (keep_current && c->x[c->xc])
        CK(cudaMemcpyAsync(nx[c->xc], c->x[c->xc], sizeof(double4) * (size_t)c->slot_cap,
                           cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int b = 0; b < 2; ++b) {
        if (c->x[b]) cudaFree(c->x[b]);
        c->x[b] = nx[b];
    }
    TRY(dalloc(c, &c->xf, cap));
    TRY(dalloc(c, &c->slot_gid, cap));
    TRY(dalloc(c, &c->gflat, (size_t)cap + c->send_extra));
    for (int b = 0; b < 2; ++b)
        TRY(dalloc(c, &c->xp[b], (size_t)3 * ((size_t)cap + c->send_extra) + 8));   // +8: bulk-copy overrun
    TRY(dalloc(c, &c->slot2t, cap));
    TRY(dalloc(c, &c->img, (size_t)cap + c->send_extra));
    TRY(dalloc(c, &c->grecv, cap));
    if (c->newton3 || c->dsl_on) {
        TRY(dalloc(c, &c->slot_t, cap));
        c->slot_t_valid = false;
    }
    c->slot_cap = cap;
    return LJMD_OK;
}

ljmd_status alloc_list(ljmd_ctx* c, int K) {
    c->K = K;
    TRY(dalloc(c, &c->nbr8, (size_t)(K / 8) * c->n_pad));
    if (c->newton3) TRY(dalloc(c, &c->nbr8h, (size_t)(K / 8) * c->n_pad));
    return LJMD_OK;
}

// ------------------------------------------------------------------ kernels launchers
// k_build_nlist dynamic shared memory: the staged fp32 halo
// (+ the per-thread x-windows of the flattened candidate loop)
inline size_t build_smem(const ljmd_ctx* c) { return 16 * (size_t)(c->stage_cap + 1) + 4 * (size_t)kBuildWinWords; }

// LJMD_SMALL_BUILD: 0 never, 2 always (measurement), default on small systems
int small_build_mode() {
    static const int m = [] {
        const char* e = getenv("LJMD_SMALL_BUILD");
        return e && *e ? atoi(e) : 1;
    }();
    return m;
}

ljmd_status launch_nlist(ljmd_ctx* c) {
    NlistArgs a;
    a.ctl = cctl(c);
    a.g = c->geo;
    a.x = c->x[c->xc];
    a.xf = c->xf;
    a.obegin = c->obegin;
    a.ocount = c->ocount;
    a.ebegin = c->ebegin;
    a.ecount = c->ecount;
    a.tr = TileRows{c->tr_begin, c->tr_off, c->tr_len};
    a.nbr8 = c->nbr8;
    a.ncount = c->ncount;
    a.n_own = c->n_own;
    a.n_pad = c->n_pad;
    a.K = c->K;
    a.ngx = (c->geo.nc[0] + 1) / 2;
    a.n_groups = a.ngx * c->geo.nc[1] * c->geo.nzl;
    a.rn2 = c->rn * c->rn;
    // Conservative fp32 band: per coordinate |x_f - x| <= 2^-24 X with
    // X = max |coordinate| <= L + 2w, the fp32 difference adds 2^-24 |dx_f|, so
    // |dx_f - dx| <= d = 2^-23 X + 2^-24 (R + 2^-23 X) for |dx| <= R = rbar_c + 1; the fp32
    // r^2 (two FMAs) then deviates from the exact r^2 by at most 3 d (2R + d) + 4 2^-24 R^2.
    // Outside [rn2 - E, rn2 + E] the fp32 value decides; inside, the canonical fp64 test.
    double X = 0.0;
    for (int d = 0; d < 3; ++d) X = std::max(X, c->geo.L[d] + 2.0 * c->geo.w[d]);
    const double R = c->rn + 1.0;
    const double dd = std::ldexp(X, -23) + std::ldexp(R + std::ldexp(X, -23), -24);
    const double E = 2.0 * (3.0 * dd * (2.0 * R + dd) + 4.0 * std::ldexp(R * R, -24)) + 1e-6;
    a.thr_lo = std::nextafter((float)(a.rn2 - E), 0.0f);
    a.thr_hi = std::nextafter((float)(a.rn2 + E), 1e30f);
    a.fl = c->d_fl;
    a.slot_gid = c->slot_gid;
    a.own_slot = c->own_slot;
    a.ocell_of = c->ocell_of;
    a.tile_oc0 = c->tile_oc0;
    a.ylo_f = c->ylo_f;
    a.zlo_f = c->zlo_f;
    // fp32 pruning margin: position conversion (2^-24 X twice), face conversion, sqrt/fma
    // roundings -- 16 x the coordinate ulp plus an absolute floor
    a.slop_f = (float)(16.0 * std::ldexp(X, -23) + 1e-5);
    a.stage_cap = c->stage_cap;
    a.parts = c->fparts;
    a.own_li = c->own_li;   // the force kernel's CTAs per tile (1 on large systems)
    if ((c->fparts > 1 && small_build_mode() == 1) || small_build_mode() == 2)   // small systems: a warp per particle
        k_build_nlist<true><<<c->n_tiles * c->fparts, kBuildThreads, build_smem(c), c->stream>>>(a);
    else
        k_build_nlist<false><<<c->n_tiles * c->fparts, kBuildThreads, build_smem(c), c->stream>>>(a);
    CKL();
    return LJMD_OK;
}

// the Newton-3 path moves particles in k_vv and refreshes every ghost slot per step instead
Images images(ljmd_ctx* c) {
    return c->newton3 ? Images{nullptr, nullptr} : Images{c->img_off, c->img};
}

ForceArgs force_args(ljmd_ctx* c) {
    ForceArgs a;
    const double s2 = c->sigma * c->sigma, s6 = s2 * s2 * s2, s12 = s6 * s6;
    a.g = c->geo;
    a.obegin = c->obegin;
    a.tile_oc0 = c->tile_oc0;
    a.tr = TileRows{c->tr_begin, c->tr_off, c->tr_len};
    a.x = c->x[c->xc];
    a.x_next = c->x[c->xc ^ 1];
    a.xp = c->xp[c->xc];
    a.xp_next = c->xp[c->xc ^ 1];
    a.own_slot = c->own_slot;
    a.own_li = c->own_li;
    a.nbr = c->nbr8;   // the last build's list, re-sequenced in place when use_rr
    a.ncount = c->ncount;
    a.fx = c->F;
    a.fy = c->F + c->own_cap;
    a.fz = c->F + 2 * (size_t)c->own_cap;
    double* v = c->v[c->oc_cur];
    a.vx = v;
    a.vy = v + c->own_cap;
    a.vz = v + 2 * (size_t)c->own_cap;
    a.e = c->e;
    a.pe_part = c->pe_part;
    a.ke_part = c->ke_part;
    a.xbuild = c->xbuild;
    a.im = images(c);
    a.fl = c->d_fl;
    a.n_own = c->n_own;
    a.n_pad = c->n_pad;
    a.rc2 = c->rc * c->rc;
    a.c12 = 48.0 * c->eps * s12;
    a.nc6 = -24.0 * c->eps * s6;
    a.a12 = 4.0 * c->eps * s12;
    a.na6 = -4.0 * c->eps * s6;
    a.a0 = 4.0 * c->eps * c->opt.energy_shift;
    a.h = 0.5 * c->dt / c->opt.mass;
    a.dt = c->dt;
    a.half_m = 0.5 * c->opt.mass;
    a.gid = c->gid[c->oc_cur];
    a.nu_dt = c->nu_dt;
    a.sd = c->thermo_sd;
    a.seed = c->thermo_seed;
    a.step = c->steps_done;
    a.ctl = c->capturing ? c->d_ctl : nullptr;
    a.parts = c->fparts;
    a.tile_base = 0;
    a.seg0 = INT_MAX;
    a.gap = 0;
    a.halo_flag = nullptr;
    a.halo_seq = 0;
    a.bfirst = 0;
    a.bdone = nullptr;
    a.nint = 0;
    a.layer = 0;
    return a;
}

constexpr size_t kStageBytes = 24;   // packed {x, y, z} per staged particle
// k_force dynamic shared memory: the staged halo (+ sentinel), then the list ring
inline size_t force_smem(const ljmd_ctx* c) {
    return (kStageBytes * (size_t)(c->stage_cap + 1) + 15) / 16 * 16 + 16 * (size_t)kRing * kForceThreads;
}

template <bool E, int M, bool C>
void force_launch(ljmd_ctx* c, const ForceArgs& a, int n_launch, cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
#if LJMD_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n_launch * c->fparts));
    cfg.blockDim = dim3(kForceThreads);
    cfg.dynamicSmemBytes = force_smem(c);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    // no programmatic overlap with a predecessor that wrote the list, the counts or the
    // halo-row tables (read before griddepcontrol.wait): only force -> force is overlapped
    cfg.numAttrs = c->pdl_ok ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_force<E, M, C>, a);
#else
    k_force<E, M, C><<<n_launch * c->fparts, kForceThreads, force_smem(c), st>>>(a);
#endif
}

template <bool E, int M, bool C>
cudaError_t force_attr() {
    return cudaFuncSetAttribute(k_force<E, M, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kMaxStageSmem);
}

ljmd_status set_force_attrs(ljmd_ctx* c) {
    cudaError_t e = cudaFuncSetAttribute(k_build_nlist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxStageSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_build_nlist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxStageSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_list_rr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRrSmem);
    constexpr int KT = kKick | kThermo, DT = kKKD | kThermo;
    for (cudaError_t r : {force_attr<true, kStore, false>(), force_attr<true, kKick, false>(),
                          force_attr<true, kKKD, false>(), force_attr<true, kKKD, true>(),
                          force_attr<false, kStore, false>(), force_attr<false, kKick, false>(),
                          force_attr<false, kKKD, false>(), force_attr<false, kKKD, true>(),
                          force_attr<true, KT, false>(), force_attr<true, DT, false>(), force_attr<true, DT, true>(),
                          force_attr<false, KT, false>(), force_attr<false, DT, false>(),
                          force_attr<false, DT, true>()})
        if (r != cudaSuccess) e = r;
    for (cudaError_t r : {cudaFuncSetAttribute(k_force_half<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               kMaxStageSmem),
                          cudaFuncSetAttribute(k_force_half<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               kMaxStageSmem)})
        if (r != cudaSuccess) e = r;
    if (e != cudaSuccess) return set_err(c, LJMD_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return LJMD_OK;
}

template <bool K2, bool E, bool KD, bool C, bool TH>
void vv_launch(ljmd_ctx* c, const VvArgs& v) {
    k_vv<K2, E, KD, C, TH><<<c->n_tiles, 256, 0, c->stream>>>(v);
}

// Newton-3 path (NEXT-1): zero F (and e), half-list force with reaction reductions, then
// the velocity-Verlet updates of `mode` on the completed F.
ljmd_status launch_half(ljmd_ctx* c, bool energy, int mode, bool check, cudaEvent_t e0, cudaEvent_t e1) {
    const size_t oc = c->own_cap;
    if (e0) CK(cudaEventRecord(e0, c->stream));
    TRY(zero_async(c, c->F, sizeof(double) * 3 * oc));
    if (energy) TRY(zero_async(c, c->e, sizeof(double) * oc));
    const double s2 = c->sigma * c->sigma, s6 = s2 * s2 * s2, s12 = s6 * s6;
    HalfArgs h;
    h.g = c->geo;
    h.x = c->x[c->xc];
    h.own_slot = c->own_slot;
    h.nbr = c->nbr8h;
    h.ncount = c->ncount_h;
    h.obegin = c->obegin;
    h.tile_oc0 = c->tile_oc0;
    h.slot_t = c->slot_t;
    h.tr = TileRows{c->tr_begin, c->tr_off, c->tr_len};
    h.fx = c->F;
    h.fy = c->F + oc;
    h.fz = c->F + 2 * oc;
    h.e = c->e;
    h.pe_part = c->pe_part;
    h.n_own = c->n_own;
    h.n_pad = c->n_pad;
    h.rc2 = c->rc * c->rc;
    h.c12 = 48.0 * c->eps * s12;
    h.nc6 = -24.0 * c->eps * s6;
    h.a12 = 4.0 * c->eps * s12;
    h.na6 = -4.0 * c->eps * s6;
    h.a0 = 4.0 * c->eps * c->opt.energy_shift;
    const size_t smem = (kStageBytes + sizeof(int)) * (size_t)(c->max_staged + 1) + 8;
    if (energy) k_force_half<true><<<c->n_tiles, kForceThreads, smem, c->stream>>>(h);
    else k_force_half<false><<<c->n_tiles, kForceThreads, smem, c->stream>>>(h);
    CKL();
    if (e1) CK(cudaEventRecord(e1, c->stream));
    double* v = c->v[c->oc_cur];
    VvArgs a;
    a.n_own = c->n_own;
    a.x = c->x[c->xc];
    a.x_next = c->x[c->xc ^ 1];
    a.own_slot = c->own_slot;
    a.vx = v;
    a.vy = v + oc;
    a.vz = v + 2 * oc;
    a.fx = c->F;
    a.fy = c->F + oc;
    a.fz = c->F + 2 * oc;
    a.ke_part = c->ke_part;
    a.xbuild = c->xbuild;
    a.fl = c->d_fl;
    a.gid = c->gid[c->oc_cur];
    a.h = 0.5 * c->dt / c->opt.mass;
    a.dt = c->dt;
    a.half_m = 0.5 * c->opt.mass;
    a.nu_dt = c->nu_dt;
    a.sd = c->thermo_sd;
    a.seed = c->thermo_seed;
    a.step = c->steps_done;
    const bool th = c->nu_dt > 0.0;
    if (mode == kStore) {
        if (!energy) return LJMD_OK;
        vv_launch<false, true, false, false, false>(c, a);
    } else if (mode == kKick) {
        if (energy) th ? vv_launch<true, true, false, false, true>(c, a) : vv_launch<true, true, false, false, false>(c, a);
        else th ? vv_launch<true, false, false, false, true>(c, a) : vv_launch<true, false, false, false, false>(c, a);
    } else if (check) {
        if (energy) th ? vv_launch<true, true, true, true, true>(c, a) : vv_launch<true, true, true, true, false>(c, a);
        else th ? vv_launch<true, false, true, true, true>(c, a) : vv_launch<true, false, true, true, false>(c, a);
    } else {
        if (energy) th ? vv_launch<true, true, true, false, true>(c, a) : vv_launch<true, true, true, false, false>(c, a);
        else th ? vv_launch<true, false, true, false, true>(c, a) : vv_launch<true, false, true, false, false>(c, a);
    }
    CKL();
    return LJMD_OK;
}

template <bool E, int M, bool C>
void force_range(ljmd_ctx* c, ForceArgs a, int first, int count, cudaStream_t st = nullptr, int seg0 = INT_MAX,
                 int gap = 0) {
    if (count <= 0) return;
    a.tile_base = first;
    a.seg0 = seg0;
    a.gap = gap;
    force_launch<E, M, C>(c, a, count, st);
}

// One force evaluation.  halo_pending (nranks > 1): the halo exchange of this step is in
// flight on aux_stream; the interior tile layers go first, the first and last z layers
// (whose halos hold the received planes) after ev_halo.  (Launching the boundary layers on
// aux_stream, concurrently with the interior, measured slower.)
template <bool E, int M, bool C>
void force_all(ljmd_ctx* c, const ForceArgs& a, bool halo_pending) {
    const int layer = c->geo.ntx * c->geo.nty;
    if (c->bdone) {
        // nranks > 1 (aux stream): one launch, boundary tile layers first; their completion
        // count lets the next halo exchange start while the interior tiles compute
        if (halo_pending) cudaStreamWaitEvent(c->stream, c->ev_halo, 0);
        ForceArgs g = a;
        g.bfirst = 1;
        g.bdone = c->bdone;
        g.nint = c->n_tiles - 2 * layer;
        g.layer = layer;
        c->bdone_issued += (unsigned)(2 * layer * c->fparts);
        force_range<E, M, C>(c, g, 0, c->n_tiles);
        return;
    }
    if (!halo_pending) {
        force_range<E, M, C>(c, a, 0, c->n_tiles);
        return;
    }
#if LJMD_HALO_GATE
    // one launch, interior tiles first; the boundary tiles wait in-kernel for the halo flag
    // (no programmatic overlap: an early-started next launch must not hold the SMs the halo
    // stream needs while boundary tiles wait)
    ForceArgs g = a;
    g.halo_flag = c->halo_flag;
    g.halo_seq = c->halo_seq;
    g.nint = c->n_tiles - 2 * layer;
    g.layer = layer;
    c->pdl_ok = false;
    force_range<E, M, C>(c, g, 0, c->n_tiles);
#else
    force_range<E, M, C>(c, a, layer, c->n_tiles - 2 * layer);
    cudaStreamWaitEvent(c->stream, c->ev_halo, 0);
    // both boundary layers in one launch (one wave instead of two)
    force_range<E, M, C>(c, a, 0, 2 * layer, nullptr, layer, c->n_tiles - 2 * layer);
#endif
}

ljmd_status launch_force(ljmd_ctx* c, bool energy, int mode, bool check, bool halo_pending = false) {
    if (c->newton3) {
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (c->opt.profile) {
            size_t k = (size_t)c->force_launches * 2;
            while (c->ev.size() < k + 2) {
                cudaEvent_t ev;
                CK(cudaEventCreate(&ev));
                c->ev.push_back(ev);
            }
            e0 = c->ev[k];
            e1 = c->ev[k + 1];
            ++c->force_launches;
        }
        return launch_half(c, energy, mode, check, e0, e1);
    }
    ForceArgs a = force_args(c);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->opt.profile) {
        size_t k = (size_t)c->force_launches * 2;
        while (c->ev.size() < k + 2) {
            cudaEvent_t ev;
            CK(cudaEventCreate(&ev));
            c->ev.push_back(ev);
        }
        e0 = c->ev[k];
        e1 = c->ev[k + 1];
        CK(cudaEventRecord(e0, c->stream));
    }
    constexpr int KT = kKick | kThermo, DT = kKKD | kThermo;
    const bool th = c->nu_dt > 0.0 && mode != kStore;
    const bool h = halo_pending;
    if (energy) {
        if (mode == kStore) force_all<true, kStore, false>(c, a, h);
        else if (mode == kKick) th ? force_all<true, KT, false>(c, a, h) : force_all<true, kKick, false>(c, a, h);
        else if (check) th ? force_all<true, DT, true>(c, a, h) : force_all<true, kKKD, true>(c, a, h);
        else th ? force_all<true, DT, false>(c, a, h) : force_all<true, kKKD, false>(c, a, h);
    } else {
        if (mode == kStore) force_all<false, kStore, false>(c, a, h);
        else if (mode == kKick) th ? force_all<false, KT, false>(c, a, h) : force_all<false, kKick, false>(c, a, h);
        else if (check) th ? force_all<false, DT, true>(c, a, h) : force_all<false, kKKD, true>(c, a, h);
        else th ? force_all<false, DT, false>(c, a, h) : force_all<false, kKKD, false>(c, a, h);
    }
    CKL();
    c->pdl_ok = true;
    if (c->opt.profile) {
        CK(cudaEventRecord(e1, c->stream));
        ++c->force_launches;
    }
    return LJMD_OK;
}

ljmd_status collect_profile(ljmd_ctx* c, int64_t first_launch) {
    if (!c->opt.profile) return LJMD_OK;
    for (int64_t k = first_launch; k < c->force_launches; ++k) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev[2 * k], c->ev[2 * k + 1]));
        c->force_ms += ms;
    }
    return LJMD_OK;
}

// cuStreamWaitValue32 through the runtime's driver entry point (no link against libcuda)
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32Fn stream_wait_value() {
    static const WaitValue32Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (WaitValue32Fn) nullptr;
        return reinterpret_cast<WaitValue32Fn>(p);
    }();
    return fn;
}

int getenv_int(const char* k, int d) {
    const char* v = getenv(k);
    return v && *v ? atoi(v) : d;
}

// Grouped exchange with the z neighbours, in the fixed order that also pairs correctly for
// nranks = 2 (both neighbours are the same rank): send (up, down), receive (from below,
// from above).  hi/lo payloads: what goes to the upper / lower neighbour.
ljmd_status exchange(ljmd_ctx* c, void* to_hi, size_t b_hi, void* to_lo, size_t b_lo, void* from_lo, size_t r_lo,
                     void* from_hi, size_t r_hi, cudaStream_t st = nullptr) {
    std::vector<Xfer> sends{{c->hi_rank, to_hi, b_hi}, {c->lo_rank, to_lo, b_lo}};
    std::vector<Xfer> recvs{{c->lo_rank, from_lo, r_lo}, {c->hi_rank, from_hi, r_hi}};
    std::string err;
    if (!c->tr->exchange(st ? st : c->stream, sends, recvs, err)) return set_err(c, LJMD_E_NCCL, "%s", err.c_str());
    return LJMD_OK;
}

ljmd_status allreduce(ljmd_ctx* c, double* dbuf, int n, bool max) {
    if (!c->tr) return LJMD_OK;
    std::string err;
    if (!c->tr->allreduce(c->stream, dbuf, n, max, err)) return set_err(c, LJMD_E_NCCL, "%s", err.c_str());
    return LJMD_OK;
}

// Halo: the boundary planes' positions travel to the neighbours' ghost planes, received
// after the slot range of the current position buffer (nranks > 1, every step).
ljmd_status halo_exchange(ljmd_ctx* c, cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    const int ns = c->n_send[0] + c->n_send[1];
    if (ns) {
        k_pack<<<nblk(ns, 256), 256, 0, st>>>(ns, c->send_idx, c->x[c->xc], c->slot_gid, c->send_buf);
        CKL();
    }
    double4* rx = c->x[c->xc] + c->n_slots;
    const size_t e = sizeof(double4);
    return exchange(c, c->send_buf + c->n_send[0], e * c->n_send[1], c->send_buf, e * c->n_send[0], rx,
                    e * c->n_recv[0], rx + c->n_recv[0], e * c->n_recv[1], st);
}

// Per step (nranks > 1): the send areas (written by the kernels that moved the particles)
// go to the neighbours and land in their ghost planes, positions and packed positions; the
// posting order pairs correctly also when both neighbours are one rank (p = 2).
ljmd_status halo_direct(ljmd_ctx* c, cudaStream_t st = nullptr, int buf = -1) {
    // double4 records (32 B: every slot aligned for the transfer); the packed copy the force
    // kernel stages is written for the two received planes right after
    if (!st) st = c->stream;
    if (buf < 0) buf = c->xc;
    double4* X = c->x[buf];
    const size_t base = (size_t)c->slot_cap;
    const size_t e4 = sizeof(double4);
    const size_t a0 = (size_t)c->area[0], a1 = (size_t)c->area[1];
    std::vector<Xfer> sends{{c->hi_rank, X + base + a0, e4 * a1}, {c->lo_rank, X + base, e4 * a0}};
    std::vector<Xfer> recvs{{c->lo_rank, X + c->gbeg[0], e4 * c->glen[0]}, {c->hi_rank, X + c->gbeg[1], e4 * c->glen[1]}};
    std::string err;
    if (!c->tr->exchange(st, sends, recvs, err)) return set_err(c, LJMD_E_NCCL, "%s", err.c_str());
    const int nr = c->glen[0] + c->glen[1];
    if (nr > 0) {
        k_xp_from_x<<<nblk(nr, 256), 256, 0, st>>>(c->gbeg[0], c->glen[0], c->gbeg[1], c->glen[1], X, c->xp[buf]);
        CKL();
    }
    return LJMD_OK;
}

// At a rebuild (nranks > 1): the send map of the direct-landing halo, appended to the image
// list gflat (so the kernels that move a boundary particle also write its send-area copies),
// and the send / ghost-plane extents (read by the host at the rebuild's next synchronisation).
ljmd_status send_map(ljmd_ctx* c) {
    const Geo& g = c->geo;
    const int np = g.ex * g.ey;
    if (!c->pl_cnt) {
        TRY(dalloc(c, &c->pl_cnt, 2 * (size_t)np));
        TRY(dalloc(c, &c->pl_off, 2 * (size_t)np + 1));
        CK(cudaHostAlloc(&c->h_pl, sizeof(int) * 8, cudaHostAllocMapped));
    }
    k_plane_ext_counts<<<nblk(2 * np, 256), 256, 0, c->stream>>>(g, c->ecount, c->pl_cnt);
    CKL();
    TRY(scan(c, c->pl_cnt, 2 * np, c->pl_off));
    const int zs0 = g.z0 == 0 ? 1 : 0, zs1 = g.z0 + g.nzl == g.nc[2] ? -1 : 0;
    k_send_map<<<nblk((int64_t)2 * np * 32, 256), 256, 0, c->stream>>>(g, c->ebegin, c->ecount, c->pl_off, c->slot_cap,
                                                                       zs0, zs1, c->gflat,
                                                                       c->slot_cap + c->send_extra, c->d_fl);
    CKL();
    TRY(to_host(c, c->h_pl + 0, c->pl_off + 2 * np, sizeof(int)));
    TRY(to_host(c, c->h_pl + 1, c->pl_off + np, sizeof(int)));
    TRY(to_host(c, c->h_pl + 2, c->ebegin, sizeof(int)));
    TRY(to_host(c, c->h_pl + 3, c->ebegin + np, sizeof(int)));
    TRY(to_host(c, c->h_pl + 4, c->ebegin + (size_t)(g.nzl + 1) * np, sizeof(int)));
    TRY(to_host(c, c->h_pl + 5, c->ebegin + c->n_ecell, sizeof(int)));
    return LJMD_OK;
}

ljmd_status refresh_ghosts(ljmd_ctx* c, bool at_build) {
    GhostCells gc{c->gc_dst, c->gc_src, c->gc_shift, c->n_gcell};
    int blocks = nblk((int64_t)c->n_gcell * 32, 256);
    if (c->n_gcell == 0) return LJMD_OK;
    if (at_build)
        k_ghost_refresh<true><<<blocks, 256, 0, c->stream>>>(gc, c->ebegin, c->ecount, c->geo, c->x[c->xc],
                                                             c->xf, c->slot_gid, c->recv_cnt, c->recv_off,
                                                             c->n_slots, c->gflat, c->xp[c->xc], c->d_fl, cctl(c));
    else if (c->n_gflat > 0)
        k_ghost_flat<<<nblk(c->n_gflat, 256), 256, 0, c->stream>>>(c->n_gflat, c->gflat, c->geo, c->x[c->xc],
                                                                    c->xp[c->xc]);
    CKL();
    return LJMD_OK;
}

// CSR of the ghost images of every owned particle (written by the kernels that move it) and
// the list of received-plane images; from the build-time ghost list
ljmd_status build_images(ljmd_ctx* c) {
    if (c->newton3 || (!dev_caps(c) && c->n_gflat == 0)) {
        TRY(zero_async(c, c->img_off, sizeof(int) * ((size_t)c->n_own + 1)));
        return LJMD_OK;
    }
    k_slot2t<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->own_slot, c->slot2t, c->img_cnt, cctl(c));
    CKL();
    // captured: the ghost count is only known on the device (grid over the slot capacity)
    const int ng = dev_caps(c) ? c->slot_cap : c->n_gflat;
    const int* ndev = dev_caps(c) ? &c->d_fl->n_gflat : nullptr;
    const int nsl = dev_caps(c) ? INT_MAX : c->n_slots;   // single rank: every source is local
    k_img_build<false><<<nblk(ng, 256), 256, 0, c->stream>>>(ng, c->gflat, nsl, c->slot2t, c->img_cnt, c->img_off,
                                                             c->img, c->grecv, c->d_fl, ndev, cctl(c));
    CKL();
    TRY(scan(c, c->img_cnt, c->n_own, c->img_off));
    k_img_build<true><<<nblk(ng, 256), 256, 0, c->stream>>>(ng, c->gflat, nsl, c->slot2t, c->img_cnt, c->img_off,
                                                            c->img, c->grecv, c->d_fl, ndev, cctl(c));
    CKL();
    return LJMD_OK;
}

// Particle migration: leavers of the slab go to the adjacent rank; stayers and
// arrivals are compacted into (xs, vs, gs), the input of the binning below.
ljmd_status migrate(ljmd_ctx* c) {
    const int n = c->n_own;
    CK(cudaMemsetAsync(c->mig_cnt, 0, sizeof(int) * 6, c->stream));
    const double* v = c->v[c->oc_cur];
    const size_t oc = c->own_cap;
    k_migrate_mark<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->x[c->xc], c->own_slot, v, v + oc, v + 2 * oc,
                                                       c->gid[c->oc_cur], c->geo, c->xs, c->vs, c->vs + oc,
                                                       c->vs + 2 * oc, c->gs, c->mig_send[0], c->mig_send[1],
                                                       c->mig_cap, c->mig_cnt, c->d_fl, c->stay_t);
    CKL();
    TRY(exchange(c, c->mig_cnt + 2, sizeof(int), c->mig_cnt + 1, sizeof(int), c->mig_cnt + 3, sizeof(int),
                 c->mig_cnt + 4, sizeof(int)));
    CK(cudaMemcpyAsync(c->h_mig, c->mig_cnt, sizeof(int) * 6, cudaMemcpyDeviceToHost, c->stream));
    TRY(sync_flags(c));
    if (c->h_fl->migrate_gid != INT_MAX)
        return set_err(c, LJMD_E_ARG, "particle %d moved more than one cell plane between rebuilds",
                       c->h_fl->migrate_gid);
    const int stay = c->h_mig[0], out_lo = c->h_mig[1], out_hi = c->h_mig[2];
    const int in_lo = c->h_mig[3], in_hi = c->h_mig[4];
    if (out_lo > c->mig_cap || out_hi > c->mig_cap || in_lo > c->mig_cap || in_hi > c->mig_cap)
        return set_err(c, LJMD_E_CAPACITY, "migration buffer overflow (%d/%d/%d/%d > %d)", out_lo, out_hi, in_lo,
                       in_hi, c->mig_cap);
    if (stay + in_lo + in_hi > c->own_cap)
        return set_err(c, LJMD_E_CAPACITY, "rank %d would own %d particles (capacity %d)", c->rank,
                       stay + in_lo + in_hi, c->own_cap);
    const size_t r = sizeof(MigRec);
    TRY(exchange(c, c->mig_send[1], r * out_hi, c->mig_send[0], r * out_lo, c->mig_recv[0], r * in_lo,
                 c->mig_recv[1], r * in_hi));
    if (in_lo) {
        k_migrate_append<<<nblk(in_lo, 256), 256, 0, c->stream>>>(in_lo, stay, c->mig_recv[0], c->xs, c->vs,
                                                                  c->vs + oc, c->vs + 2 * oc, c->gs);
        CKL();
    }
    if (in_hi) {
        k_migrate_append<<<nblk(in_hi, 256), 256, 0, c->stream>>>(in_hi, stay + in_lo, c->mig_recv[1], c->xs,
                                                                  c->vs, c->vs + oc, c->vs + 2 * oc, c->gs);
        CKL();
    }
    c->n_own = stay + in_lo + in_hi;
    TRY(dsl_migrate(c, stay, out_lo, out_hi, in_lo, in_hi));
    return LJMD_OK;
}

// Cell binning (counting sort + gid order), ghost images and the Verlet list
// (Sec. 3.4; IntegratorRange rebuild).
ljmd_status rebuild_dev_body(ljmd_ctx* c);

// the eager rebuild may run speculatively (one rank, no Newton-3 half list / DSL data hooks)
bool spec_ok(const ljmd_ctx* c) {
    return !c->split && !c->newton3 && !c->dsl_on && c->stage_cap > 0 && !c->capturing &&
           getenv_int("LJMD_SPEC_REBUILD", 1) != 0;
}

ljmd_status rebuild(ljmd_ctx* c, bool danger = true) {
    // Bank-aware re-ordering costs about 1.4 force launches and saves about 13 % of each
    // launch it serves (C2: 225 us against 21 us per step), so it pays for lists that serve
    // >= kRrMinSteps steps: always under the paper's fixed Ns = 20; under the displacement-
    // checked policy as long as the recent lists have lasted that long (running estimate of
    // the steps between rebuilds, starting at Ns).
    // The decision depends only on the rebuild history, so it is deterministic and the same
    // on every rank.
    constexpr double kRrMinSteps = 10.0;
    c->pdl_ok = false;   // the next force launch reads the new list: no programmatic overlap
    if (danger && c->last_build_step >= 0 && c->steps_done > c->last_build_step) {
        // dangerous-build test on the last step the old list served (x(s-1) in the other
        // position buffer, old layout), before the binning overwrites it
        k_maxdisp<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->x[c->xc ^ 1], c->own_slot,
                                                              c->xbuild, &c->d_st->disp_bits);
        CKL();
        TRY(allreduce(c, reinterpret_cast<double*>(&c->d_st->disp_bits), 1, true));
        k_dangerous<<<1, 1, 0, c->stream>>>(c->d_st, c->opt.delta * c->opt.delta);
        CKL();
    }
    if (c->last_build_step >= 0 && c->steps_done > c->last_build_step)
        c->interval_ema = 0.5 * c->interval_ema + 0.5 * (double)(c->steps_done - c->last_build_step);
    else if (c->interval_ema == 0.0)
        c->interval_ema = (double)c->opt.rebuild_every;
    c->last_build_step = c->steps_done;
    (void)kRrMinSteps;   // the list order is chosen per ljmd_step call (decide_list_order)
    TRY(reset_flags(c));
    TRY(zero_async(c, c->ocount, sizeof(int) * c->n_ocell));
    if (spec_ok(c)) {
        // speculative: the captured rebuild's kernels (capacities checked on the device), one
        // host wait at the end instead of three; a shortfall falls through to the sequence
        // below, which regrows it (abort 1: nothing permuted; 2: the new layout is in place)
        TRY(zero_async(c, c->d_ctl, offsetof(DevCtl, since)));
        c->spec = true;
        const ljmd_status r = rebuild_dev_body(c);
        c->spec = false;
        TRY(r);
        TRY(to_host(c, c->h_slots, c->ebegin + c->n_ecell, sizeof(int)));
        TRY(to_host(c, c->h_sctl, c->d_ctl, sizeof(DevCtl)));
        TRY(sync_flags(c));
        if (c->h_fl->nonfinite_gid != INT_MAX)
            return set_err(c, LJMD_E_NONFINITE, "non-finite position or velocity at particle %d",
                           c->h_fl->nonfinite_gid);
        if (!c->h_sctl->abort) {
            if (c->h_fl->overlap_pair != ~0ull)
                return set_err(c, LJMD_E_OVERLAP, "particles %d and %d coincide (r^2 == 0)",
                               (int)(c->h_fl->overlap_pair >> 32), (int)(c->h_fl->overlap_pair & 0xffffffffu));
            c->n_slots = *c->h_slots;
            c->max_staged = c->h_fl->max_staged;
            c->n_gflat = c->h_fl->n_gflat;
            c->n_grecv = c->h_fl->n_grecv;
            c->max_nbr = c->h_fl->max_nbr;
            c->total_nbr = c->h_fl->total_nbr;
            return LJMD_OK;
        }
        ++c->spec_aborts;
        TRY(zero_async(c, c->d_ctl, offsetof(DevCtl, since)));
        TRY(reset_flags(c));
        TRY(zero_async(c, c->ocount, sizeof(int) * c->n_ocell));
    }
    // input of the binning: the current owned particles, or the post-migration compaction
    const double4* xin = c->x[c->xc];
    const int* slot_in = c->own_slot;
    const double* vo = c->v[c->oc_cur];
    const int* gid_old = c->gid[c->oc_cur];
    if (c->split) {
        TRY(migrate(c));
        k_iota<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->iota);
        CKL();
        xin = c->xs;
        slot_in = c->iota;
        vo = c->vs;
        gid_old = c->gs;
    }
    const int n = c->n_own;
    const size_t oc = c->own_cap;
    // single rank: v and gid copied aside (v[1], gid[1]) for the in-place permutation below
    double* vcopy = c->split ? nullptr : c->v[1];
    int* gcopy = c->split ? nullptr : c->gid[1];
    k_wrap_bin<<<nblk(n, 256), 256, 0, c->stream>>>(n, xin, slot_in, c->geo, c->xw, c->ocount, c->cell_of,
                                                    c->rank_in, gid_old, c->d_fl, vo, vcopy, gcopy, (int)oc, nullptr);
    CKL();
    if (!c->split) {
        vo = c->v[1];
        gid_old = c->gid[1];
    }
    if (c->split) {   // boundary-plane cell counts -> the neighbours' ghost planes
        const int npc = c->npc;
        k_plane_counts<<<nblk(2 * npc, 256), 256, 0, c->stream>>>(c->geo, c->ocount, c->send_cnt);
        CKL();
        TRY(exchange(c, c->send_cnt + npc, sizeof(int) * npc, c->send_cnt, sizeof(int) * npc, c->recv_cnt,
                     sizeof(int) * npc, c->recv_cnt + npc, sizeof(int) * npc));
        TRY(scan(c, c->send_cnt, 2 * npc, c->send_off));
        TRY(scan(c, c->recv_cnt, 2 * npc, c->recv_off));
        CK(cudaMemcpyAsync(c->h_tot, c->send_off + npc, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(c->h_tot + 1, c->send_off + 2 * npc, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(c->h_tot + 2, c->recv_off + npc, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(c->h_tot + 3, c->recv_off + 2 * npc, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    }
    TRY(bin_offsets(c));
    TRY(to_host(c, c->h_slots, c->ebegin + c->n_ecell, sizeof(int)));
    TRY(sync_flags(c));
    if (c->h_fl->nonfinite_gid != INT_MAX)
        return set_err(c, LJMD_E_NONFINITE, "non-finite position or velocity at particle %d",
                       c->h_fl->nonfinite_gid);
    const int need = *c->h_slots;
    int n_recv_tot = 0;
    if (c->split) {
        c->n_send[0] = c->h_tot[0];
        c->n_send[1] = c->h_tot[1] - c->h_tot[0];
        c->n_recv[0] = c->h_tot[2];
        c->n_recv[1] = c->h_tot[3] - c->h_tot[2];
        n_recv_tot = c->h_tot[3];
        const int ns = c->h_tot[1];
        if (ns > c->send_cap) {
            c->send_cap = ns * 5 / 4 + 1024;
            TRY(dalloc(c, &c->send_idx, c->send_cap));
            TRY(dalloc(c, &c->send_buf, c->send_cap));
        }
    }
    if (need + n_recv_tot > c->slot_cap) {
        TRY(alloc_slots(c, (int)std::min<int64_t>((int64_t)(need + n_recv_tot) * 5 / 4 + 1024, INT_MAX), true));
        ++c->regrows;
    }
    c->n_slots = need;
    k_scatter<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->cell_of, c->rank_in, c->obegin, c->perm, cctl(c));
    CKL();
    // in place: the new layout goes into the current buffers (positions from xw, velocities
    // and gids from the copies), so no buffer pointer changes at a rebuild
    double* vn = c->v[0];
    double4* xn = c->x[c->xc];
    TRY(dsl_before_sort(c, gid_old));
    k_cell_sort<<<nblk((int64_t)c->n_ocell * 32, 256), 256, 0, c->stream>>>(
        c->n_ocell, c->geo, c->obegin, c->ocount, c->ebegin, c->perm, gid_old, c->xw, vo, vo + oc, vo + 2 * oc,
        xn, c->xf, vn, vn + oc, vn + 2 * oc, c->gid[0], c->own_slot, c->ocell_of, c->slot_gid,
        c->xbuild, c->xp[c->xc], c->d_fl, cctl(c));
    CKL();
    TRY(dsl_after_sort(c));
    if (c->split) {   // ghost planes: positions + gids of the neighbours' boundary planes
        k_plane_index<<<nblk((int64_t)2 * c->npc * 32, 256), 256, 0, c->stream>>>(c->geo, c->send_cnt,
                                                                                  c->send_off, c->ebegin,
                                                                                  c->send_idx);
        CKL();
        TRY(halo_exchange(c));
        if (n_recv_tot) {
            k_unpack_gid<<<nblk(n_recv_tot, 256), 256, 0, c->stream>>>(n_recv_tot, c->x[c->xc] + c->n_slots,
                                                                        c->slot_gid + c->n_slots);
            CKL();
        }
    }
    TRY(refresh_ghosts(c, true));
    if (c->split) TRY(send_map(c));
    k_tile_rows<<<nblk((int64_t)c->n_tiles * 32, 256), 256, 0, c->stream>>>(
        c->n_tiles, c->geo, c->ebegin, c->ecount, TileRows{c->tr_begin, c->tr_off, c->tr_len}, c->d_fl, cctl(c));
    CKL();
    TRY(sync_flags(c));
    c->max_staged = c->h_fl->max_staged;
    c->n_gflat = c->h_fl->n_gflat;
    if (c->split) {
        const int* h = c->h_pl;
        c->area[0] = h[1];
        c->area[1] = h[0] - h[1];
        c->gbeg[0] = h[2];
        c->glen[0] = h[3] - h[2];
        c->gbeg[1] = h[4];
        c->glen[1] = h[5] - h[4];
        // the send area (after slot_cap) and its image-list entries need room: regrow keeping
        // the current positions (the rebuild is past every read of the old ones)
        if (h[0] > c->send_extra || c->n_gflat > c->slot_cap + c->send_extra) {
            c->send_extra = std::max(h[0], c->n_gflat - c->slot_cap) * 5 / 4 + 1024;
            TRY(alloc_slots(c, c->slot_cap, true));
            ++c->regrows;
            return rebuild(c, false);   // the new layout is in place: bin it again with room
        }
    }
    if (c->max_staged > c->stage_cap) {   // launches are sized for stage_cap (also in graphs)
        c->stage_cap = c->max_staged + c->max_staged / LJMD_STAGE_MARGIN + 16;
        drop_graphs(c);
    }
    TRY(build_images(c));
    if (build_smem(c) > kMaxStageSmem || force_smem(c) > kMaxStageSmem || c->max_staged > 65535)
        return set_err(c, LJMD_E_CAPACITY,
                       "a force tile needs %d staged particles (> %zu B of shared memory): density too high",
                       c->max_staged, kMaxStageSmem);
    TRY(launch_nlist(c));
    TRY(sync_flags(c));
    c->n_grecv = c->h_fl->n_grecv;
    if (c->h_fl->overlap_pair != ~0ull)
        return set_err(c, LJMD_E_OVERLAP, "particles %d and %d coincide (r^2 == 0)",
                       (int)(c->h_fl->overlap_pair >> 32), (int)(c->h_fl->overlap_pair & 0xffffffffu));
    if (c->h_fl->max_nbr > c->K) {
        int K = (c->h_fl->max_nbr * 5 / 4 + 8) / 8 * 8;
        TRY(alloc_list(c, K));
        ++c->regrows;
        TRY(reset_flags(c));
        TRY(launch_nlist(c));
        TRY(sync_flags(c));
    }
    c->max_nbr = c->h_fl->max_nbr;
    c->total_nbr = c->h_fl->total_nbr;
    if (c->newton3) {
        const int* g = c->gid[c->oc_cur];
        k_cna_tmap<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, g, c->tmap);
        CKL();
        k_slot_owner<<<nblk(c->n_slots, 256), 256, 0, c->stream>>>(c->n_slots, c->slot_gid, c->tmap, c->slot_t);
        CKL();
        k_list_half<<<nblk(c->n_own, 128), 128, 0, c->stream>>>(c->n_own, c->n_pad, c->geo, c->nbr8, c->ncount,
                                                                 c->ocell_of, TileRows{c->tr_begin, c->tr_off, c->tr_len},
                                                                 c->slot_gid, g, c->nbr8h, c->ncount_h);
        CKL();
    } else if (c->use_rr) {
        k_list_rr<<<nblk(c->n_own, kRrThreads), kRrThreads, kRrSmem, c->stream>>>(
            c->n_own, c->n_pad, c->K, c->geo, c->nbr8, c->ncount, c->ocell_of, c->obegin, c->tile_oc0, c->nbr8, cctl(c));   // in place
        CKL();
    }

    return LJMD_OK;
}

// Validation mode: missed pairs of this step's positions (k_val_* in kernels.cuh), into row
// vslot of vhist.  Single rank, full list (checked at init).
ljmd_status validate_step(ljmd_ctx* c, int vslot) {
    const Geo& g = c->geo;
    const int ncell = g.nc[0] * g.nc[1] * g.nc[2];
    if (!c->vcount) {
        TRY(dalloc(c, &c->vcount, ncell));
        TRY(dalloc(c, &c->vbegin, (size_t)ncell + 1));
        TRY(dalloc(c, &c->vcell, c->own_cap));
        TRY(dalloc(c, &c->vrank, c->own_cap));
        TRY(dalloc(c, &c->vpos, c->own_cap));
    }
    const int n = c->n_own;
    CK(cudaMemsetAsync(c->vcount, 0, sizeof(int) * (size_t)ncell, c->stream));
    k_val_bin<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->x[c->xc], c->own_slot, g, c->vcount, c->vcell, c->vrank);
    CKL();
    TRY(scan(c, c->vcount, ncell, c->vbegin));
    k_val_scatter<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->x[c->xc], c->own_slot, c->vcell, c->vrank, c->vbegin,
                                                       c->vpos);
    CKL();
    ValArgs a;
    a.g = g;
    a.x = c->x[c->xc];
    a.own_slot = c->own_slot;
    a.vcell = c->vcell;
    a.vbegin = c->vbegin;
    a.vpos = c->vpos;
    a.nbr = reinterpret_cast<const unsigned short*>(c->nbr8);
    a.ncount = c->ncount;
    a.ocell_of = c->ocell_of;
    a.tr = TileRows{c->tr_begin, c->tr_off, c->tr_len};
    a.n_own = n;
    a.n_pad = c->n_pad;
    a.rc2 = c->rc * c->rc;
    a.vhist = c->vhist;
    a.vslot = vslot;
    a.fl = c->d_fl;
    k_val_count<<<nblk(n, 256), 256, 0, c->stream>>>(a);
    CKL();
    return LJMD_OK;
}


// ---------------------------------------------------------------------- graph mode (one rank)
// ljmd_step as a CUDA graph: the step sequence of a call is captured once per shape (steps,
// buffer parity, schedule phase, list order) and replayed.  The rebuild is a conditional node
// whose condition is set on the device (reading R7: fixed Ns, or the displacement check), and
// its capacity checks are device-side too, so a call runs without a single host round trip;
// the host reads the step control (rebuild steps, samples, abort) at the end of the call.  A
// capacity shortfall aborts the rest of the sequence and the host resumes at that step on
// the eager path with regrown buffers (same arithmetic, same results).
// Profilers and sanitizers cannot see the kernels of a graph with conditional nodes (ncu:
// "not supported for profiling"), so under a CUDA injection tool (ncu, compute-sanitizer:
// detected by the environment they give the target) -- or with LJMD_GRAPHS=0 -- the same kernels
// run on the eager path instead.
bool graphs_allowed() {
    static const bool ok = [] {
        // ncu sets NV_NSIGHT_INJECTION_TRANSPORT_TYPE, compute-sanitizer
        // NV_SANITIZER_INJECTION_TRANSPORT_TYPE (measured on the B200 box; neither exports
        // CUDA_INJECTION64_PATH to the target)
        for (const char* v : {"CUDA_INJECTION64_PATH", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                              "NV_SANITIZER_INJECTION_TRANSPORT_TYPE"}) {
            const char* e = getenv(v);
            if (e && *e) return false;
        }
        const char* env = getenv("LJMD_GRAPHS");
        return !(env && env[0] == '0');
    }();
    return ok;
}

bool graph_ok(const ljmd_ctx* c) {
    return c->opt.graphs && graphs_allowed() && !c->split && !c->newton3 && !c->opt.validate && !c->opt.profile &&
           c->nu_dt == 0.0 && !c->dsl_on && c->stage_cap > 0;
}

// Launch `setter(handle)` on c->stream (being captured), then an IF node after it whose body is
// captured from `fn` on `body` (c->stream points there while fn runs).
template <class Setter, class Body>
ljmd_status cond_if(ljmd_ctx* c, cudaStream_t body, Setter setter, Body fn) {
    cudaStream_t st = c->stream;
    cudaStreamCaptureStatus cs;
    cudaGraph_t g;
    const cudaGraphNode_t* deps;
    size_t nd;
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    setter(h);
    CKL();
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams prm = {};
    prm.type = cudaGraphNodeTypeConditional;
    prm.conditional.handle = h;
    prm.conditional.type = cudaGraphCondTypeIf;
    prm.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, deps, nd, &prm));
    CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(body, prm.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    c->stream = body;
    const ljmd_status r = fn();
    c->stream = st;
    cudaGraph_t tmp;
    const cudaError_t e = cudaStreamEndCapture(body, &tmp);
    if (r != LJMD_OK) return r;
    if (e != cudaSuccess) return set_err(c, LJMD_E_CUDA, "capture of a conditional body: %s", cudaGetErrorString(e));
    return LJMD_OK;
}

// The rebuild of one step inside a captured sequence (single rank): the eager rebuild's
// kernels without its host synchronisations, capacities checked on the device in three
// stages (slots before anything is permuted; staging after the tile tables; list width
// after the build); a failed check makes the rest return at entry.
// record_step > 0: the fixed schedule's rebuild of that step (the decision record folded in)
ljmd_status rebuild_captured(ljmd_ctx* c, int record_step) {
    const int n = c->n_own;
    k_maxdisp_z<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->x[c->xc ^ 1], c->own_slot, c->xbuild,
                                                     &c->d_st->disp_bits, c->ocount, c->n_ocell, c->d_ctl, c->d_fl,
                                                     c->d_rstep, record_step);
    CKL();
    k_dangerous_reset<<<1, 1, 0, c->stream>>>(c->d_st, c->opt.delta * c->opt.delta, c->d_fl, c->d_ctl);
    CKL();
    return rebuild_dev_body(c);
}

// The rebuild from the binning on, capacities checked on the device (a failed check makes the
// rest return at entry): the body of a captured rebuild and of the speculative eager one.
ljmd_status rebuild_dev_body(ljmd_ctx* c) {
    const int n = c->n_own;
    const size_t oc = c->own_cap;
    k_wrap_bin<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->x[c->xc], c->own_slot, c->geo, c->xw, c->ocount, c->cell_of,
                                                    c->rank_in, c->gid[0], c->d_fl, c->v[0], c->v[1], c->gid[1],
                                                    (int)oc, c->d_ctl);
    CKL();
    TRY(bin_offsets(c));
    DevCtl* ctl = c->d_ctl;
    DevFlags* fl = c->d_fl;
    const int* need = c->ebegin + c->n_ecell;
    const int slot_cap = c->slot_cap, stage_cap = c->stage_cap, K = c->K;
    // stage 1 before anything is permuted; a failed check makes every later kernel of the
    // sequence return at entry (round 2: in-kernel checks instead of two nested conditional
    // nodes, whose body launches cost ~4 us each on the device timeline)
    if (!(c->n_ocell <= kScanSingle && c->n_ecell <= kScanSingle)) {   // else folded into the offsets
        k_check_caps<<<1, 1, 0, c->stream>>>(ctl, fl, need, slot_cap, stage_cap, K, 1);
        CKL();
    }
    k_scatter<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->cell_of, c->rank_in, c->obegin, c->perm, cctl(c));
    CKL();
    double* vo = c->v[1];
    k_cell_sort<<<nblk((int64_t)c->n_ocell * 32, 256), 256, 0, c->stream>>>(
        c->n_ocell, c->geo, c->obegin, c->ocount, c->ebegin, c->perm, c->gid[1], c->xw, vo, vo + oc,
        vo + 2 * oc, c->x[c->xc], c->xf, c->v[0], c->v[0] + oc, c->v[0] + 2 * oc, c->gid[0], c->own_slot,
        c->ocell_of, c->slot_gid, c->xbuild, c->xp[c->xc], c->d_fl, cctl(c));
    CKL();
    TRY(refresh_ghosts(c, true));
    k_tile_rows<<<nblk((int64_t)c->n_tiles * 32, 256), 256, 0, c->stream>>>(
        c->n_tiles, c->geo, c->ebegin, c->ecount, TileRows{c->tr_begin, c->tr_off, c->tr_len}, c->d_fl, cctl(c));
    CKL();
    k_check_caps<<<1, 1, 0, c->stream>>>(ctl, fl, need, slot_cap, stage_cap, K, 2);
    CKL();
    TRY(build_images(c));
    TRY(launch_nlist(c));
    k_check_caps<<<1, 1, 0, c->stream>>>(ctl, fl, need, slot_cap, stage_cap, K, 3);
    CKL();
    if (c->use_rr) {
        k_list_rr<<<nblk(n, kRrThreads), kRrThreads, kRrSmem, c->stream>>>(
            n, c->n_pad, c->K, c->geo, c->nbr8, c->ncount, c->ocell_of, c->obegin, c->tile_oc0, c->nbr8, cctl(c));   // in place
        CKL();
    }
    return LJMD_OK;
}

// The list order of the rebuilds of one ljmd_step call (eager and graph paths alike): the
// bank-aware pass costs ~1.4 force launches and saves ~13 % of each launch it serves, so it is
// used while the recent lists have served >= 10 steps (running estimate of the rebuild
// interval, starting at Ns): always under the paper's fixed Ns = 20.  Deterministic, the same
// on every rank.
// Small systems (several force CTAs per tile) keep the build order: their pair loops are
// latency-bound, not shared-memory-bound, and the pass is a per-thread chain of ~5000
// instructions (C1: 17.2 -> 16.7 us per MD step without it).
void decide_list_order(ljmd_ctx* c, int64_t call) {
    if (c->interval_ema == 0.0) c->interval_ema = (double)c->opt.rebuild_every;
    // call k (or a new state before call k): the estimate as of the end of call k - 2, known
    // before call k is queued also while call k - 1 is unsettled (deferred settlement), so the
    // eager, synchronous-graph and deferred paths take the same decision
    const double e = call >= 2 ? c->ema_after[(call - 2) & 3] : (double)c->opt.rebuild_every;
    c->use_rr = c->bank_order && e >= 10.0 && c->fparts == 1;
}

// bookkeeping of one rebuild at MD step `step` (eager and graph paths)
void note_rebuild(ljmd_ctx* c, int64_t step) {
    ++c->n_rebuilds;
    c->rebuild_steps.push_back(step);
}

ljmd_status ensure_hist(ljmd_ctx* c, int64_t need) {
    if (need <= c->hist_cap) return LJMD_OK;
    int64_t cap = std::max<int64_t>(need, 64);
    TRY(dalloc(c, &c->hist, (size_t)2 * cap));
    c->hist_cap = cap;
    return LJMD_OK;
}

ljmd_status finalize_energy(ljmd_ctx* c, double* dst) {
    k_finalize_energy<<<1, 1024, 0, c->stream>>>(c->pe_part, c->ke_part, c->n_tiles * (c->newton3 ? 1 : c->fparts), dst,
                                                 c->capturing ? c->d_ctl : nullptr);
    CKL();
    return LJMD_OK;
}

ljmd_status pull_hist(ljmd_ctx* c, int64_t count) {
    if (count <= 0) return LJMD_OK;
    if (count > c->h_histm_cap) {
        if (c->h_histm) cudaFreeHost(c->h_histm);
        c->h_histm = nullptr;
        c->h_histm_cap = 0;
        CK(cudaHostAlloc(&c->h_histm, sizeof(double) * 2 * (size_t)count, cudaHostAllocMapped));
        c->h_histm_cap = count;
    }
    TRY(to_host(c, c->h_histm, c->hist, sizeof(double) * 2 * (size_t)count));
    CK(cudaStreamSynchronize(c->stream));
    c->h_hist.insert(c->h_hist.end(), c->h_histm, c->h_histm + 2 * count);
    return LJMD_OK;
}

// init sequence shared by ljmd_init and ljmd_set_state; dpos/dvel != null: the state is
// already on the device (a staged state, single rank)
ljmd_status load_state(ljmd_ctx* c, const double* pos, const double* vel, const double* dpos_in = nullptr,
                       const double* dvel_in = nullptr) {
    int64_t n = c->n_global;
    std::vector<double> fp, fv;
    std::vector<int> fg;
    if (c->split) {
        // initial owner by z plane, computed on the host; the first rebuild's migration
        // corrects the rare plane-boundary disagreement with the device binning
        const Geo& g = c->geo;
        for (int64_t i = 0; i < n; ++i) {
            double z = pos[3 * i + 2];
            if (!std::isfinite(z)) return set_err(c, LJMD_E_NONFINITE, "non-finite position at particle %lld",
                                                  (long long)i);
            z = z - g.L[2] * std::floor(z / g.L[2]);
            int cz = (int)std::floor(z / g.w[2]);
            cz = std::min(std::max(cz, 0), g.nc[2] - 1);
            if (cz < g.z0 || cz >= g.z0 + g.nzl) continue;
            for (int d = 0; d < 3; ++d) {
                fp.push_back(pos[3 * i + d]);
                fv.push_back(vel[3 * i + d]);
            }
            fg.push_back((int)i);
        }
        n = (int64_t)fg.size();
        if (n > c->own_cap) return set_err(c, LJMD_E_CAPACITY, "slab holds %lld particles (capacity %d)",
                                           (long long)n, c->own_cap);
        pos = fp.data();
        vel = fv.data();
    }
    // persistent staging (allocated once: a per-call cudaMalloc/cudaFree would serialise the
    // device and dominate set_state)
    if (!c->ld_pos) {
        TRY(dalloc(c, &c->ld_pos, (size_t)3 * c->n_global));
        TRY(dalloc(c, &c->ld_vel, (size_t)3 * c->n_global));
        if (c->split) TRY(dalloc(c, &c->ld_gid, (size_t)c->n_global));
    }
    const double* dpos = c->ld_pos;
    const double* dvel = c->ld_vel;
    int* dg = nullptr;
    if (dpos_in) {
        dpos = dpos_in;
        dvel = dvel_in;
    } else {
        CK(cudaMemcpyAsync(c->ld_pos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->ld_vel, vel, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    }
    if (c->split) {
        dg = c->ld_gid;
        CK(cudaMemcpyAsync(dg, fg.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    }
    TRY(dsl_to_gid_order(c));   // particle data keeps its rows across a new state
    TRY(reset_flags(c));
    c->oc_cur = 0;
    c->xc = 0;
    double* v = c->v[0];
    const size_t oc = c->own_cap;
    k_load_rows<<<nblk(n, 256), 256, 0, c->stream>>>((int)n, dpos, dvel, c->x[0], v, v + oc, v + 2 * oc,
                                                    c->gid[0], c->own_slot, dg, c->d_fl);
    CKL();
    if (dpos_in) {   // the staged buffer may be refilled once this kernel has read it
        const int b = dpos_in == c->stg[0] ? 0 : 1;
        CK(cudaEventRecord(c->stg_used[b], c->stream));
    }
    // one rank: the non-finite flag (kept by reset_flags) is read at the rebuild's first
    // synchronisation (k_wrap_bin bins a non-finite particle harmlessly); several ranks
    // check before the migration
    if (c->split) {
        TRY(sync_flags(c));
        if (c->h_fl->nonfinite_gid != INT_MAX)
            return set_err(c, LJMD_E_NONFINITE, "non-finite position or velocity at particle %d",
                           c->h_fl->nonfinite_gid);
    }
    c->init_pending = false;
    c->n_own = (int)n;
    c->since = 0;
    c->dev_since_ok = false;
    c->steps_done = 0;
    c->n_rebuilds = 0;
    c->rebuild_steps.clear();
    c->h_hist.clear();
    c->h_val.clear();
    c->last_build_step = -1;
    TRY(zero_async(c, c->d_st, sizeof(DevStats)));
    decide_list_order(c, c->ncalls);
    TRY(rebuild(c));
    TRY(ensure_hist(c, 1));
    TRY(launch_force(c, true, kStore, false));
    TRY(finalize_energy(c, c->hist));
    TRY(allreduce(c, c->hist, 2, false));
    if (!c->h_init) CK(cudaHostAlloc(&c->h_init, sizeof(double) * 2, cudaHostAllocMapped));
    TRY(to_host(c, c->h_init, c->hist, sizeof(double) * 2));   // no host wait (settle_init)
    c->init_pending = true;
    c->init_current = true;
    c->energy_current = true;
    return LJMD_OK;
}

// The init sequence's energies: first entry of the history; the current PE/KE while no step
// has run since.  Waits for the stream (callers are at a synchronisation point anyway).
ljmd_status settle_init(ljmd_ctx* c) {
    if (!c->init_pending) return LJMD_OK;
    CK(cudaStreamSynchronize(c->stream));
    c->h_hist.insert(c->h_hist.begin(), c->h_init, c->h_init + 2);
    if (c->init_current) {
        c->cur_pe = c->h_init[0];
        c->cur_ke = c->h_init[1];
    }
    c->init_pending = false;
    return LJMD_OK;
}

// PE, KE and e_i of the current state: reused when the last step of the previous
// ljmd_step call (or the init sequence) sampled them, otherwise one Energy force pass
ljmd_status energy_now(ljmd_ctx* c) {
    TRY(settle_init(c));
    if (c->energy_current) return LJMD_OK;
    TRY(launch_force(c, true, kStore, false));
    TRY(ensure_hist(c, 1));
    double* tmp = c->hist + 2 * (c->hist_cap - 1);
    TRY(finalize_energy(c, tmp));
    TRY(allreduce(c, tmp, 2, false));
    if (c->h_histm_cap < 1) {
        CK(cudaHostAlloc(&c->h_histm, sizeof(double) * 2, cudaHostAllocMapped));
        c->h_histm_cap = 1;
    }
    TRY(to_host(c, c->h_histm, tmp, sizeof(double) * 2));
    CK(cudaStreamSynchronize(c->stream));
    c->cur_pe = c->h_histm[0];
    c->cur_ke = c->h_histm[1];
    c->energy_current = true;
    return LJMD_OK;
}

ljmd_status check_ctx(ljmd_ctx* c) {
    if (!c) return LJMD_E_ARG;
    if (c->err != LJMD_OK) return LJMD_E_STATE;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return set_err(c, LJMD_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    return LJMD_OK;
}

// host scatter of a compact owned-space [n_own][3] (or [n_own]) array into caller rows
ljmd_status readback(ljmd_ctx* c, const double* dsrc, int width, double* out) {
    if (!c->split && c->ld_pos && c->n_own == c->n_global) {
        // single rank: scatter into caller order on the device, one D2H copy into `out`
        k_rows_to_gid<<<nblk((int64_t)c->n_own * width, 256), 256, 0, c->stream>>>(c->n_own, width,
                                                                                    c->gid[c->oc_cur], dsrc,
                                                                                    c->ld_pos);
        CKL();
        CK(cudaMemcpyAsync(out, c->ld_pos, sizeof(double) * width * (size_t)c->n_own, cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return LJMD_OK;
    }
    std::vector<double> tmp((size_t)width * c->n_own);
    std::vector<int> g(c->n_own);
    CK(cudaMemcpyAsync(tmp.data(), dsrc, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g.data(), c->gid[c->oc_cur], sizeof(int) * g.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int t = 0; t < c->n_own; ++t)
        for (int k = 0; k < width; ++k) out[(size_t)g[t] * width + k] = tmp[(size_t)t * width + k];
    return LJMD_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

// the last ljmd_step call's results on the host (deferred settlement); defined below
ljmd_status settle(ljmd_ctx* c);

// API entry that reads or changes the state: the context is usable and every queued
// ljmd_step call has been settled (its errors surface here)
static ljmd_status check_ready(ljmd_ctx* c) {
    TRY(check_ctx(c));
    return settle(c);
}

const char* ljmd_version(void) { return "ljmd 0.1 sm_100a"; }

ljmd_status ljmd_default_options(ljmd_options* o) {
    if (!o) return LJMD_E_ARG;
    std::memset(o, 0, sizeof *o);
    o->delta = 0.25;
    o->rebuild_every = 20;
    o->rebuild_check = 0;
    o->mass = 1.0;
    o->energy_shift = 0.25;
    o->energy_every = 10;
    o->device = -1;
    o->nbr_capacity = 0;
    o->rank = 0;
    o->nranks = 1;
    o->nccl_id = nullptr;
    o->stream = nullptr;
    o->profile = 0;
    o->list_order = 1;
    o->split_self = 0;
    o->newton3 = 0;
    o->validate = 0;
    o->graphs = 1;
    return LJMD_OK;
}

ljmd_status ljmd_plan_cells(const double box[3], double rbar_c, int64_t nc[3]) {
    if (!box || !nc || !(rbar_c > 0.0)) return LJMD_E_ARG;
    for (int d = 0; d < 3; ++d) {
        if (!(box[d] > 0.0) || !std::isfinite(box[d])) return LJMD_E_ARG;
        double q = std::floor(box[d] / (rbar_c * (1.0 + 1e-12)));
        if (q < 3.0) return LJMD_E_BOX;
        if (q > 1e6) return LJMD_E_ARG;
        nc[d] = (int64_t)q;
    }
    return LJMD_OK;
}

ljmd_status ljmd_plan_slab(int64_t ncz, int64_t nranks, int64_t rank, int64_t* z0, int64_t* z1) {
    if (!z0 || !z1 || nranks < 1 || rank < 0 || rank >= nranks) return LJMD_E_ARG;
    if (ncz < 3 || ncz < nranks) return LJMD_E_BOX;
    int64_t base = ncz / nranks, extra = ncz % nranks;
    *z0 = rank * base + std::min(rank, extra);
    *z1 = *z0 + base + (rank < extra ? 1 : 0);
    return LJMD_OK;
}

ljmd_status ljmd_init(ljmd_ctx** out, int64_t n, const double* pos, const double* vel, const double box[3],
                      double rc, double epsilon, double sigma, double dt, const ljmd_options* opt) {
    if (out) *out = nullptr;
    if (!out || !pos || !vel || !box || n <= 0 || n > INT_MAX / 2)
        return set_err(nullptr, LJMD_E_ARG, "ljmd_init: bad pointer or n = %lld", (long long)n);
    if (!(rc > 0.0) || !(epsilon > 0.0) || !(sigma > 0.0) || !(dt > 0.0) || !std::isfinite(rc) ||
        !std::isfinite(dt))
        return set_err(nullptr, LJMD_E_ARG, "ljmd_init: rc, epsilon, sigma and dt must be positive and finite");
    ljmd_options o;
    ljmd_default_options(&o);
    if (opt) o = *opt;
    if (!(o.delta >= 0.0) || o.rebuild_every < 1 || !(o.mass > 0.0) || o.energy_every < 0)
        return set_err(nullptr, LJMD_E_ARG, "ljmd_init: bad options (delta >= 0, rebuild_every >= 1, mass > 0)");
    if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks)
        return set_err(nullptr, LJMD_E_ARG, "ljmd_init: bad rank %lld / nranks %lld", (long long)o.rank,
                       (long long)o.nranks);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(nullptr, LJMD_E_CUDA, "ljmd_init: no CUDA device");
    }
    ljmd_ctx* c = new ljmd_ctx();
    c->opt = o;
    c->n_global = n;
    c->rc = rc;
    c->eps = epsilon;
    c->sigma = sigma;
    c->dt = dt;
    c->rn = rc + o.delta;
    c->bank_order = o.list_order != 0;
    c->newton3 = o.newton3 != 0;
    if (c->newton3 && (o.nranks > 1 || o.split_self)) {
        delete c;
        return set_err(nullptr, LJMD_E_ARG, "ljmd_init: newton3 needs nranks = 1 (no reverse halo)");
    }
    if (o.validate && (o.nranks > 1 || o.split_self || o.newton3)) {
        delete c;
        return set_err(nullptr, LJMD_E_ARG, "ljmd_init: validate needs nranks = 1 and the full list");
    }
    auto fail = [&](ljmd_status s) {
        g_init_error = c->msg.empty() ? std::string("ljmd_init failed") : c->msg;
        ljmd_destroy(c);
        return s;
    };
    if (o.device >= 0) {
        if (cudaSetDevice((int)o.device) != cudaSuccess) {
            set_err(c, LJMD_E_CUDA, "cudaSetDevice(%lld) failed", (long long)o.device);
            return fail(LJMD_E_CUDA);
        }
    }
    cudaGetDevice(&c->device);
    if (o.stream) {
        c->stream = (cudaStream_t)o.stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            set_err(c, LJMD_E_CUDA, "cudaStreamCreate failed");
            return fail(LJMD_E_CUDA);
        }
        c->own_stream = true;
    }
    ljmd_status s;
    c->rank = (int)o.rank;
    c->nranks = (int)o.nranks;
    c->lo_rank = (c->rank - 1 + c->nranks) % c->nranks;
    c->hi_rank = (c->rank + 1) % c->nranks;
    c->split = c->nranks > 1 || o.split_self != 0;
    if (c->split) {
        std::string terr;
        c->tr = make_transport(o.nccl_id, c->rank, c->nranks, c->device, terr);
        if (!c->tr) {
            set_err(c, LJMD_E_NCCL, "%s", terr.c_str());
            return fail(LJMD_E_NCCL);
        }
    }
    if ((s = plan_geometry(c, box)) != LJMD_OK) return fail(s);
    // overlapped halo (nranks > 1, not Newton-3): needs interior tile layers besides the two
    // boundary ones
    if (c->split && !c->newton3 && c->geo.ntz >= 3) {
        if (cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming) != cudaSuccess) {
            set_err(c, LJMD_E_CUDA, "aux stream creation failed");
            return fail(LJMD_E_CUDA);
        }
        if (cudaMalloc(&c->halo_flag, sizeof(unsigned)) != cudaSuccess ||
            cudaMemset(c->halo_flag, 0, sizeof(unsigned)) != cudaSuccess) {
            set_err(c, LJMD_E_CUDA, "halo flag allocation failed");
            return fail(LJMD_E_CUDA);
        }
        // boundary-first launches with the halo started from a stream memory wait (when the
        // driver offers cuStreamWaitValue32; else the interior / boundary split launches)
        if (stream_wait_value() && getenv_int("LJMD_BFIRST", 1)) {
            if (cudaMalloc(&c->bdone, sizeof(unsigned)) != cudaSuccess ||
                cudaMemset(c->bdone, 0, sizeof(unsigned)) != cudaSuccess) {
                set_err(c, LJMD_E_CUDA, "halo counter allocation failed");
                return fail(LJMD_E_CUDA);
            }
        }
    }
    if ((s = set_force_attrs(c)) != LJMD_OK) return fail(s);
    if (cudaMalloc(&c->d_fl, sizeof(DevFlags)) != cudaSuccess ||
        cudaMalloc(&c->d_ctl, sizeof(DevCtl)) != cudaSuccess ||
        cudaMalloc(&c->d_st, sizeof(DevStats)) != cudaSuccess ||
        cudaHostAlloc(&c->h_st, sizeof(DevStats), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostAlloc(&c->h_fl, sizeof(DevFlags), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostAlloc(&c->h_slots, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostAlloc(&c->h_sctl, sizeof(DevCtl), cudaHostAllocMapped) != cudaSuccess) {
        set_err(c, LJMD_E_CUDA, "flag allocation failed");
        return fail(LJMD_E_CUDA);
    }
    k_reset_flags<<<1, 1, 0, c->stream>>>(c->d_fl, 0);
    cudaMemsetAsync(c->d_ctl, 0, sizeof(DevCtl), c->stream);
    for (int k = 0; k < 3; ++k)
        if (cudaStreamCreateWithFlags(&c->cap_stream[k], cudaStreamNonBlocking) != cudaSuccess) {
            set_err(c, LJMD_E_CUDA, "capture stream creation failed");
            return fail(LJMD_E_CUDA);
        }
    // owned capacity: the whole system on one rank; a slab's share + 25 % headroom otherwise
    const double share = (double)c->geo.nzl / (double)c->geo.nc[2];
    const int cap = c->nranks == 1 ? (int)n : (int)std::min<int64_t>(n, (int64_t)(n * share * 1.25) + 4096);
    if ((s = alloc_owned(c, cap)) != LJMD_OK) return fail(s);
    if (c->split) {
        c->mig_cap = cap / 8 + 1024;
        for (int b = 0; b < 2; ++b) {
            if ((s = dalloc(c, &c->mig_send[b], c->mig_cap)) != LJMD_OK) return fail(s);
            if ((s = dalloc(c, &c->mig_recv[b], c->mig_cap)) != LJMD_OK) return fail(s);
        }
        if ((s = dalloc(c, &c->mig_cnt, 8)) != LJMD_OK || (s = dalloc(c, &c->xs, cap)) != LJMD_OK ||
            (s = dalloc(c, &c->vs, (size_t)3 * cap)) != LJMD_OK || (s = dalloc(c, &c->gs, cap)) != LJMD_OK ||
            (s = dalloc(c, &c->iota, cap)) != LJMD_OK || (s = dalloc(c, &c->stay_t, cap)) != LJMD_OK)
            return fail(s);
        if (cudaMallocHost(&c->h_mig, sizeof(int) * 8) != cudaSuccess ||
            cudaMallocHost(&c->h_tot, sizeof(int) * 4) != cudaSuccess) {
            set_err(c, LJMD_E_CUDA, "pinned allocation failed");
            return fail(LJMD_E_CUDA);
        }
    }
    if (c->split) {   // send areas: the two boundary planes with their x/y images, generous
        const double per_plane = (double)cap / (double)c->geo.nzl;
        const double img = (double)(c->geo.ex * c->geo.ey) / (double)(c->geo.nc[0] * c->geo.nc[1]);
        c->send_extra = (int)std::min<double>(2.0 * per_plane * img * 1.5 + 4096, (double)INT_MAX / 4);
    }
    const double ghost_ratio = (double)c->n_ecell / (double)c->n_ocell;
    int64_t scap = (int64_t)std::ceil(cap * ghost_ratio * 1.15) + 4096;
    if ((s = alloc_slots(c, (int)std::min<int64_t>(scap, INT_MAX / 2), false)) != LJMD_OK) return fail(s);
    // list width K: expected 4/3 pi rbar_c^3 rho neighbours with headroom
    double vol = box[0] * box[1] * box[2];
    double expect = 4.0 / 3.0 * M_PI * c->rn * c->rn * c->rn * (double)n / vol;
    int K = o.nbr_capacity > 0 ? ((int)o.nbr_capacity + 7) / 8 * 8 : ((int)std::ceil(expect * 1.4) + 16 + 7) / 8 * 8;
    if ((s = alloc_list(c, K)) != LJMD_OK) return fail(s);
    if ((s = load_state(c, pos, vel)) != LJMD_OK) return fail(s);
    if (o.tight_caps) {
        // testing: every capacity exactly what this state needs, so that a later rebuild inside
        // a captured step sequence runs short and takes the abort / eager-resume path
        c->stage_cap = c->max_staged;
        if ((s = alloc_list(c, std::max(8, (c->max_nbr + 7) / 8 * 8))) != LJMD_OK ||
            (s = alloc_slots(c, c->n_slots, false)) != LJMD_OK || (s = load_state(c, pos, vel)) != LJMD_OK)
            return fail(s);
    }
    *out = c;
    return LJMD_OK;
}

ljmd_status ljmd_set_state(ljmd_ctx* c, const double* pos, const double* vel) {
    TRY(check_ready(c));
    if (!pos && !vel) {
        if (c->stg_queued == 0) return set_err(c, LJMD_E_ARG, "ljmd_set_state(NULL, NULL): no staged state queued");
        const int b = (c->stg_next + 2 - c->stg_queued) & 1;   // oldest queued buffer
        --c->stg_queued;
        CK(cudaStreamWaitEvent(c->stream, c->stg_ev[b], 0));
        const size_t n3 = (size_t)3 * c->n_global;
        return load_state(c, nullptr, nullptr, c->stg[b], c->stg[b] + n3);
    }
    if (!pos || !vel) return LJMD_E_ARG;
    return load_state(c, pos, vel);
}

static ljmd_status transfers_init(ljmd_ctx* c) {
    if (c->split || c->n_own != c->n_global)
        return set_err(c, LJMD_E_ARG, "overlapped transfers need a single rank (nranks = 1, no split_self)");
    if (c->copy_stream) return LJMD_OK;
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    const size_t n3 = (size_t)3 * c->n_global;
    for (int b = 0; b < 2; ++b) {
        TRY(dalloc(c, &c->stg[b], 2 * n3));
        TRY(dalloc(c, &c->rb[b], n3));
        CK(cudaEventCreateWithFlags(&c->stg_ev[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->stg_used[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->rb_ev[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->rb_done[b], cudaEventDisableTiming));
        CK(cudaEventRecord(c->stg_used[b], c->stream));
        CK(cudaEventRecord(c->rb_done[b], c->copy_stream));
    }
    return LJMD_OK;
}

ljmd_status ljmd_stage_state(ljmd_ctx* c, const double* pos, const double* vel) {
    TRY(check_ctx(c));
    if (!pos || !vel) return LJMD_E_ARG;
    TRY(transfers_init(c));
    if (c->stg_queued >= 2) return set_err(c, LJMD_E_ARG, "ljmd_stage_state: two states already queued");
    const int b = c->stg_next;
    const size_t n3 = (size_t)3 * c->n_global;
    CK(cudaStreamWaitEvent(c->copy_stream, c->stg_used[b], 0));   // its last consumer has read it
    CK(cudaMemcpyAsync(c->stg[b], pos, sizeof(double) * n3, cudaMemcpyHostToDevice, c->copy_stream));
    CK(cudaMemcpyAsync(c->stg[b] + n3, vel, sizeof(double) * n3, cudaMemcpyHostToDevice, c->copy_stream));
    CK(cudaEventRecord(c->stg_ev[b], c->copy_stream));
    c->stg_next = b ^ 1;
    ++c->stg_queued;
    return LJMD_OK;
}

ljmd_status ljmd_get_positions_async(ljmd_ctx* c, double* out) {
    TRY(check_ready(c));
    if (!out) return LJMD_E_ARG;
    TRY(transfers_init(c));
    const int b = c->rb_next;
    c->rb_next = b ^ 1;
    CK(cudaStreamWaitEvent(c->stream, c->rb_done[b], 0));   // its previous copy-out has finished
    k_gather_pos<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->x[c->xc], c->own_slot, c->d_stage);
    CKL();
    k_rows_to_gid<<<nblk((int64_t)c->n_own * 3, 256), 256, 0, c->stream>>>(c->n_own, 3, c->gid[c->oc_cur],
                                                                          c->d_stage, c->rb[b]);
    CKL();
    CK(cudaEventRecord(c->rb_ev[b], c->stream));
    CK(cudaStreamWaitEvent(c->copy_stream, c->rb_ev[b], 0));
    CK(cudaMemcpyAsync(out, c->rb[b], sizeof(double) * 3 * (size_t)c->n_own, cudaMemcpyDeviceToHost,
                       c->copy_stream));
    CK(cudaEventRecord(c->rb_done[b], c->copy_stream));
    return LJMD_OK;
}

ljmd_status ljmd_wait_transfers(ljmd_ctx* c) {
    TRY(check_ctx(c));
    if (c->copy_stream) CK(cudaStreamSynchronize(c->copy_stream));
    return LJMD_OK;
}

ljmd_status kick_drift(ljmd_ctx* c) {
    // Alg. alg:VelocityVerlet line 6 of the first step of a call (uses the stored F)
    const bool check = c->opt.rebuild_check != 0;
    if (check) TRY(zero_async(c, &c->d_fl->maxdisp2, sizeof(unsigned long long)));
    double* v = c->v[c->oc_cur];
    const size_t oc = c->own_cap;
    const double h = 0.5 * c->dt / c->opt.mass;
    if (check)
        k_kick_drift<true><<<nblk(c->n_own, 256), 256, 0, c->stream>>>(
            c->n_own, c->x[c->xc], c->own_slot, v, v + oc, v + 2 * oc, c->F, c->F + oc, c->F + 2 * oc, h, c->dt,
            c->xbuild, c->d_fl, images(c), c->geo, c->xp[c->xc], c->x[c->xc ^ 1], c->capturing ? c->d_ctl : nullptr);
    else
        k_kick_drift<false><<<nblk(c->n_own, 256), 256, 0, c->stream>>>(
            c->n_own, c->x[c->xc], c->own_slot, v, v + oc, v + 2 * oc, c->F, c->F + oc, c->F + 2 * oc, h, c->dt,
            c->xbuild, c->d_fl, images(c), c->geo, c->xp[c->xc], c->x[c->xc ^ 1], c->capturing ? c->d_ctl : nullptr);
    CKL();
    return LJMD_OK;
}

// Steps s_first .. n of a call on the eager path (host decides each rebuild).  rebuilt_first:
// step s_first's drift and rebuild are already done (resumption after a graph abort).
ljmd_status step_eager(ljmd_ctx* c, int64_t s_first, int64_t nsteps, bool rebuilt_first) {
    c->dev_since_ok = false;   // the host decides these steps
    const bool check = c->opt.rebuild_check != 0;
    const int64_t ee = c->opt.energy_every;
    const double delta2 = c->opt.delta * c->opt.delta;
    for (int64_t s = s_first; s <= nsteps; ++s) {
        bool halo_pending = false;
        if (!(rebuilt_first && s == s_first)) {
            ++c->since;
            ++c->steps_done;
            bool due = c->since >= c->opt.rebuild_every;
            if (!due && check) {
                // global max displacement (non-negative doubles: max of the bit patterns)
                TRY(allreduce(c, reinterpret_cast<double*>(&c->d_fl->maxdisp2), 1, true));
                TRY(sync_flags(c));
                double m2;
                std::memcpy(&m2, &c->h_fl->maxdisp2, sizeof m2);
                due = 4.0 * m2 > delta2;
            }
            if (due) {
                if (c->halo_queued) {   // the rebuild re-exchanges: let the queued halo land first
                    CK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
                    c->halo_queued = false;
                }
                TRY(rebuild(c));
                c->since = 0;
                note_rebuild(c, c->steps_done);
            } else {
                // ghost images of owned particles were written with the positions (force
                // epilogue / kick-drift); received halo planes need theirs after the exchange
                if (c->halo_queued) {   // started by the previous launch's boundary tiles
                    c->halo_queued = false;
                    halo_pending = true;
                } else if (c->split && c->aux_stream) {
                    // the halo travels on aux_stream while the interior tiles compute
                    CK(cudaEventRecord(c->ev_ready, c->stream));
                    CK(cudaStreamWaitEvent(c->aux_stream, c->ev_ready, 0));
                    TRY(halo_direct(c, c->aux_stream));
#if LJMD_HALO_GATE
                    ++c->halo_seq;
                    k_set_flag<<<1, 1, 0, c->aux_stream>>>(c->halo_flag, c->halo_seq);
                    CKL();
#endif
                    CK(cudaEventRecord(c->ev_halo, c->aux_stream));
                    halo_pending = true;
                } else if (c->split) {
                    TRY(halo_direct(c));
                }
                if (c->newton3) TRY(refresh_ghosts(c, false));
            }
        }
        const bool sample = ee > 0 && (c->steps_done % ee) == 0;
        const bool last = s == nsteps;
        if (check && !last) TRY(zero_async(c, &c->d_fl->maxdisp2, sizeof(unsigned long long)));
        if (c->opt.validate) TRY(validate_step(c, (int)(s - 1)));
        TRY(launch_force(c, sample, last ? kKick : kKKD, check && !last, halo_pending));
        if (last) c->energy_current = sample && ee > 0;
        if (sample) {
            TRY(finalize_energy(c, c->hist + 2 * c->call_nsamp));
            TRY(allreduce(c, c->hist + 2 * c->call_nsamp, 2, false));
            ++c->call_nsamp;
        }
        if (!last) c->xc ^= 1;
        // the next step's halo: x(n+1) of the boundary planes is in the send areas once the
        // boundary CTAs of this launch have counted themselves done -- exchanged on aux_stream
        // while the interior tiles compute (not before a known rebuild, which re-exchanges)
        if (!last && c->bdone && !(!check && c->since + 1 >= c->opt.rebuild_every)) {
            if (stream_wait_value()(reinterpret_cast<CUstream>(c->aux_stream), reinterpret_cast<CUdeviceptr>(c->bdone),
                                    c->bdone_issued, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return set_err(c, LJMD_E_CUDA, "cuStreamWaitValue32 failed");
            TRY(halo_direct(c, c->aux_stream, c->xc));
            CK(cudaEventRecord(c->ev_halo, c->aux_stream));
            c->halo_queued = true;
        }
    }
    return LJMD_OK;
}

// The step sequence of one call, captured (graph mode): kick-drift, then per step the
// device decision + conditional rebuild (safe policy: every step; fixed policy: the
// host-known due steps), the force with its fused velocity-Verlet epilogue, the samples.
ljmd_status capture_call(ljmd_ctx* c, int64_t nsteps, ljmd_ctx::GraphEntry& ge) {
    const bool check = c->opt.rebuild_check != 0;
    const int64_t ee = c->opt.energy_every;
    const int ns = (int)c->opt.rebuild_every;
    const double delta2 = c->opt.delta * c->opt.delta;
    const int xc0 = c->xc;
    const int64_t step0 = c->steps_done;
    const int64_t k0 = c->kernel_launches;
    int64_t body_k = 0, nconds = 0;
    c->capturing = true;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    ljmd_status r = [&]() -> ljmd_status {
        // the per-call control (since persists across calls; an earlier call's abort too)
        k_call_begin<<<1, 1, 0, c->stream>>>(c->d_ctl);
        CKL();
        TRY(kick_drift(c));
        int64_t sim_since = c->since;
        for (int64_t s = 1; s <= nsteps; ++s) {
            bool cond = check;
            bool forced = false;
            if (!check) {
                ++sim_since;
                if (sim_since >= ns) {
                    sim_since = 0;
                    cond = forced = true;
                }
            }
            if (forced) {
                // the fixed schedule's rebuild: no conditional node (its kernels skip themselves
                // after an abort), the decision record in its first kernel; counted in the
                // graph's launches
                TRY(rebuild_captured(c, (int)s));
                c->pdl_ok = false;   // the force after the rebuild reads the new list
            } else if (cond) {
                const int64_t kb = c->kernel_launches;
                TRY(cond_if(
                    c, c->cap_stream[0],
                    [&](cudaGraphConditionalHandle h) {
                        k_decide<<<1, 1, 0, c->stream>>>(c->d_ctl, c->d_fl, ns, check ? 1 : 0, 0, delta2,
                                                        c->d_rstep, (int)s, h, 1);
                    },
                    [&]() { return rebuild_captured(c, 0); }));
                body_k = c->kernel_launches - kb - 1;
                ++nconds;
                c->pdl_ok = false;   // the force after the rebuild node reads the new list
            }
            const bool sample = ee > 0 && ((step0 + s) % ee) == 0;
            const bool last = s == nsteps;
            TRY(launch_force(c, sample, last ? kKick : kKKD, check && !last, false));
            if (sample) TRY(finalize_energy(c, c->hist));
            if (!last) c->xc ^= 1;
        }
        return LJMD_OK;
    }();
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    c->xc = xc0;
    c->pdl_ok = false;
    if (r != LJMD_OK) {
        if (g) cudaGraphDestroy(g);
        return r;
    }
    if (e != cudaSuccess) return set_err(c, LJMD_E_CUDA, "graph capture of ljmd_step: %s", cudaGetErrorString(e));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&ex, g, 0);
    if (ei != cudaSuccess) {
        cudaGraphDestroy(g);
        return set_err(c, LJMD_E_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ei));
    }
    ge.g = g;
    ge.ex = ex;
    ge.launches = (c->kernel_launches - k0) - nconds * body_k;   // without the conditional bodies
    ge.body_k = body_k;
    c->kernel_launches = k0;   // counted per replay below
    return LJMD_OK;
}

// Host side of a settled graph call p: rebuild bookkeeping, errors, energies; a capacity abort
// resumes the call on the eager path.  next: a call queued after p (deferred), which ran as
// no-ops if p aborted (k_call_begin) and is then re-run here.
ljmd_status step_call(ljmd_ctx* c, int64_t nsteps, bool defer, int64_t call = -1);

ljmd_status settle_call(ljmd_ctx* c, const ljmd_ctx::Pending& p, ljmd_ctx::Pending* next) {
    const int64_t ee = c->opt.energy_every;
    CK(cudaEventSynchronize(c->ev_call[p.buf]));
    if (c->init_pending) {   // the init sequence ran before this call: its energies are in place
        c->h_hist.insert(c->h_hist.begin(), c->h_init, c->h_init + 2);
        c->init_pending = false;
    }
    const CallOut o = *c->h_out[p.buf];
    const DevCtl& ctl = o.ctl;
    c->kernel_launches += p.launches + (int64_t)ctl.nreb * p.body_k;
    for (int k = 0; k < ctl.nreb; ++k) {
        const int64_t st = p.step0 + c->h_orstep[p.buf][k];
        if (c->last_build_step >= 0 && st > c->last_build_step)
            c->interval_ema = 0.5 * c->interval_ema + 0.5 * (double)(st - c->last_build_step);
        c->last_build_step = st;
        note_rebuild(c, st);
    }
    if (o.fl.nonfinite_gid != INT_MAX)
        return set_err(c, LJMD_E_NONFINITE, "non-finite position or velocity at particle %d", o.fl.nonfinite_gid);
    if (o.fl.overlap_pair != ~0ull)
        return set_err(c, LJMD_E_OVERLAP, "particles %d and %d coincide (r^2 == 0)",
                       (int)(o.fl.overlap_pair >> 32), (int)(o.fl.overlap_pair & 0xffffffffu));
    if (ctl.nreb > 0) {
        c->n_slots = o.slots;
        c->max_staged = o.fl.max_staged;
        c->n_gflat = o.fl.n_gflat;
        c->max_nbr = o.fl.max_nbr;
        c->total_nbr = o.fl.total_nbr;
    }
    if (!ctl.abort) {
        c->h_hist.insert(c->h_hist.end(), c->h_ohist[p.buf], c->h_ohist[p.buf] + 2 * (size_t)ctl.nsamp);
        if (!p.deferred) {   // else advanced at launch
            c->steps_done = p.step0 + p.nsteps;
            c->xc = p.xc0 ^ (int)((p.nsteps - 1) & 1);
            c->since = p.sim_since;
            c->energy_current = ee > 0 && (c->steps_done % ee) == 0;
        }
        if (c->opt.rebuild_check) c->since = ctl.since;   // decided on the device
        c->ema_after[p.call & 3] = c->interval_ema;
        // the current energies: from this call unless a later one is queued
        if (!(next && next->on) && ee > 0 && ((p.step0 + p.nsteps) % ee) == 0 && ctl.nsamp > 0) {
            c->cur_pe = c->h_ohist[p.buf][2 * ctl.nsamp - 2];
            c->cur_ke = c->h_ohist[p.buf][2 * ctl.nsamp - 1];
        }
        return LJMD_OK;
    }
    // a capacity ran short in the rebuild of step sa: steps 1 .. sa-1 are complete, step sa
    // has drifted; resume there on the eager path (its rebuild regrows what is short)
    ljmd_ctx::Pending skipped;
    if (next && next->on) {
        skipped = *next;
        next->on = false;
    }
    // a skipped call may still be on the stream: let it drain before buffers (and the graphs
    // holding their pointers) are regrown
    CK(cudaStreamSynchronize(c->stream));
    const int64_t sa = ctl.abort_step;
    ++c->graph_aborts;
    c->steps_done = p.step0 + sa;
    c->since = 0;
    c->xc = p.xc0 ^ (int)((sa - 1) & 1);
    c->call_nsamp = ctl.nsamp;
    TRY(zero_async(c, c->d_ctl, offsetof(DevCtl, since)));
    TRY(rebuild(c, /*danger=*/false));   // the dangerous-build test of this rebuild already ran
    TRY(step_eager(c, sa, p.nsteps, true));
    TRY(pull_hist(c, c->call_nsamp));    // the graph's samples and the eager steps'
    if (c->energy_current) {
        c->cur_pe = c->h_hist[c->h_hist.size() - 2];
        c->cur_ke = c->h_hist[c->h_hist.size() - 1];
    }
    c->ema_after[p.call & 3] = c->interval_ema;
    if (skipped.on) TRY(step_call(c, skipped.nsteps, false, skipped.call));
    return LJMD_OK;
}

ljmd_status settle(ljmd_ctx* c) {
    if (!c->pend.on) return LJMD_OK;
    const ljmd_ctx::Pending p = c->pend;
    c->pend.on = false;
    return settle_call(c, p, nullptr);
}

// mapped per-call output buffers for calls of up to n steps
static ljmd_status ensure_out(ljmd_ctx* c, int64_t n) {
    if (!c->ev_call[0]) {
        for (int b = 0; b < 2; ++b) {
            CK(cudaEventCreateWithFlags(&c->ev_call[b], cudaEventDisableTiming));
            CK(cudaHostAlloc(&c->h_out[b], sizeof(CallOut), cudaHostAllocMapped));
        }
    }
    if (n <= c->out_cap) return LJMD_OK;
    const int64_t cap = std::max<int64_t>(n, 64);
    for (int b = 0; b < 2; ++b) {
        if (c->h_orstep[b]) cudaFreeHost(c->h_orstep[b]);
        if (c->h_ohist[b]) cudaFreeHost(c->h_ohist[b]);
        c->h_orstep[b] = nullptr;
        c->h_ohist[b] = nullptr;
        CK(cudaHostAlloc(&c->h_orstep[b], sizeof(int) * (size_t)cap, cudaHostAllocMapped));
        CK(cudaHostAlloc(&c->h_ohist[b], sizeof(double) * 2 * (size_t)(cap + 2), cudaHostAllocMapped));
    }
    c->out_cap = cap;
    return LJMD_OK;
}

ljmd_status step_graph(ljmd_ctx* c, int64_t nsteps, bool defer, int64_t call) {
    const bool check = c->opt.rebuild_check != 0;
    const int64_t ee = c->opt.energy_every;
    if (c->rstep_cap < nsteps) {
        TRY(dalloc(c, &c->d_rstep, (size_t)nsteps));
        c->rstep_cap = nsteps;
    }
    TRY(ensure_out(c, nsteps));
    auto key_of = [&](bool rr) {
        char key[160];
        snprintf(key, sizeof key, "n%lld x%d s%lld e%lld c%d r%d", (long long)nsteps, c->xc,
                 check ? -1LL : (long long)c->since, ee > 0 ? (long long)(c->steps_done % ee) : 0LL, check ? 1 : 0,
                 rr ? 1 : 0);
        return std::string(key);
    };
    const std::string key = key_of(c->use_rr);
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        ljmd_ctx::GraphEntry ge;
        TRY(capture_call(c, nsteps, ge));
        it = c->graphs.emplace(key, ge).first;
        // the displacement check's list order can change from call to call (decide_list_order):
        // the other variant is captured now as well, so a later change costs no capture
        if (check && c->bank_order && c->fparts == 1 && !c->graphs.count(key_of(!c->use_rr))) {
            c->use_rr = !c->use_rr;
            ljmd_ctx::GraphEntry g2;
            const ljmd_status r = capture_call(c, nsteps, g2);
            c->use_rr = !c->use_rr;
            TRY(r);
            c->graphs.emplace(key_of(!c->use_rr), g2);
            it = c->graphs.find(key);
        }
    }
    ljmd_ctx::Pending p;
    p.on = true;
    p.step0 = c->steps_done;
    p.nsteps = nsteps;
    p.xc0 = c->xc;
    p.launches = it->second.launches;
    p.body_k = it->second.body_k;
    p.buf = c->out_next;
    p.call = call;
    c->out_next ^= 1;
    if (check && !c->dev_since_ok) {   // after eager steps or a new state: the host's count
        k_set_since<<<1, 1, 0, c->stream>>>(c->d_ctl, (int)c->since);
        CKL();
    }
    c->dev_since_ok = true;
    CK(cudaGraphLaunch(it->second.ex, c->stream));
    ++c->graph_calls;
    k_call_out<<<1, 256, 0, c->stream>>>(c->d_ctl, c->d_fl, c->ebegin + c->n_ecell, c->d_rstep, c->hist,
                                         c->h_out[p.buf], c->h_orstep[p.buf], c->h_ohist[p.buf]);
    CKL();
    CK(cudaEventRecord(c->ev_call[p.buf], c->stream));
    p.sim_since = c->since;
    for (int64_t s = 1; s <= nsteps; ++s)
        if (++p.sim_since >= c->opt.rebuild_every) p.sim_since = 0;
    if (!defer) return settle_call(c, p, nullptr);   // one host wait per call
    // the step count, buffer parity and sample phase after the call are known in advance (the
    // displacement-checked schedule's since is read at settlement): advance now, settle the
    // previous call
    p.deferred = true;
    const ljmd_ctx::Pending prev = c->pend;
    c->pend = p;
    c->steps_done = p.step0 + nsteps;
    if (!check) c->since = p.sim_since;
    c->xc = p.xc0 ^ (int)((nsteps - 1) & 1);
    c->energy_current = ee > 0 && (c->steps_done % ee) == 0;
    if (prev.on) TRY(settle_call(c, prev, &c->pend));
    return LJMD_OK;
}

// One ljmd_step call.  defer: graph mode returns once the call is queued (LJMD_DEFER=0 turns
// that off).  call: the call's index (a call re-run after an abort keeps its own)
ljmd_status step_call(ljmd_ctx* c, int64_t nsteps, bool defer, int64_t call) {
    if (call < 0) call = c->ncalls++;
    const int64_t ee = c->opt.energy_every;
    const int64_t need_hist = nsteps / std::max<int64_t>(ee, 1) + 2;
    const bool graph = graph_ok(c);
    defer = defer && graph;
    // buffers a queued call uses are regrown only after it has been settled
    if (c->pend.on && (!defer || need_hist > c->hist_cap || nsteps > c->rstep_cap || nsteps > c->out_cap))
        TRY(settle(c));
    if (!defer) TRY(settle_init(c));   // deferred: the init energies are read when this call settles
    TRY(ensure_hist(c, need_hist));
    c->call_nsamp = 0;
    const int64_t first_launch = c->force_launches;
    const int64_t step0 = c->steps_done;
    c->energy_current = false;
    c->init_current = false;
    if (c->opt.validate) {
        if (c->vhist_cap < nsteps) {
            TRY(dalloc(c, &c->vhist, (size_t)2 * nsteps));
            c->vhist_cap = nsteps;
        }
        CK(cudaMemsetAsync(c->vhist, 0, sizeof(int) * 2 * (size_t)nsteps, c->stream));
    }
    decide_list_order(c, call);
    if (graph) return step_graph(c, nsteps, defer, call);   // settled there unless deferred
    TRY(kick_drift(c));
    TRY(step_eager(c, 1, nsteps, false));
    TRY(pull_hist(c, c->call_nsamp));
    if (c->energy_current) {
        c->cur_pe = c->h_hist[c->h_hist.size() - 2];
        c->cur_ke = c->h_hist[c->h_hist.size() - 1];
    }
    c->ema_after[call & 3] = c->interval_ema;
    TRY(collect_profile(c, first_launch));
    TRY(sync_flags(c));
    if (c->h_fl->halo_timeout) return set_err(c, LJMD_E_NCCL, "a boundary force tile timed out waiting for the halo");
    if (c->opt.validate) {
        if (c->h_fl->val_error)
            return set_err(c, LJMD_E_STATE, "validation: a listed in-range pair was not found by the cell search");
        std::vector<int> h((size_t)2 * nsteps);
        CK(cudaMemcpyAsync(h.data(), c->vhist, sizeof(int) * h.size(), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int64_t k = 0; k < nsteps; ++k) {
            c->h_val.push_back(step0 + k + 1);
            c->h_val.push_back(h[2 * k]);
            c->h_val.push_back(h[2 * k + 1]);
        }
    }
    return LJMD_OK;
}

ljmd_status ljmd_step(ljmd_ctx* c, int64_t nsteps) {
    TRY(check_ctx(c));
    if (nsteps < 0) return set_err(c, LJMD_E_ARG, "ljmd_step: nsteps < 0");
    if (nsteps == 0) return LJMD_OK;
    return step_call(c, nsteps, getenv_int("LJMD_DEFER", 1) != 0);
}

ljmd_status ljmd_get_forces(ljmd_ctx* c, double* out) {
    TRY(check_ready(c));
    if (!out) return LJMD_E_ARG;
    const size_t oc = c->own_cap;
    k_gather_soa<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->F, c->F + oc, c->F + 2 * oc, c->d_stage);
    CKL();
    return readback(c, c->d_stage, 3, out);
}

ljmd_status ljmd_get_velocities(ljmd_ctx* c, double* out) {
    TRY(check_ready(c));
    if (!out) return LJMD_E_ARG;
    const size_t oc = c->own_cap;
    const double* v = c->v[c->oc_cur];
    k_gather_soa<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, v, v + oc, v + 2 * oc, c->d_stage);
    CKL();
    return readback(c, c->d_stage, 3, out);
}

ljmd_status ljmd_get_positions(ljmd_ctx* c, double* out, int64_t wrapped) {
    TRY(check_ready(c));
    if (!out) return LJMD_E_ARG;
    k_gather_pos<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->x[c->xc], c->own_slot, c->d_stage);
    CKL();
    if (!wrapped) return readback(c, c->d_stage, 3, out);
    std::vector<double> tmp((size_t)3 * c->n_own);
    std::vector<int> g(c->n_own);
    CK(cudaMemcpyAsync(tmp.data(), c->d_stage, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g.data(), c->gid[c->oc_cur], sizeof(int) * g.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int t = 0; t < c->n_own; ++t)
        for (int k = 0; k < 3; ++k) {
            double x = tmp[(size_t)3 * t + k];
            if (wrapped) {
                double L = c->geo.L[k];
                x = x - L * std::floor(x / L);
                if (x < 0.0) x += L;
                if (x >= L) x -= L;
            }
            out[(size_t)g[t] * 3 + k] = x;
        }
    return LJMD_OK;
}

ljmd_status ljmd_get_particle_energy(ljmd_ctx* c, double* out) {
    TRY(check_ready(c));
    if (!out) return LJMD_E_ARG;
    TRY(energy_now(c));
    return readback(c, c->e, 1, out);
}

ljmd_status ljmd_get_energy(ljmd_ctx* c, double* pe, double* ke) {
    TRY(check_ready(c));
    TRY(energy_now(c));
    if (pe) *pe = c->cur_pe;
    if (ke) *ke = c->cur_ke;
    return LJMD_OK;
}

#if LJMD_PHASES
// measurement build only: the force kernel's per-CTA phase timers of the last launch
extern "C" int ljmd_debug_phases(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, ljmd::ljmd_phase_buf, sizeof(unsigned long long) * 10 * (size_t)n) ==
                   cudaSuccess ? 0 : -1;
}
#endif

ljmd_status ljmd_get_energy_history(ljmd_ctx* c, double* pe, double* ke, int64_t cap, int64_t* count) {
    TRY(check_ready(c));
    TRY(settle_init(c));
    int64_t avail = (int64_t)c->h_hist.size() / 2;
    if (count) *count = avail;
    for (int64_t i = 0; i < std::min(cap, avail); ++i) {
        if (pe) pe[i] = c->h_hist[2 * i];
        if (ke) ke[i] = c->h_hist[2 * i + 1];
    }
    return LJMD_OK;
}

ljmd_status ljmd_get_neighbours(ljmd_ctx* c, int64_t* offsets, int64_t* gids, int64_t cap) {
    TRY(check_ready(c));
    if (!offsets) return LJMD_E_ARG;
    const int n = c->n_own;
    std::vector<int> cnt(n), g(n);
    CK(cudaMemcpyAsync(cnt.data(), c->ncount, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g.data(), c->gid[c->oc_cur], sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<int64_t> rowcnt(c->n_global, 0);
    for (int t = 0; t < n; ++t) rowcnt[g[t]] = std::min(cnt[t], c->K);
    offsets[0] = 0;
    for (int64_t i = 0; i < c->n_global; ++i) offsets[i + 1] = offsets[i] + rowcnt[i];
    if (!gids || cap < offsets[c->n_global]) return LJMD_OK;
    std::vector<long long> toff(n + 1, 0);
    for (int t = 0; t < n; ++t) toff[t + 1] = toff[t] + std::min(cnt[t], c->K);
    long long* d_off = nullptr;
    long long* d_out = nullptr;
    TRY(dalloc(c, &d_off, n + 1));
    TRY(dalloc(c, &d_out, (size_t)std::max<long long>(toff[n], 1)));
    CK(cudaMemcpyAsync(d_off, toff.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, c->stream));
    k_list_gids<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->n_pad, c->geo, (const unsigned short*)c->nbr8,
                                                     c->ncount, c->ocell_of,
                                                     TileRows{c->tr_begin, c->tr_off, c->tr_len}, c->slot_gid, d_off, d_out);
    CKL();
    std::vector<long long> h((size_t)toff[n]);
    CK(cudaMemcpyAsync(h.data(), d_out, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d_off);
    cudaFree(d_out);
    for (int t = 0; t < n; ++t)
        for (long long k = toff[t]; k < toff[t + 1]; ++k) gids[offsets[g[t]] + (k - toff[t])] = h[(size_t)k];
    return LJMD_OK;
}

ljmd_status ljmd_get_rebuild_steps(ljmd_ctx* c, int64_t* out, int64_t cap, int64_t* count) {
    TRY(check_ready(c));
    int64_t n = (int64_t)c->rebuild_steps.size();
    if (count) *count = n;
    for (int64_t i = 0; out && i < std::min(n, cap); ++i) out[i] = c->rebuild_steps[(size_t)i];
    return LJMD_OK;
}

ljmd_status ljmd_get_stats(ljmd_ctx* c, ljmd_stats* s) {
    TRY(check_ready(c));
    if (!s) return LJMD_E_ARG;
    std::memset(s, 0, sizeof *s);
    s->steps_done = c->steps_done;
    s->n_rebuilds = c->n_rebuilds;
    s->n_owned = c->n_own;
    s->n_ghost = c->n_slots - c->n_own;
    s->nbr_capacity = c->K;
    s->max_neighbours = c->max_nbr;
    s->total_neighbours = (int64_t)c->total_nbr;
    for (int d = 0; d < 3; ++d) s->n_cells[d] = c->geo.nc[d];
    s->regrows = c->regrows;
    s->force_launches = c->force_launches;
    s->force_ms = c->force_ms;
    TRY(settle_init(c));
    s->energy_samples = (int64_t)c->h_hist.size() / 2;
    s->kernel_launches = c->kernel_launches;
    TRY(to_host(c, c->h_st, c->d_st, sizeof(DevStats)));
    CK(cudaStreamSynchronize(c->stream));
    s->dangerous_builds = (int64_t)c->h_st->dangerous;
    s->max_build_disp = std::sqrt(c->h_st->max_disp2);
    s->graph_calls = c->graph_calls;
    s->graph_aborts = c->graph_aborts;
    s->graphs_cached = (int64_t)c->graphs.size();
    const int64_t nv = (int64_t)c->h_val.size() / 3;
    s->validated_steps = nv;
    for (int64_t k = 0; k < nv; ++k) {
        s->missed_particle_steps += c->h_val[3 * k + 1];
        s->missed_pairs += c->h_val[3 * k + 2];
        s->max_missed_particles = std::max(s->max_missed_particles, c->h_val[3 * k + 1]);
    }
    return LJMD_OK;
}

ljmd_status ljmd_get_validation(ljmd_ctx* c, int64_t* out, int64_t cap, int64_t* count) {
    TRY(check_ready(c));
    if (!c->opt.validate) return set_err(c, LJMD_E_ARG, "ljmd_get_validation: validation mode is off");
    const int64_t nv = (int64_t)c->h_val.size() / 3;
    if (count) *count = nv;
    for (int64_t k = 0; out && k < std::min(nv, cap); ++k)
        for (int q = 0; q < 3; ++q) out[3 * k + q] = c->h_val[3 * k + q];
    return LJMD_OK;
}

const char* ljmd_last_error(const ljmd_ctx* c) {
    if (!c) return g_init_error.c_str();
    return c->msg.c_str();
}

void ljmd_destroy(ljmd_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    // a step that failed after queueing the halo exchange on aux_stream may still have NCCL
    // work or copies in flight on it: drain both streams before the comm and buffers go
    if (c->aux_stream) cudaStreamSynchronize(c->aux_stream);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    void* ptrs[] = {c->x[0], c->x[1], c->xf, c->slot_gid, c->v[0], c->v[1], c->gid[0], c->gid[1],
                    c->own_slot, c->own_li, c->ocell_of, c->F, c->e, c->xbuild, c->xw, c->cell_of, c->rank_in, c->perm,
                    c->ocount, c->obegin, c->ecount, c->ebegin, c->ecell_src, c->gc_dst, c->gc_src, c->gc_shift,
                    c->scan_tmp, c->nbr8, c->ncount, c->oc_of_lex, c->lex_of_oc, c->tile_oc0, c->tr_begin, c->ylo_f, c->zlo_f,
                    c->tr_off, c->pe_part, c->ke_part, c->hist, c->d_fl, c->d_stage};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    dsl_destroy(c);
    for (void* p : {(void*)c->nbr8h, (void*)c->ncount_h, (void*)c->slot_t, (void*)c->tmap, (void*)c->tile_R,
                    (void*)c->ld_pos, (void*)c->ld_vel, (void*)c->ld_gid, (void*)c->stay_t, (void*)c->gflat,
                    (void*)c->slot2t, (void*)c->img_cnt, (void*)c->img_off, (void*)c->img, (void*)c->grecv,
                    (void*)c->xp[0], (void*)c->xp[1], (void*)c->tr_len})
        if (p) cudaFree(p);
    void* ptrs2[] = {c->send_cnt, c->send_off, c->recv_cnt, c->recv_off, c->send_idx, c->send_buf, c->mig_send[0],
                     c->mig_send[1], c->mig_recv[0], c->mig_recv[1], c->mig_cnt, c->xs, c->vs, c->gs, c->iota};
    for (void* p : ptrs2)
        if (p) cudaFree(p);
    if (c->h_mig) cudaFreeHost(c->h_mig);
    if (c->h_tot) cudaFreeHost(c->h_tot);
    delete c->tr;
    if (c->h_fl) cudaFreeHost(c->h_fl);
    if (c->h_st) cudaFreeHost(c->h_st);
    drop_graphs(c);
    for (int b = 0; b < 2; ++b) {
        if (c->h_out[b]) cudaFreeHost(c->h_out[b]);
        if (c->h_orstep[b]) cudaFreeHost(c->h_orstep[b]);
        if (c->h_ohist[b]) cudaFreeHost(c->h_ohist[b]);
        if (c->ev_call[b]) cudaEventDestroy(c->ev_call[b]);
    }
    for (void* p : {(void*)c->d_ctl, (void*)c->d_rstep, (void*)c->halo_flag})
        if (p) cudaFree(p);
    for (cudaStream_t st : c->cap_stream)
        if (st) cudaStreamDestroy(st);
    for (void* p : {(void*)c->d_st, (void*)c->vcount, (void*)c->vbegin, (void*)c->vcell, (void*)c->vrank,
                    (void*)c->vpos, (void*)c->vhist})
        if (p) cudaFree(p);
    if (c->h_histm) cudaFreeHost(c->h_histm);
    if (c->h_init) cudaFreeHost(c->h_init);
    if (c->h_slots) cudaFreeHost(c->h_slots);
    if (c->h_sctl) cudaFreeHost(c->h_sctl);
    for (auto e : c->ev) cudaEventDestroy(e);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        for (int b = 0; b < 2; ++b) {
            cudaFree(c->stg[b]);
            cudaFree(c->rb[b]);
            for (cudaEvent_t e : {c->stg_ev[b], c->stg_used[b], c->rb_ev[b], c->rb_done[b]})
                if (e) cudaEventDestroy(e);
        }
        cudaStreamDestroy(c->copy_stream);
    }
    if (c->aux_stream) {
        cudaStreamSynchronize(c->aux_stream);
        cudaStreamDestroy(c->aux_stream);
    }
    if (c->ev_ready) cudaEventDestroy(c->ev_ready);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    if (c->bdone) cudaFree(c->bdone);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // extern "C"


template <int L>
void boa_launch(ljmd_ctx* c, const BoaArgs& a, size_t smem) {
    cudaFuncSetAttribute(k_boa<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxStageSmem);
    k_boa<L><<<c->n_tiles, kForceThreads, smem, c->stream>>>(a);
}

extern "C" ljmd_status ljmd_boa(ljmd_ctx* c, int64_t ell, double rcut, double* Q, int64_t* nnb) {
    TRY(check_ready(c));
    if (!Q || ell < 0 || ell > kBoaMaxL || !(rcut > 0.0))
        return set_err(c, LJMD_E_ARG, "ljmd_boa: need 0 <= ell <= %d and rcut > 0", kBoaMaxL);
    if (rcut > c->rc)
        return set_err(c, LJMD_E_ARG, "ljmd_boa: rcut %g exceeds the force cutoff rc = %g (list validity)", rcut,
                       c->rc);
    BoaArgs a;
    a.g = c->geo;
    a.x = c->x[c->xc];
    a.own_slot = c->own_slot;
    a.nbr = c->nbr8;
    a.ncount = c->ncount;
    a.obegin = c->obegin;
    a.tile_oc0 = c->tile_oc0;
    a.tr = TileRows{c->tr_begin, c->tr_off, c->tr_len};
    a.Q = c->d_stage;
    a.nnb = c->d_stage + c->own_cap;
    a.n_own = c->n_own;
    a.n_pad = c->n_pad;
    a.rcut2 = rcut * rcut;
    for (int m = 0; m <= kBoaMaxL; ++m) {
        double f = 1.0;   // (l-m)!/(l+m)!
        for (int k = (int)ell - m + 1; k <= (int)ell + m; ++k) f /= (double)k;
        a.K[m] = m <= ell ? std::sqrt((2.0 * ell + 1.0) / (4.0 * M_PI) * f) : 0.0;
    }
    const size_t smem = 24 * (size_t)(c->max_staged + 1);
    switch (ell) {
        case 0: boa_launch<0>(c, a, smem); break;
        case 1: boa_launch<1>(c, a, smem); break;
        case 2: boa_launch<2>(c, a, smem); break;
        case 3: boa_launch<3>(c, a, smem); break;
        case 4: boa_launch<4>(c, a, smem); break;
        case 5: boa_launch<5>(c, a, smem); break;
        case 6: boa_launch<6>(c, a, smem); break;
        case 7: boa_launch<7>(c, a, smem); break;
        case 8: boa_launch<8>(c, a, smem); break;
        case 9: boa_launch<9>(c, a, smem); break;
        case 10: boa_launch<10>(c, a, smem); break;
        case 11: boa_launch<11>(c, a, smem); break;
        default: boa_launch<12>(c, a, smem); break;
    }
    CKL();
    TRY(readback(c, c->d_stage, 1, Q));
    if (nnb) {
        std::vector<double> tmp(c->n_global, -1.0);
        TRY(readback(c, c->d_stage + c->own_cap, 1, tmp.data()));
        for (int64_t i = 0; i < c->n_global; ++i)
            if (tmp[i] >= 0.0) nnb[i] = (int64_t)tmp[i];
    }
    return LJMD_OK;
}


extern "C" ljmd_status ljmd_set_thermostat(ljmd_ctx* c, double nu, double temperature, uint64_t seed) {
    TRY(check_ready(c));
    if (!(nu >= 0.0) || !(temperature >= 0.0) || !(nu * c->dt <= 1.0))
        return set_err(c, LJMD_E_ARG, "ljmd_set_thermostat: need nu >= 0, T >= 0 and nu*dt <= 1 (nu*dt = %g)",
                       nu * c->dt);
    c->nu_dt = nu * c->dt;
    c->thermo_sd = std::sqrt(temperature / c->opt.mass);
    c->thermo_seed = seed;
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_set_profile(ljmd_ctx* c, int64_t profile) {
    TRY(check_ready(c));
    if (profile != 0 && profile != 1) return set_err(c, LJMD_E_ARG, "ljmd_set_profile: profile must be 0 or 1");
    c->opt.profile = profile;
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_cna(ljmd_ctx* c, double rcut, int32_t* cls, int32_t* trip, int64_t* nnb) {
    TRY(check_ready(c));
    if (!cls || !(rcut > 0.0)) return set_err(c, LJMD_E_ARG, "ljmd_cna: cls and rcut > 0 required");
    if (rcut > c->rc)
        return set_err(c, LJMD_E_ARG, "ljmd_cna: rcut %g exceeds the force cutoff rc = %g (list validity)", rcut,
                       c->rc);
    if (c->nranks > 1 || c->split) return set_err(c, LJMD_E_ARG, "ljmd_cna: single rank only");
    const int n = c->n_own;
    int *tab = nullptr, *tcnt = nullptr, *tmap = nullptr, *dtrip = nullptr, *dcls = nullptr;
    TRY(dalloc(c, &tab, (size_t)n * kCnaMax));
    TRY(dalloc(c, &tcnt, n));
    TRY(dalloc(c, &tmap, (size_t)c->n_global));
    TRY(dalloc(c, &dtrip, (size_t)n * kCnaMax));
    TRY(dalloc(c, &dcls, n));
    TRY(reset_flags(c));
    CnaArgs a;
    a.g = c->geo;
    a.x = c->x[c->xc];
    a.own_slot = c->own_slot;
    a.nbr = c->nbr8;
    a.ncount = c->ncount;
    a.ocell_of = c->ocell_of;
    a.slot_gid = c->slot_gid;
    a.gid = c->gid[c->oc_cur];
    a.tr = TileRows{c->tr_begin, c->tr_off, c->tr_len};
    a.tab = tab;
    a.tcnt = tcnt;
    a.tmap = tmap;
    a.trip = dtrip;
    a.cls = dcls;
    a.fl = c->d_fl;
    a.n_own = n;
    a.n_pad = c->n_pad;
    a.rcut2 = rcut * rcut;
    k_cna_tmap<<<nblk(n, 256), 256, 0, c->stream>>>(n, a.gid, tmap);
    CKL();
    k_cna_bonds<<<nblk(n, 128), 128, 0, c->stream>>>(a);
    CKL();
    k_cna_triplets<<<nblk(n, 128), 128, 0, c->stream>>>(a);
    CKL();
    TRY(sync_flags(c));
    ljmd_status st = LJMD_OK;
    if (c->h_fl->overflow)
        st = set_err(c, LJMD_E_CAPACITY, "ljmd_cna: more than %d bonded neighbours inside rcut", kCnaMax);
    if (st == LJMD_OK) {
        std::vector<int> hc(n), hcnt(n), ht(trip ? (size_t)n * kCnaMax : 0), g(n);
        cudaMemcpyAsync(hc.data(), dcls, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(hcnt.data(), tcnt, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream);
        if (trip) cudaMemcpyAsync(ht.data(), dtrip, sizeof(int) * ht.size(), cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(g.data(), c->gid[c->oc_cur], sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream);
        if (cudaStreamSynchronize(c->stream) != cudaSuccess) st = set_err(c, LJMD_E_CUDA, "ljmd_cna readback");
        for (int t = 0; st == LJMD_OK && t < n; ++t) {
            cls[g[t]] = hc[t];
            if (nnb) nnb[g[t]] = hcnt[t];
            if (trip)
                for (int k = 0; k < kCnaMax; ++k)
                    trip[(size_t)g[t] * kCnaMax + k] = k < hcnt[t] ? ht[(size_t)t * kCnaMax + k] : 0;
        }
    }
    for (void* p : {(void*)tab, (void*)tcnt, (void*)tmap, (void*)dtrip, (void*)dcls}) cudaFree(p);
    return st;
}

extern "C" ljmd_status ljmd_nccl_unique_id(void* out128) {
    if (!out128) return LJMD_E_ARG;
    std::string err;
    if (!nccl_unique_id(out128, err)) return set_err(nullptr, LJMD_E_NCCL, "%s", err.c_str());
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_measure_fp64_peak(int64_t device, double* tflops) {
    ljmd_ctx* c = nullptr;
    if (!tflops) return LJMD_E_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(nullptr, LJMD_E_CUDA, "no CUDA device");
    }
    if (device >= 0) CK(cudaSetDevice((int)device));
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* out = nullptr;
    CK(cudaMalloc(&out, sizeof(double) * 4096));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = sms * 8, iters = 2048;
    k_fp64_peak<<<blocks, 256>>>(out, 64, 0.999999, 1e-7);   // warm-up (clocks)
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        k_fp64_peak<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    double flops = 2.0 * 8.0 * 16.0 * iters * (double)blocks * 256.0;
    *tflops = flops / (best * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return LJMD_OK;
}

#include "dsl.cuh"
