// dsl.cuh -- PairLoop / ParticleLoop front end, included at the end of
// ljmd.cu (it needs the context).  The paper's code generation (Sec. 2.4):
// a user C kernel plus access descriptors (Tab. tab:DSL_access) is inserted into a template
// for the target, compiled, and launched over all particles / particle pairs.  Here the
// target is sm_100a: the template is the engine's tile-staged neighbour-list loop (one CTA per
// tile, positions of the tile's halo rows in shared memory, thread per particle over its
// Verlet list), compiled at run time with NVRTC to a cubin and loaded with
// cudaLibraryLoadData.  One rank: the j side of a dat is read through slot -> owner; several
// ranks: data migrates with its particles and j-side data is brought into the halo first.
#include <dlfcn.h>
#include <nvrtc.h>

#include <cctype>
#include <map>
#include <sstream>

namespace ljmd {
// ----------------------------------------------------------------------------- helper kernels
// rows of `words` 32-bit words: new owned order from the old one, through gid
__global__ void k_dat_permute(int n, int words, const int* __restrict__ gid_new, const int* __restrict__ tmap_old,
                              const unsigned* __restrict__ src, unsigned* __restrict__ dst) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)n * words) return;
    const int t = (int)(idx / words), w = (int)(idx % words);
    dst[(size_t)t * words + w] = src[(size_t)tmap_old[gid_new[t]] * words + w];
}

// caller (gid) order <-> owned order
__global__ void k_dat_from_gid(int n, int words, const int* __restrict__ gid, const unsigned* __restrict__ src,
                               unsigned* __restrict__ dst) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)n * words) return;
    const int t = (int)(idx / words), w = (int)(idx % words);
    dst[(size_t)t * words + w] = src[(size_t)gid[t] * words + w];
}

__global__ void k_dat_to_gid(int n, int words, const int* __restrict__ gid, const unsigned* __restrict__ src,
                             unsigned* __restrict__ dst) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)n * words) return;
    const int t = (int)(idx / words), w = (int)(idx % words);
    dst[(size_t)gid[t] * words + w] = src[(size_t)t * words + w];
}

// ScalarArray INC: fixed-order sum of the per-block partials (deterministic)
template <class T>
__global__ void k_dsl_fin(const T* __restrict__ part, int nb, int nc, T* __restrict__ out, int zero) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    T s = 0;
    for (int b = 0; b < nb; ++b) s += part[(size_t)b * nc + c];
    out[c] = zero ? s : out[c] + s;
}

__global__ void k_tile_R(int n_tiles, Geo g, int* __restrict__ out) {
    const int tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile < n_tiles) out[tile] = tile_geo(g, tile).R;
}

// ---- several ranks: particle data travels with its particle, and the data a
// pair loop reads on the j side is brought into the halo
// migration: compact rows of the stayers (in the engine's compaction order), rows of leavers
__global__ void k_dat_gather_idx(int n, int words, const int* __restrict__ idx, const unsigned* __restrict__ src,
                                 unsigned* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n * words) return;
    const int k = (int)(i / words), w = (int)(i % words);
    dst[i] = src[(size_t)idx[k] * words + w];
}

__global__ void k_dat_gather_mig(int n, int words, const MigRec* __restrict__ rec, const unsigned* __restrict__ src,
                                 unsigned* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n * words) return;
    const int k = (int)(i / words), w = (int)(i % words);
    dst[i] = src[(size_t)rec[k].pad * words + w];
}

// slot-space copy of argument data: owned rows (any stride) -> their slots
template <class T>
__global__ void k_elems_to_slots(int n, int nc, const int* __restrict__ own_slot, const T* __restrict__ src,
                                 long long st, long long sc, T* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n * nc) return;
    const int t = (int)(i / nc), c = (int)(i % nc);
    dst[(size_t)own_slot[t] * nc + c] = src[(size_t)t * st + (size_t)c * sc];
}

__global__ void k_slot_pack_words(int n, int words, const int* __restrict__ idx, const unsigned* __restrict__ src,
                                  unsigned* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n * words) return;
    const int k = (int)(i / words), w = (int)(i % words);
    dst[i] = src[(size_t)idx[k] * words + w];
}

// ghost cells of the slot-space copy: rows of the source cell (local) or of the received
// plane cell, as k_ghost_refresh does for positions (no periodic shift for data)
__global__ void k_slot_ghosts_words(GhostCells gc, const int* __restrict__ ebegin, const int* __restrict__ ecount,
                                    const int* __restrict__ recv_cnt, const int* __restrict__ recv_off, int n_slots,
                                    int words, unsigned* __restrict__ d) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= gc.n) return;
    const int dst = gc.dst[warp], s = gc.src[warp];
    const int db = ebegin[dst];
    int sb, m;
    if (s >= 0) {
        sb = ebegin[s];
        m = ecount[s];
    } else {
        sb = n_slots + recv_off[-s - 1];
        m = recv_cnt[-s - 1];
    }
    for (int i = lane; i < m * words; i += 32) d[(size_t)db * words + i] = d[(size_t)sb * words + i];
}

// ScalarArray INC: this launch's sums as doubles (exact for integers below 2^53), all-reduced
// over the ranks, then applied
template <class T>
__global__ void k_dsl_fin_delta(const T* __restrict__ part, int nb, int nc, double* __restrict__ delta) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    T s = 0;
    for (int b = 0; b < nb; ++b) s += part[(size_t)b * nc + c];
    delta[c] = (double)s;
}

template <class T>
__global__ void k_dsl_apply(const double* __restrict__ delta, int nc, T* __restrict__ out, int zero) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    out[c] = zero ? (T)delta[c] : (T)(out[c] + (T)delta[c]);
}
}  // namespace ljmd

namespace {

// --------------------------------------------------------------------------- NVRTC (dlopen)
struct Nvrtc {
    bool ok = false;
    std::string why;
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
    nvrtcResult (*log_size)(nvrtcProgram, size_t*);
    nvrtcResult (*log)(nvrtcProgram, char*);
    nvrtcResult (*cubin_size)(nvrtcProgram, size_t*);
    nvrtcResult (*cubin)(nvrtcProgram, char*);
    nvrtcResult (*destroy)(nvrtcProgram*);
};

Nvrtc& nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        void* h = nullptr;
        for (const char* nm : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
            h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
            if (!h) h = dlopen(nm, RTLD_NOW);
            if (h) break;
        }
        if (!h) {
            r.why = "libnvrtc.so.12 not found";
            return r;
        }
        r.create = (decltype(r.create))dlsym(h, "nvrtcCreateProgram");
        r.compile = (decltype(r.compile))dlsym(h, "nvrtcCompileProgram");
        r.log_size = (decltype(r.log_size))dlsym(h, "nvrtcGetProgramLogSize");
        r.log = (decltype(r.log))dlsym(h, "nvrtcGetProgramLog");
        r.cubin_size = (decltype(r.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
        r.cubin = (decltype(r.cubin))dlsym(h, "nvrtcGetCUBIN");
        r.destroy = (decltype(r.destroy))dlsym(h, "nvrtcDestroyProgram");
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        if (!r.ok) r.why = "libnvrtc lacks nvrtcGetCUBIN";
        return r;
    }();
    return n;
}

const char* ctype_of(int dt) { return dt == kDslF64 ? "double" : (dt == kDslI32 ? "int" : "long long"); }

bool valid_label(const std::string& s) {
    if (s.empty() || !(std::isalpha((unsigned char)s[0]) || s[0] == '_')) return false;
    for (char ch : s)
        if (!(std::isalnum((unsigned char)ch) || ch == '_')) return false;
    return true;
}

// generated-code prelude: the parameter block, a ScalarArray accumulator (S[k] and S += x of
// Listing lst:simple-kernel), a strided j-side accessor, deterministic block sums
const char* kDslPrelude = R"(
struct DslParams { )" LJMD_DSL_STR(LJMD_DSL_PARAMS_BODY) R"( };
template <typename T, int N> struct DslAcc {
    T v[N];
    __device__ DslAcc() { for (int k = 0; k < N; ++k) v[k] = T(0); }
    __device__ T& operator[](int k) { return v[k]; }
    __device__ DslAcc& operator+=(T x) { v[0] += x; return *this; }
    __device__ DslAcc& operator-=(T x) { v[0] -= x; return *this; }
};
template <typename T> struct DslStrided {
    const T* p; long long s;
    __device__ T operator[](int k) const { return p[(long long)k * s]; }
};
template <typename T> __device__ T dsl_block_sum(T v) {
    __shared__ T sh[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    T r = T(0);
    if (threadIdx.x < 32) {
        r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : T(0);
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;
}
)";

// Source of one loop.  Pair loop: CTA per tile, the tile's halo rows staged in shared memory
// (positions, and the owner index for j-side dat reads), thread per owned particle i over its
// Verlet list, kernel body run for every entry with canonical r^2 < shell_cutoff^2.
std::string generate(const DslLoop& L, const std::string& code, const std::string& consts) {
    // every name the template declares starts with ljmd_ so it cannot shadow a user label
    std::ostringstream s;
    s << kDslPrelude << "\n" << consts << "\n";
    const bool pair = L.kind == 1;
    s << "extern \"C\" __global__ void __launch_bounds__(" << L.block << ") " << L.name << "(DslParams ljmd_p) {\n";
    if (pair) {
        s << "  extern __shared__ double ljmd_smem[];\n"
             "  const int ljmd_tile = blockIdx.x;\n"
             "  const int ljmd_t0 = ljmd_p.obegin[ljmd_p.tile_oc0[ljmd_tile]];\n"
             "  const int ljmd_m = ljmd_p.obegin[ljmd_p.tile_oc0[ljmd_tile + 1]] - ljmd_t0;\n"
             "  const int ljmd_R = ljmd_p.tile_R[ljmd_tile];\n"
             "  const int* ljmd_rb = ljmd_p.tr_begin + ljmd_tile * ljmd_p.rows_max;\n"
             "  const int* ljmd_ro = ljmd_p.tr_off + ljmd_tile * (ljmd_p.rows_max + 1);\n"
             "  const int ljmd_total = ljmd_ro[ljmd_R];\n"
             "  double* ljmd_sP = ljmd_smem;\n"
             "  int* ljmd_sO = (int*)(ljmd_sP + 3 * ljmd_total);\n"
             "  for (int ljmd_r = 0; ljmd_r < ljmd_R; ++ljmd_r) {\n"
             "    const int ljmd_b0 = ljmd_rb[ljmd_r], ljmd_o0 = ljmd_ro[ljmd_r];\n"
             "    const int ljmd_len = ljmd_p.tr_len[ljmd_tile * ljmd_p.rows_max + ljmd_r];\n"
             "    for (int ljmd_k = threadIdx.x; ljmd_k < ljmd_len; ljmd_k += blockDim.x) {\n"
             "      const double* ljmd_q = ljmd_p.x + 4 * (long long)(ljmd_b0 + ljmd_k);\n"
             "      ljmd_sP[3 * (ljmd_o0 + ljmd_k)] = ljmd_q[0];\n"
             "      ljmd_sP[3 * (ljmd_o0 + ljmd_k) + 1] = ljmd_q[1];\n"
             "      ljmd_sP[3 * (ljmd_o0 + ljmd_k) + 2] = ljmd_q[2];\n"
             "      ljmd_sO[ljmd_o0 + ljmd_k] = ljmd_p.slot_t ? ljmd_p.slot_t[ljmd_b0 + ljmd_k] : (ljmd_b0 + ljmd_k);\n"
             "    }\n"
             "  }\n"
             "  __syncthreads();\n";
    }
    // ScalarArray accumulators live across the particles a thread handles
    for (size_t k = 0; k < L.args.size(); ++k) {
        const DslArg& a = L.args[k];
        if (a.global && a.access != LJMD_READ)
            s << "  DslAcc<" << ctype_of(a.dtype) << ", " << a.ncomp << "> " << a.label << ";\n";
    }
    if (pair)
        s << "  for (int ljmd_qq = threadIdx.x; ljmd_qq < ljmd_m; ljmd_qq += blockDim.x) {\n"
             "    const int ljmd_t = ljmd_t0 + ljmd_qq;\n";
    else
        s << "  {\n    const int ljmd_t = blockIdx.x * blockDim.x + threadIdx.x;\n    if (ljmd_t < ljmd_p.n_own) {\n";
    s << "    const double* ljmd_xip = ljmd_p.x + 4 * (long long)ljmd_p.own_slot[ljmd_t];\n"
         "    const double ljmd_xi[3] = {ljmd_xip[0], ljmd_xip[1], ljmd_xip[2]};\n";
    const std::string P = "ljmd_p.";
    auto K = [](size_t k) { return std::to_string(k); };
    // i-side copies
    for (size_t k = 0; k < L.args.size(); ++k) {
        const DslArg& a = L.args[k];
        if (a.handle == LJMD_DAT_POSITION || a.global || !a.local) continue;
        const char* T = ctype_of(a.dtype);
        s << "    " << T << " ljmd_" << a.label << "_i[" << a.ncomp << "];\n";
        if (a.access == LJMD_INC_ZERO) {
            s << "    for (int ljmd_c = 0; ljmd_c < " << a.ncomp << "; ++ljmd_c) ljmd_" << a.label << "_i[ljmd_c] = ("
              << T << ")0;\n";
        } else {
            s << "    for (int ljmd_c = 0; ljmd_c < " << a.ncomp << "; ++ljmd_c) ljmd_" << a.label
              << "_i[ljmd_c] = ((const " << T << "*)" << P << "ptr[" << K(k) << "])[(long long)ljmd_t * " << P
              << "st[" << K(k) << "] + (long long)ljmd_c * " << P << "sc[" << K(k) << "]];\n";
        }
    }
    std::ostringstream bind;   // the labels seen by the user code
    for (size_t k = 0; k < L.args.size(); ++k) {
        const DslArg& a = L.args[k];
        const std::string T = ctype_of(a.dtype);
        const std::string q = a.access == LJMD_READ ? "const " : "";
        if (a.global) {
            if (a.access == LJMD_READ)
                bind << "      const " << T << "* " << a.label << " = (const " << T << "*)" << P << "ptr[" << K(k)
                     << "];\n";
            continue;
        }
        const bool jside = pair && (a.access == LJMD_READ || a.access == LJMD_RW || a.access == LJMD_WRITE);
        std::string ival;
        if (a.handle == LJMD_DAT_POSITION) ival = "ljmd_xi";
        else if (a.local) ival = "ljmd_" + a.label + "_i";
        else ival = "((" + T + "*)" + P + "ptr[" + K(k) + "]) + (long long)ljmd_t * " + P + "st[" + K(k) + "]";
        if (!jside) {
            bind << "      struct { " << q << T << "* i; } " << a.label << " = { " << ival << " };\n";
            continue;
        }
        std::string jt, jval;
        if (a.handle == LJMD_DAT_POSITION) {
            jt = "const double*";
            jval = "ljmd_sP + 3 * ljmd_l";
        } else if (a.ncomp == 1 || a.handle >= 0) {   // AoS rows (user dats) or one component
            jt = "const " + T + "*";
            jval = "((const " + T + "*)" + P + "jptr[" + K(k) + "]) + (long long)ljmd_tj * " + P + "jst[" + K(k) + "]";
        } else {                                      // engine SoA (velocities, forces)
            jt = "DslStrided<" + T + ">";
            jval = "DslStrided<" + T + ">{((const " + T + "*)" + P + "jptr[" + K(k) + "]) + ljmd_tj * " + P + "jst[" +
                   K(k) + "], " + P + "jsc[" + K(k) + "]}";
        }
        bind << "      struct { " << q << T << "* i; " << jt << " j; } " << a.label << " = { " << ival << ", " << jval
             << " };\n";
    }
    if (pair) {
        // the list in its 16-byte blocks of 8 indices (one load per block, the next block in
        // flight while the current one is evaluated), as the engine's force kernel reads it
        s << "    const int ljmd_cnt = ljmd_p.ncount[ljmd_t];\n"
             "    const uint4* ljmd_nb = (const uint4*)ljmd_p.nbr + ljmd_t;\n"
             "    const int ljmd_nblk = (ljmd_cnt + 7) >> 3;\n"
             "    uint4 ljmd_cur = ljmd_nblk > 0 ? ljmd_nb[0] : make_uint4(0u, 0u, 0u, 0u);\n"
             "    for (int ljmd_b = 0; ljmd_b < ljmd_nblk; ++ljmd_b) {\n"
             "     const uint4 ljmd_nxt = ljmd_b + 1 < ljmd_nblk ? ljmd_nb[(long long)(ljmd_b + 1) * ljmd_p.n_pad]\n"
             "                                                   : make_uint4(0u, 0u, 0u, 0u);\n"
             "     const unsigned ljmd_w[4] = {ljmd_cur.x, ljmd_cur.y, ljmd_cur.z, ljmd_cur.w};\n"
             "     ljmd_cur = ljmd_nxt;\n"
             "     #pragma unroll\n"
             "     for (int ljmd_e = 0; ljmd_e < 8; ++ljmd_e) {\n"
             "      if (ljmd_b * 8 + ljmd_e >= ljmd_cnt) break;\n"
             "      const int ljmd_l = (ljmd_e & 1) ? (int)(ljmd_w[ljmd_e >> 1] >> 16) : (int)(ljmd_w[ljmd_e >> 1] & 0xffffu);\n"
             "      const double* ljmd_xj = ljmd_sP + 3 * ljmd_l;\n"
             "      const double ljmd_dx = ljmd_xi[0] - ljmd_xj[0], ljmd_dy = ljmd_xi[1] - ljmd_xj[1];\n"
             "      const double ljmd_dz = ljmd_xi[2] - ljmd_xj[2];\n"
             "      const double ljmd_r2 = __dadd_rn(__dadd_rn(__dmul_rn(ljmd_dx, ljmd_dx), __dmul_rn(ljmd_dy, ljmd_dy)),\n"
             "                                       __dmul_rn(ljmd_dz, ljmd_dz));\n"
             "      if (!(ljmd_r2 < ljmd_p.cut2)) continue;\n"
             "      const int ljmd_tj = ljmd_sO[ljmd_l];\n"
             "      (void)ljmd_tj;\n"
          << bind.str() << "      {\n" << code << "\n      }\n     }\n    }\n";
    } else {
        s << "    {\n" << bind.str() << "      {\n" << code << "\n      }\n    }\n";
    }
    // write back the i-side copies of written dats
    for (size_t k = 0; k < L.args.size(); ++k) {
        const DslArg& a = L.args[k];
        if (a.handle == LJMD_DAT_POSITION || a.global || !a.local || a.access == LJMD_READ) continue;
        s << "    for (int ljmd_c = 0; ljmd_c < " << a.ncomp << "; ++ljmd_c) ((" << ctype_of(a.dtype) << "*)" << P
          << "ptr[" << K(k) << "])[(long long)ljmd_t * " << P << "st[" << K(k) << "] + (long long)ljmd_c * " << P
          << "sc[" << K(k) << "]] = ljmd_" << a.label << "_i[ljmd_c];\n";
    }
    s << (pair ? "  }\n" : "    }\n  }\n");
    // ScalarArray INC: deterministic block sums into per-block partials
    for (size_t k = 0; k < L.args.size(); ++k) {
        const DslArg& a = L.args[k];
        if (!a.global || a.access == LJMD_READ) continue;
        const char* T = ctype_of(a.dtype);
        s << "  for (int ljmd_c = 0; ljmd_c < " << a.ncomp << "; ++ljmd_c) {\n"
          << "    const " << T << " ljmd_v = dsl_block_sum<" << T << ">(" << a.label << ".v[ljmd_c]);\n"
          << "    if (threadIdx.x == 0) ((" << T << "*)" << P << "part[" << K(k) << "])[(long long)blockIdx.x * "
          << a.ncomp << " + ljmd_c] = ljmd_v;\n  }\n";
    }
    s << "}\n";
    return s.str();
}

ljmd_status dsl_enable(ljmd_ctx* c) {
    if (c->dsl_on) return LJMD_OK;
    if (!c->split && !c->slot_t) TRY(dalloc(c, &c->slot_t, (size_t)c->slot_cap));
    if (!c->tmap) TRY(dalloc(c, &c->tmap, (size_t)c->n_global));
    TRY(dalloc(c, &c->tile_R, (size_t)c->n_tiles));
    k_tile_R<<<nblk(c->n_tiles, 256), 256, 0, c->stream>>>(c->n_tiles, c->geo, c->tile_R);
    CKL();
    c->dsl_on = true;
    c->slot_t_valid = false;
    return LJMD_OK;
}

ljmd_status dsl_slot_owner(ljmd_ctx* c) {
    if (c->slot_t_valid || c->split) return LJMD_OK;
    k_cna_tmap<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->gid[c->oc_cur], c->tmap);
    CKL();
    k_slot_owner<<<nblk(c->n_slots, 256), 256, 0, c->stream>>>(c->n_slots, c->slot_gid, c->tmap, c->slot_t);
    CKL();
    c->slot_t_valid = true;
    return LJMD_OK;
}

}  // namespace

// rebuild hooks (called from rebuild() around the owned-order permutation)
ljmd_status dsl_before_sort(ljmd_ctx* c, const int* gid_old) {
    if (!c->dsl_on) return LJMD_OK;
    k_cna_tmap<<<nblk(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, gid_old, c->tmap);
    CKL();
    return LJMD_OK;
}

ljmd_status dsl_after_sort(ljmd_ctx* c) {
    if (!c->dsl_on) return LJMD_OK;
    const int n = c->n_own;
    for (DslDat& d : c->dats) {
        if (!d.alive || d.global) continue;
        const int words = d.ncomp * d.esize / 4;
        k_dat_permute<<<nblk((int64_t)n * words, 256), 256, 0, c->stream>>>(
            n, words, c->gid[c->oc_cur], c->tmap, (const unsigned*)d.d, (unsigned*)d.tmp);
        CKL();
        std::swap(d.d, d.tmp);
    }
    c->slot_t_valid = false;
    return LJMD_OK;
}

// load_state: dats to caller (gid) order, which is the owned order right after loading
ljmd_status dsl_to_gid_order(ljmd_ctx* c) {
    if (!c->dsl_on || c->n_own == 0) return LJMD_OK;
    for (DslDat& d : c->dats) {
        if (!d.alive || d.global) continue;
        if (c->split) {   // a new state may give this slab particles whose rows live elsewhere
            CK(cudaMemsetAsync(d.d, 0, (size_t)c->own_cap * d.ncomp * d.esize, c->stream));
            continue;
        }
        const int words = d.ncomp * d.esize / 4;
        k_dat_to_gid<<<nblk((int64_t)c->n_own * words, 256), 256, 0, c->stream>>>(
            c->n_own, words, c->gid[c->oc_cur], (const unsigned*)d.d, (unsigned*)d.tmp);
        CKL();
        std::swap(d.d, d.tmp);
    }
    return LJMD_OK;
}

// migration ("the State object will automatically move all data owned by the
// particle to the receiving processor"): rows follow the engine's compaction of (x, v, gid)
ljmd_status dsl_migrate(ljmd_ctx* c, int stay, int out_lo, int out_hi, int in_lo, int in_hi) {
    if (!c->dsl_on) return LJMD_OK;
    for (DslDat& d : c->dats) {
        if (!d.alive || d.global) continue;
        const size_t row = (size_t)d.ncomp * d.esize;
        const int words = (int)(row / 4);
        if ((size_t)c->mig_cap > d.msend_cap) {
            for (int b = 0; b < 2; ++b) TRY(dalloc(c, (char**)&d.msend[b], row * (size_t)c->mig_cap));
            d.msend_cap = (size_t)c->mig_cap;
        }
        if (stay) {
            k_dat_gather_idx<<<nblk((int64_t)stay * words, 256), 256, 0, c->stream>>>(
                stay, words, c->stay_t, (const unsigned*)d.d, (unsigned*)d.tmp);
            CKL();
        }
        const int outs[2] = {out_lo, out_hi};
        for (int b = 0; b < 2; ++b) {
            if (!outs[b]) continue;
            k_dat_gather_mig<<<nblk((int64_t)outs[b] * words, 256), 256, 0, c->stream>>>(
                outs[b], words, c->mig_send[b], (const unsigned*)d.d, (unsigned*)d.msend[b]);
            CKL();
        }
        char* dst = (char*)d.tmp;
        TRY(exchange(c, d.msend[1], row * out_hi, d.msend[0], row * out_lo, dst + row * stay, row * in_lo,
                     dst + row * (stay + in_lo), row * in_hi));
        std::swap(d.d, d.tmp);
    }
    return LJMD_OK;
}

namespace {
ljmd_status dat_lookup(ljmd_ctx* c, int64_t h, DslDat** out) {
    if (h < 0 || h >= (int64_t)c->dats.size() || !c->dats[h].alive)
        return set_err(c, LJMD_E_ARG, "bad dat handle %lld", (long long)h);
    *out = &c->dats[h];
    return LJMD_OK;
}
}  // namespace

extern "C" ljmd_status ljmd_dat_create(ljmd_ctx* c, int64_t ncomp, int64_t dtype, int64_t global, int64_t* handle) {
    TRY(check_ready(c));
    if (!handle || ncomp < 1 || ncomp > (1 << 20) || dtype < 0 || dtype > 2)
        return set_err(c, LJMD_E_ARG, "ljmd_dat_create: ncomp >= 1 and dtype in {0 f64, 1 i32, 2 i64}");
    TRY(dsl_enable(c));
    DslDat d;
    d.alive = true;
    d.global = global != 0;
    d.ncomp = (int)ncomp;
    d.dtype = (int)dtype;
    d.esize = dtype == kDslI32 ? 4 : 8;
    const size_t rows = d.global ? 1 : (size_t)std::max<int64_t>(c->own_cap, c->n_global);
    const size_t bytes = rows * (size_t)ncomp * d.esize;
    TRY(dalloc(c, (char**)&d.d, bytes));
    TRY(dalloc(c, (char**)&d.tmp, bytes));
    CK(cudaMemsetAsync(d.d, 0, bytes, c->stream));
    c->dats.push_back(d);
    *handle = (int64_t)c->dats.size() - 1;
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_dat_set(ljmd_ctx* c, int64_t h, const void* host) {
    TRY(check_ready(c));
    c->energy_current = false;   // engine velocities may change: no cached energies
    DslDat* d;
    TRY(dat_lookup(c, h, &d));
    if (!host) return set_err(c, LJMD_E_ARG, "ljmd_dat_set: NULL");
    const size_t row = (size_t)d->ncomp * d->esize;
    if (d->global) {
        CK(cudaMemcpyAsync(d->d, host, row, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return LJMD_OK;
    }
    CK(cudaMemcpyAsync(d->tmp, host, row * (size_t)c->n_global, cudaMemcpyHostToDevice, c->stream));
    const int words = (int)(row / 4);
    k_dat_from_gid<<<nblk((int64_t)c->n_own * words, 256), 256, 0, c->stream>>>(
        c->n_own, words, c->gid[c->oc_cur], (const unsigned*)d->tmp, (unsigned*)d->d);
    CKL();
    CK(cudaStreamSynchronize(c->stream));
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_dat_get(ljmd_ctx* c, int64_t h, void* host) {
    TRY(check_ready(c));
    DslDat* d;
    TRY(dat_lookup(c, h, &d));
    if (!host) return set_err(c, LJMD_E_ARG, "ljmd_dat_get: NULL");
    const size_t row = (size_t)d->ncomp * d->esize;
    if (d->global) {
        CK(cudaMemcpyAsync(host, d->d, row, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return LJMD_OK;
    }
    const int words = (int)(row / 4);
    k_dat_to_gid<<<nblk((int64_t)c->n_own * words, 256), 256, 0, c->stream>>>(
        c->n_own, words, c->gid[c->oc_cur], (const unsigned*)d->d, (unsigned*)d->tmp);
    CKL();
    if (!c->split) {
        CK(cudaMemcpyAsync(host, d->tmp, row * (size_t)c->n_global, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return LJMD_OK;
    }
    // several ranks: only the rows of this rank's particles are written
    std::vector<char> all(row * (size_t)c->n_global);
    std::vector<int> g(c->n_own);
    CK(cudaMemcpyAsync(all.data(), d->tmp, all.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g.data(), c->gid[c->oc_cur], sizeof(int) * g.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int t = 0; t < c->n_own; ++t)
        std::memcpy((char*)host + row * (size_t)g[t], all.data() + row * (size_t)g[t], row);
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_dat_free(ljmd_ctx* c, int64_t h) {
    TRY(check_ready(c));
    DslDat* d;
    TRY(dat_lookup(c, h, &d));
    CK(cudaStreamSynchronize(c->stream));
    for (void* q : {d->d, d->tmp, d->msend[0], d->msend[1]})
        if (q) cudaFree(q);
    *d = DslDat{};
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_loop_create(ljmd_ctx* c, int64_t kind, const char* name, const char* code,
                                        const char* constants, double shell_cutoff, int64_t nargs,
                                        const char* const* labels, const int64_t* handles, const int64_t* access,
                                        int64_t flags, int64_t* loop) {
    TRY(check_ready(c));
    if (!loop || !name || !code || (nargs > 0 && (!labels || !handles || !access)) || nargs < 0 ||
        nargs > kDslMaxArgs || (kind != 0 && kind != 1))
        return set_err(c, LJMD_E_ARG, "ljmd_loop_create: bad arguments (kind 0/1, at most %d dats)", kDslMaxArgs);
    if (kind == 1 && !(shell_cutoff > 0.0 && shell_cutoff <= c->rc))
        return set_err(c, LJMD_E_ARG,
                       "ljmd_loop_create: pair loops need 0 < shell_cutoff <= rc = %g (the Verlet list covers rc)",
                       c->rc);
    TRY(dsl_enable(c));
    Nvrtc& nv = nvrtc();
    if (!nv.ok) return set_err(c, LJMD_E_CUDA, "ljmd_loop_create: %s", nv.why.c_str());
    DslLoop L;
    L.kind = (int)kind;
    L.cut2 = shell_cutoff * shell_cutoff;
    L.block = 256;
    std::string nm = "ljmd_dsl_";
    for (const char* p = name; *p; ++p) nm += std::isalnum((unsigned char)*p) ? *p : '_';
    L.name = nm + "_" + std::to_string(c->loops.size());
    for (int64_t k = 0; k < nargs; ++k) {
        DslArg a;
        a.label = labels[k] ? labels[k] : "";
        a.handle = handles[k];
        a.access = (int)access[k];
        if (!valid_label(a.label))
            return set_err(c, LJMD_E_ARG, "ljmd_loop_create: label '%s' is not a C identifier", a.label.c_str());
        for (int64_t q = 0; q < k; ++q)
            if (L.args[q].label == a.label)
                return set_err(c, LJMD_E_ARG, "ljmd_loop_create: label '%s' used twice", a.label.c_str());
        if (a.access < LJMD_READ || a.access > LJMD_INC_ZERO)
            return set_err(c, LJMD_E_ARG, "ljmd_loop_create: bad access descriptor for '%s'", a.label.c_str());
        if (a.handle >= 0) {
            DslDat* d;
            TRY(dat_lookup(c, a.handle, &d));
            a.ncomp = d->ncomp;
            a.dtype = d->dtype;
            a.global = d->global;
            a.local = a.global || d->ncomp <= kDslLocalMax;
            if (a.global && (a.access == LJMD_WRITE || a.access == LJMD_RW))
                return set_err(c, LJMD_E_ARG, "ljmd_loop_create: ScalarArray '%s' allows READ, INC, INC_ZERO",
                               a.label.c_str());
        } else {
            a.local = true;
            switch (a.handle) {
                case LJMD_DAT_POSITION: a.ncomp = 3; a.dtype = kDslF64; break;
                case LJMD_DAT_VELOCITY: a.ncomp = 3; a.dtype = kDslF64; break;
                case LJMD_DAT_FORCE: a.ncomp = 3; a.dtype = kDslF64; break;
                case LJMD_DAT_GID: a.ncomp = 1; a.dtype = kDslI32; break;
                case LJMD_DAT_ENERGY: a.ncomp = 1; a.dtype = kDslF64; break;
                default: return set_err(c, LJMD_E_ARG, "ljmd_loop_create: bad engine dat %lld", (long long)a.handle);
            }
            if (a.handle != LJMD_DAT_VELOCITY && a.access != LJMD_READ)
                return set_err(c, LJMD_E_ARG, "ljmd_loop_create: engine dat '%s' is READ only (velocities: any)",
                               a.label.c_str());
        }
        L.args.push_back(a);
    }
    // constants: "name=value" per line -> #define (Constant objects, Tab. tab:DSL_data)
    std::string consts;
    if (constants) {
        std::istringstream in(constants);
        std::string line;
        while (std::getline(in, line)) {
            if (line.empty()) continue;
            const size_t eq = line.find('=');
            if (eq == std::string::npos || !valid_label(line.substr(0, eq)))
                return set_err(c, LJMD_E_ARG, "ljmd_loop_create: constant '%s' is not name=value", line.c_str());
            consts += "#define " + line.substr(0, eq) + " (" + line.substr(eq + 1) + ")\n";
        }
    }
    L.source = generate(L, code, consts);
    nvrtcProgram prog;
    if (nv.create(&prog, L.source.c_str(), (L.name + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
        return set_err(c, LJMD_E_CUDA, "nvrtcCreateProgram failed");
    const bool fmad = (flags & 1) != 0;
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", fmad ? "--fmad=true" : "--fmad=false",
                          "-lineinfo"};
    const nvrtcResult cr = nv.compile(prog, 4, opts);
    size_t ls = 0;
    nv.log_size(prog, &ls);
    L.log.assign(ls, '\0');
    if (ls) nv.log(prog, &L.log[0]);
    if (cr != NVRTC_SUCCESS) {
        nv.destroy(&prog);
        return set_err(c, LJMD_E_ARG, "ljmd_loop_create: kernel '%s' does not compile: %.400s", name,
                       L.log.c_str());
    }
    size_t cs = 0;
    nv.cubin_size(prog, &cs);
    std::vector<char> cubin(cs);
    nv.cubin(prog, cubin.data());
    nv.destroy(&prog);
    CK(cudaLibraryLoadData(&L.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    CK(cudaLibraryGetKernel(&L.kernel, L.lib, L.name.c_str()));
    if (L.kind == 1)
        CK(cudaKernelSetAttributeForDevice(L.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kMaxStageSmem, c->device));
    L.part.assign(L.args.size(), nullptr);
    L.part_cap.assign(L.args.size(), 0);
    L.jbuf.assign(L.args.size(), nullptr);
    L.jbuf_cap.assign(L.args.size(), 0);
    L.jsend.assign(L.args.size(), nullptr);
    L.jsend_cap.assign(L.args.size(), 0);
    L.alive = true;
    c->loops.push_back(new DslLoop(L));
    *loop = (int64_t)c->loops.size() - 1;
    return LJMD_OK;
}

namespace {
// Halo update of one argument the pair loop reads on the j side ("before the
// execution of the loop halo regions have to be updated for all variables which have a
// READ access descriptor"): owned rows to their slots, boundary-plane rows exchanged with
// the z neighbours exactly like the positions, then the ghost cells filled.
ljmd_status dsl_halo(ljmd_ctx* c, DslLoop& L, size_t k, DslParams& p) {
    const DslArg& a = L.args[k];
    const int es = a.dtype == kDslI32 ? 4 : 8;
    const size_t row = (size_t)a.ncomp * es;
    const int words = (int)(row / 4);
    if ((size_t)c->slot_cap > L.jbuf_cap[k]) {
        TRY(dalloc(c, (char**)&L.jbuf[k], row * (size_t)c->slot_cap));
        L.jbuf_cap[k] = (size_t)c->slot_cap;
    }
    const int ns = c->n_send[0] + c->n_send[1];
    if ((size_t)std::max(ns, 1) > L.jsend_cap[k]) {
        TRY(dalloc(c, (char**)&L.jsend[k], row * (size_t)std::max(ns, 1)));
        L.jsend_cap[k] = (size_t)std::max(ns, 1);
    }
    const int n = c->n_own, g = nblk((int64_t)n * a.ncomp, 256);
    if (a.dtype == kDslF64)
        k_elems_to_slots<double><<<g, 256, 0, c->stream>>>(n, a.ncomp, c->own_slot, (const double*)p.ptr[k],
                                                           p.st[k], p.sc[k], (double*)L.jbuf[k]);
    else if (a.dtype == kDslI64)
        k_elems_to_slots<long long><<<g, 256, 0, c->stream>>>(n, a.ncomp, c->own_slot, (const long long*)p.ptr[k],
                                                              p.st[k], p.sc[k], (long long*)L.jbuf[k]);
    else
        k_elems_to_slots<int><<<g, 256, 0, c->stream>>>(n, a.ncomp, c->own_slot, (const int*)p.ptr[k], p.st[k],
                                                        p.sc[k], (int*)L.jbuf[k]);
    CKL();
    if (ns) {
        k_slot_pack_words<<<nblk((int64_t)ns * words, 256), 256, 0, c->stream>>>(
            ns, words, c->send_idx, (const unsigned*)L.jbuf[k], (unsigned*)L.jsend[k]);
        CKL();
    }
    char* sb = (char*)L.jsend[k];
    char* rb = (char*)L.jbuf[k] + row * (size_t)c->n_slots;
    TRY(exchange(c, sb + row * c->n_send[0], row * c->n_send[1], sb, row * c->n_send[0], rb, row * c->n_recv[0],
                 rb + row * c->n_recv[0], row * c->n_recv[1]));
    if (c->n_gcell) {
        GhostCells gc{c->gc_dst, c->gc_src, c->gc_shift, c->n_gcell};
        k_slot_ghosts_words<<<nblk((int64_t)c->n_gcell * 32, 256), 256, 0, c->stream>>>(
            gc, c->ebegin, c->ecount, c->recv_cnt, c->recv_off, c->n_slots, words, (unsigned*)L.jbuf[k]);
        CKL();
    }
    p.jptr[k] = L.jbuf[k];
    p.jst[k] = a.ncomp;
    p.jsc[k] = 1;
    return LJMD_OK;
}
}  // namespace

extern "C" ljmd_status ljmd_loop_execute(ljmd_ctx* c, int64_t loop) {
    TRY(check_ready(c));
    if (loop < 0 || loop >= (int64_t)c->loops.size() || !c->loops[loop] || !c->loops[loop]->alive)
        return set_err(c, LJMD_E_ARG, "bad loop handle %lld", (long long)loop);
    DslLoop& L = *c->loops[loop];
    c->energy_current = false;   // a loop may write the engine's velocities
    if (L.kind == 1) TRY(dsl_slot_owner(c));
    DslParams p;
    std::memset(&p, 0, sizeof p);
    p.x = reinterpret_cast<const double*>(c->x[c->xc]);
    p.own_slot = c->own_slot;
    p.nbr = reinterpret_cast<const unsigned short*>(c->nbr8);
    p.ncount = c->ncount;
    p.obegin = c->obegin;
    p.tile_oc0 = c->tile_oc0;
    p.tr_begin = c->tr_begin;
    p.tr_off = c->tr_off;
    p.tr_len = c->tr_len;
    p.tile_R = c->tile_R;
    p.slot_t = c->slot_t;
    p.n_own = c->n_own;
    p.n_pad = c->n_pad;
    p.rows_max = kRowsMax;
    p.cut2 = L.cut2;
    p.slot_t = c->split ? nullptr : c->slot_t;
    const int nblocks = L.kind == 1 ? c->n_tiles : std::max(1, nblk(c->n_own, L.block));
    const size_t oc = c->own_cap;
    for (size_t k = 0; k < L.args.size(); ++k) {
        const DslArg& a = L.args[k];
        if (a.handle >= 0) {
            DslDat* d;
            TRY(dat_lookup(c, a.handle, &d));
            p.ptr[k] = d->d;
            p.st[k] = d->ncomp;
            p.sc[k] = 1;
            if (!a.global && !a.local && a.access == LJMD_INC_ZERO)
                CK(cudaMemsetAsync(d->d, 0, (size_t)c->n_own * d->ncomp * d->esize, c->stream));
            if (a.global && a.access != LJMD_READ) {
                const size_t need = (size_t)nblocks * a.ncomp * d->esize;
                if (need > L.part_cap[k]) {
                    if (L.part[k]) cudaFree(L.part[k]);
                    L.part[k] = nullptr;
                    TRY(dalloc(c, (char**)&L.part[k], need));
                    L.part_cap[k] = need;
                }
                p.part[k] = L.part[k];
            }
        } else {
            switch (a.handle) {
                case LJMD_DAT_POSITION: p.ptr[k] = nullptr; break;
                case LJMD_DAT_VELOCITY: p.ptr[k] = c->v[c->oc_cur]; p.st[k] = 1; p.sc[k] = (long long)oc; break;
                case LJMD_DAT_FORCE: p.ptr[k] = c->F; p.st[k] = 1; p.sc[k] = (long long)oc; break;
                case LJMD_DAT_GID: p.ptr[k] = c->gid[c->oc_cur]; p.st[k] = 1; p.sc[k] = 1; break;
                case LJMD_DAT_ENERGY: p.ptr[k] = c->e; p.st[k] = 1; p.sc[k] = 1; break;
            }
        }
    }
    for (size_t k = 0; k < L.args.size(); ++k) {   // j-side data (pair loops)
        p.jptr[k] = p.ptr[k];
        p.jst[k] = p.st[k];
        p.jsc[k] = p.sc[k];
        const DslArg& a = L.args[k];
        const bool jside = L.kind == 1 && !a.global && a.handle != LJMD_DAT_POSITION &&
                           (a.access == LJMD_READ || a.access == LJMD_RW || a.access == LJMD_WRITE);
        if (!jside || !c->split) continue;
        if (a.handle == LJMD_DAT_GID) {   // slot-space gids exist for every slot already
            p.jptr[k] = c->slot_gid;
            p.jst[k] = 1;
            p.jsc[k] = 1;
            continue;
        }
        TRY(dsl_halo(c, L, k, p));
    }
    void* args[] = {&p};
    const size_t smem = L.kind == 1 ? (3 * sizeof(double) + sizeof(int)) * (size_t)(c->max_staged + 1) : 0;
    CK(cudaLaunchKernel((const void*)L.kernel, dim3(nblocks), dim3(L.block), args, smem, c->stream));
    CKL();
    for (size_t k = 0; k < L.args.size(); ++k) {   // ScalarArray INC: sum, all-reduce, apply
        const DslArg& a = L.args[k];
        if (!a.global || a.access == LJMD_READ) continue;
        DslDat* d = &c->dats[a.handle];
        const int zero = a.access == LJMD_INC_ZERO;
        if ((size_t)a.ncomp > L.delta_cap) {
            TRY(dalloc(c, &L.delta, (size_t)a.ncomp));
            L.delta_cap = (size_t)a.ncomp;
        }
        const int g = nblk(a.ncomp, 128);
        if (a.dtype == kDslF64)
            k_dsl_fin_delta<double><<<g, 128, 0, c->stream>>>((const double*)L.part[k], nblocks, a.ncomp, L.delta);
        else if (a.dtype == kDslI64)
            k_dsl_fin_delta<long long><<<g, 128, 0, c->stream>>>((const long long*)L.part[k], nblocks, a.ncomp,
                                                                  L.delta);
        else
            k_dsl_fin_delta<int><<<g, 128, 0, c->stream>>>((const int*)L.part[k], nblocks, a.ncomp, L.delta);
        CKL();
        if (c->split) TRY(allreduce(c, L.delta, a.ncomp, false));
        if (a.dtype == kDslF64)
            k_dsl_apply<double><<<g, 128, 0, c->stream>>>(L.delta, a.ncomp, (double*)d->d, zero);
        else if (a.dtype == kDslI64)
            k_dsl_apply<long long><<<g, 128, 0, c->stream>>>(L.delta, a.ncomp, (long long*)d->d, zero);
        else
            k_dsl_apply<int><<<g, 128, 0, c->stream>>>(L.delta, a.ncomp, (int*)d->d, zero);
        CKL();
    }
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_loop_source(ljmd_ctx* c, int64_t loop, char* out, int64_t cap, int64_t* len) {
    TRY(check_ready(c));
    if (loop < 0 || loop >= (int64_t)c->loops.size() || !c->loops[loop])
        return set_err(c, LJMD_E_ARG, "bad loop handle %lld", (long long)loop);
    const std::string& s = c->loops[loop]->source;
    if (len) *len = (int64_t)s.size();
    if (out && cap > 0) {
        const size_t m = std::min<size_t>((size_t)cap - 1, s.size());
        std::memcpy(out, s.data(), m);
        out[m] = '\0';
    }
    return LJMD_OK;
}

extern "C" ljmd_status ljmd_loop_free(ljmd_ctx* c, int64_t loop) {
    TRY(check_ready(c));
    if (loop < 0 || loop >= (int64_t)c->loops.size() || !c->loops[loop])
        return set_err(c, LJMD_E_ARG, "bad loop handle %lld", (long long)loop);
    CK(cudaStreamSynchronize(c->stream));
    DslLoop* L = c->loops[loop];
    for (auto* v : {&L->part, &L->jbuf, &L->jsend})
        for (void* q : *v)
            if (q) cudaFree(q);
    if (L->delta) cudaFree(L->delta);
    if (L->lib) cudaLibraryUnload(L->lib);
    delete L;
    c->loops[loop] = nullptr;
    return LJMD_OK;
}

void dsl_destroy(ljmd_ctx* c) {
    for (DslDat& d : c->dats)
        for (void* q : {d.d, d.tmp, d.msend[0], d.msend[1]})
            if (q) cudaFree(q);
    c->dats.clear();
    for (DslLoop* L : c->loops) {
        if (!L) continue;
        for (auto* v : {&L->part, &L->jbuf, &L->jsend})
            for (void* q : *v)
                if (q) cudaFree(q);
        if (L->delta) cudaFree(L->delta);
        if (L->lib) cudaLibraryUnload(L->lib);
        delete L;
    }
    c->loops.clear();
}
