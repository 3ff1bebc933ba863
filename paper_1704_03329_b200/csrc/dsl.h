// dsl.h -- types of the PairLoop / ParticleLoop front end (the paper's
// DSL, Sec. 2.2-2.4): particle data registered with a context, user C
// kernels compiled at run time with NVRTC into a tile-staged template for sm_100a.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace ljmd {

// Kernel parameter block, shared verbatim by the host (this struct) and the generated CUDA
// source (the same text, stringified), so the two layouts cannot drift apart.
#define LJMD_DSL_PARAMS_BODY                                                                  \
    const double* x;             /* slot-space positions, 4 doubles per slot          */     \
    const int* own_slot;                                                                      \
    const unsigned short* nbr;   /* blocked 16-bit local indices (build order)        */     \
    const int* ncount;                                                                        \
    const int* obegin;                                                                        \
    const int* tile_oc0;                                                                      \
    const int* tr_begin;                                                                      \
    const int* tr_off;                                                                        \
    const int* tr_len;           /* true row lengths (rows are padded in the layout)  */     \
    const int* tile_R;                                                                        \
    const int* slot_t;           /* slot -> owned index (one rank); null: j by slot    */     \
    void* ptr[24];               /* argument k: data base pointer                     */     \
    long long st[24];            /* element (t, c) at ptr[k][t * st[k] + c * sc[k]]   */     \
    long long sc[24];                                                                         \
    void* jptr[24];              /* j-side data: owned arrays (one rank) or the        */     \
    long long jst[24];           /* slot-space halo copy (several ranks), indexed by   */     \
    long long jsc[24];           /* the staged sO[l]                                   */     \
    void* part[24];              /* argument k (ScalarArray INC): per-block partials  */     \
    int n_own;                                                                                \
    int n_pad;                                                                                \
    int rows_max;                                                                             \
    int pad_;                                                                                 \
    double cut2;                 /* shell_cutoff^2 (pair loops)                       */

struct DslParams {
    LJMD_DSL_PARAMS_BODY
};

#define LJMD_DSL_STR2(...) #__VA_ARGS__
#define LJMD_DSL_STR(x) LJMD_DSL_STR2(x)

constexpr int kDslMaxArgs = 24;
constexpr int kDslLocalMax = 16;   // i-side copies in registers up to this many components

enum DslDtype { kDslF64 = 0, kDslI32 = 1, kDslI64 = 2 };

struct DslDat {
    bool alive = false;
    bool global = false;   // ScalarArray (one row)
    int ncomp = 1;
    int dtype = kDslF64;
    int esize = 8;
    void* d = nullptr;     // owned order [own_cap][ncomp] (global: [ncomp])
    void* tmp = nullptr;   // permutation / host-order staging, same size
    void* msend[2] = {nullptr, nullptr};   // migration send rows (nranks > 1)
    size_t msend_cap = 0;
};

struct DslArg {
    std::string label;
    long long handle = 0;  // >= 0 user dat; < 0 engine dat (LJMD_DAT_*)
    int access = 0;        // LJMD_READ ..
    int ncomp = 1;
    int dtype = kDslF64;
    bool global = false;
    bool local = true;     // i-side copy in registers (else direct global access)
};

struct DslLoop {
    bool alive = false;
    int kind = 0;          // 0 particle loop, 1 pair loop
    std::string name, source, log;
    double cut2 = 0.0;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    int block = 256;
    std::vector<DslArg> args;
    std::vector<void*> part;      // per-argument partial buffers (ScalarArray INC)
    std::vector<size_t> part_cap;
    std::vector<void*> jbuf;      // per-argument slot-space halo copy (nranks > 1)
    std::vector<size_t> jbuf_cap;
    std::vector<void*> jsend;     // per-argument boundary-plane send rows
    std::vector<size_t> jsend_cap;
    double* delta = nullptr;      // ScalarArray INC: this launch's sums (all-reduced)
    size_t delta_cap = 0;
};

}  // namespace ljmd
