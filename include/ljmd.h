/*
 * ljmd.h -- C ABI of the B200-native Lennard-Jones PairLoop engine
 * (hot path of arXiv 1704.03329, PPMD: cell binning, Verlet neighbour list
 * within rbar_c = rc + delta, fp64 LJ force/energy, velocity-Verlet updates).
 *
 * The calls follow the paper's statement of the problem:
 *   - State / Domain / PositionDat / ParticleDat (Sec. 3.1, PAPER.md:234-299,
 *     Listing lst:state-example PAPER.md:385-402)      -> ljmd_init
 *   - IntegratorRange(Ni, dt, v, Ns, delta) driving Algorithm
 *     alg:VelocityVerlet   -> ljmd_step
 *   - PairLoop of Listing lst:LJ-loop returning F and u
 *                                                    -> ljmd_get_forces/energy
 *
 * Conventions (all calls):
 *   - Return ljmd_status; LJMD_OK == 0.  The first error puts the context in
 *     the error state: every later call except ljmd_last_error/ljmd_destroy
 *     returns LJMD_E_STATE.  ljmd_last_error names the particle (global index,
 *     "gid" = row in the caller's arrays) where one applies.
 *   - Host arrays are owned by the caller, row-major [n][3] float64 in the
 *     caller's particle order (gid = row).  They are copied in by ljmd_init /
 *     ljmd_set_state and written by the getters; the library never keeps a
 *     pointer to them.  The library owns all device memory, the CUDA stream it
 *     creates (unless one is passed in ljmd_options.stream) and the NCCL
 *     communicator, and releases them in ljmd_destroy.
 *   - Periodic orthorhombic box [0,Lx) x [0,Ly) x [0,Lz) only (reading R10).
 *   - Not thread-safe per context; one context per rank/GPU.
 *   - No CPU fallback: every computation runs in the sm_100a kernels of
 *     libljmd.so; a missing GPU returns LJMD_E_CUDA.
 */
#ifndef LJMD_H
#define LJMD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ljmd_ctx ljmd_ctx;

typedef enum {
    LJMD_OK = 0,
    LJMD_E_ARG = -1,       /* bad argument (NULL pointer, n <= 0, rc <= 0, ...)            */
    LJMD_E_BOX = -2,       /* fewer than 3 cells of width >= rbar_c in some dimension       */
    LJMD_E_NONFINITE = -3, /* non-finite position/velocity; message names the gid           */
    LJMD_E_OVERLAP = -4,   /* two particles at r^2 == 0; message names both gids            */
    LJMD_E_CAPACITY = -5,  /* device allocation for a regrown buffer failed                 */
    LJMD_E_CUDA = -6,      /* CUDA runtime error / no device                                 */
    LJMD_E_NCCL = -7,      /* NCCL error (nranks > 1)                                        */
    LJMD_E_STATE = -8      /* context poisoned by an earlier error                           */
} ljmd_status;

/* Every field is 8 bytes wide so the struct has no padding (ctypes-friendly). */
typedef struct {
    double  delta;          /* shell thickness delta = rbar_c - rc; default 0.25 = 0.1 rc
                               (Tab. 7.2T1)                      */
    int64_t rebuild_every;  /* list reuse count Ns; default 20               */
    int64_t rebuild_check;  /* 0: fixed Ns only (paper); 1: also rebuild when
                               2 max_i |x_i - x_i(build)| > delta (reading R7)              */
    double  mass;           /* scalar particle mass m; default 1 (reading R11)              */
    double  energy_shift;   /* s in V = 4 eps[(sigma/r)^12 - (sigma/r)^6 + s]; default 0.25
                               = the paper's Eq. eqn:LJpotential (R3)         */
    int64_t energy_every;   /* sample PE/KE every k steps inside ljmd_step; default 10
                               (PAPER.md:866); 0 disables in-loop sampling                  */
    int64_t device;         /* CUDA device ordinal; -1 = current device (default)           */
    int64_t nbr_capacity;   /* initial neighbour-list width K; 0 = automatic. Grown
                               transparently (and the list rebuilt) on overflow             */
    int64_t rank;           /* this rank in [0, nranks); default 0                          */
    int64_t nranks;         /* number of z-slab ranks; 1 = single GPU (no NCCL)             */
    const void* nccl_id;    /* nranks > 1: pointer to a 128-byte ncclUniqueId, identical on
                               every rank (broadcast by the caller, e.g. torch.distributed) */
    void*   stream;         /* cudaStream_t to launch on; NULL = library-created stream    */
    int64_t profile;        /* 1: time every force launch with CUDA events (ljmd_get_stats) */
    int64_t list_order;     /* 1 (default): bank-aware neighbour order (fastest) for lists
                               expected to serve >= 10 steps (always with the fixed Ns = 20;
                               with rebuild_check as long as recent lists lasted that long) on
                               systems with one force CTA per tile, build order otherwise; 0: always the build order (stencil
                               row, slot) -- results then do not depend on the number of
                               slabs (bitwise), at ~13 % more force-kernel time             */
    int64_t split_self;     /* 1: with nranks = 1, still run the slab-exchange path (halo
                               planes sent to itself through the transport; testing)        */
    int64_t newton3;        /* 1: Newton-3 half list: each pair
                               evaluated once, reactions added with fp64 global reductions,
                               velocity Verlet in a separate pass; nranks = 1 only.  Slower
                               than the default on B200; sums not bitwise
                               reproducible (reduction order)                                */
    int64_t validate;       /* 1: validation mode (single rank, full list): before every force
                               evaluation inside ljmd_step, count the ordered pairs with
                               r^2 < rc^2 (canonical r^2, minimum image, R9) that the Verlet
                               list does not serve -- a fresh cell search minus the in-range
                               list entries, per particle.  Per-step counts from
                               ljmd_get_validation; totals in ljmd_stats.  Costs about one list
                               build per step; 0 (default) off.  The paper's fixed Ns = 20
                                keeps a list past the skin guarantee of
                               Eq. eqn:extended_cutoff when particles move
                               fast: this measures what that costs in missed interactions.  */
    int64_t graphs;         /* 1 (default): on one rank (no newton3 / validate / profile /
                               thermostat / DSL data), ljmd_step runs as a captured CUDA graph:
                               the rebuild decision (fixed Ns or the displacement check) and the
                               capacity checks are taken on the device, no host round trip per
                               step or per rebuild; a capacity shortfall resumes on the eager
                               path at that step.  0: eager launches (host decides each step). */
    int64_t tight_caps;     /* testing: after init, shrink the slot, staging and list capacities
                               to exactly what the initial state needs (the next larger rebuild
                               then exercises the capacity checks); 0 (default)               */
} ljmd_options;

typedef struct {
    int64_t steps_done;        /* MD steps since init / set_state                           */
    int64_t n_rebuilds;        /* cell + neighbour rebuilds after init                      */
    int64_t n_owned;           /* particles owned by this rank                              */
    int64_t n_ghost;           /* ghost (periodic image / halo) particles                   */
    int64_t nbr_capacity;      /* current list width K                                      */
    int64_t max_neighbours;    /* longest list at the last build                            */
    int64_t total_neighbours;  /* sum of list lengths at the last build (this rank)         */
    int64_t n_cells[3];        /* global cell grid                                          */
    int64_t regrows;           /* capacity regrowths so far                                 */
    int64_t force_launches;    /* force launches timed (profile = 1)                        */
    double  force_ms;          /* summed CUDA-event time of those launches (profile = 1)    */
    int64_t energy_samples;    /* samples available from ljmd_get_energy_history            */
    int64_t kernel_launches;   /* kernels of this library launched since init               */
    /* Rebuild certification (Eq. eqn:extended_cutoff; reading R7): a
     * rebuild is "dangerous" when 2 max_i |x_i(s-1) - x_i(build)| > delta on the last step
     * s-1 the old list served, i.e. the skin no longer guaranteed that list (counted over
     * all ranks, since init / set_state; never under rebuild_check = 1). */
    int64_t dangerous_builds;
    double  max_build_disp;    /* largest max_i |x_i(s-1) - x_i(build)| seen at a rebuild     */
    /* Validation mode (ljmd_options.validate) totals since init / set_state: */
    int64_t validated_steps;
    int64_t missed_pairs;      /* ordered pairs with r < rc not in the list, summed over steps */
    int64_t missed_particle_steps;  /* (particle, step) with at least one missed pair          */
    int64_t max_missed_particles;   /* largest number of such particles in one step           */
    int64_t graph_calls;       /* ljmd_step calls run as a captured graph                       */
    int64_t graph_aborts;      /* of those, resumed eagerly after a device capacity check      */
    int64_t graphs_cached;     /* captured step graphs currently instantiated                  */
} ljmd_stats;

/* Fill *o with the defaults listed above. */
ljmd_status ljmd_default_options(ljmd_options* o);

/* Create a context: copies pos/vel ([n][3] fp64, host) to the device, wraps
 * positions into the box (half-open, reading R10), bins them into cells of
 * width >= rbar_c (Sec. 3.4), builds the neighbour list at
 * rbar_c = rc + delta (Eq. eqn:extended_cutoff PAPER.md:406-408)
 * and computes F(r0) (reading R6) plus PE/KE at step 0.
 *   box     : [3] box lengths (Lx, Ly, Lz) > 0
 *   rc      : force cutoff (> 0); epsilon, sigma > 0; dt > 0
 *   opt     : NULL -> ljmd_default_options
 * With nranks > 1 every rank passes the same global arrays and keeps the
 * particles of its z-slab.  On failure *out is NULL and the message is
 * available from ljmd_last_error(NULL). */
ljmd_status ljmd_init(ljmd_ctx** out, int64_t n, const double* pos, const double* vel,
                      const double box[3], double rc, double epsilon, double sigma, double dt,
                      const ljmd_options* opt);

/* Replace positions and velocities (same n, box and parameters as init) and
 * redo the init sequence (wrap, bin, list, F(r0), step-0 energies).
 * pos = vel = NULL: take the state most recently queued by ljmd_stage_state (single
 * rank; LJMD_E_ARG if none is queued). */
ljmd_status ljmd_set_state(ljmd_ctx* c, const double* pos, const double* vel);

/* Overlapped host transfers for a stream of states (single rank, nranks = 1 without
 * split_self; LJMD_E_ARG otherwise).  The context owns a copy stream and two device
 * staging buffers per direction, so a transfer runs while the previous state computes.
 *
 * ljmd_stage_state: queue the host->device copy of pos and vel ([n][3] fp64, caller
 *   order; page-locked memory for a truly asynchronous copy) and return.  The host arrays
 *   must stay valid and unchanged until the ljmd_set_state(c, NULL, NULL) that consumes
 *   them has returned.  At most two states may be queued ahead of their consumption.
 * ljmd_get_positions_async: queue the device->host copy of the current positions
 *   ([n][3], caller order, unwrapped as ljmd_get_positions) into out and return; out is
 *   complete after ljmd_wait_transfers.
 * ljmd_wait_transfers: block until every queued copy has completed. */
ljmd_status ljmd_stage_state(ljmd_ctx* c, const double* pos, const double* vel);
ljmd_status ljmd_get_positions_async(ljmd_ctx* c, double* out);
ljmd_status ljmd_wait_transfers(ljmd_ctx* c);

/* Advance nsteps velocity-Verlet steps (Alg. alg:VelocityVerlet lines 5-9):
 * v += dt/(2m) F; r += dt v; [rebuild every Ns steps, after the drift, R8];
 * F <- sum over the list of Eq. eqn:LJforce (INC_ZERO, R5); v += dt/(2m) F.
 * PE and KE are sampled every energy_every steps.  After the call x, v and F are
 * synchronised at the final step (velocities at full step).
 * Asynchronous in graph mode (either rebuild policy): the call returns
 * once its steps are queued on the stream, and the host reads its outcome (rebuild steps,
 * energy samples, capacity aborts, error flags) when the NEXT ljmd_step call has been
 * queued, or at the next call of any other function of this header that reads or changes
 * the state -- so an error of one call (non-finite coordinates, coincident particles) is
 * returned by the following call, and a call queued behind a capacity abort runs as no-ops
 * and is re-run after the aborted one is resumed.  Work queued on the engine's stream after
 * ljmd_step (events, copies) is ordered after the steps.  LJMD_DEFER=0 in the environment
 * makes every call wait for its outcome (one host synchronisation per call). */
ljmd_status ljmd_step(ljmd_ctx* c, int64_t nsteps);

/* Readback in the caller's order ([n][3] / [n]; with nranks > 1 only rows of
 * particles owned by this rank are written).  Positions are the raw device
 * positions (wrapped at the last rebuild, R10) unless wrapped != 0. */
ljmd_status ljmd_get_forces(ljmd_ctx* c, double* out);
ljmd_status ljmd_get_positions(ljmd_ctx* c, double* out, int64_t wrapped);
ljmd_status ljmd_get_velocities(ljmd_ctx* c, double* out);
/* e_i = 1/2 sum_j V(r_ij) over the list, r_ij < rc (reading R2). */
ljmd_status ljmd_get_particle_energy(ljmd_ctx* c, double* out);
/* Global PE = sum_i e_i and KE = 1/2 m sum_i |v_i|^2 (Example 1)
 * at the current state (deterministic fixed-order sums; summed over ranks). */
ljmd_status ljmd_get_energy(ljmd_ctx* c, double* pe, double* ke);
/* In-loop samples recorded by ljmd_step since init/set_state (index 0 = step 0).
 * Writes min(cap, available) entries of pe/ke and *count = available. */
ljmd_status ljmd_get_energy_history(ljmd_ctx* c, double* pe, double* ke, int64_t cap,
                                    int64_t* count);
/* The current Verlet list as gid pairs: offsets[n+1] (CSR over the caller's
 * order; empty rows for particles not owned) and, if gids != NULL and
 * cap >= offsets[n], the neighbour gids of each row in list order. */
ljmd_status ljmd_get_neighbours(ljmd_ctx* c, int64_t* offsets, int64_t* gids, int64_t cap);
/* MD step index of each rebuild after init (min(cap, n_rebuilds) entries). */
ljmd_status ljmd_get_rebuild_steps(ljmd_ctx* c, int64_t* out, int64_t cap, int64_t* count);
ljmd_status ljmd_get_stats(ljmd_ctx* c, ljmd_stats* s);
/* Validation mode: per validated step since init / set_state, out[k] = {step index,
 * particles with at least one missed pair, missed ordered pairs} (min(cap, available)
 * rows of 3 int64; *count = available).  LJMD_E_ARG if validation is off. */
ljmd_status ljmd_get_validation(ljmd_ctx* c, int64_t* out, int64_t cap, int64_t* count);

/* Message of the last error of c (or of the last failed ljmd_init if c == NULL). */
const char* ljmd_last_error(const ljmd_ctx* c);
void ljmd_destroy(ljmd_ctx* c);

/* Library version string, e.g. "ljmd 0.1 sm_100a". */
const char* ljmd_version(void);

/* Bond-order analysis (Sec. 4.1): Steinhardt
 * Q_ell of every owned particle at the current positions,
 *   q_lm(i) = (1/|N(i)|) sum_{j in N(i)} Y_l^m(r_hat_ij)          (Eq. eqn:qellm)
 *   Q_l(i)  = sqrt(4 pi/(2 l + 1) sum_m |q_lm(i)|^2)             (Eq. eqn:Qell)
 * with N(i) = { j : r_ij < rcut } taken from the engine's Verlet list, so rcut <= rc is
 * required (LJMD_E_ARG otherwise); 0 <= ell <= 12.  Q[n] (and nnb[n] = |N(i)| if non-NULL)
 * in the caller's order; with nranks > 1 only owned rows are written; |N(i)| = 0 -> 0;
 * at most 160 neighbours inside rcut are used per particle. */
ljmd_status ljmd_boa(ljmd_ctx* c, int64_t ell, double rcut, double* Q, int64_t* nnb);

/* Andersen thermostat ("coupled the system to an Andersen thermostat"; SPEC
 * S:346-354; reading R19).  From the next ljmd_step on, at the end of every step (after
 * line 8 of Alg. alg:VelocityVerlet, before the energy sample) each particle is, with
 * probability nu*dt, given a new velocity drawn from N(0, T/m) per component.  The draws
 * are Philox4x32-10 keyed by (seed, gid, step index since init/set_state), so they do not
 * depend on the number of ranks.  nu = 0 switches it off (NVE, the default).
 * LJMD_E_ARG if nu < 0, T < 0 or nu*dt > 1. */
ljmd_status ljmd_set_thermostat(ljmd_ctx* c, double nu, double temperature, uint64_t seed);

/* Switch the per-launch force timing (ljmd_options.profile) on (1) or off (0) between
 * ljmd_step calls: the CUDA events around every force launch cost a few microseconds per
 * step, so a benchmark times its headline region without them.  LJMD_E_ARG if profile is
 * not 0 or 1. */
ljmd_status ljmd_set_profile(ljmd_ctx* c, int64_t profile);

/* Common-neighbour analysis (Sec. 4.2, Algs. alg:cna_I-III, alg:max_cluster_size,
 * PAPER.md:522-653, 1151-1174) at the current positions, single rank:
 * bonds = pairs with r < rcut (rcut <= rc: taken from the Verlet list).  For every bond
 * (i, j): n_nb = |common neighbours|, n_b = bonds among them, n_lcb = bonds in their
 * largest connected cluster.  cls[n]: 1 fcc (12 x (4,2,1)), 2 hcp (6 x (4,2,1) +
 * 6 x (4,2,2)), 3 bcc (14 bonds: 8 x (6,6,6) + 6 x (4,4,4)), 0 other.  Optional
 * trip[n][24]: triplet of the k-th bond of i in ascending neighbour gid, packed
 * n_nb | n_b << 8 | n_lcb << 16 (0 past the last bond); nnb[n]: bonds per particle.
 * LJMD_E_CAPACITY if a particle has more than 24 bonds. */
ljmd_status ljmd_cna(ljmd_ctx* c, double rcut, int32_t* cls, int32_t* trip, int64_t* nnb);

/* ---------------------------------------------------------------------------------------
 * PairLoop / ParticleLoop front end (the paper's DSL, Sec. 2.2-2.4; Tabs.
 * tab:DSL_data, tab:DSL_looping, tab:DSL_access).
 * With nranks > 1 particle data migrates with its particles at every rebuild, data read on
 * the j side of a pair loop is exchanged into the halo before the loop (only for READ / RW /
 * WRITE arguments: the access descriptors decide), and ScalarArray increments
 * are all-reduced over the ranks.  ljmd_dat_set takes the full [n][ncomp] array on every
 * rank; ljmd_dat_get writes the rows of this rank's particles; ljmd_set_state on several
 * ranks zeroes particle data (its rows may now belong to another rank).
 *
 * Particle data ("ParticleDat"): ncomp components of dtype (0 double, 1 int32,
 * 2 int64) per particle, zero-initialised, owned by the context, kept in the engine's
 * particle order on the device (permuted at every rebuild); ljmd_dat_set/get copy
 * [n][ncomp] host arrays in the caller's particle order.  global = 1 makes a ScalarArray
 * (P:166): one row of ncomp values, shared by all particles.
 * Engine data usable in loops (handles < 0): positions (the PositionDat, READ), velocities
 * (any access), forces, global ids (int32), per-particle energies (READ).
 *
 * Loops (ljmd_loop_create): kind 0 = ParticleLoop, 1 = PairLoop.  `code` is the user's C
 * kernel (Listing lst:simple-kernel style): for every argument k, labels[k] is visible as a
 * struct with member i (pointer to particle i's components) and, in pair loops for READ /
 * RW / WRITE data, member j (particle j's; reading R20); a ScalarArray is used as label[k]
 * (and label += x for INC).  access[k]: LJMD_READ .. LJMD_INC_ZERO (Tab. tab:DSL_access;
 * INC_ZERO zeroes first).  constants: "name=value" lines, substituted as #defines (the
 * Constant class).  A PairLoop visits the ordered pairs (i, j) of the neighbour list with
 * canonical r^2 < shell_cutoff^2, 0 < shell_cutoff <= rc (Listing lst:LJ-loop).  flags bit 0:
 * allow FMA contraction (default: every operation rounded as written, like the oracle).
 * The kernel is compiled with NVRTC for sm_100a at creation; a compile error returns
 * LJMD_E_ARG with the compiler log in ljmd_last_error. */
#define LJMD_DAT_POSITION (-1)
#define LJMD_DAT_VELOCITY (-2)
#define LJMD_DAT_FORCE (-3)
#define LJMD_DAT_GID (-4)
#define LJMD_DAT_ENERGY (-5)
enum { LJMD_READ = 0, LJMD_WRITE = 1, LJMD_RW = 2, LJMD_INC = 3, LJMD_INC_ZERO = 4 };

ljmd_status ljmd_dat_create(ljmd_ctx* c, int64_t ncomp, int64_t dtype, int64_t global, int64_t* handle);
ljmd_status ljmd_dat_set(ljmd_ctx* c, int64_t handle, const void* host);
ljmd_status ljmd_dat_get(ljmd_ctx* c, int64_t handle, void* host);
ljmd_status ljmd_dat_free(ljmd_ctx* c, int64_t handle);
ljmd_status ljmd_loop_create(ljmd_ctx* c, int64_t kind, const char* name, const char* code,
                             const char* constants, double shell_cutoff, int64_t nargs,
                             const char* const* labels, const int64_t* handles,
                             const int64_t* access, int64_t flags, int64_t* loop);
ljmd_status ljmd_loop_execute(ljmd_ctx* c, int64_t loop);
/* the generated CUDA source (len = its length; copied into out when cap > 0) */
ljmd_status ljmd_loop_source(ljmd_ctx* c, int64_t loop, char* out, int64_t cap, int64_t* len);
ljmd_status ljmd_loop_free(ljmd_ctx* c, int64_t loop);

/* Multi-GPU plumbing: fill out128 with a fresh ncclUniqueId (NCCL is loaded with dlopen;
 * the copy torch already mapped is reused).  Rank 0 calls it and broadcasts the 128
 * bytes (e.g. with torch.distributed) into ljmd_options.nccl_id on every rank.  An id
 * that starts with "LJMDLOCAL" instead selects the in-process loopback transport (several
 * contexts of one process exchanging through device copies; used by the tests to run the
 * multi-rank path on one GPU), and one that starts with "LJMDSHM:<key>" the host-staged
 * multi-PROCESS transport (ranks in separate processes on one GPU, transfers staged through
 * files under /dev/shm; correctness path for the multi-process flow, synchronous). */
ljmd_status ljmd_nccl_unique_id(void* out128);

/* Measurement utility (bench.py roofline denominator): FP64 FMA throughput of the
 * device, from a DFMA-chain probe kernel timed with CUDA events (best of 5), in
 * TFLOP/s (2 flops per FMA).  device = -1: current device. */
ljmd_status ljmd_measure_fp64_peak(int64_t device, double* tflops);

/* ---- host-side decomposition planning (pure host code, no GPU needed) ----
 * Cell grid of Sec. 3.4: n_d = floor(L_d / (rbar_c (1 + 1e-12))) (>= 3 required)
 * and the z-slab split used for nranks > 1 (slab boundaries on global cell
 * planes; the first (ncz mod nranks) ranks get one extra plane).
 * Returns LJMD_E_BOX if a dimension has fewer than 3 cells or a slab has
 * fewer than 1 plane.... */
ljmd_status ljmd_plan_cells(const double box[3], double rbar_c, int64_t nc[3]);
ljmd_status ljmd_plan_slab(int64_t ncz, int64_t nranks, int64_t rank, int64_t* z0, int64_t* z1);

#ifdef __cplusplus
}
#endif
#endif /* LJMD_H */
