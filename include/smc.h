/*
 * smc.h — C ABI of libsmc: B200-native (sm_100a) data-parallel hot path of
 * sequential Monte Carlo over PPL control-flow graphs (PCFGs), after
 * Lunden et al., "Compiling Universal Probabilistic Programming Languages
 * with Efficient Parallel Sequential Monte Carlo Inference" (arXiv
 * 2112.00364).  Citation keys: P:n = PAPER.md line n; DESIGN.md §R-x = a
 * documented reading where the paper is silent.
 *
 * What one handle computes: Algorithm 1 with the RootPPL loop
 * order: N particles start at block b0; each epoch every particle
 * runs its PCFG blocks up to the next checkpoint drawing
 * from counter-based Philox streams keyed by (seed, global particle, epoch,
 * draw) and accumulating a log-weight; if every particle reached b_stop the
 * run ends with a final log Z update and no resample (§R-6);
 * otherwise the weights are normalised (log-sum-exp; log Z += LSE - log N,
 * P:655, §R-7), scanned, mapped to ancestors by systematic resampling
 * (§R-8/§R-9: exact integer weights) and the particle states are
 * gathered.
 *
 * Conventions
 *  - All functions are extern "C"; no torch types cross the boundary.
 *  - A handle owns all device memory it allocates; model data and params are
 *    COPIED at create.  Host output buffers are caller-owned.  Functions
 *    taking device pointers (smc_resample_device) never take ownership.
 *  - Errors: every int-returning function returns an smc_status; the message
 *    is available from smc_errmsg(h) (or smc_errmsg(NULL) for the last
 *    failed create on this thread).  A failed handle stays valid for
 *    smc_stats/smc_errmsg/smc_destroy.
 *  - Thread-compatible: one handle per host thread.
 *  - Determinism: for fixed (model, total N, seed) every output is
 *    bit-identical across runs and across shard counts (reading R1).
 *  - There is no CPU fallback: without a CUDA device smc_create fails with
 *    SMC_ECUDA.
 */
#ifndef SMC_H
#define SMC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMC_ABI_VERSION 2

typedef enum {
  SMC_OK = 0,
  SMC_EINVAL = 1,     /* bad argument: N = 0 or total N >= 2^32, malformed data, unknown kind */
  SMC_ECUDA = 2,      /* CUDA runtime error (message has the CUDA error string)               */
  SMC_ENCCL = 3,      /* NCCL error or NCCL unavailable                                         */
  SMC_EREJECTED = 4,  /* every particle has log-weight -inf (log Z = -inf)               */
  SMC_ENAN = 5,       /* a log-weight became NaN or +inf (model bug), §R-10                     */
  SMC_EOVERFLOW = 6,  /* helper stack/event cap overflow with SMC_FLAG_STRICT, §R-12            */
  SMC_ESTATE = 7      /* call not valid in the handle's current state                           */
} smc_status;

/* Model kinds (block tables; DESIGN.md "Models" gives each spec). */
typedef enum {
  SMC_CRBD = 1,            /* constant-rate birth-death on a fixed tree (§R-11)   */
  SMC_CLADS2 = 2,          /* lineage-specific-rate birth-death (BASELINE configs[2], §R-14)   */
  SMC_SEIR = 3,            /* vector-borne disease SEIR (§R-15)                   */
  SMC_GEOMETRIC = 10,      /* weighted geometric, Fig. 2                    */
  SMC_SSM = 11,            /* linear-Gaussian state-space model, Eq. (2) / Fig. 4  */
  SMC_CONSTW = 12,         /* weight(log w); checkpoint; ... K times                   */
  SMC_FIG3 = 13,           /* the PCFG of Fig. 3(a), blocks b0..b4 (DESIGN R-23)    */
  SMC_STACKF = 14,         /* Fig. 5(c) recursion with a PSTATE byte stack (R-24)   */
  SMC_RESAMPLE_BENCH = 20  /* no blocks: resampler only, opaque state (BASELINE configs[4])    */
} smc_model_kind;

#define SMC_FLAG_STRICT 1u   /* helper-stack overflow is an error instead of weight -inf */
/* CRBD / CLADS2: lineage-keyed side trees: every hidden-tree
 * node draws from its own Philox counter, so a CTA evaluates one particle's
 * side trees in parallel (cooperative kernel).  Same model, different (equally
 * valid) stream layout; results match the oracle's lineage-keyed kinds. */
#define SMC_FLAG_LINEAGE_RNG 2u
/* CRBD only: the §5.3 variance reduction:
 * each hidden speciation event at age t contributes ln 2 + ln E(t), E(t) the
 * probability that a lineage alive at age t leaves no sampled descendant,
 * instead of a simulated side tree.  Overrides SMC_FLAG_LINEAGE_RNG (no side
 * trees are simulated).  CLADS2 with this flag: SMC_EINVAL (lineage-specific
 * rates have no closed-form E). */
#define SMC_FLAG_ANALYTIC_UNDETECTED 4u
/* Any kind: in-place resampling: the sorted
 * systematic ancestors are permuted so that every particle with offspring
 * keeps its slot and its extra copies fill the slots without offspring in
 * ascending order; the state is updated in place (one state buffer, copies
 * only into slots without offspring).  smc_ancestors returns the permuted
 * ancestors.  Single shard only: smc_create_virtual with shards > 1 or
 * smc_create_sharded with world > 1 -> SMC_EINVAL.  smc_resample_device:
 * d_state_out must be NULL or equal to d_state_in. */
#define SMC_FLAG_INPLACE 8u

/*
 * Model description (all arrays COPIED at create).
 *  CRBD, CLADS2  data = tree: [M, root, (parent, left, right, age) x M] as
 *                doubles (tips: left = right = -1; ages in time units before
 *                present).  params CRBD: [rho, lambda_fixed, mu_fixed]
 *                (fixed < 0: draw from the prior); CLADS2: [rho, lambda0,
 *                sigma, alpha, eps] (each < 0: prior).
 *  SEIR          data = observed daily cases y[T]; params optional:
 *                [lam_h, del_h, gam_h, lam_m, del_m, rho] (lam_h < 0: priors),
 *                [6] n_h, [7] initial susceptible mosquitoes, [8] initial
 *                exposed humans, [9] initial infectious mosquitoes.
 *  SSM           data = y[T]; params [m0, s0, drift, q, r] (std devs).
 *  GEOMETRIC     params [p, w].      CONSTW  params [log w, K].
 *  FIG3          params [p_loop, p3, w1, w2, w3, w4] (defaults 0.5, 0.3, 2,
 *                1.2, 1.2, 0.5): b2 loops with probability p_loop (weight w2),
 *                goes to b3 with p3 (weight w3, checkpoint, back to b2), else
 *                to b4 (weight w4, checkpoint, b_stop); b1 weighs w1.
 *  STACKF        data = y[D] (observation per recursion depth, may be empty);
 *                params [p0, p_rec, sigma, cap] (defaults 2, 2, 0.5, 768):
 *                the recursive f of Fig. 5 made terminating (recurse iff
 *                s1 >= 1), a byte stack of cap bytes (multiple of 16, 48-byte
 *                frames) plus a stack pointer; state = 16-byte header +
 *                cap/16 stack planes, of which resampling copies only the
 *                planes below the stack pointer.
 *  RESAMPLE_BENCH state_bytes = bytes per particle (multiple of 16, <= 512).
 */
typedef struct {
  int32_t kind;            /* smc_model_kind                                  */
  uint32_t state_bytes;    /* SMC_RESAMPLE_BENCH only                         */
  const double* data;      /* host pointer, may be NULL when data_len == 0    */
  uint64_t data_len;       /* number of doubles in data                       */
  const double* params;    /* host pointer, may be NULL when n_params == 0    */
  int32_t n_params;
  uint32_t flags;          /* SMC_FLAG_*                                      */
} smc_model;

typedef struct smc_ctx* smc_handle;

/* Run statistics (this rank / the whole virtual group). */
typedef struct {
  uint64_t n_total;                 /* particles over all shards/ranks                       */
  uint64_t n_local;                 /* particles owned by this handle (all virtual shards)    */
  uint64_t epochs;                  /* propagation epochs completed                          */
  uint64_t resamples;               /* resampling steps completed                            */
  uint64_t alive_particle_steps;    /* sum over epochs of particles with pc != b_stop at the
                                       start of the epoch (this handle's particles)          */
  uint64_t overflow;                /* particles set to -inf by a helper-stack/event cap     */
  int64_t first_error_particle;     /* global index of the first overflow/NaN particle, -1   */
  int32_t status;                   /* smc_status of the run so far                          */
  int32_t rank, world, shards;      /* process rank/world and virtual shards in this handle  */
  uint32_t state_bytes;             /* bytes of SoA state per particle                       */
  uint32_t done;                    /* 1 when the run reached b_stop (or failed)             */
  uint64_t draws;                   /* uniforms drawn by propagation (this handle)           */
  double ms_propagate;              /* CUDA-event time of propagation (smc_set_timing on)    */
  double ms_resample;               /* ... of the resampling chain (reduce, gather, finalize) */
  uint64_t timed_epochs;            /* epochs covered by the two timers                      */
  uint64_t side_roots;              /* lineage-keyed kernels: hidden events (side-tree roots) */
  uint32_t max_rounds;              /* ... longest cooperative phase of a batch (rounds)      */
  uint32_t max_side_nodes;          /* ... largest side-tree node count of one particle-step  */
  uint64_t distinct;                /* distinct ancestors, summed over the resamples since
                                       reset (per call for smc_resample_*)                   */
  double ms_kernel[4];              /* resample-only path with timing on: CUDA-event ms of
                                       max, reduce, anc_gather, finalize (accumulated)       */
  uint64_t stack_planes;            /* stack models (ClaDS2, STACKF): 16-byte state planes the
                                       out-of-place gathers copied, summed since reset (the
                                       stack prefix only, R-22/R-24)                          */
  uint64_t guard_kills;             /* ClaDS2: particle-steps set to -inf by the rate guard
                                       (R-14b; under SMC_FLAG_LINEAGE_RNG a step
                                       whose side trees both detect and break the guard may
                                       be counted either way)                               */
  uint32_t deferred_gather;         /* 1: resampling writes ancestors only and the next
                                       propagation reads each state from its ancestor's slot
                                       (DESIGN.md 7.7); 0: the resampling step copies states  */
  uint32_t reserved0;
} smc_stats_t;

/* --- lifetime --------------------------------------------------------------- */

/* One GPU, N particles.  Returns NULL on error (smc_errmsg(NULL)).
 * N in [1, 2^32).  Uses the current CUDA device. */
smc_handle smc_create(const smc_model* model, uint64_t n_particles, uint64_t seed);

/* One GPU emulating `n_shards` ranks of `n_per_shard` particles each (global
 * index = shard * n_per_shard + local).  Runs the multi-GPU resampler path
 * (per-shard records, global offsets, cross-shard migration) in one process;
 * results are identical to smc_create with N = n_shards * n_per_shard. */
smc_handle smc_create_virtual(const smc_model* model, uint64_t n_per_shard, uint64_t seed,
                              int32_t n_shards);

/* Collective hooks for one-process-per-GPU runs.
 *  nccl_id    128-byte ncclUniqueId (smc_get_nccl_id on rank 0, broadcast by the
 *             caller), or NULL to use `allgather` for the small exchanges.
 *  allgather  host-staged all-gather: gathers `bytes` from every rank into
 *             recv[world * bytes] in rank order; returns 0 on success.  Used
 *             when nccl_id is NULL (e.g. torch.distributed gloo in tests). */
typedef struct {
  const void* nccl_id;
  int (*allgather)(const void* send, void* recv, uint64_t bytes, void* user);
  void* user;
} smc_comm;

/* Rank `rank` of `world`, n_per_rank particles each.  After creation each
 * rank exports its peer-memory handle (smc_ipc_export), the caller
 * all-gathers the blobs, and every rank calls smc_ipc_import before running.
 * Migration of particles between ranks is done by the gather kernel with
 * stores into peer memory (CUDA IPC over NVLink). */
smc_handle smc_create_sharded(const smc_model* model, uint64_t n_per_rank, uint64_t seed,
                              int32_t rank, int32_t world, const smc_comm* comm);
/* Writes this rank's IPC blob (smc_ipc_blob_bytes() bytes) to out. */
int smc_ipc_export(smc_handle h, void* out);
uint64_t smc_ipc_blob_bytes(void);
/* blobs = world concatenated blobs in rank order. */
int smc_ipc_import(smc_handle h, const void* blobs);

/* rank 0: writes a fresh 128-byte ncclUniqueId (NCCL loaded at run time). */
int smc_get_nccl_id(void* out128);

void smc_destroy(smc_handle h);

/* CUDA stream (cudaStream_t as void*) for all subsequent work; NULL = the
 * handle's own non-blocking stream. */
int smc_set_stream(smc_handle h, void* cuda_stream);

/* --- running ---------------------------------------------------------------- */

/* ESS-adaptive resampling: resample at a
 * checkpoint only if ESS < tau N, tau = a / b, decided exactly in integers
 * (b W^2 < a N sum q^2); otherwise weights accumulate and log Z is not
 * updated until the next resample or the end.  a >= b (default 1/1):
 * resample at every checkpoint (plain Algorithm 1).  Persists across
 * smc_reset. */
int smc_set_ess_threshold(smc_handle h, uint32_t a, uint32_t b);

/* smc_run as ONE CUDA graph launch (default on): a WHILE conditional node
 * repeats {epoch, epoch} until the device sets done; no host round trip per
 * epoch.  Off: a host loop of smc_step (needed with a host all-gather comm or
 * per-phase timing, which force the host loop automatically). */
int smc_set_graph(smc_handle h, int32_t on);

/* Resampling launch shape.  *grid_out = the CTA count of the
 * single cooperative launch that performs a whole resampling step (rows
 * a6-a10: quantise + exact u128 sum, grid barrier, ancestors + gather,
 * log Z), chosen at create time when the handle holds one shard, resamples
 * out of place and its particles fit the co-resident grid's shared memory
 * (12 B each); 0 = the split reduce / anc_gather / finalize kernels (several
 * shards, in-place, large N, or env SMC_NO_FUSED_RESAMPLE=1 at create).
 * Both paths give bit-identical results.  Returns SMC_EINVAL on NULL. */
int smc_resample_grid(smc_handle h, int32_t* grid_out);

/* Per-phase CUDA-event timing of every epoch (off by default).  The times
 * accumulate into smc_stats_t.ms_propagate / ms_resample until smc_reset. */
int smc_set_timing(smc_handle h, int32_t on);

/* Replace the model data (tree / series) with new data of the SAME shape
 * (host pointer; copied to the device on the handle's stream); parameters
 * are kept.  With smc_reset this runs a new sweep without re-creating the
 * handle (the per-step input upload of bench.py's e2e figure). */
int smc_set_data(smc_handle h, const double* data, uint64_t data_len);

/* Re-initialise for a fresh sweep: pc = b0, log Z = 0, epoch = 0, new seed. */
int smc_reset(smc_handle h, uint64_t seed);

/* Run epochs until every particle reached b_stop.  Synchronises the stream.
 * Returns SMC_OK, SMC_EREJECTED, SMC_ENAN or SMC_EOVERFLOW (strict). */
int smc_run(smc_handle h);

/* One epoch (propagate, then resample or finish).  *done = 1 at the end. */
int smc_step(smc_handle h, int32_t* done);

/* --- results (synchronise the stream) -------------------------------------- */

/* log of the normalising-constant estimate; NaN before the first epoch. */
double smc_log_z(smc_handle h);
/* Ancestor (global index) of each of this handle's slots from the LAST
 * resample (identity before the first); out has n = n_local entries. */
int smc_ancestors(smc_handle h, uint32_t* out, uint64_t n);
/* Log-weights accumulated since the last resample (the final normalised
 * weights are exp(lw - LSE(lw))); out has n_local entries. */
int smc_log_weights(smc_handle h, double* out, uint64_t n);
/* Raw SoA state: plane-major, bytes = state_bytes * n_local. */
int smc_state(smc_handle h, void* out, uint64_t bytes);
/* Decoded state: n_local x smc_nfields(h) doubles, in the field order of
 * DESIGN.md "Observable state" (pc first). */
int smc_nfields(smc_handle h);
int smc_fields(smc_handle h, double* out, uint64_t n_doubles);
int smc_stats(smc_handle h, smc_stats_t* out);
/* Message for the last error on h, or for the last failed create on this
 * thread when h is NULL.  Never NULL. */
const char* smc_errmsg(smc_handle h);

/* --- resampler alone (BASELINE configs[4]) --------------------------------- */

/* One resampling step on caller-owned DEVICE buffers (handle of kind
 * SMC_RESAMPLE_BENCH with n particles): d_lw[n] log-weights; d_state_in /
 * d_state_out SoA planes (plane p of particle k at byte offset
 * (p * n + k) * 16), state_bytes / 16 planes; d_anc[n] receives global
 * ancestors.  `epoch` selects the resampling uniform (Philox counter
 * (0, epoch, 0, 1)).  Enqueued on the handle's stream, no synchronisation.
 * Reads back the log Z increment into *logz_inc only if logz_inc != NULL
 * (synchronises).  d_lw, d_state_in and d_state_out must be 16-byte aligned
 * (128-bit loads/stores; SMC_EINVAL otherwise).  The caller's pointers are
 * used for this call only (the handle's own buffers are not redirected). */
int smc_resample_device(smc_handle h, const double* d_lw, const void* d_state_in,
                        void* d_state_out, uint32_t* d_anc, uint32_t epoch, double* logz_inc);
/* Same with HOST buffers: copies in, resamples, copies anc and states out
 * (pageable or pinned host memory; synchronises). */
int smc_resample_host(smc_handle h, const double* lw, const void* state_in, void* state_out,
                      uint32_t* anc, uint32_t epoch, double* logz_inc);

/* Resampling of the handle's OWN buffers, global across shards/ranks (the
 * multi-GPU form of configs[4]).  smc_load copies n_local log-weights and the
 * SoA state (plane-major per shard) into the handle (device_ptrs != 0: device
 * pointers, else host); smc_resample_step then runs max, reduce, the two
 * all-gathers, anc_gather with peer-store migration, the barrier and
 * finalize, and swaps buffers; smc_state / smc_ancestors read the result.
 * Enqueued on the handle's stream (host-staged comm synchronises). */
int smc_load(smc_handle h, const double* lw, const void* state, int32_t device_ptrs);
int smc_resample_step(smc_handle h, uint32_t epoch);

/* Number of distinct ancestors in the last smc_resample_* call (for the
 * algorithmic-bytes count); synchronises. */
int smc_last_distinct(smc_handle h, uint64_t* out);

/* Host-side planner of the global systematic grid (no device needed): given
 * the all-gathered integer shard totals W_g (w_lohi[2g] = low 64 bits, [2g+1]
 * = high), world shards of n_per particles and the resampling integer z
 * (u = (2z+1) 2^-54), writes out[0..world] with out[g] = #{grid points j :
 * (j + u) W < N P_g}, P_g = W_0 + ... + W_{g-1}: shard g's particles fill the
 * global output slots [out[g], out[g+1]).  Identical integer arithmetic to the
 * device kernels; used for migration accounting and by the CPU tests. */
int smc_plan_ranges(const uint64_t* w_lohi, int32_t world, uint64_t n_per, uint64_t z,
                    uint64_t* out);

/* Measured draw-rate ceiling of propagation (the roofline
 * denominator of the "alu"-bound propagation kernels): launches a
 * divergence-free microkernel on the current device in which every lane of a
 * full-occupancy grid draws draws_per_thread Exp(rate) variates from its own
 * Philox4x32-10 stream (hq conversion, the kernels' table-driven fp64 log of a
 * uniform times a precomputed 1/rate; R-1..R-3, §7)
 * and writes their sum.  *draws_per_s = uniforms consumed per second, best of
 * three timed launches (CUDA events).  SMC_EINVAL for a NULL output or 0
 * draws; SMC_ECUDA without a device.  Allocates and frees its own buffer. */
int smc_draw_peak(uint32_t draws_per_thread, double* draws_per_s);

/* Symbols-only helper: ABI version of the loaded library. */
int smc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SMC_H */
