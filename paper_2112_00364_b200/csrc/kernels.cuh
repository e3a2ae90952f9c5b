// kernels.cuh — the sm_100a hot path:
//   propagate<M>   Alg. 1 step 2: one particle per thread,
//                  blocks dispatched by pc until the next checkpoint; epilogue
//                  = CTA max of the log-weights (order-preserving int64
//                  atomicMax), alive count (termination), NaN flag
//   reduce         exact integer weights q = rint(2^62 exp(lw - m)) summed per
//                  2048-particle tile in u128; the last CTA scans the tile sums
//                  (normalising sum; reading R1)
//   anc_gather     per tile: exclusive u128 scan, systematic ancestor map
//                  a_j = min{k : (j+u) W < N C_k} evaluated as offspring
//                  boundaries O_k = F(C_k) (fp64 estimate + exact 192-bit fix-
//                  up near integers), then the coalesced 128-bit state gather
//                  of the tile's output slots, written straight into the
//                  destination shard's buffers (multi-GPU: peer
//                  memory), plus the ancestor array
//   finalize       log Z += m + log W - 62 ln 2 - log N, termination,
//                  epoch advance (single thread)
#pragma once
#include <climits>
#include "models.cuh"

namespace smc {

typedef unsigned __int128 u128;

constexpr int kThreads = 256;
#ifndef SMC_PROP_THREADS
#define SMC_PROP_THREADS 256
#endif
constexpr int kPThreads = SMC_PROP_THREADS;   // propagate_kernel CTA size (register cap kept: kMinBlocks x 256 threads)
constexpr int kItems = 8;                  // particles per thread in a resampling tile (large N)
constexpr int kItemsSmall = 2;             // ... below kSmallN particles per shard (more CTAs)
constexpr unsigned long long kSmallN = 0;   // small tiles measured slower at 10^6 (per-CTA fixed costs dominate)
constexpr int kTile = kThreads * kItems;

// Record all-gathered after propagation (16 B per shard).
struct RecA {
  long long key;       // order-preserving key of the shard's max log-weight
  unsigned alive;      // particles with pc != b_stop after propagation
  unsigned flags;      // bit 0: NaN or +inf log-weight seen
};

// Record all-gathered after the reduce pass (48 B per shard): integer total
// weight W and, for ESS-adaptive resampling, sum of q^2 (192-bit).
struct RecB {
  u128 W;
  unsigned long long q2[3];
  unsigned long long pad;
};

struct Ctrl {
  double logz;
  double last_inc;
  unsigned epoch;
  unsigned done;
  int status;
  unsigned counter;                  // last-block-done ticket for reduce
  unsigned long long resamples;
  unsigned long long epochs;
  unsigned long long alive_steps;
  unsigned long long overflow;
  unsigned long long first_err;      // ULLONG_MAX = none
  unsigned long long distinct;       // distinct ancestors in the last resample
  unsigned long long draws;          // uniforms drawn by propagation (all epochs)
  unsigned long long seed;           // Philox key of the run (device-resident: graphs survive reset)
  unsigned batch;                    // next 256-particle batch (persistent propagation grids)
  unsigned ess_a, ess_b;             // ESS threshold tau = a / b (a >= b: always resample, R-19)
  unsigned carry;                    // 1: the last checkpoint did not resample, lw accumulates
  unsigned max_rounds;               // diag: longest cooperative phase (rounds) in a batch
  unsigned long long side_roots;     // diag: hidden events (side-tree roots) generated
  unsigned max_side_nodes;           // diag: largest per-particle side-tree node count
  unsigned holes;                    // in-place resampling (R-21): slots without offspring
  unsigned bar_count, bar_gen;       // grid barrier of resample_fused_kernel
  unsigned long long guard_kills;    // ClaDS2 rate guard (R-14b): killed particle-steps
  unsigned long long stack_planes;   // stack models: 16-byte planes copied by the gathers (R-22/R-24)
  unsigned gmap_id;                  // deferred gather: 1 = the next propagation reads its own slot
};

enum { ST_OK = 0, ST_REJECTED = 4, ST_NAN = 5, ST_OVERFLOW = 6 };

// ---------------------------------------------------------------- u128 helpers
__device__ __forceinline__ u128 shfl_up_u128(u128 v, int d) {
  unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  lo = __shfl_up_sync(0xffffffffu, lo, d);
  hi = __shfl_up_sync(0xffffffffu, hi, d);
  return ((u128)hi << 64) | lo;
}
__device__ __forceinline__ u128 shfl_idx_u128(u128 v, int src) {
  unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  lo = __shfl_sync(0xffffffffu, lo, src);
  hi = __shfl_sync(0xffffffffu, hi, src);
  return ((u128)hi << 64) | lo;
}
__device__ __forceinline__ u128 shfl_xor_u128(u128 v, int d) {
  unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  lo = __shfl_xor_sync(0xffffffffu, lo, d);
  hi = __shfl_xor_sync(0xffffffffu, hi, d);
  return ((u128)hi << 64) | lo;
}
// u128 -> double by truncation to 53 significant bits: every
// step exact, so log W is bit-identical wherever it is evaluated.
__host__ __device__ __forceinline__ double u128_trunc_double(u128 x) {
  const unsigned long long hi = (unsigned long long)(x >> 64), lo = (unsigned long long)x;
  int bl;
#ifdef __CUDA_ARCH__
  bl = hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
#else
  bl = hi ? 128 - __builtin_clzll(hi) : (lo ? 64 - __builtin_clzll(lo) : 0);
#endif
  const int s = bl > 53 ? bl - 53 : 0;
  const unsigned long long top = (unsigned long long)(x >> s);
  return ldexp((double)top, s);
}
__device__ __forceinline__ u128 ld_cg_u128(const u128* p) {
  const unsigned long long* q = (const unsigned long long*)p;
  return ((u128)__ldcg(q + 1) << 64) | __ldcg(q);
}
__device__ __forceinline__ double u128_approx(u128 x) {
  return __ull2double_rn((unsigned long long)(x >> 64)) * 0x1p64 +
         __ull2double_rn((unsigned long long)x);
}

// 128 x 128 -> 256-bit product, limbs little-endian.
struct U256 { unsigned long long w[4]; };
__device__ __forceinline__ U256 mul_u128(u128 a, u128 b) {
  const unsigned long long a0 = (unsigned long long)a, a1 = (unsigned long long)(a >> 64);
  const unsigned long long b0 = (unsigned long long)b, b1 = (unsigned long long)(b >> 64);
  const u128 p00 = (u128)a0 * b0, p01 = (u128)a0 * b1, p10 = (u128)a1 * b0, p11 = (u128)a1 * b1;
  U256 r;
  r.w[0] = (unsigned long long)p00;
  u128 mid = (p00 >> 64) + (unsigned long long)p01 + (unsigned long long)p10;
  r.w[1] = (unsigned long long)mid;
  u128 hi = (mid >> 64) + (p01 >> 64) + (p10 >> 64) + (unsigned long long)p11;
  r.w[2] = (unsigned long long)hi;
  r.w[3] = (unsigned long long)(hi >> 64) + (unsigned long long)(p11 >> 64);
  return r;
}
__device__ __forceinline__ bool lt_u256(const U256& a, const U256& b) {
#pragma unroll
  for (int i = 3; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  return false;
}

// 192-bit accumulation of q^2 (q < 2^62+1, N < 2^32: sum < 2^157).
struct U192 { unsigned long long w[3]; };
__device__ __forceinline__ void add_u192(U192& a, const U192& b) {
  const u128 s0 = (u128)a.w[0] + b.w[0];
  const u128 s1 = (u128)a.w[1] + b.w[1] + (unsigned long long)(s0 >> 64);
  a.w[0] = (unsigned long long)s0;
  a.w[1] = (unsigned long long)s1;
  a.w[2] = a.w[2] + b.w[2] + (unsigned long long)(s1 >> 64);
}
__device__ __forceinline__ void add_u192_u128(U192& a, u128 b) {
  U192 t;
  t.w[0] = (unsigned long long)b; t.w[1] = (unsigned long long)(b >> 64); t.w[2] = 0;
  add_u192(a, t);
}
__device__ __forceinline__ U192 shfl_xor_u192(const U192& v, int d) {
  U192 r;
#pragma unroll
  for (int i = 0; i < 3; ++i) r.w[i] = __shfl_xor_sync(0xffffffffu, v.w[i], d);
  return r;
}
// 4-limb (256-bit) product x * m.
__device__ __forceinline__ void mul_limbs(const unsigned long long* x, int n, unsigned long long m,
                                          unsigned long long* out /*[4]*/) {
  u128 carry = 0;
  for (int i = 0; i < 4; ++i) {
    const u128 cur = (i < n ? (u128)x[i] * m : 0) + carry;
    out[i] = (unsigned long long)cur;
    carry = cur >> 64;
  }
}
// ESS gate (R-19): resample iff tau >= 1 or b W^2 < a N sum q^2, exactly.
__device__ __forceinline__ bool ess_resample(u128 W, const U192& Q2, unsigned long long N,
                                             unsigned a, unsigned b) {
  if (a >= b) return true;
  const unsigned long long w[2] = {(unsigned long long)W, (unsigned long long)(W >> 64)};
  unsigned long long W2[4] = {0, 0, 0, 0};
  {   // W^2 (< 2^190)
    const u128 p00 = (u128)w[0] * w[0], p01 = (u128)w[0] * w[1], p11 = (u128)w[1] * w[1];
    W2[0] = (unsigned long long)p00;
    const u128 mid = (p00 >> 64) + 2 * (u128)(unsigned long long)p01;
    W2[1] = (unsigned long long)mid;
    const u128 hi = (mid >> 64) + 2 * (p01 >> 64) + (unsigned long long)p11;
    W2[2] = (unsigned long long)hi;
    W2[3] = (unsigned long long)(hi >> 64) + (unsigned long long)(p11 >> 64);
  }
  unsigned long long lhs[4], t[4], rhs[4];
  mul_limbs(W2, 4, b, lhs);
  mul_limbs(Q2.w, 3, a, t);
  mul_limbs(t, 4, N, rhs);
#pragma unroll
  for (int i = 3; i >= 0; --i)
    if (lhs[i] != rhs[i]) return lhs[i] < rhs[i];
  return false;
}

// Systematic grid of one resampling step: positions (j + u)/N, u = (2z+1)/2^54.
struct Grid {
  u128 W;                    // total integer weight (all shards)
  u128 Nsc;                  // N * 2^54
  unsigned long long z2p1;   // 2z + 1
  unsigned long long N;
  double Wd, Nd, ud;
  double NdWd;               // N / W (fp64)
  // P(j, C): grid point j lies strictly below cumulative weight C.
  __device__ __forceinline__ bool below(unsigned long long j, u128 C) const {
    const u128 A = ((u128)j << 54) + z2p1;
    return lt_u256(mul_u128(A, W), mul_u128(Nsc, C));
  }
  // F(C) = #{j in [0, N) : (j + u) W < N C} = clamp(ceil(N C / W - u), 0, N).
  // The fp64 estimate (relative error a few ulps, i.e. < 2^-19 absolute for
  // N < 2^32) only selects the exact 192-bit fix-up near integers.
  __device__ __forceinline__ unsigned long long count_below(u128 C) const {
    const double x = u128_approx(C) * NdWd - ud;
    const double r = rint(x);
    if (fabs(x - r) > 0x1p-12) {
      double c = ceil(x);
      c = c < 0.0 ? 0.0 : (c > Nd ? Nd : c);
      return (unsigned long long)c;
    }
    long long j = (long long)r;                      // exact fix-up near integers
    if (j < 0) j = 0;
    if (j > (long long)N) j = (long long)N;
    while (j < (long long)N && below((unsigned long long)j, C)) ++j;
    while (j > 0 && !below((unsigned long long)(j - 1), C)) --j;
    return (unsigned long long)j;
  }
};

// q = rint(2^62 exp(x)), x = lw - m <= 0 (reading R9).  exp specialised to
// this domain: q = 0 below x = -44 (2^62 e^-44 = 0.36 < 1/2); otherwise
// x = k ln2 + r (Cody-Waite, |r| <= ln2/2), e^r by a degree-13 Horner
// polynomial (truncation 6e-18), scaled by 2^(k+62) in [2^-2, 2^62] — no
// over/underflow paths.  Within ~2 ulp of exp(); both resampling passes use
// this one function, so W and the prefixes are consistent.
// Coefficients in constant memory: DFMA takes a constant-bank operand
// directly, whereas 64-bit immediates cost two UMOVs per use (ncu: the reduce
// pass was issue-bound with ~24 UMOVs per particle).
__constant__ double kQuantC[16] = {
    1.4426950408889634074,        // 1/ln 2
    -6.93147180369123816490e-01,  // -ln 2 (high part)
    -1.90821492927058770002e-10,  // -ln 2 (low part)
    1.6059043836821614599e-10,    // 1/13!
    2.0876756987868098979e-09,    // 1/12!
    2.5052108385441718775e-08,
    2.7557319223985890653e-07,
    2.7557319223985890653e-06,
    2.4801587301587301587e-05,
    1.9841269841269841270e-04,
    1.3888888888888888889e-03,
    8.3333333333333333333e-03,
    4.1666666666666666667e-02,
    1.6666666666666666667e-01,
    0.5,
    -44.0};
__device__ __forceinline__ unsigned long long quantize(double lw, double m) {
  const double x0 = lw - m;
  const bool ok = x0 >= kQuantC[15];                // false for lw = -inf
  const double x = ok ? x0 : 0.0;                   // branch-free: independent chains interleave
  const double k = rint(x * kQuantC[0]);
  double r = fma(k, kQuantC[1], x);
  r = fma(k, kQuantC[2], r);
  double p = kQuantC[3];
#pragma unroll
  for (int i = 4; i <= 14; ++i) p = fma(p, r, kQuantC[i]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int e2 = (int)k + 62 + 1023;                // 2^(k+62), k in [-64, 0]
  const double scale = __hiloint2double(e2 << 20, 0);
  const unsigned long long q = __double2ull_rn(p * scale);
  return ok ? q : 0ull;
}

// ============================================================================
// propagate
// ============================================================================
struct PropArgs {
  uint4* planes;                 // current SoA planes of this shard (the epoch's output)
  // deferred gather (single shard): the epoch reads particle
  // i's state from src_planes at its ancestor gmap[i] (at i when
  // ctrl->gmap_id) and writes it to planes[i]; lazy = 0: in place (src = planes)
  const uint4* src_planes;
  const uint32_t* gmap;
  int lazy;
  double* lw;                    // [n_local]
  unsigned long long n_local;    // also the plane stride
  unsigned long long shard_base; // global index of local particle 0
  RecA* recA;                    // gathered records, both parities [2][world]
  int world, rank;
  Ctrl* ctrl;
};

// Per-thread accumulators of propagate_kernel's epilogue.
struct PropAcc {
  int start_alive = 0, end_alive = 0;
  bool bad = false;
  unsigned long long drw = 0, first_bad = ~0ull;
  long long key = LLONG_MIN;
};

// Deferred gather: the source slot of output particle i (gmap holds global
// ancestor indices; lazy runs have one shard, base 0), and the relocation of
// state a model keeps in global memory while it runs (stack planes): copied
// from the ancestor's slot below the stack pointer, then the model works on
// its own slot.  Models that hold their whole state in registers: nothing.
__device__ __forceinline__ unsigned long long gmap_src(const PropArgs& a, unsigned long long i) {
  return (*(volatile unsigned*)&a.ctrl->gmap_id) ? i : (unsigned long long)__ldg(a.gmap + i);
}
template <class M> struct HasRelocate {
  template <class T> static auto test(int) -> decltype(&T::relocate, char());
  template <class T> static long test(...);
  static constexpr bool value = sizeof(test<M>(0)) == sizeof(char);
};
template <class M>
__device__ __forceinline__ void relocate(typename M::State& s, const uint4* src, uint4* dst,
                                         unsigned long long st, unsigned long long si, unsigned long long di) {
  if constexpr (HasRelocate<M>::value) M::relocate(s, src, dst, st, si, di);
}

// One particle: load, run blocks to the next checkpoint (or STOP), store.
template <class M>
__device__ __forceinline__ void propagate_one(const PropArgs& a, const ModelConst& C, unsigned long long i,
                                              unsigned epoch, bool carry, unsigned long long seed,
                                              PropAcc& acc, Diag& dg) {
  double lw = carry ? a.lw[i] : 0.0;
  const unsigned long long ovf0 = dg.overflow;
  typename M::State s;
  if (a.lazy) {                                   // the resampled state: ancestor's slot of the previous buffer
    const unsigned long long si = gmap_src(a, i);
    M::load(s, a.src_planes, a.n_local, si);
    relocate<M>(s, a.src_planes, a.planes, a.n_local, si, i);
  } else {
    M::load(s, a.planes, a.n_local, i);
  }
  if (M::pc(s) != kStop) {
    ++acc.start_alive;
    Rng r(seed, (uint32_t)(a.shard_base + i), epoch);
    for (;;) {
      const bool ck = M::step(s, lw, r, C, dg);
      if (ck || M::pc(s) == kStop) break;
    }
    M::store(s, a.planes, a.n_local, i);
    acc.drw += 2ull * r.blk - (r.has_spare ? 1ull : 0ull);
  } else if (a.lazy) {
    M::store(s, a.planes, a.n_local, i);          // finished particles move too
  }
  acc.end_alive += M::pc(s) != kStop;
  a.lw[i] = lw;
  const bool b = isnan(lw) || lw == INFINITY;
  acc.bad |= b;
  if ((b || dg.overflow != ovf0) && acc.first_bad == ~0ull) acc.first_bad = a.shard_base + i;
  const long long k = order_key(lw);
  acc.key = k > acc.key ? k : acc.key;
}

// Register cap per model (M::kMinBlocks resident CTAs per SM), measured on
// B200: CRBD 4 (64 regs), SEIR 4 (64 regs, samplers out of line; 3 CTAs at 80 regs measured 1.7% slower), ClaDS2 2.
// Grid (M::kOneWave): light models run one wave of resident CTAs and
// grid-stride, so the epilogue's same-address atomics run once per CTA;
// uneven models run one particle per thread and let the block scheduler
// balance the load.
template <class M>
__global__ void __launch_bounds__(kPThreads, M::kMinBlocks * (256 / kPThreads)) propagate_kernel(PropArgs a, ModelConst C) {
  __shared__ long long s_key[kPThreads / 32];
  __shared__ unsigned long long s_ovf[kPThreads / 32];
  __shared__ unsigned long long s_drw[kPThreads / 32];
  if (*(volatile unsigned*)&a.ctrl->done) return;
  const unsigned epoch = a.ctrl->epoch;
  const bool carry = a.ctrl->carry != 0;               // R-19: no resample at the last checkpoint
  const unsigned long long seed = a.ctrl->seed;
  PropAcc acc;
  Diag dg;
  const unsigned long long i0 = (unsigned long long)blockIdx.x * kPThreads + threadIdx.x;
  if constexpr (M::kOneWave) {
    for (unsigned long long i = i0; i < a.n_local; i += (unsigned long long)gridDim.x * kPThreads)
      propagate_one<M>(a, C, i, epoch, carry, seed, acc, dg);
  } else {
    if (i0 < a.n_local) propagate_one<M>(a, C, i0, epoch, carry, seed, acc, dg);
  }
  int start_alive = acc.start_alive, end_alive = acc.end_alive;
  const bool bad = acc.bad;
  unsigned long long drw = acc.drw;
  const unsigned long long first_bad = acc.first_bad;
  long long key = acc.key;
  // epilogue: CTA max key, counts, flags
  unsigned long long ovf = dg.overflow;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, key, d);
    key = o > key ? o : key;
    ovf += __shfl_xor_sync(0xffffffffu, ovf, d);
    drw += __shfl_xor_sync(0xffffffffu, drw, d);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_key[warp] = key; s_ovf[warp] = ovf; s_drw[warp] = drw; }
  if (first_bad != ~0ull) atomicMin(&a.ctrl->first_err, first_bad);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    end_alive += __shfl_xor_sync(0xffffffffu, end_alive, d);
    start_alive += __shfl_xor_sync(0xffffffffu, start_alive, d);
  }
  __shared__ int s_cnt2[2][kPThreads / 32];
  if (lane == 0) { s_cnt2[0][warp] = end_alive; s_cnt2[1][warp] = start_alive; }
  __syncwarp();   // bar.red needs a converged warp (synccheck)
  const int any_bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    long long k = s_key[0];
    unsigned long long o = s_ovf[0], dr = s_drw[0];
    int n_end = s_cnt2[0][0], n_start = s_cnt2[1][0];
    for (int w = 1; w < kPThreads / 32; ++w) {
      k = s_key[w] > k ? s_key[w] : k;
      o += s_ovf[w];
      dr += s_drw[w];
      n_end += s_cnt2[0][w];
      n_start += s_cnt2[1][w];
    }
    RecA* rec = a.recA + (epoch & 1) * a.world + a.rank;
    atomicMax(&rec->key, k);
    if (n_end) atomicAdd(&rec->alive, (unsigned)n_end);
    if (any_bad) atomicOr(&rec->flags, 1u);
    if (n_start) atomicAdd(&a.ctrl->alive_steps, (unsigned long long)n_start);
    if (o) atomicAdd(&a.ctrl->overflow, o);
    if (dr) atomicAdd(&a.ctrl->draws, dr);
  }
  if (dg.guard) atomicAdd(&a.ctrl->guard_kills, dg.guard);   // rare (ClaDS2 only)
}

// Deferred gather, state dumps only (smc_state / smc_fields): materialise the
// resampled states dst[i] = src[anc[i]] (every plane) into the buffer the next
// propagation will overwrite anyway.
__global__ void gather_view_kernel(const uint4* src, uint4* dst, const uint32_t* anc,
                                   unsigned long long n, int planes, unsigned long long base) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long a = (unsigned long long)anc[i] - base;
    for (int p = 0; p < planes; ++p) dst[(unsigned long long)p * n + i] = src[(unsigned long long)p * n + a];
  }
}

// anc[i] = base + i (identity before the first resample)
__global__ void iota_kernel(uint32_t* anc, unsigned long long n, unsigned long long base) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    anc[i] = (uint32_t)(base + i);
}

// ============================================================================
// resampling: shared argument block
// ============================================================================
struct ResArgs {
  const double* lw;
  unsigned long long n_local;         // particles in this shard (= plane stride)
  unsigned long long shard_base;
  unsigned long long n_total;
  int world, rank;
  RecA* recA;                         // [2][world]
  RecB* recB;                         // [2][world] shard totals (W, sum q^2)
  U192* tile_q2;                      // [n_chunks] chunk sums of q^2 (ESS only)
  u128* tile_sum;                     // [n_chunks] chunk sums, then their exclusive prefix
  u128* tile_excl;                    // [n_tiles] exclusive prefix of tile t within its chunk
  int n_tiles;
  int chunk_tiles;                    // tiles per reduce chunk (one warp each)
  int n_chunks;
  const uint4* src_planes;
  int planes;
  uint4* const* dst_planes;           // [world] destination buffers (peer pointers)
  uint32_t* const* dst_anc;           // [world]
  Ctrl* ctrl;
  // in-place resampling (R-21; single shard)
  uint32_t* offs;                     // [n] O_k: output boundary after particle k
  uint32_t* tile_nz;                  // [n_tiles] particles with offspring per tile
  uint32_t* tile_nz_excl;             // [n_tiles] exclusive prefix of tile_nz
  uint32_t* hole_dst;                 // [n] slot of the h-th particle without offspring
  uint32_t* extra_src;                // [n] source of the h-th extra copy
  // stack-prefix copy (R-22): planes [stk0, stk0 + stk_n) hold a stack of
  // stk_per entries per plane whose pointer is word sp_word of the particle's
  // planes; only the first ceil(sp / stk_per) stack planes are copied
  int stk0, stk_n, stk_per, sp_word;
  int lazy;                           // deferred gather: ancestors only, no state copies (§7.7)
};

// First stack plane of particle `src` that need not be copied (planes
// [skip_lo, stk0 + stk_n) are beyond the stack pointer); a.stk_n == 0: none.
__device__ __forceinline__ int stack_skip_lo(const ResArgs& a, const uint4* planes, unsigned long long src) {
  if (a.stk_n == 0) return 1 << 30;
  const uint4 w = __ldg(planes + (unsigned long long)(a.sp_word >> 2) * a.n_local + src);
  const int c = a.sp_word & 3;
  const unsigned sp = c == 0 ? w.x : c == 1 ? w.y : c == 2 ? w.z : w.w;
  const int need = (int)min((unsigned)a.stk_n, (sp + (unsigned)a.stk_per - 1u) / (unsigned)a.stk_per);
  return a.stk0 + need;
}
__device__ __forceinline__ bool copy_plane(const ResArgs& a, int p, int skip_lo) {
  return p < skip_lo || p >= a.stk0 + a.stk_n;
}
// planes a slot copies (stack models: the planes below the stack pointer)
__device__ __forceinline__ unsigned planes_copied(const ResArgs& a, int skip_lo) {
  const int hi = a.stk0 + a.stk_n;
  return (unsigned)(a.planes - (hi - min(max(skip_lo, a.stk0), hi)));
}
// next plane to copy after p (run-time plane loops skip the planes beyond the
// stack pointer in one step)
__device__ __forceinline__ int next_plane(const ResArgs& a, int p, int skip_lo) {
  return p + 1 == skip_lo ? max(p + 1, a.stk0 + a.stk_n) : p + 1;
}

struct Global {
  double m;
  unsigned alive;
  unsigned flags;
  bool ok;          // finite max and no NaN: resampling quantities are defined
};
__device__ __forceinline__ Global read_global(const RecA* A, int world) {
  long long k = LLONG_MIN;
  unsigned alive = 0, flags = 0;
  for (int g = 0; g < world; ++g) {
    k = A[g].key > k ? A[g].key : k;
    alive += A[g].alive;
    flags |= A[g].flags;
  }
  Global G;
  G.m = key_to_double(k);
  G.alive = alive;
  G.flags = flags;
  G.ok = !flags && G.m != -INFINITY && k != LLONG_MIN;
  return G;
}

// ============================================================================
// reduce: one warp per chunk of chunk_tiles consecutive tiles.  The warp walks
// its tiles in order: 8 coalesced 16-byte loads per lane in flight, quantise,
// warp-sum in u128, record the tile's exclusive prefix within the chunk and
// advance the running chunk sum — no CTA barriers.  The last CTA (ticket)
// scans the n_chunks chunk sums (exclusive prefix written back in place) and
// publishes the shard total W (and sum q^2 for the ESS gate).  A tile's
// exclusive prefix = tile_sum[t / chunk_tiles] + tile_excl[t].
// ============================================================================
__device__ __forceinline__ u128 tile_prefix(const ResArgs& a, int t) {
  return ld_cg_u128(a.tile_sum + t / a.chunk_tiles) + ld_cg_u128(a.tile_excl + t);
}

template <int ITEMS>
__global__ void __launch_bounds__(kThreads, 3) reduce_kernel(ResArgs a) {
  constexpr int kTile = kThreads * ITEMS;              // particles per tile
  constexpr int kB = 4;                                // double2 loads per lane per batch (+ the next batch prefetched)
  constexpr int kPerBatch = 32 * 2 * kB;               // 512 particles per warp batch
  static_assert(kTile % kPerBatch == 0, "tile = whole batches");
  __shared__ U192 s_q2[kThreads / 32];
  __shared__ unsigned s_ticket;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = blockIdx.x * (kThreads / 32) + warp;
  const int t_lo = chunk * a.chunk_tiles;
  const int t_hi = min(a.n_tiles, t_lo + a.chunk_tiles);
  const double2* lw2 = reinterpret_cast<const double2*>(a.lw);
  auto load_batch = [&](unsigned long long p0, double2 (&x)[kB]) {
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const unsigned long long p = p0 + (unsigned long long)(b * 32 + lane) * 2;
      if (p + 1 < a.n_local) x[b] = __ldg(lw2 + p / 2);
      else {
        x[b].x = p < a.n_local ? __ldg(a.lw + p) : -INFINITY;
        x[b].y = -INFINITY;
      }
    }
  };
  double2 x[kB];
  if (t_lo < t_hi) load_batch((unsigned long long)t_lo * kTile, x);   // before the control reads
  if (*(volatile unsigned*)&a.ctrl->done) return;
  const unsigned par = a.ctrl->epoch & 1;
  const bool ess = a.ctrl->ess_a < a.ctrl->ess_b;      // uniform
  const Global G = read_global(a.recA + par * a.world, a.world);
  if (!G.ok) return;
  u128 run = 0;                                        // chunk sum (warp-uniform)
  U192 q2 = {{0, 0, 0}};                               // lane's sum of q^2
  for (int t = t_lo; t < t_hi; ++t) {
    u128 ts = 0;
    const unsigned long long p0 = (unsigned long long)t * kTile;
    for (int bb = 0; bb < kTile / kPerBatch; ++bb) {
      double2 y[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) y[b] = x[b];
      // prefetch the next batch (next tile's first at the end of this tile)
      const bool last = bb == kTile / kPerBatch - 1;
      if (!last) load_batch(p0 + (unsigned long long)(bb + 1) * kPerBatch, x);
      else if (t + 1 < t_hi) load_batch(p0 + kTile, x);
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const unsigned long long q0 = quantize(y[b].x, G.m), q1 = quantize(y[b].y, G.m);
        ts += (u128)q0 + q1;
        if (ess) add_u192_u128(q2, (u128)q0 * q0 + (u128)q1 * q1);   // q <= 2^62: < 2^125
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) ts += shfl_xor_u128(ts, d);
    if (lane == 0) a.tile_excl[t] = run;
    run += ts;
  }
  if (lane == 0 && chunk < a.n_chunks) a.tile_sum[chunk] = run;
  if (ess) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) add_u192(q2, shfl_xor_u192(q2, d));
    if (lane == 0 && chunk < a.n_chunks) a.tile_q2[chunk] = q2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_ticket = atomicAdd(&a.ctrl->counter, 1u);
  }
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  // ---- last CTA: exclusive scan of the chunk sums (in place), shard total -> recB
  __threadfence();
  const int nc = a.n_chunks;
  const int per = (nc + kThreads - 1) / kThreads;
  const int lo = threadIdx.x * per;
  const int hi = min(nc, lo + per);
  u128 local = 0;
#pragma unroll 4
  for (int c = lo; c < hi; ++c) local += ld_cg_u128(a.tile_sum + c);
  u128 incl = local;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u128 o = shfl_up_u128(incl, d);
    if (lane >= d) incl += o;
  }
  __shared__ u128 s_w[kThreads / 32];
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  u128 woff = 0;
  for (int w = 0; w < warp; ++w) woff += s_w[w];
  u128 rr = woff + incl - local;
  u128 sums[4];
  for (int c0 = lo; c0 < hi; c0 += 4) {                // batched reloads, then in-place prefixes
#pragma unroll
    for (int u = 0; u < 4; ++u) sums[u] = c0 + u < hi ? ld_cg_u128(a.tile_sum + c0 + u) : (u128)0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + u < hi) { a.tile_sum[c0 + u] = rr; rr += sums[u]; }
  }
  if (threadIdx.x == kThreads - 1) {
    a.recB[par * a.world + a.rank].W = rr;             // shard total
    a.ctrl->counter = 0;
  }
  if (ess) {                                           // uniform: whole CTA
    U192 q = {{0, 0, 0}};
    for (int c = lo; c < hi; ++c) {
      U192 v;
      const unsigned long long* src = (const unsigned long long*)(a.tile_q2 + c);
      v.w[0] = __ldcg(src); v.w[1] = __ldcg(src + 1); v.w[2] = __ldcg(src + 2);
      add_u192(q, v);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) add_u192(q, shfl_xor_u192(q, d));
    if (lane == 0) s_q2[warp] = q;
    __syncthreads();
    if (threadIdx.x == 0) {
      U192 t = s_q2[0];
      for (int w = 1; w < kThreads / 32; ++w) add_u192(t, s_q2[w]);
      RecB* rb = a.recB + par * a.world + a.rank;
      rb->q2[0] = t.w[0]; rb->q2[1] = t.w[1]; rb->q2[2] = t.w[2];
    }
  }
}

// ============================================================================
// anc_gather: ancestors of the tile's output slots + fused state gather
// ============================================================================
__device__ __forceinline__ U192 total_q2(const RecB* B, int world) {
  U192 q = {{0, 0, 0}};
  for (int g = 0; g < world; ++g) {
    U192 v;
    v.w[0] = B[g].q2[0]; v.w[1] = B[g].q2[1]; v.w[2] = B[g].q2[2];
    add_u192(q, v);
  }
  return q;
}
__device__ __forceinline__ Grid make_grid(const ResArgs& a, const RecB* B, unsigned epoch,
                                          u128& prefix) {
  u128 W = 0;
  prefix = 0;
  for (int g = 0; g < a.world; ++g) {
    if (g < a.rank) prefix += B[g].W;
    W += B[g].W;
  }
  const unsigned long long seed = a.ctrl->seed;
  const uint4 r = philox4x32_10(make_uint4(0u, epoch, 0u, 1u), (uint32_t)seed, (uint32_t)(seed >> 32));
  const unsigned long long z = hq_bits(r.x, r.y);
  Grid gr;
  gr.W = W;
  gr.N = a.n_total;
  gr.Nsc = (u128)a.n_total << 54;
  gr.z2p1 = 2ull * z + 1ull;
  gr.Wd = u128_approx(W);
  gr.Nd = (double)a.n_total;
  gr.ud = (double)gr.z2p1 * 0x1p-54;
  gr.NdWd = gr.Nd / gr.Wd;
  return gr;
}
__device__ __forceinline__ Grid make_grid_w(u128 W, unsigned long long n_total, unsigned long long z) {
  Grid gr;
  gr.W = W;
  gr.N = n_total;
  gr.Nsc = (u128)n_total << 54;
  gr.z2p1 = 2ull * z + 1ull;
  gr.Wd = u128_approx(W);
  gr.Nd = (double)n_total;
  gr.ud = (double)gr.z2p1 * 0x1p-54;
  gr.NdWd = gr.Nd / gr.Wd;
  return gr;
}

template <int P, int ITEMS>   // P = planes per particle (<= 0: runtime a.planes)
__global__ void __launch_bounds__(kThreads, 4) anc_gather_kernel(ResArgs a) {
  constexpr int kTile = kThreads * ITEMS;
  constexpr int kItems = ITEMS;
  __shared__ double s_lw[kTile];
  __shared__ unsigned s_O[kTile];
  __shared__ u128 s_w[kThreads / 32];
  __shared__ unsigned long long s_jlo;
  const unsigned long long base = (unsigned long long)blockIdx.x * kTile;
  const int cnt = (int)min((unsigned long long)kTile, a.n_local - base);
  double lwv[kItems];                      // striped (coalesced) loads, before the control reads
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int k = r * kThreads + threadIdx.x;
    lwv[r] = k < cnt ? __ldg(a.lw + base + k) : -INFINITY;
  }
  if (*(volatile unsigned*)&a.ctrl->done) return;
  const unsigned epoch = a.ctrl->epoch;
  const unsigned par = epoch & 1;
  const Global G = read_global(a.recA + par * a.world, a.world);
  if (!G.ok || G.alive == 0) return;       // error, or final epoch: no resample
  u128 prefix;
  const Grid gr = make_grid(a, a.recB + par * a.world, epoch, prefix);
  if (!ess_resample(gr.W, total_q2(a.recB + par * a.world, a.world), a.n_total, a.ctrl->ess_a,
                    a.ctrl->ess_b)) {
    // ESS high enough: no resample (R-19); keep the states (copy to the other
    // buffer so the epoch's buffer parity holds), ancestors unchanged
    uint4* dst = a.dst_planes[a.rank];
    const int np = P > 0 ? P : a.planes;
    for (int k = threadIdx.x; k < (a.lazy ? 0 : cnt); k += kThreads) {   // deferred gather: none
      const int lo = stack_skip_lo(a, a.src_planes, base + k);
      for (int p = 0; p < np; p = next_plane(a, p, lo))
        if (copy_plane(a, p, lo))
          dst[(unsigned long long)p * a.n_local + base + k] =
              __ldg(a.src_planes + (unsigned long long)p * a.n_local + base + k);
    }
    return;
  }
  // striped load, blocked use
#pragma unroll
  for (int r = 0; r < kItems; ++r) s_lw[r * kThreads + threadIdx.x] = lwv[r];
  __syncthreads();
  unsigned long long q[kItems];
  u128 tsum = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    q[r] = quantize(s_lw[threadIdx.x * kItems + r], G.m);
    tsum += q[r];
  }
  // CTA exclusive scan of per-thread sums
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u128 incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u128 o = shfl_up_u128(incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  u128 woff = 0;
  for (int w = 0; w < warp; ++w) woff += s_w[w];
  const u128 tile_start = prefix + tile_prefix(a, blockIdx.x);
  u128 C = tile_start + woff + incl - tsum;   // exclusive prefix of this thread's first item
  if (threadIdx.x == 0) s_jlo = gr.count_below(tile_start);
  unsigned long long prevO = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    C += q[r];
    // zero weight: C_k = C_{k-1}, hence O_k = O_{k-1} (no offspring)
    const unsigned long long O = (q[r] == 0 && r > 0) ? prevO : gr.count_below(C);
    s_O[threadIdx.x * kItems + r] = (unsigned)O;
    prevO = O;
  }
  __syncthreads();
  const unsigned long long jlo = s_jlo;
  unsigned distinct = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int k = threadIdx.x * kItems + r;
    if (k < cnt) distinct += s_O[k] > (k ? s_O[k - 1] : (unsigned)jlo);
  }
  // distinct-ancestor count (for the algorithmic-bytes figure)
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) distinct += __shfl_xor_sync(0xffffffffu, distinct, d);
  if (lane == 0 && distinct) atomicAdd(&a.ctrl->distinct, (unsigned long long)distinct);

  const unsigned long long jhi = cnt > 0 ? s_O[cnt - 1] : jlo;
  // Output slots.  Warp w's particles [w*32*kItems, (w+1)*32*kItems) (its
  // lanes' blocked items) fill the contiguous slots [O_{first-1}, O_last): the
  // lanes take consecutive slots and binary-search the warp's O values.  If a
  // warp owns more than 8 slots per particle (a few dominant weights), the
  // whole CTA shares the tile's slots instead.
  const int wk0 = warp * 32 * kItems, wn = 32 * kItems;
  const unsigned wA = wk0 ? s_O[wk0 - 1] : (unsigned)jlo;
  const unsigned wB = s_O[wk0 + wn - 1];
#ifdef SMC_ANC_WARP
  const bool heavy = __syncthreads_or(wB - wA > 8u * (unsigned)wn);
#else
  const bool heavy = true;                  // measured: CTA-wide striping balances better
#endif
  const unsigned long long j_first = heavy ? jlo + threadIdx.x : wA + lane;
  const unsigned long long j_end = heavy ? jhi : wB;
  const unsigned j_step = heavy ? kThreads : 32;
  const int s_lo = heavy ? 0 : wk0, s_hi = heavy ? kTile - 1 : wk0 + wn - 1;
  unsigned long long stk_copied = 0;        // stack models: planes copied (bench bytes)
  for (unsigned long long j = j_first; j < j_end; j += j_step) {
    int lo = s_lo, hi = s_hi;               // first item with O_k > j
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_O[mid] > j) hi = mid; else lo = mid + 1;
    }
    const unsigned long long src = base + lo;
    unsigned long long dshard = 0, dl = j;
    if (a.world > 1) {
      dshard = j / a.n_local;
      dl = j - dshard * a.n_local;
    }
    uint4* dst = a.dst_planes[dshard];
    const int skip = stack_skip_lo(a, a.src_planes, src);     // R-22: stack prefix only
    if (a.stk_n) stk_copied += planes_copied(a, skip);
    if (a.lazy) {                                             // deferred gather: ancestors only
      a.dst_anc[dshard][dl] = (uint32_t)(a.shard_base + src);
      continue;
    }
    if (P > 0) {
      uint4 v[P > 0 ? P : 1];
#pragma unroll
      for (int p = 0; p < (P > 0 ? P : 1); ++p)
        if (copy_plane(a, p, skip)) v[p] = __ldg(a.src_planes + (unsigned long long)p * a.n_local + src);
#pragma unroll
      for (int p = 0; p < (P > 0 ? P : 1); ++p)
        if (copy_plane(a, p, skip)) dst[(unsigned long long)p * a.n_local + dl] = v[p];
    } else {
      for (int p = 0; p < a.planes; p = next_plane(a, p, skip))
        if (copy_plane(a, p, skip))
          dst[(unsigned long long)p * a.n_local + dl] = __ldg(a.src_planes + (unsigned long long)p * a.n_local + src);
    }
    a.dst_anc[dshard][dl] = (uint32_t)(a.shard_base + src);
  }
  if (a.stk_n) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) stk_copied += __shfl_xor_sync(0xffffffffu, stk_copied, d);
    if ((threadIdx.x & 31) == 0 && stk_copied) atomicAdd(&a.ctrl->stack_planes, stk_copied);
  }
  if (a.world > 1) __threadfence_system();   // peer stores visible before the epoch barrier
}

// ============================================================================
// in-place resampling (single shard).  From
// the sorted ancestors of the systematic grid: particles with offspring keep
// their slot; their extra copies fill the slots without offspring in order.
//   offspring_kernel  O_k per particle (stored), survivors per tile, last CTA:
//                     tile prefix of survivors and the hole count H
//   permute_kernel    anc[k] = k for survivors, hole list, extra-copy list
//   fill_holes_kernel for h < H: anc[hole_h] = extra_h, copy the state planes
//                     in place (holes are never sources)
// ============================================================================
__device__ __forceinline__ bool inplace_active(const ResArgs& a, unsigned epoch, Global& G) {
  const unsigned par = epoch & 1;
  G = read_global(a.recA + par * a.world, a.world);
  if (!G.ok || G.alive == 0) return false;           // error, or final epoch: no resample
  u128 W = 0;
  for (int g = 0; g < a.world; ++g) W += a.recB[par * a.world + g].W;
  return ess_resample(W, total_q2(a.recB + par * a.world, a.world), a.n_total, a.ctrl->ess_a,
                      a.ctrl->ess_b);                 // ESS skip: state stays where it is
}

template <int ITEMS>
__global__ void __launch_bounds__(kThreads) offspring_kernel(ResArgs a) {
  constexpr int kTile = kThreads * ITEMS;
  constexpr int kItems = ITEMS;
  __shared__ double s_lw[kTile];
  __shared__ unsigned s_O[kTile];
  __shared__ u128 s_w[kThreads / 32];
  __shared__ unsigned s_n[kThreads / 32];
  __shared__ unsigned long long s_jlo;
  __shared__ unsigned s_ticket;
  if (*(volatile unsigned*)&a.ctrl->done) return;
  const unsigned epoch = a.ctrl->epoch;
  Global G;
  if (!inplace_active(a, epoch, G)) return;
  u128 prefix;
  const Grid gr = make_grid(a, a.recB + (epoch & 1) * a.world, epoch, prefix);
  const unsigned long long base = (unsigned long long)blockIdx.x * kTile;
  const int cnt = (int)min((unsigned long long)kTile, a.n_local - base);
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int k = r * kThreads + threadIdx.x;
    s_lw[k] = k < cnt ? __ldg(a.lw + base + k) : -INFINITY;
  }
  __syncthreads();
  unsigned long long q[kItems];
  u128 tsum = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    q[r] = quantize(s_lw[threadIdx.x * kItems + r], G.m);
    tsum += q[r];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u128 incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u128 o = shfl_up_u128(incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  u128 woff = 0;
  for (int w = 0; w < warp; ++w) woff += s_w[w];
  const u128 tile_start = prefix + tile_prefix(a, blockIdx.x);
  u128 C = tile_start + woff + incl - tsum;
  if (threadIdx.x == 0) s_jlo = gr.count_below(tile_start);
  unsigned long long prevO = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    C += q[r];
    const unsigned long long O = (q[r] == 0 && r > 0) ? prevO : gr.count_below(C);
    s_O[threadIdx.x * kItems + r] = (unsigned)O;
    prevO = O;
  }
  __syncthreads();
  const unsigned jlo = (unsigned)s_jlo;
  unsigned nz = 0;
  for (int k = threadIdx.x; k < cnt; k += kThreads) {     // striped: coalesced store
    const unsigned O = s_O[k];
    a.offs[base + k] = O;
    nz += O > (k ? s_O[k - 1] : jlo);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, d);
  if (lane == 0) s_n[warp] = nz;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += s_n[w];
    a.tile_nz[blockIdx.x] = t;
    if (t) atomicAdd(&a.ctrl->distinct, (unsigned long long)t);
    __threadfence();
    s_ticket = atomicAdd(&a.ctrl->counter, 1u);
  }
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  // ---- last CTA: exclusive scan of the per-tile survivor counts
  __threadfence();
  const int nt = a.n_tiles;
  const int per = (nt + kThreads - 1) / kThreads;
  const int lo = threadIdx.x * per, hi = min(nt, lo + per);
  unsigned local = 0;
  for (int t = lo; t < hi; ++t) local += __ldcg(a.tile_nz + t);
  unsigned inc2 = local;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, inc2, d);
    if (lane >= d) inc2 += o;
  }
  __syncthreads();                                       // s_n reused
  if (lane == 31) s_n[warp] = inc2;
  __syncthreads();
  unsigned wo = 0;
  for (int w = 0; w < warp; ++w) wo += s_n[w];
  unsigned run = wo + inc2 - local;
  for (int t = lo; t < hi; ++t) {
    a.tile_nz_excl[t] = run;
    run += __ldcg(a.tile_nz + t);
  }
  if (threadIdx.x == kThreads - 1) {
    a.ctrl->holes = (unsigned)(a.n_local - run);        // run = survivors (distinct ancestors)
    a.ctrl->counter = 0;
  }
}

template <int ITEMS>
__global__ void __launch_bounds__(kThreads) permute_kernel(ResArgs a) {
  constexpr int kTile = kThreads * ITEMS;
  constexpr int kItems = ITEMS;
  __shared__ unsigned s_O[kTile];
  __shared__ unsigned s_E[kTile];
  __shared__ unsigned s_n[kThreads / 32];
  __shared__ unsigned s_prev;
  if (*(volatile unsigned*)&a.ctrl->done) return;
  Global G;
  if (!inplace_active(a, a.ctrl->epoch, G)) return;
  const unsigned long long base = (unsigned long long)blockIdx.x * kTile;
  const int cnt = (int)min((unsigned long long)kTile, a.n_local - base);
  for (int k = threadIdx.x; k < cnt; k += kThreads) s_O[k] = a.offs[base + k];
  if (threadIdx.x == 0) s_prev = base ? a.offs[base - 1] : 0u;    // O_{-1} = 0 (single shard)
  __syncthreads();
  // survivors before each item: blocked per thread, CTA scan, tile prefix
  const unsigned prev0 = s_prev;
  unsigned c = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int k = threadIdx.x * kItems + r;
    if (k < cnt) c += s_O[k] > (k ? s_O[k - 1] : prev0);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_n[warp] = incl;
  __syncthreads();
  unsigned wo = 0;
  for (int w = 0; w < warp; ++w) wo += s_n[w];
  const unsigned tile_d = a.tile_nz_excl[blockIdx.x];
  unsigned D = tile_d + wo + incl - c;                  // survivors before this thread's first item
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int k = threadIdx.x * kItems + r;
    if (k < cnt) {
      D += s_O[k] > (k ? s_O[k - 1] : prev0);
      s_E[k] = s_O[k] - D;                               // extra copies through particle k
    }
  }
  __syncthreads();
  uint32_t* anc = a.dst_anc[a.rank];
  for (int k = threadIdx.x; k < cnt; k += kThreads) {   // striped: coalesced anc stores
    const unsigned O = s_O[k];
    const unsigned gk = (unsigned)(a.shard_base + base + k);
    if (O > (k ? s_O[k - 1] : prev0)) anc[base + k] = gk;     // survivor keeps its slot
    else a.hole_dst[(base + k) - (O - s_E[k])] = gk;          // rank among the holes
  }
  // extra copies of this tile: ranks [E_{base-1}, E_{last}); rank e belongs to
  // the first item with s_E > e
  const unsigned elo = prev0 - tile_d, ehi = cnt > 0 ? s_E[cnt - 1] : elo;
  for (unsigned e = elo + threadIdx.x; e < ehi; e += kThreads) {
    int lo = 0, hi = cnt - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_E[mid] > e) hi = mid; else lo = mid + 1;
    }
    a.extra_src[e] = (unsigned)(a.shard_base + base + lo);
  }
}

template <int P>   // P = planes per particle (<= 0: runtime a.planes)
__global__ void __launch_bounds__(kThreads) fill_holes_kernel(ResArgs a) {
  if (*(volatile unsigned*)&a.ctrl->done) return;
  Global G;
  if (!inplace_active(a, a.ctrl->epoch, G)) return;
  const unsigned H = a.ctrl->holes;
  uint4* pl = const_cast<uint4*>(a.src_planes);          // the one state buffer
  uint32_t* anc = a.dst_anc[a.rank];
  const int np = P > 0 ? P : a.planes;
  for (unsigned long long h = (unsigned long long)blockIdx.x * kThreads + threadIdx.x; h < H;
       h += (unsigned long long)gridDim.x * kThreads) {
    const unsigned dst = a.hole_dst[h], src = a.extra_src[h];
    anc[dst] = src;
    const int lo = stack_skip_lo(a, pl, src);               // R-22: stack prefix only
    if (P > 0) {
      uint4 v[P > 0 ? P : 1];
#pragma unroll
      for (int p = 0; p < (P > 0 ? P : 1); ++p)
        if (copy_plane(a, p, lo)) v[p] = __ldg(pl + (unsigned long long)p * a.n_local + src);
#pragma unroll
      for (int p = 0; p < (P > 0 ? P : 1); ++p)
        if (copy_plane(a, p, lo)) pl[(unsigned long long)p * a.n_local + dst] = v[p];
    } else {
      for (int p = 0; p < np; p = next_plane(a, p, lo))
        if (copy_plane(a, p, lo))
          pl[(unsigned long long)p * a.n_local + dst] = __ldg(pl + (unsigned long long)p * a.n_local + src);
    }
  }
}

// ============================================================================
// finalize: log Z, termination, epoch advance (one thread)
// ============================================================================
struct FinArgs {
  RecA* recA;
  RecB* recB;
  int world, rank;
  unsigned long long n_total;
  int strict;
  Ctrl* ctrl;
};
__device__ __noinline__ void finalize_body(const FinArgs& a) {
  Ctrl* c = a.ctrl;
  if (c->done) return;
  const unsigned epoch = c->epoch;
  const unsigned par = epoch & 1;
  const Global G = read_global(a.recA + par * a.world, a.world);
  if (G.flags) {
    c->status = (G.flags & 1u) ? ST_NAN : ST_OVERFLOW;   // bit 1: side-tree task stack full
    c->done = 1;
    c->epochs = c->epochs + 1;
  } else if (!(G.m > -INFINITY)) {
    c->status = ST_REJECTED;
    c->logz = -INFINITY;
    c->done = 1;
    c->epochs = c->epochs + 1;
  } else {
    u128 W = 0;
    for (int g = 0; g < a.world; ++g) W += a.recB[par * a.world + g].W;
    const double lwd = log(u128_trunc_double(W));
    const double inc = G.m + ((lwd - 62.0 * kLn2) - log((double)a.n_total));
    c->last_inc = inc;
    c->epochs = c->epochs + 1;
    if (a.strict && c->overflow) {
      c->logz = c->logz + inc;
      c->status = ST_OVERFLOW;
      c->done = 1;
    } else if (G.alive == 0) {
      c->logz = c->logz + inc;                         // final: no resample (R-6)
      c->done = 1;
      c->gmap_id = 1;
    } else if (ess_resample(W, total_q2(a.recB + par * a.world, a.world), a.n_total, c->ess_a,
                            c->ess_b)) {
      c->logz = c->logz + inc;
      c->resamples = c->resamples + 1;
      c->carry = 0;
      c->epoch = epoch + 1;
      c->gmap_id = 0;                                  // next epoch reads through the ancestors
    } else {
      c->carry = 1;                                    // weights accumulate (R-19)
      c->epoch = epoch + 1;
      c->gmap_id = 1;                                  // states stay where they are
    }
  }
  c->batch = 0;
  // reset this shard's records of the other parity for the next epoch
  RecA* nx = a.recA + (par ^ 1) * a.world + a.rank;
  nx->key = LLONG_MIN;
  nx->alive = 0;
  nx->flags = 0;
  RecB* nb = a.recB + (par ^ 1) * a.world + a.rank;
  nb->W = 0;
  nb->q2[0] = nb->q2[1] = nb->q2[2] = 0;
}
__global__ void finalize_kernel(FinArgs a) {
  if (threadIdx.x == 0) finalize_body(a);
}

// ============================================================================
// whole-run CUDA graph: the WHILE node's condition = "not done"
// ============================================================================
__global__ void set_condition_kernel(cudaGraphConditionalHandle hdl, const Ctrl* c,
                                     unsigned max_epochs) {
  if (threadIdx.x == 0) {
    const bool more = !c->done && c->epoch < max_epochs;
    cudaGraphSetConditional(hdl, more ? 1u : 0u);
  }
}

// ============================================================================
// resampler-only helpers (BASELINE configs[4])
// ============================================================================
// Set the epoch and clear the records of a standalone resampling step.
__global__ void prep_resample_kernel(Ctrl* c, RecA* recA, RecB* recB, int world, int rank,
                                     unsigned epoch) {
  if (threadIdx.x != 0) return;
  c->epoch = epoch;
  c->done = 0;
  c->status = 0;
  c->distinct = 0;
  RecA* r = recA + (epoch & 1) * world + rank;
  r->key = LLONG_MIN;
  r->alive = 1;          // a standalone step always resamples
  r->flags = 0;
  RecB* b = recB + (epoch & 1) * world + rank;
  b->W = 0;
  b->q2[0] = b->q2[1] = b->q2[2] = 0;
  c->ess_a = 1;              // a standalone step always resamples
  c->ess_b = 1;
}
// Max of lw (the propagation epilogue's job in a full SMC run).
__global__ void __launch_bounds__(kThreads) max_kernel(const double* lw, unsigned long long n,
                                                       RecA* recA, int world, int rank, Ctrl* c) {
  __shared__ long long s_key[kThreads / 32];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const unsigned par = c->epoch & 1;
  long long key = LLONG_MIN;
  bool bad = false;
  const unsigned long long n2 = n / 2;
  const double2* p = reinterpret_cast<const double2*>(lw);
  const unsigned long long stride = (unsigned long long)gridDim.x * kThreads;
  unsigned long long i = (unsigned long long)blockIdx.x * kThreads + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {       // 4 x 16-byte loads in flight
    double2 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = __ldg(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bad |= isnan(t[u].x) || t[u].x == INFINITY || isnan(t[u].y) || t[u].y == INFINITY;
      const long long k0 = order_key(t[u].x), k1 = order_key(t[u].y);
      key = max(key, max(k0, k1));
    }
  }
  for (; i < n2; i += stride) {
    const double2 t = __ldg(p + i);
    bad |= isnan(t.x) || t.x == INFINITY || isnan(t.y) || t.y == INFINITY;
    key = max(key, max(order_key(t.x), order_key(t.y)));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
    const double t = __ldg(lw + n - 1);
    bad |= isnan(t) || t == INFINITY;
    key = max(key, order_key(t));
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, key, d);
    key = o > key ? o : key;
  }
  if ((threadIdx.x & 31) == 0) s_key[threadIdx.x >> 5] = key;
  if (bad) s_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long k = s_key[0];
    for (int w = 1; w < kThreads / 32; ++w) k = s_key[w] > k ? s_key[w] : k;
    RecA* r = recA + par * world + rank;
    atomicMax(&r->key, k);
    if (s_bad) atomicOr(&r->flags, 1u);
  }
}


// ============================================================================
// resample_fused: the whole resampling step of a single-shard run in ONE
// cooperative launch (rows a6-a10 + finalize), for shards whose particles fit
// the grid's shared memory (12 B each: 10^6 particles = 12 MB over 148 SMs).  Phase 1: each CTA
// loads its contiguous block of log-weights once, quantises them in shared
// memory (the same q = quantize(lw, m) as reduce) and publishes its u128 block
// sum (and sum q^2 for the ESS gate); grid barrier; phase 2: every CTA derives
// the identical exact total W and its block's exclusive prefix from the block
// sums, CTA 0 folds the epoch into log Z (finalize_body), and each CTA maps its
// particles to offspring boundaries O_k = F(C_k) and gathers the output slots
// they own — the second weight pass reads shared memory, not HBM, and one
// launch replaces reduce + anc_gather + finalize.  Results are identical to
// the split path (same integers, same grid, same slot ownership).
// ============================================================================
#ifndef SMC_FUSED_THREADS
#define SMC_FUSED_THREADS 512
#endif
#ifndef SMC_FUSED_GALLOP
#define SMC_FUSED_GALLOP 0
#endif
#ifndef SMC_FUSED_SCAN
#define SMC_FUSED_SCAN 0      // warp-local mark + max-scan slot map: measured no faster (CRBD resampling 7.25 -> 7.35 ms/sweep), off
#endif
constexpr int kFT = SMC_FUSED_THREADS;   // threads per fused CTA
#ifndef SMC_FUSED_MINB
#define SMC_FUSED_MINB 2                 // resident CTAs per SM (register cap 64)
#endif
constexpr int kMaxFusedGrid = 1024;

struct FusedArgs {
  u128* blk_sum;                         // [grid]
  U192* blk_q2;                          // [grid]
  int ipt;                               // particles per thread (block = kFT * ipt)
  FinArgs fin;
};

__device__ __forceinline__ void grid_barrier(Ctrl* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = &c->bar_gen;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(&c->bar_count, 1u) == gridDim.x - 1) {
      c->bar_count = 0;
      __threadfence();
      atomicExch(&c->bar_gen, g + 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// One output slot: copy particle `src`'s planes (stack prefix only, R-22).
template <int P>
__device__ __forceinline__ void copy_particle(const ResArgs& a, uint4* dst, unsigned long long src,
                                              unsigned long long slot, int skip) {
  if (P > 0) {
    uint4 v[P > 0 ? P : 1];
#pragma unroll
    for (int p = 0; p < (P > 0 ? P : 1); ++p)
      if (copy_plane(a, p, skip)) v[p] = __ldg(a.src_planes + (unsigned long long)p * a.n_local + src);
#pragma unroll
    for (int p = 0; p < (P > 0 ? P : 1); ++p)
      if (copy_plane(a, p, skip)) dst[(unsigned long long)p * a.n_local + slot] = v[p];
  } else {
    for (int p = 0; p < a.planes; p = next_plane(a, p, skip))
      if (copy_plane(a, p, skip))
        dst[(unsigned long long)p * a.n_local + slot] = __ldg(a.src_planes + (unsigned long long)p * a.n_local + src);
  }
}

// Layout: CTA b owns particles [b*kFT*ipt, (b+1)*kFT*ipt); round r of a CTA
// covers its particles r*kFT + t (t = thread), so every round is a contiguous
// run of kFT particles, scanned across the CTA, and a thread writes the
// offspring slots [O_{k-1}, O_k) of its own particle k (consecutive threads,
// consecutive slots: coalesced; no search).
template <int P>   // planes per particle (<= 0: runtime a.planes)
__global__ void __launch_bounds__(kFT, SMC_FUSED_MINB) resample_fused_kernel(ResArgs a, FusedArgs f) {
  extern __shared__ unsigned long long s_q[];          // [kFT * ipt] quantised weights
  __shared__ u128 s_w[2][kFT / 32];
  __shared__ u128 s_w2[kFT / 32];
  __shared__ U192 s_q2[kFT / 32];
  Ctrl* c = a.ctrl;
  const int ipt = f.ipt;
  const int blk = kFT * ipt;
  const unsigned long long base = (unsigned long long)blockIdx.x * blk;
  const int cnt = base < a.n_local ? (int)min((unsigned long long)blk, a.n_local - base) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- phase 1: striped (coalesced) load into shared memory, issued before
  // the control reads it does not depend on; each thread then quantises its
  // blocked items k = t*ipt + r in place and sums them; one CTA scan gives
  // every thread the exclusive prefix of its items and the block sum
  for (int r0 = 0; r0 < ipt; r0 += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = (r0 + u) * kFT + threadIdx.x;
      v[u] = (r0 + u < ipt && k < cnt) ? __ldg(a.lw + base + k) : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r0 + u < ipt) s_q[(r0 + u) * kFT + threadIdx.x] = (unsigned long long)__double_as_longlong(v[u]);
  }
  if (*(volatile unsigned*)&c->done) return;          // read by every CTA before the barrier
  const unsigned epoch = c->epoch;
  const unsigned par = epoch & 1;
  const bool ess = c->ess_a < c->ess_b;
  const Global G = read_global(a.recA + par * a.world, a.world);
  // the last CTA (fewest particles: the ragged tail) folds the epoch into log Z
  const bool fin_cta = blockIdx.x == gridDim.x - 1;
  if (!G.ok) {                                          // error / all rejected: finalize only
    if (fin_cta && threadIdx.x == 0) finalize_body(f.fin);
    return;
  }
  __syncthreads();
  u128 tsum = 0, tq2 = 0;
  for (int r = 0; r < ipt; ++r) {
    const int k = threadIdx.x * ipt + r;
    const unsigned long long q = quantize(__longlong_as_double((long long)s_q[k]), G.m);
    s_q[k] = q;
    tsum += q;
    if (ess) tq2 += (u128)q * q;
  }
  u128 incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u128 o = shfl_up_u128(incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_w[0][warp] = incl;
  if (ess) {
    U192 q2;
    q2.w[0] = (unsigned long long)tq2; q2.w[1] = (unsigned long long)(tq2 >> 64); q2.w[2] = 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) add_u192(q2, shfl_xor_u192(q2, d));
    if (lane == 0) s_q2[warp] = q2;
  }
  __syncthreads();
  // warp totals -> their inclusive scan across the 16 warps, in every warp's
  // lanes 0..15 (4 shuffle steps instead of 16 shared loads per thread)
  u128 ws = lane < kFT / 32 ? s_w[0][lane] : (u128)0;
#pragma unroll
  for (int d = 1; d < kFT / 32; d <<= 1) {
    const u128 o = shfl_up_u128(ws, d);
    if (lane >= d) ws += o;
  }
  const u128 woff = warp ? shfl_idx_u128(ws, warp - 1) : (u128)0;
  const u128 bsum = shfl_idx_u128(ws, kFT / 32 - 1);
  const u128 texcl = woff + incl - tsum;                // exclusive prefix of this thread's items
  if (threadIdx.x == 0) {
    f.blk_sum[blockIdx.x] = bsum;
    if (ess) {
      U192 q = s_q2[0];
      for (int w = 1; w < kFT / 32; ++w) add_u192(q, s_q2[w]);
      f.blk_q2[blockIdx.x] = q;
    }
  }
  grid_barrier(c);
  // ---- phase 2: exact totals (identical in every CTA), finalize, ancestors + gather
  u128 tot = 0, pre = 0;
  U192 q2t = {{0, 0, 0}};
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kFT) {
    const u128 v = ld_cg_u128(f.blk_sum + b);
    tot += v;
    if (b < (int)blockIdx.x) pre += v;
    if (ess) {
      const unsigned long long* src = (const unsigned long long*)(f.blk_q2 + b);
      U192 t;
      t.w[0] = __ldcg(src); t.w[1] = __ldcg(src + 1); t.w[2] = __ldcg(src + 2);
      add_u192(q2t, t);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    tot += shfl_xor_u128(tot, d);
    pre += shfl_xor_u128(pre, d);
    if (ess) add_u192(q2t, shfl_xor_u192(q2t, d));
  }
  if (lane == 0) { s_w[1][warp] = tot; s_w2[warp] = pre; if (ess) s_q2[warp] = q2t; }
  __syncthreads();
  tot = lane < kFT / 32 ? s_w[1][lane] : (u128)0;
  pre = lane < kFT / 32 ? s_w2[lane] : (u128)0;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    tot += shfl_xor_u128(tot, d);
    pre += shfl_xor_u128(pre, d);
  }
  if (ess) {
    q2t = {{0, 0, 0}};
    for (int w = 0; w < kFT / 32; ++w) add_u192(q2t, s_q2[w]);
  }
  if (fin_cta && threadIdx.x == 0) {
    RecB* rb = a.recB + par * a.world + a.rank;
    rb->W = tot;
    rb->q2[0] = q2t.w[0]; rb->q2[1] = q2t.w[1]; rb->q2[2] = q2t.w[2];
    finalize_body(f.fin);                               // log Z, termination, epoch advance
  }
  if (G.alive == 0) return;                             // final epoch: no resample
  uint4* dst = a.dst_planes[a.rank];
  if (!ess_resample(tot, q2t, a.n_total, c->ess_a, c->ess_b)) {
    if (!a.lazy)                                        // (deferred gather: states stay put)
      for (int k = threadIdx.x; k < cnt; k += kFT)      // ESS high: identity copy (R-19)
        copy_particle<P>(a, dst, base + k, base + k, stack_skip_lo(a, a.src_planes, base + k));
    return;
  }
  const unsigned long long seed = c->seed;
  const uint4 rr = philox4x32_10(make_uint4(0u, epoch, 0u, 1u), (uint32_t)seed, (uint32_t)(seed >> 32));
  const Grid gr = make_grid_w(tot, a.n_total, hq_bits(rr.x, rr.y));
  uint32_t* anc = a.dst_anc[a.rank];
  unsigned* s_O = reinterpret_cast<unsigned*>(s_q + blk);   // [blk] offspring boundaries O_k
  // 2a: O_k = F(C_k) for the thread's blocked items (shared memory only)
  u128 C = pre + texcl;
  unsigned distinct = 0;                                // particles with offspring
  unsigned prevO = (unsigned)gr.count_below(C);
  for (int r = 0; r < ipt; ++r) {
    const int k = threadIdx.x * ipt + r;
    C += s_q[k];
    const unsigned O = (unsigned)gr.count_below(C);     // zero weight: O_k = O_{k-1}
    s_O[k] = O;
    distinct += O > prevO;
    prevO = O;
  }
  if (threadIdx.x == 0) s_O[blk] = (unsigned)gr.count_below(pre);   // O before the block
  __syncthreads();
#ifdef SMC_DIAG_FUSED_NO_GATHER
  return;   // diagnostics only (timing of phases 1-2a; results invalid)
#endif
  // 2b: output slots.  Warp w's particles [w*32*ipt, (w+1)*32*ipt) (the
  // blocked items of its lanes) fill the contiguous slots [O_{first-1},
  // O_last); the lanes take consecutive slots and find their source by a
  // binary search over the warp's O values (coalesced stores, no barriers).
  // If one warp owns more than kHeavy slots per particle on average (a few
  // dominant weights), the whole CTA instead shares the block's slots, so a
  // single heavy particle is copied by kFT threads, not 32.
  constexpr unsigned kHeavy = 8;
  unsigned long long stk_copied = 0;                    // stack models: planes copied (bench bytes)
  __shared__ unsigned s_heavy;
  if (threadIdx.x == 0) s_heavy = 0;
  __syncthreads();
  const int wk0 = warp * 32 * ipt, wn = 32 * ipt;       // the warp's particles
  const unsigned wA = wk0 ? s_O[wk0 - 1] : s_O[blk];
  const unsigned wB = s_O[wk0 + wn - 1];
#ifdef SMC_FUSED_CTA_STRIPE
  if (threadIdx.x == 0) s_heavy = 1u;
#else
  if (lane == 0 && wB - wA > kHeavy * (unsigned)wn) atomicOr(&s_heavy, 1u);
#endif
  __syncthreads();
  if (!s_heavy) {
    // U chunks of 32 slots per iteration: U independent searches, then all
    // loads, then all stores (U*P 16-byte loads in flight per lane)
#ifndef SMC_FUSED_U2
#define SMC_FUSED_U2 2
#endif
    constexpr int U = P == 1 ? 4 : P == 2 ? SMC_FUSED_U2 : 1;
#if SMC_FUSED_GALLOP
    const unsigned wspan = wB - wA;
#endif
#if SMC_FUSED_SCAN
    // Slot -> source map without searches when the warp's slots fit the
    // shared memory its particles' quantised weights occupied (dead after 2a:
    // 8 B per particle = 2 slots): each particle with offspring marks the
    // first slot of its run, an inclusive max-scan over the warp's slots
    // carries the mark to every slot of the run (no barrier: warp-local).
    const unsigned span = wB - wA;
    const bool use_map = span <= 2u * (unsigned)wn;
    // (volatile: 32-bit accesses only — the region held 64-bit weights, and
    // ptxas must not pair neighbouring entries into 64-bit loads)
    volatile unsigned* buf = reinterpret_cast<volatile unsigned*>(s_q + wk0);
    if (use_map) {
      for (unsigned i = lane; i < span; i += 32) buf[i] = 0u;
      __syncwarp();
      const int k0 = wk0 + lane * ipt;
      unsigned Op = k0 ? s_O[k0 - 1] : s_O[blk];
      for (int r = 0; r < ipt; ++r) {
        const unsigned Ok = s_O[k0 + r];
        if (Ok > Op) buf[Op - wA] = (unsigned)(k0 + r - wk0) + 1u;
        Op = Ok;
      }
      __syncwarp();
      const unsigned per = (span + 31u) / 32u;
      const unsigned lo = min(span, lane * per), hi = min(span, lo + per);
      unsigned mx = 0;
      for (unsigned i = lo; i < hi; ++i) { mx = max(mx, buf[i]); buf[i] = mx; }
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, mx, d);
        if (lane >= d) mx = max(mx, t);
      }
      unsigned ex = __shfl_up_sync(0xffffffffu, mx, 1);
      if (lane == 0) ex = 0u;
      for (unsigned i = lo; i < hi; ++i) buf[i] = max(buf[i], ex);
      __syncwarp();
    }
#endif
    for (unsigned j0 = wA + lane; j0 < wB; j0 += 32 * U) {
      int src[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned j = j0 + 32 * u;
#if SMC_FUSED_SCAN
        if (use_map) {
          src[u] = j < wB ? wk0 + (int)buf[j - wA] - 1 : wk0;
          continue;
        }
#endif
        int lo = wk0, hi = wk0 + wn - 1;                // first particle with O_k > j
#if SMC_FUSED_GALLOP
        // start at the proportional guess and gallop to a bracket (sources
        // sit near their proportional position when weights are even)
        if (j < wB) {
          int g = wk0 + (int)(((unsigned long long)(j - wA) * (unsigned)wn) / max(1u, wspan));
          g = min(max(g, wk0), wk0 + wn - 1);
          if (s_O[g] > j) {
            int st = 1;
            hi = g;
            while (g - st >= wk0 && s_O[g - st] > j) { hi = g - st; st <<= 1; }
            lo = max(wk0, g - st);
          } else {
            int st = 1;
            lo = g + 1;
            while (g + st < wk0 + wn - 1 && s_O[g + st] <= j) { lo = g + st + 1; st <<= 1; }
            hi = min(wk0 + wn - 1, g + st);
          }
        }
#endif
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_O[mid] > j) hi = mid; else lo = mid + 1;
        }
        src[u] = lo;
      }
      if (P > 0 && P <= 2 && a.stk_n == 0) {            // whole-particle copies
        uint4 v[U][P > 0 && P <= 2 ? P : 1];
        if (!a.lazy) {
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int p = 0; p < (P > 0 && P <= 2 ? P : 1); ++p)
              if (j0 + 32 * u < wB)
                v[u][p] = __ldg(a.src_planes + (unsigned long long)p * a.n_local + base + src[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const unsigned j = j0 + 32 * u;
          if (j < wB) {
            if (!a.lazy) {
#pragma unroll
              for (int p = 0; p < (P > 0 && P <= 2 ? P : 1); ++p) dst[(unsigned long long)p * a.n_local + j] = v[u][p];
            }
            anc[j] = (uint32_t)(a.shard_base + base + src[u]);
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const unsigned j = j0 + 32 * u;
          if (j < wB) {
            const unsigned long long sp = base + src[u];
            const int skip = stack_skip_lo(a, a.src_planes, sp);
            if (a.stk_n) stk_copied += planes_copied(a, skip);
            if (!a.lazy) copy_particle<P>(a, dst, sp, j, skip);
            anc[j] = (uint32_t)(a.shard_base + sp);
          }
        }
      }
    }
  } else {
    const unsigned A = s_O[blk], B = s_O[blk - 1];
    for (unsigned j = A + threadIdx.x; j < B; j += kFT) {
      int lo = 0, hi = blk - 1;                         // first item with O_k > j
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_O[mid] > j) hi = mid; else lo = mid + 1;
      }
      const unsigned long long src = base + lo;
      const int skip = stack_skip_lo(a, a.src_planes, src);
      if (a.stk_n) stk_copied += planes_copied(a, skip);
      if (!a.lazy) copy_particle<P>(a, dst, src, j, skip);
      anc[j] = (uint32_t)(a.shard_base + src);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) distinct += __shfl_xor_sync(0xffffffffu, distinct, d);
  if (lane == 0 && distinct) atomicAdd(&c->distinct, (unsigned long long)distinct);
  if (a.stk_n) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) stk_copied += __shfl_xor_sync(0xffffffffu, stk_copied, d);
    if (lane == 0 && stk_copied) atomicAdd(&c->stack_planes, stk_copied);
  }
}

}  // namespace smc
