// device_rng.cuh — Philox4x32-10, the hq uniform conversion, fp64 samplers and
// log-densities for the sm_100a propagation kernel.
//
// The paper asks for a unique seed per state and per-thread seeds in
// CUDA; we replace seed state by a stateless counter-based stream
// (DESIGN.md §R-1): draw d of particle n in epoch t is half (d & 1) of Philox
// block (d >> 1, t, n, tag=0) under key (seed_lo, seed_hi).  Samplers and draw
// counts follow DESIGN.md §R-3 (the oracle implements the same written spec
// independently; nothing here is shared with oracle/).
#pragma once
#include <cstdint>
#include <cstring>

namespace smc {

constexpr double kLn2 = 0.6931471805599453094172321214581766;
constexpr double kTwoPi = 6.283185307179586476925286766559006;
constexpr double kHalfLog2Pi = 0.9189385332046727417803297364056176;

// U = rounds per loop iteration: 10 = straight-line code; a partly rolled loop
// trades two loop instructions per iteration for code size.  Measured (B200,
// ms per sweep): the sequential stream rolled to 5: SEIR 82.7 -> 80.4 (its
// sampler code is instruction-fetch bound), sequential-stream CRBD 198 -> 213;
// every Philox rolled to 5: CRBD 53.6 -> 58.4, ClaDS2 181.4 -> 197.6.  So only
// the binomial samplers use the rolled form (Rng::uniform_compact).
#ifndef SMC_PHILOX_UNROLL_SEQ
#define SMC_PHILOX_UNROLL_SEQ 5
#endif
template <int U = 10>
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll U
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;                    // key schedule (the bump after round 10 is unused)
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Out-of-line Philox for call sites where code size matters more than the
// call (the ClaDS2 kernel was instruction-fetch bound, ncu no_instruction
// stalls): SMC_PHILOX_OOL=1 routes Rng::uniform and the side-tree blocks
// through one copy of the rounds.  Same values either way.
#ifndef SMC_PHILOX_OOL
#define SMC_PHILOX_OOL 0
#endif
__device__ __noinline__ uint4 philox_call(uint4 c, uint32_t k0, uint32_t k1) { return philox4x32_10(c, k0, k1); }
__device__ __forceinline__ uint4 philox_site(uint4 c, uint32_t k0, uint32_t k1) {
#if SMC_PHILOX_OOL
  return philox_call(c, k0, k1);
#else
  return philox4x32_10(c, k0, k1);
#endif
}

// log of a uniform u in (0, 1) (an hq draw: normal, never 0 or 1) for the
// Exp and Box-Muller draws: u = 2^k z, z in [sqrt(1/2), sqrt(2)); a 128-entry
// table (invc ~ 1/c, logc = -ln invc; tools/gen_logu_table.py) reduces to
// r = fma(z, invc, -1), |r| < 2^-8; log1p(r) by Taylor to degree 7.  Worst
// error 1.23 ulp against 60-digit logs (CUDA's log: <= 1 ulp; glibc's, the
// oracle's: < 1 ulp) — ulp-level differences of the class the parity bars
// already admit, for ~12 instead of ~30 fp64 operations.
#ifndef SMC_FAST_LOGU
#define SMC_FAST_LOGU 1
#endif
#include "logu_table.cuh"
__device__ __forceinline__ double log_table(double u) {
  const long long ix = __double_as_longlong(u);
  const long long tmp = ix - 0x3fe6a09e667f3bcdLL;
  const int i = (int)((tmp >> 45) & 127);
  const double kd = (double)(tmp >> 52);
  const double z = __longlong_as_double(ix - (tmp & (long long)0xfff0000000000000ULL));
  const double2 t = __ldg(&c_logu_tab[i]);
  const double r = fma(z, t.x, -1.0);
  double p = fma(r, 1.0 / 7.0, -1.0 / 6.0);
  p = fma(r, p, 1.0 / 5.0);
  p = fma(r, p, -0.25);
  p = fma(r, p, 1.0 / 3.0);
  p = fma(r, p, -0.5);
  const double l1 = fma(r * r, p, r);
  return fma(kd, SMC_LOGU_LN2_HI, t.y) + fma(kd, SMC_LOGU_LN2_LO, l1);
}
__device__ __forceinline__ double log_u(double u) {
#if SMC_FAST_LOGU
  return log_table(u);
#else
  return log(u);
#endif
}
// The same for any x: the table path serves positive normal finite x (the
// reduction holds for any exponent); 0, subnormals, inf and NaN take the
// library log out of line (one copy).  Used for log(lambda) weight terms.
__device__ __noinline__ double log_far(double x) { return log(x); }
#ifndef SMC_FAST_LOGPOS
#define SMC_FAST_LOGPOS 0      // measured neutral (CRBD 48.5 vs 48.6, ClaDS2 156.5 vs 157.0 ms): library log for weight terms
#endif
__device__ __forceinline__ double log_pos(double x) {
#if SMC_FAST_LOGU && SMC_FAST_LOGPOS
  if (!(x >= 0x1p-1022 && x <= 0x1.fffffffffffffp+1023)) return log_far(x);
  return log_table(x);
#else
  return log(x);
#endif
}

// e^x by a 128-entry table of 2^(j/128) and a degree-5 expm1 (Tang's method;
// tools/gen_expt_table.py: worst 0.99 ulp against 60-digit exponentials), for
// the ClaDS2 rate factors e^{sigma z}; |x| > 700 (overflow / underflow
// territory) is clamped (or, SMC_FAST_EXP=1, goes to exp()).  ~10 instead of
// ~17 fp64 operations.
#ifndef SMC_FAST_EXP
#define SMC_FAST_EXP 2      // 2: clamped to |x| <= 700 (ClaDS2 156.6 -> 153.6 ms/sweep); 1: out-of-line
#endif                      // library exp beyond 700 (measured slower, 160.7 -> 165.2); 0: library exp
#include "expt_table.cuh"
__device__ __noinline__ double exp_far(double x) { return exp(x); }   // rare: one out-of-line copy
__device__ __forceinline__ double exp_t(double x) {
#if SMC_FAST_EXP
#if SMC_FAST_EXP == 2
  // clamped instead of a far path: e^{+-700} stands in for inf / 0 (a rate
  // factor that large breaks the rate guard either way; one that small makes
  // every event time exceed the branch, as a zero rate does)
  x = fmin(fmax(x, -700.0), 700.0);
#else
  if (!(fabs(x) <= 700.0)) return exp_far(x);
#endif
  const double kd = rint(x * SMC_EXPT_INV);
  const int k = (int)kd;
  double r = fma(-kd, SMC_EXPT_C_HI, x);
  r = fma(-kd, SMC_EXPT_C_LO, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r * r, p, r);                             // expm1(r)
  const double tj = __ldg(&c_expt_tab[k & 127]);
  const double scale = __hiloint2double(((k >> 7) + 1023) << 20, 0);
  return fma(tj, p, tj) * scale;
#else
  return exp(x);
#endif
}

// cos and sin of 2 pi t for a uniform t in (0, 1) (the Box-Muller angle):
// j = rint(256 t), r = t - j/256 exactly, x = 2 pi r, |x| <= pi/256;
// cos(2 pi t) = C_j cos x - S_j sin x (sin likewise) with a 256-entry table of
// (C_j, S_j) and Taylor polynomials to x^6 / x^7 (tools/gen_trig_table.py:
// absolute error <= 1.6e-16, below that of cos(fl(2 pi u)) itself).
#ifndef SMC_FAST_TRIG
#define SMC_FAST_TRIG 1
#endif
#include "trig_table.cuh"
__device__ __forceinline__ double2 sincos2pi_u(double t) {      // (sin, cos)
  const double jd = rint(t * 256.0);
  const double r = t - jd * (1.0 / 256.0);
  const double x = r * SMC_TRIG_TWO_PI;
  const double x2 = x * x;
  double cm = fma(x2, -1.0 / 720.0, 1.0 / 24.0);
  cm = fma(x2, cm, -0.5);
  cm = x2 * cm;                                     // cos x - 1
  double sp = fma(x2, -1.0 / 5040.0, 1.0 / 120.0);
  sp = fma(x2, sp, -1.0 / 6.0);
  const double sx = fma(x * x2, sp, x);             // sin x
  const double2 cs = __ldg(&c_trig_tab[(int)jd & 255]);
  return make_double2(fma(cs.y, cm, fma(cs.x, sx, cs.y)), fma(cs.x, cm, fma(-cs.y, sx, cs.x)));
}
__device__ __forceinline__ double cos2pi_u(double t) {
#if SMC_FAST_TRIG
  return sincos2pi_u(t).y;
#else
  return cospi(2.0 * t);
#endif
}

// 53-bit integer of the hq conversion and the double u = z 2^-53 + 2^-54.
__device__ __forceinline__ unsigned long long hq_bits(uint32_t x, uint32_t y) {
  return (unsigned long long)x ^ ((unsigned long long)y << 21);
}
__device__ __forceinline__ double hq(uint32_t x, uint32_t y) {
  // z 2^-53 is exact (z < 2^53), so one fma rounds exactly where the add did
  return __fma_rn(__ull2double_rn(hq_bits(x, y)), 0x1p-53, 0x1p-54);
}

// Per-particle uniform stream for one epoch (registers only; SoA state holds
// no RNG state because the stream is a pure function of the counters).
struct Rng {
  uint32_t k0, k1, t, n, blk;
  double spare;
  bool has_spare;
  __device__ __forceinline__ Rng(unsigned long long seed, uint32_t particle, uint32_t epoch)
      : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), t(epoch), n(particle), blk(0),
        spare(0.0), has_spare(false) {}
  __device__ __forceinline__ double uniform() {
    if (has_spare) { has_spare = false; return spare; }
    const uint4 r = philox_site(make_uint4(blk, t, n, 0u), k0, k1);
    ++blk;
    spare = hq(r.z, r.w);
    has_spare = true;
    return hq(r.x, r.y);
  }
  // The same stream from a partly rolled Philox (smaller code; for the
  // out-of-line binomial samplers, whose kernel is instruction-fetch bound).
  __device__ __forceinline__ double uniform_compact() {
    if (has_spare) { has_spare = false; return spare; }
    const uint4 r = philox4x32_10<SMC_PHILOX_UNROLL_SEQ>(make_uint4(blk, t, n, 0u), k0, k1);
    ++blk;
    spare = hq(r.z, r.w);
    has_spare = true;
    return hq(r.x, r.y);
  }
  // The next six uniforms of the stream, without consuming them: the three
  // Philox blocks they need are independent (instruction-level parallelism
  // instead of one block per dependent uniform() call).  consume(n, u), n <= 5,
  // then advances the stream exactly as n calls of uniform() would.
  __device__ __forceinline__ void peek6(double u[6]) const {
    const uint4 a = philox4x32_10(make_uint4(blk, t, n, 0u), k0, k1);
    const uint4 b = philox4x32_10(make_uint4(blk + 1u, t, n, 0u), k0, k1);
    const uint4 c = philox4x32_10(make_uint4(blk + 2u, t, n, 0u), k0, k1);
    const double h[6] = {hq(a.x, a.y), hq(a.z, a.w), hq(b.x, b.y), hq(b.z, b.w), hq(c.x, c.y), hq(c.z, c.w)};
    if (has_spare) {
      u[0] = spare;
#pragma unroll
      for (int k = 1; k < 6; ++k) u[k] = h[k - 1];
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) u[k] = h[k];
    }
  }
  // The next two uniforms from ONE Philox block (u[2] = the block's other half
  // when the first came from the spare): consume(cnt <= 2, u) follows.
  __device__ __forceinline__ void peek2(double u[3]) const {
    const uint4 a = philox4x32_10(make_uint4(blk, t, n, 0u), k0, k1);
    if (has_spare) { u[0] = spare; u[1] = hq(a.x, a.y); u[2] = hq(a.z, a.w); }
    else { u[0] = hq(a.x, a.y); u[1] = hq(a.z, a.w); u[2] = 0.0; }
  }
  __device__ __forceinline__ void consume(int cnt, const double* u) {
    // position of the next uniform: 2 blk - has_spare
    const uint32_t p = 2u * blk - (has_spare ? 1u : 0u) + (uint32_t)cnt;
    blk = (p + 1u) >> 1;
    has_spare = (p & 1u) != 0u;
    if (has_spare) spare = u[cnt];          // half 1 of block p >> 1 (peeked)
  }
};

// ---- samplers (draw counts: Exp 1, Bernoulli 1, Uniform 1, Normal 2,
//      Gamma k=1: 1, k>1: 3 per attempt, k<1: Gamma(k+1) then 1, Beta: two
//      Gammas, Binomial inversion 1, BTRS 2 per attempt) --------------------
__device__ __forceinline__ double d_exp(Rng& r, double rate) {
  const double u = r.uniform();
  return -log_u(u) / rate;
}
__device__ __forceinline__ bool d_bernoulli(Rng& r, double p) { return r.uniform() < p; }
__device__ __forceinline__ double d_uniform(Rng& r, double a, double b) {
  const double u = r.uniform();
  return a + (b - a) * u;
}
__device__ __forceinline__ double d_normal(Rng& r, double mu, double sigma) {
  const double u1 = r.uniform();
  const double u2 = r.uniform();
  const double rad = sqrt(-2.0 * log_u(u1));
  const double c = cos2pi_u(u2);          // cos(2 pi u2) without a 2 pi range reduction
  return mu + sigma * (rad * c);
}
__device__ __noinline__ double d_gamma_mt(Rng& r, double k, double theta) {   // k > 1, Marsaglia-Tsang
  const double d = k - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    const double x = d_normal(r, 0.0, 1.0);
    const double u = r.uniform();
    double v = 1.0 + c * x;
    if (v <= 0.0) continue;
    v = v * v * v;
    const double lhs = log(u);
    const double rhs = 0.5 * x * x + d - d * v + d * log(v);
    if (lhs < rhs) return d * v * theta;
  }
}
__device__ __forceinline__ double d_gamma(Rng& r, double k, double theta) {
  if (k == 1.0) {
    const double u = r.uniform();
    return -theta * log_u(u);
  }
  if (k < 1.0) {
    const double g = d_gamma_mt(r, k + 1.0, theta);
    const double u = r.uniform();
    return g * pow(u, 1.0 / k);
  }
  return d_gamma_mt(r, k, theta);
}
__device__ __forceinline__ double d_beta(Rng& r, double a, double b) {
  const double x = d_gamma(r, a, 1.0);
  const double y = d_gamma(r, b, 1.0);
  return x / (x + y);
}

// lgamma(k + 1) for integer k: table lookup when the model supplies one
// (host-computed log-factorials, identical to the host libm values), else the
// device lgamma.  Every lgamma in the binomial code has an integer argument.
struct LogFact {
  const double* tbl;
  long long n;
  __device__ __forceinline__ double operator()(double x1) const {   // x1 = k + 1
    const long long k = (long long)x1 - 1;
    return (tbl && k >= 0 && k < n) ? __ldg(tbl + k) : lgamma(x1);
  }
};

// Binomial: inversion (BINV) for n p < 10; BTRS (Hormann 1993) otherwise.
// The BTRS normaliser h = lgamma(m+1) + lgamma(n-m+1) is only needed when
// the squeeze fails, so it is computed lazily (same value, fewer lgammas).
// SMC_FAST_BINOM: the same formulas with the table-driven log / exp of §7.8
// (log1p(y) = log u + (y - (u - 1)) / u for u = fl(1 + y), the tiny
// correction divided by a float reciprocal), 1/x from a table in the
// inversion loop, and the BTRS acceptance log by the table: ulp-level
// differences, as the CUDA/glibc transcendentals have.
#ifndef SMC_FAST_BINOM
#define SMC_FAST_BINOM 1
#endif
struct RcpTab { double v[128]; };
constexpr RcpTab make_rcp_tab() {
  RcpTab t{};
  for (int i = 1; i < 128; ++i) t.v[i] = 1.0 / (double)i;
  return t;
}
__device__ const RcpTab c_rcp_tab = make_rcp_tab();
__device__ __forceinline__ double log1p_neg(double y) {            // y in [-1/2, 0]
  const double u = 1.0 + y;
  const double c = y - (u - 1.0);                                   // exact (Sterbenz)
  return log_table(u) + c * (double)__frcp_rn((float)u);
}
__device__ __noinline__ long long d_binomial_inv(Rng& r, long long n, double p) {
  const double q = 1.0 - p;
  const double sr = p / q;
  const double a = (double)(n + 1) * sr;
#if SMC_FAST_BINOM
  double pr = exp_t((double)n * log1p_neg(-p));
#else
  double pr = exp((double)n * log1p(-p));
#endif
  double u = r.uniform_compact();
  long long x = 0;
  while (x < n && u > pr) {
    u = u - pr;
    x = x + 1;
#if SMC_FAST_BINOM
    pr = pr * ((x < 128 ? a * c_rcp_tab.v[x] : a / (double)x) - sr);
#else
    pr = pr * (a / (double)x - sr);
#endif
  }
  return x;
}
__device__ __noinline__ long long d_binomial_btrs(Rng& r, long long n, double p, const LogFact& lf) {
  const double q = 1.0 - p;
  const double nd = (double)n;
  const double spq = sqrt(nd * p * q);
  const double b = 1.15 + 2.53 * spq;
  const double a = -0.0873 + 0.0248 * b + 0.01 * p;
  const double c = nd * p + 0.5;
  const double vr = 0.92 - 4.2 / b;
  const double m = floor((nd + 1.0) * p);
  bool have_h = false;
  double h = 0.0, alpha = 0.0, lpq = 0.0;
  for (;;) {
    const double U = r.uniform_compact() - 0.5;
    const double V = r.uniform_compact();
    const double us = 0.5 - fabs(U);
    const double kd = floor((2.0 * a / us + b) * U + c);
    if (kd < 0.0 || kd > nd) continue;
    if (us >= 0.07 && V <= vr) return (long long)kd;
    if (!have_h) {
      alpha = (2.83 + 5.1 / b) * spq;
#if SMC_FAST_BINOM
      lpq = log_table(p / q);
#else
      lpq = log(p / q);
#endif
      h = lf(m + 1.0) + lf(nd - m + 1.0);
      have_h = true;
    }
#if SMC_FAST_BINOM
    const double lv = log_table(V * alpha / (a / (us * us) + b));
#else
    const double lv = log(V * alpha / (a / (us * us) + b));
#endif
    const double rhs = h - lf(kd + 1.0) - lf(nd - kd + 1.0) + (kd - m) * lpq;
    if (lv <= rhs) return (long long)kd;
  }
}
// Out of line on purpose: SEIR calls it 11 times per day; inlining every copy
// of BTRS + inversion made the kernel thrash the instruction cache (ncu:
// "no_instruction" stalls 30 cycles per issue).
__device__ __noinline__ long long d_binomial(Rng& r, long long n, double p,
                                            const LogFact& lf = LogFact{nullptr, 0}) {
  bool flip = false;
  if (p > 0.5) { p = 1.0 - p; flip = true; }
  const long long k = ((double)n * p < 10.0) ? d_binomial_inv(r, n, p) : d_binomial_btrs(r, n, p, lf);
  return flip ? n - k : k;
}

__device__ __noinline__ double d_binomial_logpmf(long long k, long long n, double p,
                                                    const LogFact& lf = LogFact{nullptr, 0}) {
  if (k < 0 || k > n) return -INFINITY;
  double v = lf((double)n + 1.0) - lf((double)k + 1.0) - lf((double)(n - k) + 1.0);
  if (k > 0) v = v + (double)k * log(p);
  if (n - k > 0) v = v + (double)(n - k) * log1p(-p);
  return v;
}
__device__ __forceinline__ double d_normal_logpdf(double y, double mu, double sigma) {
  const double z = (y - mu) / sigma;
  return -0.5 * z * z - log(sigma) - kHalfLog2Pi;
}

// ---- order-preserving int64 key of a double (for atomicMax of log-weights)
__device__ __forceinline__ long long order_key(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFLL);
}
__host__ __device__ __forceinline__ double key_to_double(long long k) {
  const long long b = k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFLL);
  double d;
  memcpy(&d, &b, sizeof(d));
  return d;
}

}  // namespace smc
