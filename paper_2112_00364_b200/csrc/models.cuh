// models.cuh — PCFG block tables (sim : B x S -> B x S x {ckpt})
// for the propagation kernel.  Each model is a struct with
//   kPlanes                 number of 16-byte SoA state planes
//   State / load / store    registers <-> planes  (plane p of particle i at
//                           planes[p * stride + i])
//   pc(s)                   current block, kStop = -1 is b_stop
//   step(s, lw, rng, C, d)  run block pc(s) once; returns true at a checkpoint
//                           (checkpoints only at block tails)
// The specs are DESIGN.md §R-11 (CRBD), §R-14 (ClaDS2), §R-15 (SEIR),
// Fig. 2 (geometric), Eq. (2)/Fig. 4 (SSM), S:493 (constant weight).
#pragma once
#include "device_rng.cuh"

namespace smc {

constexpr int kStop = -1;
constexpr int kStackCap = 1024;          // helper DFS stack (§R-12)
constexpr unsigned kEventCap = 1u << 22; // helper DFS events per call (§R-12)

// Constant model data, passed by value to the kernel.
struct ModelConst {
  const double* table;   // device: per-model table (branches / series)
  int n;                 // number of branches / series length
  int flags;
  double p[12];          // parameters
  const double* logfact; // SEIR: lgamma(k+1), k < n_logfact (host libm values)
  long long n_logfact;
};

// Per-thread diagnostics sink.
struct Diag {
  unsigned long long overflow;
  unsigned guard;                // ClaDS2 rate-guard kills (R-14b)
  __device__ Diag() : overflow(0), guard(0) {}
};

__device__ __forceinline__ uint4 ldp(const uint4* planes, unsigned long long stride, int p,
                                     unsigned long long i) {
  return planes[(unsigned long long)p * stride + i];
}
__device__ __forceinline__ void stp(uint4* planes, unsigned long long stride, int p,
                                    unsigned long long i, uint4 v) {
  planes[(unsigned long long)p * stride + i] = v;
}
__device__ __forceinline__ uint4 pack_dd(double a, double b) {
  const unsigned long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return make_uint4((uint32_t)x, (uint32_t)(x >> 32), (uint32_t)y, (uint32_t)(y >> 32));
}
__device__ __forceinline__ double lo_d(uint4 v) {
  return __longlong_as_double(((long long)v.y << 32) | v.x);
}
__device__ __forceinline__ double hi_d(uint4 v) {
  return __longlong_as_double(((long long)v.w << 32) | v.z);
}

// ============================================================================
// CRBD (§R-11).  Table: per branch i (left-first preorder over non-root
// nodes): [t_parent, t_child, internal].  Params: rho, lambda_fixed, mu_fixed.
// Planes: P0 = {lambda, mu}; P1 = {pc, branch, 0, 0}.
// ============================================================================
struct Crbd {
  static constexpr int kPlanes = 2;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kOneWave = false;  // grid: one CTA per 256 particles (uneven work: block scheduler balances)
  struct State { double lambda, mu; int pc, branch; };
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    const uint4 a = ldp(P, st, 0, i), b = ldp(P, st, 1, i);
    s.lambda = lo_d(a); s.mu = hi_d(a); s.pc = (int)b.x; s.branch = (int)b.y;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    stp(P, st, 0, i, pack_dd(s.lambda, s.mu));
    stp(P, st, 1, i, make_uint4((uint32_t)s.pc, (uint32_t)s.branch, 0u, 0u));
  }
  __device__ static int pc(const State& s) { return s.pc; }

  // goesUndetected: DFS over the hidden side subtree born at age s0.
  // 1 undetected, 0 detected, -1 stack/event overflow.
  __device__ static int undetected(double s0, const State& st, double rho, Rng& r) {
    double stack[kStackCap];
    int sp = 0;
    stack[sp++] = s0;
    unsigned events = 0;
    const double tot = st.lambda + st.mu;
    const double pb = st.lambda / tot;
    while (sp > 0) {
      double s = stack[--sp];
      for (;;) {
        if (++events > kEventCap) return -1;
        const double d = d_exp(r, tot);
        if (d > s) {
          if (d_bernoulli(r, rho)) return 0;
          break;
        }
        s = s - d;
        if (d_bernoulli(r, pb)) {
          if (sp >= kStackCap) return -1;
          stack[sp++] = s;
          continue;
        }
        break;
      }
    }
    return 1;
  }

  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag& dg) {
    const double rho = C.p[0];
    if (s.pc == 0) {                                    // INIT, jump (no checkpoint)
      s.lambda = C.p[1] >= 0.0 ? C.p[1] : d_gamma(r, 1.0, 1.0);
      s.mu = C.p[2] >= 0.0 ? C.p[2] : d_gamma(r, 1.0, 0.5);
      s.branch = 0;
      s.pc = 1;
      return false;
    }
    const double* b = C.table + 3 * s.branch;           // BRANCH
    const double tp = __ldg(b), tc = __ldg(b + 1);
    const bool internal = __ldg(b + 2) != 0.0;
    lw = lw + (-s.mu * (tp - tc));
    lw = lw + (internal ? log_pos(s.lambda) : log(rho));
    double t = tp;
    for (;;) {
      t = t - d_exp(r, s.lambda);
      if (t <= tc) break;
      const int u = undetected(t, s, rho, r);
      if (u == 1) { lw = lw + kLn2; continue; }
      if (u < 0) ++dg.overflow;
      lw = -INFINITY;
      break;
    }
    s.branch = s.branch + 1;
    s.pc = (s.branch == C.n) ? kStop : 1;
    return true;
  }
};

// ============================================================================
// CRBD with the §5.3 variance reduction: each hidden
// speciation event at age t is weighted by 2 E(t), E = probability that a
// lineage alive at age t leaves no sampled descendant, instead of simulating
// its side tree.  Same state and planes as Crbd; no helper stack.
// ============================================================================
__device__ __forceinline__ double crbd_no_sampled_descendant(double t, double lam, double mu, double rho) {
  // one branch-free form for both signs of r = lam - mu (lanes of a warp hold
  // different particles' rates): with a = |r| t, g = (1 - e^{-a}) / |r|
  // (-> t at r = 0) and c = e^{-rt} if r > 0 else 1,
  //   E = (rho mu g + (1 - rho) c) / (rho lam g + c)
  // (r > 0: numerator and denominator of the textbook form scaled by e^{-rt})
  const double r = lam - mu, ar = fabs(r);
  const double em = expm1(-ar * t);                    // e^{-a} - 1, in (-1, 0]
  const double g = ar > 0.0 ? -em / ar : t;
  const double c = r > 0.0 ? exp(-ar * t) : 1.0;       // not em + 1: relative accuracy for large a
  return (rho * mu * g + (1.0 - rho) * c) / (rho * lam * g + c);
}

struct CrbdAE : Crbd {
  static constexpr int kMinBlocks = 4;
  static constexpr bool kOneWave = true;   // grid: one resident wave, grid-stride (light, even work)
  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag&) {
    const double rho = C.p[0];
    if (s.pc == 0) {                                    // INIT, jump (no checkpoint)
      s.lambda = C.p[1] >= 0.0 ? C.p[1] : d_gamma(r, 1.0, 1.0);
      s.mu = C.p[2] >= 0.0 ? C.p[2] : d_gamma(r, 1.0, 0.5);
      s.branch = 0;
      s.pc = 1;
      return false;
    }
    const double* b = C.table + 3 * s.branch;           // BRANCH
    const double tp = __ldg(b), tc = __ldg(b + 1);
    const bool internal = __ldg(b + 2) != 0.0;
    lw = lw + (-s.mu * (tp - tc));
    lw = lw + (internal ? log_pos(s.lambda) : log(rho));
    double t = tp;
    for (;;) {
      t = t - d_exp(r, s.lambda);
      if (t <= tc) break;
      lw = lw + kLn2;
      lw = lw + log_pos(crbd_no_sampled_descendant(t, s.lambda, s.mu, rho));
    }
    s.branch = s.branch + 1;
    s.pc = (s.branch == C.n) ? kStop : 1;
    return true;
  }
};

// ============================================================================
// ClaDS2 (§R-14).  Table: per branch i (smaller-subtree-first preorder):
// [t_parent, t_child, internal, first_left]; C.p[5] = root first_left.
// Params: rho, lambda0, sigma, alpha, eps (each < 0: prior).
// Planes: P0 {sigma, alpha} P1 {eps, lam} P2..P4 pending rates[6]
//         P5 {pc, branch, sp, 0}.
// ============================================================================
// Rate guard: any lineage rate above kMaxRate (or not
// finite) is outside the model's support -> weight -inf and the block ends
// ("kill": branch index and pc advance, nothing else).
struct Clads2 {
  static constexpr int kPlanes = 6;
  static constexpr int kMinBlocks = 2;
  static constexpr bool kOneWave = false;  // grid: one CTA per 256 particles (uneven work: block scheduler balances)
  static constexpr int kPend = 6;
  static constexpr double kMaxRate = 1e4;
  __device__ static bool bad_rate(double r) { return !(r <= kMaxRate); }

  struct State { double sigma, alpha, eps, lam; double pend[kPend]; int pc, branch, sp; };
  // The pending-rate stack is pend[0, sp): planes beyond the stack pointer are
  // neither read nor written (the copies skip them too).
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    uint4 v = ldp(P, st, 5, i); s.pc = (int)v.x; s.branch = (int)v.y; s.sp = (int)v.z;
    v = ldp(P, st, 0, i); s.sigma = lo_d(v); s.alpha = hi_d(v);
    v = ldp(P, st, 1, i); s.eps = lo_d(v); s.lam = hi_d(v);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v = 2 * k < s.sp ? ldp(P, st, 2 + k, i) : make_uint4(0u, 0u, 0u, 0u);
      s.pend[2 * k] = lo_d(v); s.pend[2 * k + 1] = hi_d(v);
    }
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    stp(P, st, 0, i, pack_dd(s.sigma, s.alpha));
    stp(P, st, 1, i, pack_dd(s.eps, s.lam));
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (2 * k < s.sp) stp(P, st, 2 + k, i, pack_dd(s.pend[2 * k], s.pend[2 * k + 1]));
    stp(P, st, 5, i, make_uint4((uint32_t)s.pc, (uint32_t)s.branch, (uint32_t)s.sp, 0u));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  __device__ static double daughter(const State& s, double lam, double z) {
    return s.alpha * lam * exp(s.sigma * z);
  }
  __device__ static void push(State& s, double v) {
    // constant-index selects keep pend[] in registers
#pragma unroll
    for (int k = 0; k < kPend; ++k) if (k == s.sp) s.pend[k] = v;
    s.sp = s.sp + 1;
  }
  __device__ static double pop(State& s) {
    s.sp = s.sp - 1;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < kPend; ++k) if (k == s.sp) v = s.pend[k];
    return v;
  }
  __device__ static int undetected(double s0, double lam0, const State& st, double rho, Rng& r) {
    double stk_s[kStackCap];
    double stk_l[kStackCap];
    int sp = 0;
    stk_s[sp] = s0; stk_l[sp] = lam0; ++sp;
    unsigned events = 0;
    const double pb = 1.0 / (1.0 + st.eps);
    while (sp > 0) {
      --sp;
      double s = stk_s[sp], lam = stk_l[sp];
      for (;;) {
        if (++events > kEventCap) return -1;
        const double d = d_exp(r, lam * (1.0 + st.eps));
        if (d > s) {
          if (d_bernoulli(r, rho)) return 0;
          break;
        }
        s = s - d;
        if (d_bernoulli(r, pb)) {
          const double za = d_normal(r, 0.0, 1.0);
          const double zb = d_normal(r, 0.0, 1.0);
          const double la = daughter(st, lam, za), lb = daughter(st, lam, zb);
          if (bad_rate(la) || bad_rate(lb)) return -2;
          if (sp >= kStackCap) return -1;
          stk_s[sp] = s; stk_l[sp] = lb; ++sp;
          lam = la;
          continue;
        }
        break;
      }
    }
    return 1;
  }
  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag& dg) {
    const double rho = C.p[0];
    if (s.pc == 0) {                                     // INIT + root split (jump)
      const double lam0 = C.p[1] >= 0.0 ? C.p[1] : d_gamma(r, 1.0, 1.0);
      s.sigma = C.p[2] >= 0.0 ? C.p[2] : sqrt(1.0 / d_gamma(r, 1.0, 1.0 / 0.2));
      s.alpha = C.p[3] >= 0.0 ? C.p[3] : exp(d_normal(r, 0.0, s.sigma));
      s.eps = C.p[4] >= 0.0 ? C.p[4] : d_uniform(r, 0.0, 1.0);
      const double zl = d_normal(r, 0.0, 1.0);
      const double zr = d_normal(r, 0.0, 1.0);
      const double rl = daughter(s, lam0, zl), rr = daughter(s, lam0, zr);
      const bool fl = C.p[5] != 0.0;
      s.sp = 0;
      push(s, fl ? rr : rl);
      s.lam = fl ? rl : rr;
      s.branch = 0;
      s.pc = 1;
      return false;
    }
    const double* b = C.table + 4 * s.branch;
    const double tp = __ldg(b), tc = __ldg(b + 1);
    const bool internal = __ldg(b + 2) != 0.0;
    const bool first_left = __ldg(b + 3) != 0.0;
    bool killed = bad_rate(s.lam), detected = false;
    double t = tp;
    while (!killed) {
      const double dt = d_exp(r, s.lam);
      if (t - dt <= tc) {
        lw = lw + (-s.eps * s.lam * (t - tc));
        break;
      }
      lw = lw + (-s.eps * s.lam * dt);
      t = t - dt;
      const double zs = d_normal(r, 0.0, 1.0);
      const double zc = d_normal(r, 0.0, 1.0);
      const double ls = daughter(s, s.lam, zs);
      if (bad_rate(ls)) { killed = true; break; }
      const int u = undetected(t, ls, s, rho, r);
      if (u != 1) {
        if (u == -1) ++dg.overflow;
        if (u != -2) detected = true;   // detected / overflow: not a guard kill
        killed = true;
        break;
      }
      lw = lw + kLn2;
      s.lam = daughter(s, s.lam, zc);
      if (bad_rate(s.lam)) { killed = true; break; }
    }
    if (!killed && internal) {
      lw = lw + log_pos(s.lam);
      const double zl = d_normal(r, 0.0, 1.0);
      const double zr = d_normal(r, 0.0, 1.0);
      const double rl = daughter(s, s.lam, zl), rr = daughter(s, s.lam, zr);
      if (bad_rate(rl) || bad_rate(rr)) {
        killed = true;
      } else {
        push(s, first_left ? rr : rl);
        s.lam = first_left ? rl : rr;
      }
    } else if (!killed) {
      lw = lw + log(rho);
      if (s.branch + 1 < C.n) s.lam = pop(s);
    }
    if (killed) {
      lw = -INFINITY;
      if (!detected) ++dg.guard;
    }
    s.branch = s.branch + 1;
    s.pc = (s.branch == C.n) ? kStop : 1;
    return true;
  }
};

// ============================================================================
// SEIR (§R-15).  Table: y[T].  Params: [lam_h, del_h, gam_h, lam_m, del_m,
// rho] (p[0] < 0: priors), p[6] n_h, p[7] s_m0, p[8] e_h0, p[9] i_m0.
// Planes: P0 {lam_h, del_h} P1 {gam_h, lam_m} P2 {del_m, rho}
//         P3 {sh, eh, ih, rh} P4 {sm, em, im, t} P5 {pc, 0, 0, 0}.
// ============================================================================
#ifndef SMC_SEIR_MINB
#define SMC_SEIR_MINB 4   // 64 registers (some spills): 86.9 vs 88.5 ms/sweep at 3 (80 registers)
#endif
struct Seir {
  static constexpr int kPlanes = 6;
  static constexpr int kMinBlocks = SMC_SEIR_MINB;
  static constexpr bool kOneWave = false;  // grid: one CTA per 256 particles (uneven work: block scheduler balances)
  struct State { double lam_h, del_h, gam_h, lam_m, del_m, rho; int sh, eh, ih, rh, sm, em, im, t, pc; };
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    uint4 v = ldp(P, st, 0, i); s.lam_h = lo_d(v); s.del_h = hi_d(v);
    v = ldp(P, st, 1, i); s.gam_h = lo_d(v); s.lam_m = hi_d(v);
    v = ldp(P, st, 2, i); s.del_m = lo_d(v); s.rho = hi_d(v);
    v = ldp(P, st, 3, i); s.sh = (int)v.x; s.eh = (int)v.y; s.ih = (int)v.z; s.rh = (int)v.w;
    v = ldp(P, st, 4, i); s.sm = (int)v.x; s.em = (int)v.y; s.im = (int)v.z; s.t = (int)v.w;
    v = ldp(P, st, 5, i); s.pc = (int)v.x;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    stp(P, st, 0, i, pack_dd(s.lam_h, s.del_h));
    stp(P, st, 1, i, pack_dd(s.gam_h, s.lam_m));
    stp(P, st, 2, i, pack_dd(s.del_m, s.rho));
    stp(P, st, 3, i, make_uint4((uint32_t)s.sh, (uint32_t)s.eh, (uint32_t)s.ih, (uint32_t)s.rh));
    stp(P, st, 4, i, make_uint4((uint32_t)s.sm, (uint32_t)s.em, (uint32_t)s.im, (uint32_t)s.t));
    stp(P, st, 5, i, make_uint4((uint32_t)s.pc, 0u, 0u, 0u));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag&) {
    const long long nh_i = (long long)C.p[6];
    if (s.pc == 0) {                                     // INIT (jump)
      if (C.p[0] >= 0.0) {
        s.lam_h = C.p[0]; s.del_h = C.p[1]; s.gam_h = C.p[2];
        s.lam_m = C.p[3]; s.del_m = C.p[4]; s.rho = C.p[5];
      } else {
        s.lam_h = d_beta(r, 1.0, 1.0);
        s.del_h = d_beta(r, 1.0 + 2.0 / 4.4, 3.0 - 2.0 / 4.4);
        s.gam_h = d_beta(r, 1.0 + 2.0 / 4.5, 3.0 - 2.0 / 4.5);
        s.lam_m = d_beta(r, 1.0, 1.0);
        s.del_m = d_beta(r, 1.0 + 2.0 / 6.5, 3.0 - 2.0 / 6.5);
        s.rho = d_beta(r, 1.0, 1.0);
      }
      const int eh0 = (int)C.p[8];
      s.sh = (int)nh_i - 1 - eh0; s.eh = eh0; s.ih = 1; s.rh = 0;
      s.sm = (int)C.p[7]; s.em = 0; s.im = (int)C.p[9];
      s.t = 0;
      s.pc = 1;
      return false;
    }
    const LogFact lf{C.logfact, C.n_logfact};
    const double nh = (double)nh_i;                      // DAY
#if SMC_FAST_BINOM
    const double ph = 1.0 - exp_t(-(double)s.im / nh);    // (table exp, §7.8)
    const double pm = 1.0 - exp_t(-(double)s.ih / nh);
#else
    const double ph = 1.0 - exp(-(double)s.im / nh);
    const double pm = 1.0 - exp(-(double)s.ih / nh);
#endif
    const long long tau_h = d_binomial(r, s.sh, ph, lf);
    const long long de_h = d_binomial(r, tau_h, s.lam_h, lf);
    const long long di_h = d_binomial(r, s.eh, s.del_h, lf);
    const long long dr_h = d_binomial(r, s.ih, s.gam_h, lf);
    s.sh = (int)(s.sh - de_h);
    s.eh = (int)(s.eh + de_h - di_h);
    s.ih = (int)(s.ih + di_h - dr_h);
    s.rh = (int)(s.rh + dr_h);
    const long long tau_m = d_binomial(r, s.sm, pm, lf);
    const long long de_m = d_binomial(r, tau_m, s.lam_m, lf);
    const long long di_m = d_binomial(r, s.em, s.del_m, lf);
    const long long nm = (long long)s.sm + s.em + s.im;
    const double nu_m = 1.0 / 7.0, mu_m = 6.0 / 7.0;
    const long long births = d_binomial(r, nm, nu_m, lf);
    const long long s2 = d_binomial(r, s.sm - de_m, mu_m, lf);
    const long long e2 = d_binomial(r, s.em + de_m - di_m, mu_m, lf);
    const long long i2 = d_binomial(r, s.im + di_m, mu_m, lf);
    s.sm = (int)(s2 + births);
    s.em = (int)e2;
    s.im = (int)i2;
    const long long y = (long long)__ldg(C.table + s.t);
    lw = lw + d_binomial_logpmf(y, di_h, s.rho, lf);
    s.t = s.t + 1;
    s.pc = (s.t == C.n) ? kStop : 1;
    return true;
  }
};

// ============================================================================
// The PCFG of Fig. 3(a): blocks b0..b4, PC
// dispatch by a switch; checkpoints on the figure's regular arrows (b0 -> b1,
// b3 -> b2, b4 -> b_stop), jumps on the open ones (b1 -> b2, b2 -> b2 | b3 |
// b4).  Params p_loop, p3, w1, w2, w3, w4 (as log weights in C.p[6..9]).
// Plane P0 {pc, n (b3 visits), x (b2 self-loops), 0}.
// ============================================================================
struct Fig3 {
  static constexpr int kPlanes = 1;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kOneWave = false;  // uneven work (geometric loops): block scheduler balances
  struct State { int pc, n, x; };
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    const uint4 v = ldp(P, st, 0, i); s.pc = (int)v.x; s.n = (int)v.y; s.x = (int)v.z;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    stp(P, st, 0, i, make_uint4((uint32_t)s.pc, (uint32_t)s.n, (uint32_t)s.x, 0u));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag&) {
    switch (s.pc) {
      case 0:                                          // b0 -> b1 (checkpoint)
        s.n = 0; s.x = 0; s.pc = 1;
        return true;
      case 1:                                          // b1: weight(w1) -> b2
        lw = lw + C.p[6]; s.pc = 2;
        return false;
      case 2: {                                        // b2 -> b2 | b3 | b4
        const double u = d_uniform(r, 0.0, 1.0);
        if (u < C.p[0]) { s.x = s.x + 1; lw = lw + C.p[7]; s.pc = 2; }
        else if (u < C.p[0] + C.p[1]) s.pc = 3;
        else s.pc = 4;
        return false;
      }
      case 3:                                          // b3: weight(w3) -> b2 (checkpoint)
        s.n = s.n + 1; lw = lw + C.p[8]; s.pc = 2;
        return true;
      default:                                         // b4: weight(w4) -> b_stop (checkpoint)
        lw = lw + C.p[9]; s.pc = kStop;
        return true;
    }
  }
};

// ============================================================================
// STACKF (§R-24): the recursive function of Fig. 5 compiled to
// blocks 1-4 of Fig. 5(c) with a PSTATE byte stack and stack pointer
// (P:905-925).  Table y[D] (observation per recursion depth); params p0,
// p_rec, sigma, cap (stack bytes).  Planes: P0 {pc, sp (bytes), result f64};
// P1 .. P(cap/16) the stack, 16 bytes per plane (SoA like every plane): frame
// j (STACK_f, 48 bytes) = planes 1+3j {ra, retValLoc, p}, 2+3j {s1, s3},
// 3+3j {s4, 0}.  The blocks read and write frame fields where they touch
// them (the stack never passes through registers); resampling copies the
// header plane and only the planes below the stack pointer (R-22).
// ============================================================================
struct Stackf {
  static constexpr int kPlanes = 0;        // 1 + cap/16, set at create
  static constexpr int kMinBlocks = 4;
  static constexpr bool kOneWave = false;  // uneven work (recursion depths): block scheduler balances
  static constexpr int kFrame = 48, kRaStop = -1;
  struct State { int pc, sp; double result; uint4* P; unsigned long long st, i; };
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    const uint4 v = ldp(P, st, 0, i);
    s.pc = (int)v.x; s.sp = (int)v.y; s.result = hi_d(v);
    s.P = const_cast<uint4*>(P); s.st = st; s.i = i;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    const unsigned long long rb = __double_as_longlong(s.result);
    stp(P, st, 0, i, make_uint4((uint32_t)s.pc, (uint32_t)s.sp, (uint32_t)rb, (uint32_t)(rb >> 32)));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  // deferred gather: the ancestor's stack planes below sp move to this slot
  __device__ static void relocate(State& s, const uint4* src, uint4* dst, unsigned long long st,
                                  unsigned long long si, unsigned long long di) {
    for (int q = 0; 16 * q < s.sp; ++q)
      dst[(unsigned long long)(1 + q) * st + di] = __ldg(src + (unsigned long long)(1 + q) * st + si);
    s.P = dst;
    s.i = di;
  }
  // the stack plane holding byte offset `off`
  __device__ static uint4* plane(const State& s, int off) {
    return s.P + (unsigned long long)(1 + off / 16) * s.st + s.i;
  }
  __device__ static bool call(State& s, int ra, int rv, double p, int cap) {
    if (s.sp + kFrame > cap) return false;
    const unsigned long long pb = __double_as_longlong(p);
    *plane(s, s.sp) = make_uint4((uint32_t)ra, (uint32_t)rv, (uint32_t)pb, (uint32_t)(pb >> 32));
    *plane(s, s.sp + 16) = make_uint4(0u, 0u, 0u, 0u);
    *plane(s, s.sp + 32) = make_uint4(0u, 0u, 0u, 0u);
    s.sp = s.sp + kFrame;
    return true;
  }
  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag& dg) {
    const int cap = (int)C.p[3];
    const int top = s.sp - kFrame;                       // current frame (sf)
    switch (s.pc) {
      case 0:                                            // main: f(p0) into the result slot
        s.sp = 0; s.result = 0.0;
        if (!call(s, kRaStop, -1, C.p[0], cap)) { ++dg.overflow; lw = -INFINITY; s.pc = kStop; return true; }
        s.pc = 1;
        return false;
      case 1: {                                          // block 1: s1 = assume Gamma p p; resample
        const uint4 a = *plane(s, top);
        const double p = hi_d(a);
        const uint4 b = *plane(s, top + 16);
        const double s1 = d_gamma(r, p, 1.0 / p);
        const unsigned long long x = __double_as_longlong(s1);
        *plane(s, top + 16) = make_uint4((uint32_t)x, (uint32_t)(x >> 32), b.z, b.w);
        s.pc = 2;
        return true;
      }
      case 2: {                                          // block 2: observe, branch, call
        const uint4 b = *plane(s, top + 16);
        const double s1 = lo_d(b);
        const int d = s.sp / kFrame - 1;
        if (d < C.n) lw = lw + d_normal_logpdf(__ldg(C.table + d), s1, C.p[2]);
        if (s1 >= 1.0) {                                 // s4 = f(p_rec)
          if (!call(s, 3, top + 32, C.p[1], cap)) { ++dg.overflow; lw = -INFINITY; s.pc = kStop; return true; }
          s.pc = 1;
        } else {                                         // s3 = 8
          const unsigned long long x = __double_as_longlong(8.0);
          *plane(s, top + 16) = make_uint4(b.x, b.y, (uint32_t)x, (uint32_t)(x >> 32));
          s.pc = 4;
        }
        return false;
      }
      case 3: {                                          // block 3: s3 = s4 + s4
        const uint4 b = *plane(s, top + 16);
        const double s4 = lo_d(*plane(s, top + 32));
        const unsigned long long x = __double_as_longlong(s4 + s4);
        *plane(s, top + 16) = make_uint4(b.x, b.y, (uint32_t)x, (uint32_t)(x >> 32));
        s.pc = 4;
        return false;
      }
      default: {                                         // block 4: return s3 * s3
        const uint4 a = *plane(s, top);
        const double s3 = hi_d(*plane(s, top + 16));
        const double t = s3 * s3;
        const int ra = (int)a.x, rv = (int)a.y;
        if (rv < 0) {
          s.result = t;
        } else {                                         // 8 bytes at retValLoc of the caller's frame
          uint4 w = *plane(s, rv);
          const unsigned long long x = __double_as_longlong(t);
          if ((rv & 15) == 0) { w.x = (uint32_t)x; w.y = (uint32_t)(x >> 32); }
          else { w.z = (uint32_t)x; w.w = (uint32_t)(x >> 32); }
          *plane(s, rv) = w;
        }
        s.sp = s.sp - kFrame;
        s.pc = ra == kRaStop ? kStop : ra;
        return false;
      }
    }
  }
};

// ============================================================================
// Weighted geometric, Fig. 2(a).  Params p, w.  Plane P0 {pc, n, 0, 0}.
// ============================================================================
struct Geometric {
  static constexpr int kPlanes = 1;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kOneWave = true;   // grid: one resident wave, grid-stride (light, even work)
  struct State { int pc, n; };
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    const uint4 v = ldp(P, st, 0, i); s.pc = (int)v.x; s.n = (int)v.y;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    stp(P, st, 0, i, make_uint4((uint32_t)s.pc, (uint32_t)s.n, 0u, 0u));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag&) {
    const bool x = d_bernoulli(r, C.p[0]);
    s.n = s.n + 1;
    if (x) { lw = lw + log(C.p[1]); s.pc = 0; }
    else { s.pc = kStop; }
    return true;
  }
};

// ============================================================================
// SSM, Eq. (2) / Fig. 4.  Table y[T]; params m0, s0, drift, q, r.
// Plane P0 {x, pc, t}.
// ============================================================================
struct Ssm {
  static constexpr int kPlanes = 1;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kOneWave = true;   // grid: one resident wave, grid-stride (light, even work)
  struct State { double x; int pc, t; };
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    const uint4 v = ldp(P, st, 0, i); s.x = lo_d(v); s.pc = (int)v.z; s.t = (int)v.w;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    const unsigned long long xb = __double_as_longlong(s.x);
    stp(P, st, 0, i, make_uint4((uint32_t)xb, (uint32_t)(xb >> 32), (uint32_t)s.pc, (uint32_t)s.t));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  __device__ static bool step(State& s, double& lw, Rng& r, const ModelConst& C, Diag&) {
    if (s.pc == 0) {
      s.x = d_normal(r, C.p[0], C.p[1]);
      s.t = 0;
      s.pc = 1;
      return false;
    }
    s.x = d_normal(r, s.x + C.p[2], C.p[3]);
    lw = lw + d_normal_logpdf(__ldg(C.table + s.t), s.x, C.p[4]);
    s.t = s.t + 1;
    s.pc = (s.t == C.n) ? kStop : 1;
    return true;
  }
};

// ============================================================================
// Constant weight: weight(log w); checkpoint; K times.  Plane P0 {pc, k}.
// ============================================================================
struct Constw {
  static constexpr int kPlanes = 1;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kOneWave = true;   // grid: one resident wave, grid-stride (light, even work)
  struct State { int pc, k; };
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    const uint4 v = ldp(P, st, 0, i); s.pc = (int)v.x; s.k = (int)v.y;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    stp(P, st, 0, i, make_uint4((uint32_t)s.pc, (uint32_t)s.k, 0u, 0u));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  __device__ static bool step(State& s, double& lw, Rng&, const ModelConst& C, Diag&) {
    lw = lw + C.p[0];
    s.k = s.k + 1;
    s.pc = (s.k == (int)C.p[1]) ? kStop : 0;
    return true;
  }
};

}  // namespace smc
