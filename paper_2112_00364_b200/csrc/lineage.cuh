// lineage.cuh — cooperative propagation for the birth-death models under the
// lineage-keyed side-tree reading (SURVEY c.2 #18).
//
// The cost of CRBD / ClaDS2 propagation is the "goes undetected" simulation of
// hidden side trees ("recursive and stochastic tree constructions").
// Its size is heavy-tailed: in early epochs one particle's tree can hold 10^5
// nodes, and with one thread per particle that single thread bounds the whole
// epoch.  Under §R-18 every tree node draws from its own Philox block (counter
// = node id, particle, epoch, tag), so a tree's nodes can be evaluated in any
// order.  This kernel therefore runs, per CTA, a batch of kLRThreads (128)
// particles:
//   phase 1  each thread walks its particle's observed branch on the
//            particle's own stream (INIT, hidden event times, node bookkeeping)
//            and pushes one root task per hidden event onto the CTA's stack;
//   phase 2  rounds: every particle ("owner") with pending tasks gets W =
//            128 / (#owners with tasks last round) lanes (its top W tasks,
//            LIFO per owner, trimmed to the lanes left at its prefix offset);
//            lanes left over take tasks from a CTA overflow stack.
//            With many busy owners each explores depth-first (the order a
//            sequential DFS uses, so a supercritical tree is detected along
//            one path instead of 128); when few remain, their trees get the
//            idle lanes.  Tasks of particles already detected are pruned;
//   phase 3  each thread finishes its particle: -inf if any node was detected
//            (or the node cap was exceeded), else + ln 2 per hidden event.
// The grid is persistent (CTAs pull 256-particle batches from a counter), so a
// CTA stuck on a giant tree does not hold back the other batches, and the giant
// tree itself is explored 128 nodes at a time.
#pragma once
#include "kernels.cuh"

namespace smc {

#ifndef SMC_LR_THREADS
#define SMC_LR_THREADS 128
#endif
#ifndef SMC_LR_MINB
#define SMC_LR_MINB 8
#endif
#ifndef SMC_LR_OPT
#define SMC_LR_OPT 1
#endif
#ifndef SMC_CRBD_SPEC_CHILD
#define SMC_CRBD_SPEC_CHILD 0   // CRBD nodes: the daughters' id block before the event test
#endif
#ifndef SMC_CRBD_RECIP
#define SMC_CRBD_RECIP 1        // CRBD branch walk: -log(u) * (1/lambda) instead of a division
#endif
#ifndef SMC_CLADS2_MERGED
#define SMC_CLADS2_MERGED 1     // ClaDS2 branch walk: one loop body for hidden events and the node split
#endif
#ifndef SMC_CLADS2_LAZYPEEK
#define SMC_CLADS2_LAZYPEEK 0   // Philox blocks only as far as used: measured slower (181.0 -> 187.0 ms; the look-ahead ILP wins)
#endif
#ifndef SMC_CLADS2_SPEC_Z
#define SMC_CLADS2_SPEC_Z 0     // daughters' noise block before the event test: 1.3% faster in round 1, 0.7% slower on the final kernel (149.8 vs 150.8 ms)
#endif
constexpr int kLRThreads = SMC_LR_THREADS;     // threads per CTA = lanes per cooperative round
constexpr int kOPT = SMC_LR_OPT;                 // particles (owners) per thread
constexpr int kOwners = kLRThreads * kOPT;       // particles per batch
constexpr unsigned kSideNodeCap = 1u << 22;      // nodes per branch (all its side trees)
constexpr int kSeg = 512 / kOPT;                 // per-owner LIFO segment (tasks)
constexpr int kOverflowCap = 1 << 17;            // CTA-wide overflow LIFO (tasks)
constexpr unsigned kTasksPerCta = (unsigned)(kOwners * kSeg + kOverflowCap);
constexpr unsigned kTagNode = 3u, kTagChild = 4u, kTagZ = 5u;

struct TaskArrays {
  double2* sid;                 // (start age of the lineage, 64-bit node id as double bits)
  double* lam;                  // lineage rate (ClaDS2 only; may be null)
  unsigned short* owner;        // particle slot within the batch (overflow region only)
  unsigned cap;                 // tasks per CTA
};

struct LRArgs {
  PropArgs p;
  TaskArrays t;
  unsigned n_batches;
};

__device__ __forceinline__ uint4 side_block(unsigned long long seed, unsigned long long id,
                                            uint32_t n, uint32_t t, uint32_t tag) {
  return philox_site(make_uint4((uint32_t)id, (uint32_t)(id >> 32), n, (tag << 28) | t),
                       (uint32_t)seed, (uint32_t)(seed >> 32));
}
__device__ __forceinline__ unsigned long long root_id(unsigned k) {
  return (unsigned long long)k | (0xFFFFFFFFull << 32);
}

// Outcome of evaluating one side-tree node.
struct NodeOut {
  double s2, la, lb;             // daughters' start age and rates (rates: ClaDS2)
  unsigned long long ida, idb;   // daughters' ids
};
enum { NODE_LEAF = 0, NODE_DETECTED = 1, NODE_BIRTH = 2, NODE_GUARD = 3 };

// Per-owner constants kept in shared memory during phase 2.
struct OwnerCrbd { double inv_tot, pb; };
struct OwnerClads2 { double opeps, alpha, sigma, pb; };   // opeps = 1 + eps

// ---------------------------------------------------------------------------
// CRBD under §R-18
// ---------------------------------------------------------------------------
struct CrbdLR {
  static constexpr int kLRMinBlocks = SMC_LR_MINB;   // 64 registers at 128 threads
#ifndef SMC_LRW_MINB_CRBD
#define SMC_LRW_MINB_CRBD 5      // 5 CTAs/SM (up to 102 regs): measured 55.8 / 55.7 / 54.7 / 53.6 / 56.4 ms at 8 / 7 / 6 / 5 / 4
#endif
  static constexpr int kLRWMinBlocks = SMC_LRW_MINB_CRBD;   // warp-level kernel (lineage_warp.cuh)
  typedef Crbd::State State;
  typedef OwnerCrbd Owner;
  static constexpr int kPlanes = Crbd::kPlanes;
  static constexpr bool kHasLam = false;
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    Crbd::load(s, P, st, i);
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    Crbd::store(s, P, st, i);
  }
  __device__ static int pc(const State& s) { return s.pc; }

  // Phase 1: INIT (if pc = b0) and the main-stream part of BRANCH.  Calls
  // push(s, lam, k) for hidden event k.  Returns false if the particle is
  // already dead (never for CRBD).
  template <class Push>
  __device__ static bool main_part(State& s, double& lw, Rng& r, const ModelConst& C, Owner& ow,
                                   int& K, Push push) {
    const double rho = C.p[0];
    if (s.pc == 0) {
      s.lambda = C.p[1] >= 0.0 ? C.p[1] : d_gamma(r, 1.0, 1.0);
      s.mu = C.p[2] >= 0.0 ? C.p[2] : d_gamma(r, 1.0, 0.5);
      s.branch = 0;
      s.pc = 1;
    }
    const double* b = C.table + 3 * s.branch;
    const double tp = __ldg(b), tc = __ldg(b + 1);
    const bool internal = __ldg(b + 2) != 0.0;
    lw = lw + (-s.mu * (tp - tc));
    lw = lw + (internal ? log_pos(s.lambda) : log(rho));
    const double tot = s.lambda + s.mu;   // before any push: phase-2 lanes read them
    ow.inv_tot = 1.0 / tot;
    ow.pb = s.lambda / tot;
    double t = tp;
    K = 0;
    // hidden event times t -= Exp(lambda) until t <= t_c (the draws of d_exp,
    // two per iteration from one Philox block, their logs side by side; the
    // division by lambda as a multiplication by 1/lambda: ulp-level
    // differences, like the CUDA/glibc log differences)
#if SMC_CRBD_RECIP
    const double il = 1.0 / s.lambda;
#endif
    for (;;) {
      double u[3];
      r.peek2(u);
#if SMC_CRBD_RECIP
      const double t1 = t - (-log_u(u[0]) * il);
      const double e1 = -log_u(u[1]) * il;
#else
      const double t1 = t - (-log_u(u[0]) / s.lambda);
      const double e1 = -log_u(u[1]) / s.lambda;
#endif
      if (t1 <= tc) { r.consume(1, u); break; }
      push(t1, 0.0, (unsigned)K);
      ++K;
      const double t2 = t1 - e1;
      r.consume(2, u);
      if (t2 <= tc) break;
      push(t2, 0.0, (unsigned)K);
      ++K;
      t = t2;
    }
    s.branch = s.branch + 1;
    s.pc = (s.branch == C.n) ? kStop : 1;
    return true;
  }

  // Phase 2: one node (lineage from its birth at age s to its next event).
  __device__ static int node(double s, double, unsigned long long id, const Owner& ow, uint32_t n,
                             uint32_t t, unsigned long long seed, double rho, NodeOut& out) {
    const uint4 B = side_block(seed, id, n, t, kTagNode);
#if SMC_CRBD_SPEC_CHILD
    const uint4 Cb = side_block(seed, id, n, t, kTagChild);    // speculative: independent of B
#endif
    const double u0 = hq(B.x, B.y), u1 = hq(B.z, B.w);
    const double d = -log_u(u0) * ow.inv_tot;   // Exp(lambda + mu)
    if (d > s) return u1 < rho ? NODE_DETECTED : NODE_LEAF;
    if (!(u1 < ow.pb)) return NODE_LEAF;                       // death
#if !SMC_CRBD_SPEC_CHILD
    const uint4 Cb = side_block(seed, id, n, t, kTagChild);
#endif
    out.s2 = s - d;
    out.la = out.lb = 0.0;
    out.ida = ((unsigned long long)Cb.y << 32) | Cb.x;
    out.idb = ((unsigned long long)Cb.w << 32) | Cb.z;
    return NODE_BIRTH;
  }
};

// ---------------------------------------------------------------------------
// ClaDS2 under §R-18 (with the §R-14b rate guard)
// ---------------------------------------------------------------------------
// ClaDS2 transcendental chains, optionally out of line (SMC_CLADS2_MATH_OOL=1,
// value arguments only: nothing is forced to local memory); same formulas.
#ifndef SMC_CLADS2_MATH_OOL
#define SMC_CLADS2_MATH_OOL 0
#endif
#if SMC_CLADS2_MATH_OOL
#define SMC_CLADS2_FN __device__ __noinline__
#else
#define SMC_CLADS2_FN __device__ __forceinline__
#endif
SMC_CLADS2_FN double clads2_bm(double u1, double u2) {            // N(0,1) (R-3, cos branch)
  return 0.0 + 1.0 * (sqrt(-2.0 * log_u(u1)) * cos2pi_u(u2));
}
SMC_CLADS2_FN double2 clads2_bm_pair(double u1, double u2) {      // Box-Muller pair (R-18)
  const double rad = sqrt(-2.0 * log_u(u1));
#if SMC_FAST_TRIG
  const double2 sc = sincos2pi_u(u2);
  return make_double2(rad * sc.y, rad * sc.x);
#else
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  return make_double2(rad * cs, rad * sn);
#endif
}
SMC_CLADS2_FN double clads2_rate(double alpha, double lam, double sigma, double z) {
  return alpha * lam * exp_t(sigma * z);
}

struct Clads2LR {
#ifndef SMC_LR_MINB_CLADS2
#define SMC_LR_MINB_CLADS2 4
#endif
  static constexpr int kLRMinBlocks = SMC_LR_MINB_CLADS2;   // larger state: avoid spills
#ifndef SMC_LRW_MINB_CLADS2
#define SMC_LRW_MINB_CLADS2 4
#endif
  static constexpr int kLRWMinBlocks = SMC_LRW_MINB_CLADS2;
  // Lean state: the pending-rate stack (planes 2..4, R-22) stays in global
  // memory; a push writes its 8-byte entry, a pop reads one, and the stack
  // never occupies registers (12 registers and 3 plane loads/stores per
  // particle-step less than Clads2::State; same planes, same values).
  struct State { double sigma, alpha, eps, lam; int pc, branch, sp; uint4* P; unsigned long long st, i; };
  typedef OwnerClads2 Owner;
  static constexpr int kPlanes = Clads2::kPlanes;
  static constexpr bool kHasLam = true;
  __device__ static void load(State& s, const uint4* P, unsigned long long st, unsigned long long i) {
    uint4 v = ldp(P, st, 5, i); s.pc = (int)v.x; s.branch = (int)v.y; s.sp = (int)v.z;
    v = ldp(P, st, 0, i); s.sigma = lo_d(v); s.alpha = hi_d(v);
    v = ldp(P, st, 1, i); s.eps = lo_d(v); s.lam = hi_d(v);
    s.P = const_cast<uint4*>(P); s.st = st; s.i = i;
  }
  __device__ static void store(const State& s, uint4* P, unsigned long long st, unsigned long long i) {
    stp(P, st, 0, i, pack_dd(s.sigma, s.alpha));
    stp(P, st, 1, i, pack_dd(s.eps, s.lam));
    stp(P, st, 5, i, make_uint4((uint32_t)s.pc, (uint32_t)s.branch, (uint32_t)s.sp, 0u));
  }
  __device__ static int pc(const State& s) { return s.pc; }
  // deferred gather: the ancestor's pending-rate planes below sp move to this slot
  __device__ static void relocate(State& s, const uint4* src, uint4* dst, unsigned long long st,
                                  unsigned long long si, unsigned long long di) {
    for (int k = 0; 2 * k < s.sp; ++k)
      dst[(unsigned long long)(2 + k) * st + di] = __ldg(src + (unsigned long long)(2 + k) * st + si);
    s.P = dst;
    s.i = di;
  }
  __device__ static double* pend_slot(const State& s, int k) {
    return reinterpret_cast<double*>(s.P + (unsigned long long)(2 + (k >> 1)) * s.st + s.i) + (k & 1);
  }
  __device__ static void push_pend(State& s, double v) { *pend_slot(s, s.sp) = v; s.sp = s.sp + 1; }
  __device__ static double pop_pend(State& s) { s.sp = s.sp - 1; return *pend_slot(s, s.sp); }
  __device__ static double daughter(const State& s, double lam, double z) {
    return clads2_rate(s.alpha, lam, s.sigma, z);
  }

  template <class Push>
  __device__ static bool main_part(State& s, double& lw, Rng& r, const ModelConst& C, Owner& ow,
                                   int& K, Push push) {
    const double rho = C.p[0];
    K = 0;
    if (s.pc == 0) {                          // INIT + root split: the draws of Clads2::step (§R-14)
      const double lam0 = C.p[1] >= 0.0 ? C.p[1] : d_gamma(r, 1.0, 1.0);
      s.sigma = C.p[2] >= 0.0 ? C.p[2] : sqrt(1.0 / d_gamma(r, 1.0, 1.0 / 0.2));
      s.alpha = C.p[3] >= 0.0 ? C.p[3] : exp(d_normal(r, 0.0, s.sigma));
      s.eps = C.p[4] >= 0.0 ? C.p[4] : d_uniform(r, 0.0, 1.0);
      const double zl = d_normal(r, 0.0, 1.0);
      const double zr = d_normal(r, 0.0, 1.0);
      const double rl = daughter(s, lam0, zl), rr = daughter(s, lam0, zr);
      const bool fl = C.p[5] != 0.0;
      s.sp = 0;
      push_pend(s, fl ? rr : rl);
      s.lam = fl ? rl : rr;
      s.branch = 0;
      s.pc = 1;
    }
    ow.opeps = 1.0 + s.eps; ow.alpha = s.alpha; ow.sigma = s.sigma;
    ow.pb = 1.0 / (1.0 + s.eps);
    const double* b = C.table + 4 * s.branch;
    const double tp = __ldg(b), tc = __ldg(b + 1);
    const bool internal = __ldg(b + 2) != 0.0;
    const bool first_left = __ldg(b + 3) != 0.0;
#if SMC_CLADS2_MERGED
    // One loop body for the hidden events of the branch and the split at its
    // end (internal child): both turn four uniforms into two normals and two
    // daughter rates of the current rate, so the Box-Muller and exp code is
    // emitted once (half the instruction footprint of this phase, and lanes
    // at a split run it together with lanes at an event).  Same draws, same
    // formulas and the same order of checks as the two-loop form below.
    bool killed = Clads2::bad_rate(s.lam);
    double t = tp;
    bool split = false;
    while (!killed) {
      double u[6];
#if SMC_CLADS2_LAZYPEEK
      // the Philox blocks of the next uniforms only as far as they are used:
      // block A always (u0, the event time); B for the normals of an event or
      // a split; C only for an event that starts on a fresh block (5 uniforms)
      const uint4 A = philox4x32_10(make_uint4(r.blk, r.t, r.n, 0u), r.k0, r.k1);
      {
        const double a0 = hq(A.x, A.y), a1 = hq(A.z, A.w);
        u[0] = r.has_spare ? r.spare : a0;
        u[1] = r.has_spare ? a0 : a1;
        u[2] = a1;
      }
      double dt = 0.0;
      if (!split) {
        dt = -log_u(u[0]) / s.lam;
        if (t - dt <= tc) {
          r.consume(1, u);
          lw = lw + (-s.eps * s.lam * (t - tc));
          if (!internal) break;
          lw = lw + log_pos(s.lam);
          split = true;
          continue;
        }
      }
      {
        const uint4 B = philox4x32_10(make_uint4(r.blk + 1u, r.t, r.n, 0u), r.k0, r.k1);
        const double b0 = hq(B.x, B.y), b1 = hq(B.z, B.w);
        if (r.has_spare) {
          u[3] = b0; u[4] = b1; u[5] = 0.0;
        } else {
          u[2] = b0; u[3] = b1; u[4] = 0.0; u[5] = 0.0;
          if (!split) {
            const uint4 Cc = philox4x32_10(make_uint4(r.blk + 2u, r.t, r.n, 0u), r.k0, r.k1);
            u[4] = hq(Cc.x, Cc.y); u[5] = hq(Cc.z, Cc.w);
          }
        }
      }
      if (!split) {
        r.consume(5, u);
        lw = lw + (-s.eps * s.lam * dt);
        t = t - dt;
      } else {
        r.consume(4, u);                     // z_l, z_r: the four uniforms of two d_normal calls
      }
#else
      r.peek6(u);
      if (!split) {
        const double dt = -log_u(u[0]) / s.lam;
        if (t - dt <= tc) {
          r.consume(1, u);
          lw = lw + (-s.eps * s.lam * (t - tc));
          if (!internal) break;
          lw = lw + log_pos(s.lam);
          split = true;
          continue;
        }
        r.consume(5, u);
        lw = lw + (-s.eps * s.lam * dt);
        t = t - dt;
      } else {
        r.consume(4, u);                     // z_l, z_r: the four uniforms of two d_normal calls
      }
#endif
      const double a1 = split ? u[0] : u[1], a2 = split ? u[1] : u[2];   // (selects: no local array)
      const double b1 = split ? u[2] : u[3], b2 = split ? u[3] : u[4];
      const double z1 = clads2_bm(a1, a2);
      const double z2 = clads2_bm(b1, b2);
      const double r1 = daughter(s, s.lam, z1), r2 = daughter(s, s.lam, z2);
      if (split) {
        if (Clads2::bad_rate(r1) || Clads2::bad_rate(r2)) {
          killed = true;
        } else {
          push_pend(s, first_left ? r2 : r1);
          s.lam = first_left ? r1 : r2;
        }
        break;
      }
      if (Clads2::bad_rate(r1)) { killed = true; break; }   // the side lineage (z_side)
      push(t, r1, (unsigned)K);
      ++K;
      s.lam = r2;                                           // the continuing lineage (z_cont)
      if (Clads2::bad_rate(s.lam)) { killed = true; break; }
    }
    if (!killed && !internal) {
      lw = lw + log(rho);
      if (s.branch + 1 < C.n) s.lam = pop_pend(s);
    }
#else
    bool killed = Clads2::bad_rate(s.lam);
    double t = tp;
    while (!killed) {
      // one hidden event = Exp(lam_cur), then z_side, z_cont ~ N(0, 1): the
      // same five uniforms and formulas as d_exp + 2 d_normal (R-3, R-14),
      // their Philox blocks and the two Box-Muller chains computed side by side
      double u[6];
      r.peek6(u);
      const double dt = -log_u(u[0]) / s.lam;
      if (t - dt <= tc) {
        r.consume(1, u);
        lw = lw + (-s.eps * s.lam * (t - tc));
        break;
      }
      r.consume(5, u);
      lw = lw + (-s.eps * s.lam * dt);
      t = t - dt;
      const double zs = clads2_bm(u[1], u[2]);
      const double zc = clads2_bm(u[3], u[4]);
      const double ls = daughter(s, s.lam, zs);
      if (Clads2::bad_rate(ls)) { killed = true; break; }
      push(t, ls, (unsigned)K);
      ++K;
      s.lam = daughter(s, s.lam, zc);
      if (Clads2::bad_rate(s.lam)) { killed = true; break; }
    }
    if (!killed && internal) {
      lw = lw + log_pos(s.lam);
      double u[6];                           // z_l, z_r: the four uniforms of two d_normal calls
      r.peek6(u);
      r.consume(4, u);
      const double zl = clads2_bm(u[0], u[1]);
      const double zr = clads2_bm(u[2], u[3]);
      const double rl = daughter(s, s.lam, zl), rr = daughter(s, s.lam, zr);
      if (Clads2::bad_rate(rl) || Clads2::bad_rate(rr)) {
        killed = true;
      } else {
        push_pend(s, first_left ? rr : rl);
        s.lam = first_left ? rl : rr;
      }
    } else if (!killed) {
      lw = lw + log(rho);
      if (s.branch + 1 < C.n) s.lam = pop_pend(s);
    }
#endif
    if (killed) lw = -INFINITY;
    s.branch = s.branch + 1;
    s.pc = (s.branch == C.n) ? kStop : 1;
    return !killed;
  }

  __device__ static int node(double s, double lam, unsigned long long id, const Owner& ow, uint32_t n,
                             uint32_t t, unsigned long long seed, double rho, NodeOut& out) {
    const uint4 B = side_block(seed, id, n, t, kTagNode);
#if SMC_CLADS2_SPEC_Z
    const uint4 Z = side_block(seed, id, n, t, kTagZ);     // speculative: independent of B
#endif
    const double u0 = hq(B.x, B.y), u1 = hq(B.z, B.w);
    // d = -log(u0) / (lam (1 + eps)) ~ Exp(lam (1 + eps)); the test d > s is
    // taken as -log(u0) > s lam (1 + eps) (no division; the same decision up
    // to rounding, like the CUDA/glibc ulp differences), d itself only for a birth
    const double rate = lam * ow.opeps;
    const double nl = -log_u(u0);
    if (nl > s * rate) return u1 < rho ? NODE_DETECTED : NODE_LEAF;
    if (!(u1 < ow.pb)) return NODE_LEAF;
#if !SMC_CLADS2_SPEC_Z
    const uint4 Z = side_block(seed, id, n, t, kTagZ);
#endif
    const double2 zz = clads2_bm_pair(hq(Z.x, Z.y), hq(Z.z, Z.w));   // angle 2 pi u
    out.la = clads2_rate(ow.alpha, lam, ow.sigma, zz.x);
    out.lb = clads2_rate(ow.alpha, lam, ow.sigma, zz.y);
    if (Clads2::bad_rate(out.la) || Clads2::bad_rate(out.lb)) return NODE_GUARD;   // rate guard
    const uint4 Cb = side_block(seed, id, n, t, kTagChild);
    out.s2 = s - nl / rate;
    out.ida = ((unsigned long long)Cb.y << 32) | Cb.x;
    out.idb = ((unsigned long long)Cb.w << 32) | Cb.z;
    return NODE_BIRTH;
  }
};

// ---------------------------------------------------------------------------
template <class M>
__global__ void __launch_bounds__(kLRThreads, M::kLRMinBlocks) propagate_lr_kernel(LRArgs a, ModelConst C) {
  __shared__ int s_cnt[kOwners];             // tasks in owner o's segment
  __shared__ int s_sel[kLRThreads];          // this round: lane -> task slot (owner-written)
  __shared__ int s_ovtop;                     // overflow stack top
  // 16-byte aligned: its vectorised read after barrier (A) must not cover the
  // neighbouring s_ovtop, which thread 0 writes after (A) (racecheck)
  __shared__ __align__(16) int s_wsum[kLRThreads / 32];
  __shared__ unsigned s_batch;
  __shared__ int s_dead[kOwners];             // 0 alive, 1 detected, 2 node cap, 3 rate guard
  __shared__ unsigned s_nodes[kOwners];
  __shared__ typename M::Owner s_own[kOwners];
  __shared__ int s_taskcap;
  __shared__ long long s_key[kLRThreads / 32];
  __shared__ unsigned long long s_acc[3][kLRThreads / 32];
  const PropArgs& p = a.p;
  if (*(volatile unsigned*)&p.ctrl->done) return;
  const unsigned epoch = p.ctrl->epoch;
  const unsigned long long seed = p.ctrl->seed;
  const bool carry = p.ctrl->carry != 0;
  const double rho = C.p[0];
  const int tid = threadIdx.x;
  const unsigned long long tbase = (unsigned long long)blockIdx.x * kTasksPerCta;
  double2* T_sid = a.t.sid + tbase;
  double* T_lam = M::kHasLam ? a.t.lam + tbase : nullptr;
  unsigned short* T_own = a.t.owner + tbase;
  constexpr unsigned long long kSegSlots = (unsigned long long)kOwners * kSeg;
  if (tid == 0) s_taskcap = 0;
  // store a task at a CTA-local slot; segment slots imply their owner
  auto put = [&](unsigned long long slot, int o, double s0, double lam0, unsigned long long id) {
    T_sid[slot] = make_double2(s0, __longlong_as_double((long long)id));
    if (M::kHasLam) T_lam[slot] = lam0;
    if (slot >= kSegSlots) T_own[slot] = (unsigned short)o;
  };
  auto overflow_slot = [&]() -> long long {
    const int q = atomicAdd(&s_ovtop, 1);
    if (q >= kOverflowCap) { s_taskcap = 1; return -1; }
    return (long long)kSegSlots + q;
  };
  // push one task for owner o: its segment, else the overflow stack
  auto push_task = [&](int o, double s0, double lam0, unsigned long long id) {
    const int pos = atomicAdd(&s_cnt[o], 1);
    const long long slot = pos < kSeg ? (long long)o * kSeg + pos : overflow_slot();
    if (slot >= 0) put((unsigned long long)slot, o, s0, lam0, id);
  };
  // push both daughters of a birth with one reservation (first daughter on top)
  auto push_pair = [&](int o, double s0, double lb, unsigned long long idb, double la,
                       unsigned long long ida) {
    const int pos = atomicAdd(&s_cnt[o], 2);
    const long long s1 = pos < kSeg ? (long long)o * kSeg + pos : overflow_slot();
    const long long s2 = pos + 1 < kSeg ? (long long)o * kSeg + pos + 1 : overflow_slot();
    if (s1 >= 0) put((unsigned long long)s1, o, s0, lb, idb);
    if (s2 >= 0) put((unsigned long long)s2, o, s0, la, ida);
  };

  long long key = LLONG_MIN;
  unsigned long long n_end = 0, n_start = 0, drw = 0, ovf = 0, roots = 0, guard = 0;
  bool bad = false;
  unsigned max_rounds = 0, max_nodes = 0;
  const int warp_id = tid >> 5, lane_id = tid & 31;

  for (;;) {
    if (tid == 0) {
      s_batch = atomicAdd(&p.ctrl->batch, 1u);
      s_ovtop = 0;
    }
#pragma unroll
    for (int q = 0; q < kOPT; ++q) {
      s_cnt[q * kLRThreads + tid] = 0;
      s_dead[q * kLRThreads + tid] = 0;
      s_nodes[q * kLRThreads + tid] = 0;
    }
    __syncthreads();
    const unsigned batch = s_batch;
    if (batch >= a.n_batches) break;
    const unsigned long long bbase = (unsigned long long)batch * kOwners;
    // ---------------- phase 1: each particle's own stream; thread tid runs
    // owners q*kLRThreads + tid (coalesced), stores the state at once and
    // keeps lw, K and flags for phase 3
    double lw[kOPT];
    int K[kOPT];
    bool act[kOPT], alive_end[kOPT];
#pragma unroll
    for (int q = 0; q < kOPT; ++q) {
      const int o = q * kLRThreads + tid;
      const unsigned long long i = bbase + o;
      const bool valid = i < p.n_local;
      lw[q] = (valid && carry) ? p.lw[i] : 0.0;   // R-19 carried weights
      K[q] = 0;
      act[q] = false;
      alive_end[q] = false;
      if (valid) {
        typename M::State st;
        M::load(st, p.planes, p.n_local, i);
        if (M::pc(st) != kStop) {
          act[q] = true;
          ++n_start;
          Rng r(seed, (uint32_t)(p.shard_base + i), epoch);
          int k = 0;
          auto push = [&](double s0, double lam0, unsigned kk) { push_task(o, s0, lam0, root_id(kk)); };
          if (!M::main_part(st, lw[q], r, C, s_own[o], k, push)) s_dead[o] = 3;   // rate guard
          K[q] = k;
          roots += (unsigned long long)k;
          drw += 2ull * r.blk - (r.has_spare ? 1ull : 0ull);
          M::store(st, p.planes, p.n_local, i);
        }
        alive_end[q] = M::pc(st) != kStop;
      }
    }
    __syncthreads();
    // ---------------- phase 2: cooperative side-tree evaluation.  Thread tid
    // manages owners kOPT*tid + q.  Four barriers per round: (A) scan, (B) lane
    // map written, (C) task records read, (D) pushes done.  The fair share W
    // uses the previous round's active-owner count; each owner trims its share
    // to the lanes left at its prefix offset, so at most kLRThreads tasks are
    // taken.  Task count and active-owner count travel packed in one scan.
    int n_act = 0;
    {
      int c0 = 0;
#pragma unroll
      for (int q = 0; q < kOPT; ++q) {
        const int o = kOPT * tid + q;
        const int c = s_cnt[o];
        if (c > kSeg) s_cnt[o] = kSeg;          // pushes beyond the segment went to overflow
        c0 += c > 0;
      }
      __syncwarp();   // bar.red needs a converged warp (synccheck)
      n_act = __syncthreads_count(c0 > 0) * kOPT;   // estimate for the first round's share
    }
    unsigned rounds = 0;
    for (;;) {
      int c[kOPT], m[kOPT];
      // lanes per owner: a heuristic (no result depends on it)
      const int W = max(1, __float2int_rz((float)kLRThreads * __frcp_rn((float)max(1, n_act)) + 1e-3f));
      int msum = 0, nact = 0;
#pragma unroll
      for (int q = 0; q < kOPT; ++q) {
        c[q] = s_cnt[kOPT * tid + q];
        m[q] = min(c[q], W);
        msum += m[q];
        nact += c[q] > 0;
      }
      int incl = msum | (nact << 16);          // msum <= kOPT * kLRThreads < 2^16
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane_id >= d) incl += o;
      }
      if (lane_id == 31) s_wsum[warp_id] = incl;
      const int ov = min(*(volatile int*)&s_ovtop, kOverflowCap);
      __syncwarp();
      __syncthreads();                                                     // (A)
      int woff = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kLRThreads / 32; ++w) {
        const int v = s_wsum[w];
        woff += w < warp_id ? (v & 0xFFFF) : 0;
        tot += v;
      }
      n_act = tot >> 16;
      if (n_act == 0 && ov == 0) break;
      const int T = min(tot & 0xFFFF, kLRThreads);
      {
        // owners write the slots of their top m tasks to lanes [off, off+m)
        int off = woff + (incl & 0xFFFF) - msum;
#pragma unroll
        for (int q = 0; q < kOPT; ++q) {
          const int o = kOPT * tid + q;
          const int me = max(0, min(m[q], kLRThreads - off));
          const int seg = o * kSeg;
          for (int j = 0; j < me; ++j) s_sel[off + j] = seg + (c[q] - 1 - j);
          s_cnt[o] = c[q] - me;
          // side-tree node count of the branch: every popped task of a live
          // owner is evaluated this round (exact for the node-cap rule)
          if (me && s_dead[o] == 0) {
            s_nodes[o] += (unsigned)me;
            if (s_nodes[o] > kSideNodeCap) atomicCAS(&s_dead[o], 0, 2);
          }
          off += m[q];
        }
        if (tid == 0) s_ovtop = ov - min(ov, kLRThreads - T);
      }
      __syncthreads();                                                     // (B)
      // lane -> task
      bool have = false;
      double ts = 0.0, tl = 0.0;
      unsigned long long tidv = 0;
      int o = 0;
      unsigned long long slot = 0;
      if (tid < T) {
        slot = (unsigned long long)s_sel[tid];
        have = true;
      } else if (tid - T < ov) {
        slot = kSegSlots + (ov - 1 - (tid - T));
        have = true;
      }
      if (have) {
        const double2 rec = T_sid[slot];
        ts = rec.x;
        tidv = (unsigned long long)__double_as_longlong(rec.y);
        if (M::kHasLam) tl = T_lam[slot];
        o = slot < kSegSlots ? (int)(slot / kSeg) : (int)T_own[slot];
      }
      __syncthreads();                                                     // (C)
      // s_dead is a sticky flag (0 -> nonzero, never back): written and read
      // with shared-memory atomics; a stale 0 only costs one pruned-late node
      if (have && atomicAdd(&s_dead[o], 0) == 0) {
        const uint32_t n_owner = (uint32_t)(p.shard_base + bbase + o);
        drw += 2;
        NodeOut out;
        const int res = M::node(ts, tl, tidv, s_own[o], n_owner, epoch, seed, rho, out);
        if (M::kHasLam && (res == NODE_BIRTH || res == NODE_GUARD)) drw += 2;   // daughters' noise block
        if (res == NODE_DETECTED || res == NODE_GUARD) {
          atomicCAS(&s_dead[o], 0, res == NODE_GUARD ? 3 : 1);
        } else if (res == NODE_BIRTH) {
          push_pair(o, out.s2, out.lb, out.idb, out.la, out.ida);   // first daughter on top
        }
      }
      __syncthreads();                                                     // (D)
#pragma unroll
      for (int q = 0; q < kOPT; ++q)
        if (s_cnt[kOPT * tid + q] > kSeg) s_cnt[kOPT * tid + q] = kSeg;
      ++rounds;
    }
    max_rounds = rounds > max_rounds ? rounds : max_rounds;
    // ---------------- phase 3: finish the particles (phase-1 mapping)
#pragma unroll
    for (int q = 0; q < kOPT; ++q) {
      const int o = q * kLRThreads + tid;
      const unsigned long long i = bbase + o;
      max_nodes = s_nodes[o] > max_nodes ? s_nodes[o] : max_nodes;
      if (i < p.n_local) {
        double w = lw[q];
        if (act[q]) {
          const int dead = s_dead[o];
          if (dead) {
            w = -INFINITY;
            if (dead == 3) ++guard;
            if (dead == 2) {
              ++ovf;
              atomicMin(&p.ctrl->first_err, (unsigned long long)(p.shard_base + i));
            }
          } else {
            for (int k = 0; k < K[q]; ++k) w = w + kLn2;
          }
        }
        p.lw[i] = w;
        if (alive_end[q]) ++n_end;
        const bool b = isnan(w) || w == INFINITY;
        bad |= b;
        const long long kk = order_key(w);
        key = kk > key ? kk : key;
      }
    }
    __syncthreads();
  }
  // ---------------- epilogue: one set of atomics per CTA
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, key, d);
    key = o > key ? o : key;
    n_end += __shfl_xor_sync(0xffffffffu, n_end, d);
    n_start += __shfl_xor_sync(0xffffffffu, n_start, d);
    drw += __shfl_xor_sync(0xffffffffu, drw, d);
    ovf += __shfl_xor_sync(0xffffffffu, ovf, d);
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
    s_key[warp] = key;
    s_acc[0][warp] = n_end;
    s_acc[1][warp] = n_start;
    s_acc[2][warp] = drw;
  }
  __syncwarp();   // bar.red needs a converged warp (synccheck)
  const int any_bad = __syncthreads_or(bad);
  __syncwarp();   // bar.red needs a converged warp (synccheck)
  const int any_ovf = __syncthreads_or(ovf != 0);
  unsigned long long ovf_sum = ovf;
  (void)ovf_sum;
  if (tid == 0) {
    long long k = s_key[0];
    unsigned long long e = 0, st = 0, dr = 0;
    for (int w = 0; w < kLRThreads / 32; ++w) {
      k = s_key[w] > k ? s_key[w] : k;
      e += s_acc[0][w];
      st += s_acc[1][w];
      dr += s_acc[2][w];
    }
    RecA* rec = p.recA + (epoch & 1) * p.world + p.rank;
    atomicMax(&rec->key, k);
    if (e) atomicAdd(&rec->alive, (unsigned)e);
    if (any_bad) atomicOr(&rec->flags, 1u);
    if (s_taskcap) atomicOr(&rec->flags, 2u);
    if (st) atomicAdd(&p.ctrl->alive_steps, st);
    if (dr) atomicAdd(&p.ctrl->draws, dr);
  }
  if (any_ovf && lane == 0 && ovf) atomicAdd(&p.ctrl->overflow, ovf);
  if (guard) atomicAdd(&p.ctrl->guard_kills, guard);   // rare (ClaDS2 only)
  // diagnostics (one atomic per warp)
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    roots += __shfl_xor_sync(0xffffffffu, roots, d);
    max_nodes = max(max_nodes, __shfl_xor_sync(0xffffffffu, max_nodes, d));
  }
  if (lane == 0) {
    if (roots) atomicAdd(&p.ctrl->side_roots, roots);
    atomicMax(&p.ctrl->max_side_nodes, max_nodes);
    if (tid == 0) atomicMax(&p.ctrl->max_rounds, max_rounds);
  }
}

}  // namespace smc
