// =============================================================================
// smc_oracle.cpp — plain, sequential, fp64 CPU oracle for SMC over PCFGs.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares NO code with the CUDA path (paper_2112_00364_b200/csrc, include/):
// its own Philox, its own samplers, its own models, its own resampler.
//
// Citation keys: P:n = /root/reference/PAPER.md line n (LaTeX source of
// arXiv 2112.00364); S:n = SPEC.md line n; DESIGN.md §R-x = a documented
// reading where the paper is silent.
//
// Pins (tests/test_oracle_*.py, -m "not gpu"):
//   philox           Random123 known-answer vectors                (pinned)
//   uniform          closed form of the hq conversion; open interval (pinned)
//   samplers         moments within 5 SE; Gamma(1,θ) ≡ Exp; binomial
//                    chi-square against the exact pmf              (pinned)
//   resample         exact big-integer brute force (Python ints),
//                    systematic invariants floor/ceil(N w)         (pinned)
//   smc loop / LSE   constant-weight log Z = K ln 3 exactly; weighted
//                    geometric E[Z] = 2; SSM vs Kalman (pinned)
//   crbd             E[Z] vs the closed-form CRBD likelihood; prior-
//                    integrated Z by quadrature                    (pinned)
//   clads2           sigma=0, alpha=1 reduces to CRBD closed form; sigma=0,
//                    alpha!=1 vs the rate-level ladder of backward ODEs;
//                    sigma>0 vs a forward simulation of a cherry; prior
//                    block by KS tests                             (pinned)
//   seir             tiny-population exact forward algorithm, fixed
//                    parameters and with priors (QMC prior integral);
//                    prior block by KS tests                       (pinned)
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared (see build()).
// =============================================================================
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <string>
#include <algorithm>

namespace {

typedef unsigned __int128 u128;

const double LN2 = 0.6931471805599453094172321214581766;
const double TWO_PI = 6.283185307179586476925286766559006;
const double HALF_LOG_2PI = 0.9189385332046727417803297364056176;

// ----------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11 / Random123).  The paper only says each
// particle needs a unique seed; counter-based Philox keyed
// by (seed, particle, draw) is the north-star choice.
// ----------------------------------------------------------------------------
struct Block { uint32_t v[4]; };

Block philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                    uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    uint64_t p0 = (uint64_t)M0 * c0;
    uint64_t p1 = (uint64_t)M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  Block b; b.v[0] = c0; b.v[1] = c1; b.v[2] = c2; b.v[3] = c3;
  return b;
}

// hq conversion of two 32-bit words to a double in (0,1):
// z = x ^ (y << 21) (53 bits);  u = z * 2^-53 + 2^-54.
uint64_t hq_bits(uint32_t x, uint32_t y) {
  return (uint64_t)x ^ ((uint64_t)y << 21);
}
double hq(uint32_t x, uint32_t y) {
  uint64_t z = hq_bits(x, y);
  double a = (double)z * 0x1p-53;
  return a + 0x1p-54;
}

enum { TAG_PARTICLE = 0, TAG_RESAMPLE = 1, TAG_DATA = 2 };

// One particle's uniform stream within one epoch: draw d comes from Philox
// block b = d/2 (counter (b, t, n, tag), key (seed_lo, seed_hi)), half d%2.
struct Stream {
  uint32_t k0, k1, t, n, tag;
  uint64_t d;
  uint64_t* counter;   // optional instrumentation: total draws
  double uniform() {
    Block b = philox4x32_10((uint32_t)(d >> 1), t, n, tag, k0, k1);
    double u = (d & 1) ? hq(b.v[2], b.v[3]) : hq(b.v[0], b.v[1]);
    ++d;
    if (counter) ++*counter;
    return u;
  }
};

Stream make_stream(uint64_t seed, uint32_t n, uint32_t t, uint32_t tag, uint64_t* counter) {
  Stream s;
  s.k0 = (uint32_t)seed; s.k1 = (uint32_t)(seed >> 32);
  s.t = t; s.n = n; s.tag = tag; s.d = 0; s.counter = counter;
  return s;
}

// ----------------------------------------------------------------------------
// Samplers (draw counts fixed per the table there).  The paper
// names the distributions in its examples
// but not the algorithms.
// ----------------------------------------------------------------------------
double sample_exp(Stream& s, double rate) {            // 1 draw
  double u = s.uniform();
  return -std::log(u) / rate;
}
bool sample_bernoulli(Stream& s, double p) {           // 1 draw
  double u = s.uniform();
  return u < p;
}
double sample_uniform(Stream& s, double a, double b) { // 1 draw
  double u = s.uniform();
  return a + (b - a) * u;
}
double sample_normal(Stream& s, double mu, double sigma) {   // 2 draws
  double u1 = s.uniform();
  double u2 = s.uniform();
  double r = std::sqrt(-2.0 * std::log(u1));
  double c = std::cos(TWO_PI * u2);
  return mu + sigma * (r * c);
}
// Gamma(shape k, scale theta)  ((shape, scale)).
double sample_gamma(Stream& s, double k, double theta) {
  if (k == 1.0) {                                      // 1 draw
    double u = s.uniform();
    return -theta * std::log(u);
  }
  if (k < 1.0) {                                       // Gamma(k+1) draws, then 1
    double g = sample_gamma(s, k + 1.0, theta);
    double u = s.uniform();
    return g * std::pow(u, 1.0 / k);
  }
  // Marsaglia & Tsang (2000): 3 draws per attempt.
  double d = k - 1.0 / 3.0;
  double c = 1.0 / std::sqrt(9.0 * d);
  for (;;) {
    double x = sample_normal(s, 0.0, 1.0);
    double u = s.uniform();
    double v = 1.0 + c * x;
    if (v <= 0.0) continue;
    v = v * v * v;
    double lhs = std::log(u);
    double rhs = 0.5 * x * x + d - d * v + d * std::log(v);
    if (lhs < rhs) return d * v * theta;
  }
}
double sample_beta(Stream& s, double a, double b) {
  double x = sample_gamma(s, a, 1.0);
  double y = sample_gamma(s, b, 1.0);
  return x / (x + y);
}

// Binomial(n, p): symmetry for p > 1/2; inversion (BINV) for n p < 10,
// 1 draw; BTRS (Hormann 1993) otherwise, 2 draws per attempt.
int64_t binomial_inversion(Stream& s, int64_t n, double p) {
  double q = 1.0 - p;
  double sr = p / q;
  double a = (double)(n + 1) * sr;
  double r = std::exp((double)n * std::log1p(-p));
  double u = s.uniform();
  int64_t x = 0;
  while (x < n && u > r) {
    u = u - r;
    x = x + 1;
    r = r * (a / (double)x - sr);
  }
  return x;
}
int64_t binomial_btrs(Stream& s, int64_t n, double p) {
  double q = 1.0 - p;
  double nd = (double)n;
  double spq = std::sqrt(nd * p * q);
  double b = 1.15 + 2.53 * spq;
  double a = -0.0873 + 0.0248 * b + 0.01 * p;
  double c = nd * p + 0.5;
  double vr = 0.92 - 4.2 / b;
  double alpha = (2.83 + 5.1 / b) * spq;
  double lpq = std::log(p / q);
  double m = std::floor((nd + 1.0) * p);
  double h = std::lgamma(m + 1.0) + std::lgamma(nd - m + 1.0);
  for (;;) {
    double U = s.uniform() - 0.5;
    double V = s.uniform();
    double us = 0.5 - std::fabs(U);
    double kd = std::floor((2.0 * a / us + b) * U + c);
    if (kd < 0.0 || kd > nd) continue;
    if (us >= 0.07 && V <= vr) return (int64_t)kd;
    double lv = std::log(V * alpha / (a / (us * us) + b));
    double rhs = h - std::lgamma(kd + 1.0) - std::lgamma(nd - kd + 1.0) + (kd - m) * lpq;
    if (lv <= rhs) return (int64_t)kd;
  }
}
int64_t sample_binomial(Stream& s, int64_t n, double p) {
  if (p > 0.5) return n - sample_binomial(s, n, 1.0 - p);
  if ((double)n * p < 10.0) return binomial_inversion(s, n, p);
  return binomial_btrs(s, n, p);
}

// log pmf of Binomial(n, p) at k; zero-count terms contribute 0.
double binomial_logpmf(int64_t k, int64_t n, double p) {
  if (k < 0 || k > n) return -INFINITY;
  double r = std::lgamma((double)n + 1.0) - std::lgamma((double)k + 1.0)
           - std::lgamma((double)(n - k) + 1.0);
  if (k > 0) r = r + (double)k * std::log(p);
  if (n - k > 0) r = r + (double)(n - k) * std::log1p(-p);
  return r;
}
double normal_logpdf(double y, double mu, double sigma) {
  double z = (y - mu) / sigma;
  return -0.5 * z * z - std::log(sigma) - HALF_LOG_2PI;
}

// ----------------------------------------------------------------------------
// Models as PCFG block tables (sim : B x S -> B x S x {ckpt}).
// pc = -1 is b_stop.
// ----------------------------------------------------------------------------
const int PC_STOP = -1;

// Phylogeny given as node arrays (parent, left, right, age); tips have left =
// right = -1.  Each model builds its own traversal ("precomputes the
// recursion order over this tree, and encodes it as an iterative procedure").
struct Tree {
  int n_nodes = 0, root = -1;
  std::vector<int> parent, left, right;
  std::vector<double> age;
  int ntips(int v) const {
    if (left[v] < 0) return 1;
    return ntips(left[v]) + ntips(right[v]);
  }
};

struct Branch { double tp, tc; bool internal; bool first_left; };

// Preorder, left child first, over non-root nodes.
void preorder_left(const Tree& T, int v, std::vector<Branch>& out) {
  if (T.left[v] < 0) return;
  int kids[2] = {T.left[v], T.right[v]};
  for (int c : kids) {
    Branch b; b.tp = T.age[v]; b.tc = T.age[c]; b.internal = T.left[c] >= 0; b.first_left = true;
    out.push_back(b);
    preorder_left(T, c, out);
  }
}
// Preorder visiting the child with fewer tips first (ties: left first).
// Returns branches with first_left describing the child order at the CHILD
// node (used by ClaDS2 to know which daughter rate continues).
void preorder_smaller(const Tree& T, int v, std::vector<Branch>& out, int& maxpend, int pend) {
  if (T.left[v] < 0) return;
  int l = T.left[v], r = T.right[v];
  bool lf = T.ntips(l) <= T.ntips(r);
  int first = lf ? l : r, second = lf ? r : l;
  // after visiting v's branch (or at the root) the second child is pending
  if (pend + 1 > maxpend) maxpend = pend + 1;
  int kids[2] = {first, second};
  for (int i = 0; i < 2; ++i) {
    int c = kids[i];
    Branch b; b.tp = T.age[v]; b.tc = T.age[c]; b.internal = T.left[c] >= 0;
    b.first_left = false;
    if (b.internal) b.first_left = T.ntips(T.left[c]) <= T.ntips(T.right[c]);
    out.push_back(b);
    preorder_smaller(T, c, out, maxpend, i == 0 ? pend + 1 : pend);
  }
}

// ---- CRBD ----------------------------
// E(t): probability that a lineage alive at age t leaves no sampled
// descendant at the present (Nee et al. 1994), the textbook
//   E(t) = 1 - rho r / (rho lam + (lam (1 - rho) - mu) e^{-r t}),  r = lam - mu,
// rewritten without cancellation or overflow: with
// h = (e^{r t} - 1)/r (h = t at r = 0),  E = (rho mu h + 1 - rho)/(rho lam h + 1);
// for r > 0 numerator and denominator are multiplied by e^{-r t}.
double crbd_E(double t, double lam, double mu, double rho) {
  const double r = lam - mu;
  if (r > 0.0) {
    const double e = std::exp(-r * t), f = -std::expm1(-r * t) / r;
    return (rho * mu * f + (1.0 - rho) * e) / (rho * lam * f + e);
  }
  const double h = r == 0.0 ? t : std::expm1(r * t) / r;
  return (rho * mu * h + (1.0 - rho)) / (rho * lam * h + 1.0);
}

struct CrbdModel {
  std::vector<Branch> br;
  double rho = 1.0, lam_fixed = -1.0, mu_fixed = -1.0;
  // §5.3 variance reduction: a hidden
  // speciation event at age t contributes 2 E(t), the probability-weighted
  // form of "2 if its side tree goes undetected, else 0", instead of a
  // simulated side tree.
  bool analytic = false;
  uint64_t stack_cap = 1024, event_cap = (1u << 22);
  struct State { int pc = 0; int branch = 0; double lambda = 0, mu = 0; };
  static const int NF = 4;
  void fields(const State& s, double* f) const {
    f[0] = s.pc; f[1] = s.branch; f[2] = s.lambda; f[3] = s.mu;
  }
  // goesUndetected(s): DFS over the hidden side subtree started at age s
  // with an explicit pending stack.  Returns 1 if undetected,
  // 0 if detected, -1 on stack/event overflow.
  int undetected(double s0, const State& st, Stream& rs) const {
    std::vector<double> stack;
    stack.push_back(s0);
    uint64_t events = 0;
    double tot = st.lambda + st.mu;
    double pb = st.lambda / tot;
    while (!stack.empty()) {
      double s = stack.back(); stack.pop_back();
      for (;;) {
        if (++events > event_cap) return -1;
        double d = sample_exp(rs, tot);
        if (d > s) {
          if (sample_bernoulli(rs, rho)) return 0;
          break;
        }
        s = s - d;
        if (sample_bernoulli(rs, pb)) {
          if (stack.size() >= stack_cap) return -1;
          stack.push_back(s);
          continue;
        }
        break;
      }
    }
    return 1;
  }
  int step(State& s, double& lw, Stream& rs, uint64_t& overflow) const {
    if (s.pc == 0) {                                   // INIT (jump, no ckpt)
      s.lambda = lam_fixed >= 0.0 ? lam_fixed : sample_gamma(rs, 1.0, 1.0);
      s.mu = mu_fixed >= 0.0 ? mu_fixed : sample_gamma(rs, 1.0, 0.5);
      s.branch = 0;
      s.pc = 1;
      return 0;
    }
    // BRANCH i: edge parent -> c
    const Branch& b = br[s.branch];
    lw = lw + (-s.mu * (b.tp - b.tc));
    lw = lw + (b.internal ? std::log(s.lambda) : std::log(rho));
    double t = b.tp;
    for (;;) {
      t = t - sample_exp(rs, s.lambda);
      if (t <= b.tc) break;
      if (analytic) {
        lw = lw + LN2;
        lw = lw + std::log(crbd_E(t, s.lambda, s.mu, rho));
        continue;
      }
      int r = undetected(t, s, rs);
      if (r == 1) { lw = lw + LN2; continue; }
      if (r < 0) ++overflow;
      lw = -INFINITY;
      break;
    }
    s.branch = s.branch + 1;
    s.pc = (s.branch == (int)br.size()) ? PC_STOP : 1;
    return 1;
  }
};

// ---- ClaDS2 (BASELINE.json configs[2]; not in PAPER.md) -----
// Rate guard: a lineage rate above kMaxRate (or not finite)
// is outside the model's support; the particle's weight becomes -inf and the
// block ends at once ("kill": branch index and pc advance, nothing else).
// The threshold is params[5] (default 1e4); every kill is counted (stats
// "guard") so runs can report how often the truncation acts.
const double CLADS2_MAX_RATE = 1e4;
struct Clads2Model {
  std::vector<Branch> br;
  double rho = 1.0, lam0_fixed = -1.0, sigma_fixed = -1.0, alpha_fixed = -1.0, eps_fixed = -1.0;
  double max_rate = CLADS2_MAX_RATE;
  mutable uint64_t* guard = nullptr;   // rate-guard kills (R-14b), owned by the Smc loop
  bool root_first_left = true;
  uint64_t stack_cap = 1024, event_cap = (1u << 22);
  static const int PEND = 6;
  struct State {
    int pc = 0, branch = 0, sp = 0;
    double sigma = 0, alpha = 0, eps = 0, lam = 0;
    double pend[PEND] = {0, 0, 0, 0, 0, 0};
  };
  static const int NF = 7 + PEND;
  // The pending-rate stack holds pend[0 .. sp); entries at or above the stack
  // pointer are not part of the state (the unused part of the stack
  // beyond the stack pointer is not copied) and read as 0.
  void fields(const State& s, double* f) const {
    f[0] = s.pc; f[1] = s.branch; f[2] = s.sp; f[3] = s.sigma; f[4] = s.alpha;
    f[5] = s.eps; f[6] = s.lam;
    for (int i = 0; i < PEND; ++i) f[7 + i] = i < s.sp ? s.pend[i] : 0.0;
  }
  bool bad_rate(double r) const { return !(r <= max_rate); }
  double daughter(const State& s, double lam, double z) const {
    return s.alpha * lam * std::exp(s.sigma * z);
  }
  // 1 undetected, 0 detected, -1 stack/event overflow, -2 rate out of range
  int undetected(double s0, double lam0, const State& st, Stream& rs) const {
    std::vector<std::pair<double, double>> stack;
    stack.push_back(std::make_pair(s0, lam0));
    uint64_t events = 0;
    double pb = 1.0 / (1.0 + st.eps);
    while (!stack.empty()) {
      double s = stack.back().first, lam = stack.back().second;
      stack.pop_back();
      for (;;) {
        if (++events > event_cap) return -1;
        double d = sample_exp(rs, lam * (1.0 + st.eps));
        if (d > s) {
          if (sample_bernoulli(rs, rho)) return 0;
          break;
        }
        s = s - d;
        if (sample_bernoulli(rs, pb)) {
          double za = sample_normal(rs, 0.0, 1.0);
          double zb = sample_normal(rs, 0.0, 1.0);
          double la = daughter(st, lam, za), lb = daughter(st, lam, zb);
          if (bad_rate(la) || bad_rate(lb)) return -2;
          if (stack.size() >= stack_cap) return -1;
          stack.push_back(std::make_pair(s, lb));
          lam = la;
          continue;
        }
        break;
      }
    }
    return 1;
  }
  int kill(State& s, double& lw) const {
    if (guard) ++*guard;
    lw = -INFINITY;
    s.branch = s.branch + 1;
    s.pc = (s.branch == (int)br.size()) ? PC_STOP : 1;
    return 1;
  }
  int step(State& s, double& lw, Stream& rs, uint64_t& overflow) const {
    if (s.pc == 0) {                                   // INIT + root split
      double lam0 = lam0_fixed >= 0.0 ? lam0_fixed : sample_gamma(rs, 1.0, 1.0);
      if (sigma_fixed >= 0.0) s.sigma = sigma_fixed;
      else s.sigma = std::sqrt(1.0 / sample_gamma(rs, 1.0, 1.0 / 0.2));   // sigma^2 ~ InvGamma(1, 0.2)
      if (alpha_fixed >= 0.0) s.alpha = alpha_fixed;
      else s.alpha = std::exp(sample_normal(rs, 0.0, s.sigma));            // log alpha ~ N(0, sigma)
      s.eps = eps_fixed >= 0.0 ? eps_fixed : sample_uniform(rs, 0.0, 1.0);
      double zl = sample_normal(rs, 0.0, 1.0);
      double zr = sample_normal(rs, 0.0, 1.0);
      double rl = daughter(s, lam0, zl), rr = daughter(s, lam0, zr);
      s.sp = 0;
      s.pend[s.sp++] = root_first_left ? rr : rl;
      s.lam = root_first_left ? rl : rr;
      s.branch = 0;
      s.pc = 1;
      return 0;
    }
    const Branch& b = br[s.branch];
    if (bad_rate(s.lam)) return kill(s, lw);
    double t = b.tp;
    for (;;) {
      double dt = sample_exp(rs, s.lam);
      if (t - dt <= b.tc) {
        lw = lw + (-s.eps * s.lam * (t - b.tc));
        break;
      }
      lw = lw + (-s.eps * s.lam * dt);
      t = t - dt;
      double zs = sample_normal(rs, 0.0, 1.0);
      double zc = sample_normal(rs, 0.0, 1.0);
      double ls = daughter(s, s.lam, zs);
      if (bad_rate(ls)) return kill(s, lw);
      int r = undetected(t, ls, s, rs);
      if (r != 1) {
        if (r == -1) ++overflow;
        if (r == -2) return kill(s, lw);            // rate guard inside the side tree
        lw = -INFINITY;
        s.branch = s.branch + 1;
        s.pc = (s.branch == (int)br.size()) ? PC_STOP : 1;
        return 1;
      }
      lw = lw + LN2;
      s.lam = daughter(s, s.lam, zc);
      if (bad_rate(s.lam)) return kill(s, lw);
    }
    if (b.internal) {
      lw = lw + std::log(s.lam);
      double zl = sample_normal(rs, 0.0, 1.0);
      double zr = sample_normal(rs, 0.0, 1.0);
      double rl = daughter(s, s.lam, zl), rr = daughter(s, s.lam, zr);
      if (bad_rate(rl) || bad_rate(rr)) return kill(s, lw);
      s.pend[s.sp++] = b.first_left ? rr : rl;
      s.lam = b.first_left ? rl : rr;
    } else {
      lw = lw + std::log(rho);
      if (s.branch + 1 < (int)br.size()) s.lam = s.pend[--s.sp];
    }
    s.branch = s.branch + 1;
    s.pc = (s.branch == (int)br.size()) ? PC_STOP : 1;
    return 1;
  }
};

// ---- Lineage-keyed side trees (SURVEY c.2 #18) ------------
// Every node of a hidden side tree (one lineage from its birth to its next
// event) draws from its OWN Philox block: counter (id0, id1, n, TAG_NODE<<28 |
// t), key = seed.  u0 = hq(B0,B1) times the event, u1 = hq(B2,B3) decides it.
// A birth's two daughters get ids from the block with tag TAG_CHILD
// (child a = (C0,C1), child b = (C2,C3)); ClaDS2 daughters' rate noises are the
// Box-Muller pair of the block with tag TAG_Z.  The root of the k-th hidden
// event of the branch has id (k, 0xFFFFFFFF).  "Undetected" is an AND over the
// tree's nodes, so it does not depend on the order nodes are visited; the
// oracle visits them depth-first.
enum { TAG_NODE = 3, TAG_CHILD = 4, TAG_Z = 5 };
const uint64_t SIDE_NODE_CAP = (1ull << 22);   // nodes per branch (all its side trees)

Block side_block(uint64_t seed, uint32_t id0, uint32_t id1, uint32_t n, uint32_t t, uint32_t tag,
                 uint64_t* draws) {
  if (draws) *draws += 2;
  return philox4x32_10(id0, id1, n, (tag << 28) | t, (uint32_t)seed, (uint32_t)(seed >> 32));
}

enum { SIDE_UNDETECTED = 0, SIDE_DETECTED = 1, SIDE_OVERFLOW = 2, SIDE_GUARD = 3 };

struct CrbdLRModel : CrbdModel {
  uint64_t seed = 0;
  mutable uint64_t* draws = nullptr;
  // whole side tree of hidden event k born at age s0
  int side_tree(uint32_t k, double s0, const State& st, uint32_t n, uint32_t t, uint64_t& count) const {
    struct Node { uint32_t a, b; double s; };
    std::vector<Node> stack;
    stack.push_back(Node{k, 0xFFFFFFFFu, s0});
    const double tot = st.lambda + st.mu;
    const double pb = st.lambda / tot;
    while (!stack.empty()) {
      Node v = stack.back(); stack.pop_back();
      if (++count > SIDE_NODE_CAP) return SIDE_OVERFLOW;
      Block B = side_block(seed, v.a, v.b, n, t, TAG_NODE, draws);
      double u0 = hq(B.v[0], B.v[1]), u1 = hq(B.v[2], B.v[3]);
      double d = -std::log(u0) / tot;
      if (d > v.s) {
        if (u1 < rho) return SIDE_DETECTED;
        continue;
      }
      double s2 = v.s - d;
      if (u1 < pb) {
        Block Cb = philox4x32_10(v.a, v.b, n, (TAG_CHILD << 28) | t, (uint32_t)seed, (uint32_t)(seed >> 32));
        stack.push_back(Node{Cb.v[0], Cb.v[1], s2});
        stack.push_back(Node{Cb.v[2], Cb.v[3], s2});
      }
    }
    return SIDE_UNDETECTED;
  }
  int step_lr(State& s, double& lw, Stream& rs, uint64_t& overflow, uint32_t n, uint32_t t) const {
    if (s.pc == 0) {
      s.lambda = lam_fixed >= 0.0 ? lam_fixed : sample_gamma(rs, 1.0, 1.0);
      s.mu = mu_fixed >= 0.0 ? mu_fixed : sample_gamma(rs, 1.0, 0.5);
      s.branch = 0;
      s.pc = 1;
      return 0;
    }
    const Branch& b = br[s.branch];
    lw = lw + (-s.mu * (b.tp - b.tc));
    lw = lw + (b.internal ? std::log(s.lambda) : std::log(rho));
    // hidden speciation times along the observed branch (the particle's own stream)
    std::vector<double> ev;
    double tt = b.tp;
    for (;;) {
      tt = tt - sample_exp(rs, s.lambda);
      if (tt <= b.tc) break;
      ev.push_back(tt);
    }
    uint64_t count = 0;
    bool dead = false;
    for (size_t k = 0; k < ev.size() && !dead; ++k) {
      int r = side_tree((uint32_t)k, ev[k], s, n, t, count);
      if (r != SIDE_UNDETECTED) {
        if (r == SIDE_OVERFLOW) ++overflow;
        dead = true;
      }
    }
    if (dead) lw = -INFINITY;
    else for (size_t k = 0; k < ev.size(); ++k) lw = lw + LN2;
    s.branch = s.branch + 1;
    s.pc = (s.branch == (int)br.size()) ? PC_STOP : 1;
    return 1;
  }
};

struct Clads2LRModel : Clads2Model {
  uint64_t seed = 0;
  mutable uint64_t* draws = nullptr;
  int side_tree(uint32_t k, double s0, double lam0, const State& st, uint32_t n, uint32_t t,
                uint64_t& count) const {
    struct Node { uint32_t a, b; double s, lam; };
    std::vector<Node> stack;
    stack.push_back(Node{k, 0xFFFFFFFFu, s0, lam0});
    const double pb = 1.0 / (1.0 + st.eps);
    while (!stack.empty()) {
      Node v = stack.back(); stack.pop_back();
      if (++count > SIDE_NODE_CAP) return SIDE_OVERFLOW;
      Block B = side_block(seed, v.a, v.b, n, t, TAG_NODE, draws);
      double u0 = hq(B.v[0], B.v[1]), u1 = hq(B.v[2], B.v[3]);
      double d = -std::log(u0) / (v.lam * (1.0 + st.eps));
      if (d > v.s) {
        if (u1 < rho) return SIDE_DETECTED;
        continue;
      }
      double s2 = v.s - d;
      if (u1 < pb) {
        Block Z = side_block(seed, v.a, v.b, n, t, TAG_Z, draws);
        double r = std::sqrt(-2.0 * std::log(hq(Z.v[0], Z.v[1])));
        double th = TWO_PI * hq(Z.v[2], Z.v[3]);
        double za = r * std::cos(th), zb = r * std::sin(th);
        double la = daughter(st, v.lam, za), lb = daughter(st, v.lam, zb);
        if (bad_rate(la) || bad_rate(lb)) return SIDE_GUARD;      // rate guard: reject
        Block Cb = philox4x32_10(v.a, v.b, n, (TAG_CHILD << 28) | t, (uint32_t)seed, (uint32_t)(seed >> 32));
        stack.push_back(Node{Cb.v[0], Cb.v[1], s2, la});
        stack.push_back(Node{Cb.v[2], Cb.v[3], s2, lb});
      }
    }
    return SIDE_UNDETECTED;
  }
  int step_lr(State& s, double& lw, Stream& rs, uint64_t& overflow, uint32_t n, uint32_t t) const {
    if (s.pc == 0) return step(s, lw, rs, overflow);        // INIT + root split (main stream)
    const Branch& b = br[s.branch];
    if (bad_rate(s.lam)) return kill(s, lw);
    struct Root { double s, lam; };
    std::vector<Root> roots;
    double tt = b.tp;
    for (;;) {
      double dt = sample_exp(rs, s.lam);
      if (tt - dt <= b.tc) {
        lw = lw + (-s.eps * s.lam * (tt - b.tc));
        break;
      }
      lw = lw + (-s.eps * s.lam * dt);
      tt = tt - dt;
      double zs = sample_normal(rs, 0.0, 1.0);
      double zc = sample_normal(rs, 0.0, 1.0);
      double ls = daughter(s, s.lam, zs);
      if (bad_rate(ls)) return kill(s, lw);
      roots.push_back(Root{tt, ls});
      s.lam = daughter(s, s.lam, zc);
      if (bad_rate(s.lam)) return kill(s, lw);
    }
    if (b.internal) {
      lw = lw + std::log(s.lam);
      double zl = sample_normal(rs, 0.0, 1.0);
      double zr = sample_normal(rs, 0.0, 1.0);
      double rl = daughter(s, s.lam, zl), rr = daughter(s, s.lam, zr);
      if (bad_rate(rl) || bad_rate(rr)) return kill(s, lw);
      s.pend[s.sp++] = b.first_left ? rr : rl;
      s.lam = b.first_left ? rl : rr;
    } else {
      lw = lw + std::log(rho);
      if (s.branch + 1 < (int)br.size()) s.lam = s.pend[--s.sp];
    }
    uint64_t count = 0;
    bool dead = false;
    for (size_t k = 0; k < roots.size() && !dead; ++k) {
      int r = side_tree((uint32_t)k, roots[k].s, roots[k].lam, s, n, t, count);
      if (r != SIDE_UNDETECTED) {
        if (r == SIDE_OVERFLOW) ++overflow;
        if (r == SIDE_GUARD && guard) ++*guard;
        dead = true;
      }
    }
    if (dead) lw = -INFINITY;
    else for (size_t k = 0; k < roots.size(); ++k) lw = lw + LN2;
    s.branch = s.branch + 1;
    s.pc = (s.branch == (int)br.size()) ? PC_STOP : 1;
    return 1;
  }
};

// ---- Vector-borne disease SEIR --------------
struct SeirParams { double lam_h, del_h, gam_h, lam_m, del_m, rho; };
struct SeirCounts { int64_t sh, eh, ih, rh, sm, em, im; };
const int64_t SEIR_NH = 7370;
const double SEIR_NU_M = 1.0 / 7.0, SEIR_MU_M = 6.0 / 7.0;

// Initial state: one infectious human, optionally eh0 exposed humans and im0
// infectious mosquitoes (defaults 0; used by the tiny-population pin).
void seir_init_counts(SeirCounts& c, int64_t nh, int64_t sm0, int64_t eh0, int64_t im0) {
  c.sh = nh - 1 - eh0; c.eh = eh0; c.ih = 1; c.rh = 0;
  c.sm = sm0; c.em = 0; c.im = im0;
}
// One day of the model; returns the new human cases z ("daily numbers
// of reported new cases").
int64_t seir_day(const SeirParams& p, SeirCounts& c, int64_t nh_count, Stream& rs) {
  double nh = (double)nh_count;
  double ph = 1.0 - std::exp(-(double)c.im / nh);
  double pm = 1.0 - std::exp(-(double)c.ih / nh);
  int64_t tau_h = sample_binomial(rs, c.sh, ph);
  int64_t de_h = sample_binomial(rs, tau_h, p.lam_h);
  int64_t di_h = sample_binomial(rs, c.eh, p.del_h);
  int64_t dr_h = sample_binomial(rs, c.ih, p.gam_h);
  c.sh = c.sh - de_h;
  c.eh = c.eh + de_h - di_h;
  c.ih = c.ih + di_h - dr_h;
  c.rh = c.rh + dr_h;
  int64_t tau_m = sample_binomial(rs, c.sm, pm);
  int64_t de_m = sample_binomial(rs, tau_m, p.lam_m);
  int64_t di_m = sample_binomial(rs, c.em, p.del_m);
  int64_t nm = c.sm + c.em + c.im;
  int64_t births = sample_binomial(rs, nm, SEIR_NU_M);
  int64_t s2 = sample_binomial(rs, c.sm - de_m, SEIR_MU_M);
  int64_t e2 = sample_binomial(rs, c.em + de_m - di_m, SEIR_MU_M);
  int64_t i2 = sample_binomial(rs, c.im + di_m, SEIR_MU_M);
  c.sm = s2 + births;
  c.em = e2;
  c.im = i2;
  return di_h;
}

struct SeirModel {
  std::vector<int64_t> y;
  bool fixed = false;
  SeirParams fp{};
  int64_t nh = SEIR_NH, sm0 = 10 * SEIR_NH, eh0 = 0, im0 = 0;
  struct State { int pc = 0; int t = 0; SeirParams p{}; SeirCounts c{}; };
  static const int NF = 15;
  void fields(const State& s, double* f) const {
    f[0] = s.pc; f[1] = s.t; f[2] = s.p.lam_h; f[3] = s.p.del_h; f[4] = s.p.gam_h;
    f[5] = s.p.lam_m; f[6] = s.p.del_m; f[7] = s.p.rho;
    f[8] = (double)s.c.sh; f[9] = (double)s.c.eh; f[10] = (double)s.c.ih; f[11] = (double)s.c.rh;
    f[12] = (double)s.c.sm; f[13] = (double)s.c.em; f[14] = (double)s.c.im;
  }
  int step(State& s, double& lw, Stream& rs, uint64_t&) const {
    if (s.pc == 0) {                                   // INIT (jump)
      if (fixed) {
        s.p = fp;
      } else {
        s.p.lam_h = sample_beta(rs, 1.0, 1.0);
        s.p.del_h = sample_beta(rs, 1.0 + 2.0 / 4.4, 3.0 - 2.0 / 4.4);
        s.p.gam_h = sample_beta(rs, 1.0 + 2.0 / 4.5, 3.0 - 2.0 / 4.5);
        s.p.lam_m = sample_beta(rs, 1.0, 1.0);
        s.p.del_m = sample_beta(rs, 1.0 + 2.0 / 6.5, 3.0 - 2.0 / 6.5);
        s.p.rho = sample_beta(rs, 1.0, 1.0);
      }
      seir_init_counts(s.c, nh, sm0, eh0, im0);
      s.t = 0;
      s.pc = 1;
      return 0;
    }
    int64_t z = seir_day(s.p, s.c, nh, rs);
    lw = lw + binomial_logpmf(y[s.t], z, s.p.rho);
    s.t = s.t + 1;
    s.pc = (s.t == (int)y.size()) ? PC_STOP : 1;
    return 1;
  }
};

// ---- The PCFG of Fig. 3(a) ---------
// Blocks b0..b4 and b_stop with the figure's transitions; regular arrows are
// checkpoint transitions, open arrows are not:
//   b0 -> b1 (ckpt)
//   b1 -> b2          weight(w1)
//   b2 -> b2 | b3 | b4  one uniform u: u < p_loop: self-loop with weight(w2);
//                       u < p_loop + p3: to b3; else to b4 (no checkpoints)
//   b3 -> b2 (ckpt)   weight(w3)
//   b4 -> b_stop (ckpt) weight(w4)
// Particles run different block sequences within one epoch and reach b_stop
// at different epochs.  State: pc, n (b3 visits), x (b2 loops).
struct Fig3Model {
  double p_loop = 0.5, p3 = 0.3, w1 = 2.0, w2 = 1.2, w3 = 1.2, w4 = 0.5;
  enum { B0 = 0, B1 = 1, B2 = 2, B3 = 3, B4 = 4 };
  struct State { int pc = 0; int n = 0; int x = 0; };
  static const int NF = 3;
  void fields(const State& s, double* f) const { f[0] = s.pc; f[1] = s.n; f[2] = s.x; }
  int step(State& s, double& lw, Stream& rs, uint64_t&) const {
    switch (s.pc) {
      case B0:
        s.n = 0; s.x = 0; s.pc = B1;
        return 1;
      case B1:
        lw = lw + std::log(w1); s.pc = B2;
        return 0;
      case B2: {
        double u = sample_uniform(rs, 0.0, 1.0);
        if (u < p_loop) { s.x = s.x + 1; lw = lw + std::log(w2); s.pc = B2; }
        else if (u < p_loop + p3) s.pc = B3;
        else s.pc = B4;
        return 0;
      }
      case B3:
        s.n = s.n + 1; lw = lw + std::log(w3); s.pc = B2;
        return 1;
      default:   // B4
        lw = lw + std::log(w4); s.pc = PC_STOP;
        return 1;
    }
  }
};

// ---- The compiled recursive function of Fig. 5(c) with a PSTATE stack -------
// (Fig. 5; Sec. 4.2: "PSTATE consists of a byte array
// stack and a pointer to the top of this stack"; the part of the
// stack beyond the stack pointer is not copied)
// f(p): s1 ~ Gamma(p, 1/p); resample; weight N(y_d; s1, sigma) at recursion
// depth d (d < |y|); if s1 >= 1 then s4 = f(p_rec); s3 = s4 + s4 else s3 = 8;
// return s3 * s3.  Blocks as Fig. 5(c): b0 calls f(p0); b1 = block 1 (sample,
// checkpoint); b2 = block 2 (branch, call); b3 = block 3 (s3 = s4 + s4); b4 =
// block 4 (return: write s3*s3 at retValLoc, pop, jump to ra).  The frame
// STACK_f (48 bytes) holds ra, retValLoc (byte offset in the stack; -1: the
// program's result slot), p, s1, s3, s4.  A push beyond the user-defined stack
// size (params[3] bytes) sets the weight to -inf (counted as overflow, R-12).
struct StackfModel {
  std::vector<double> y;
  double p0 = 2.0, prec = 2.0, sigma = 0.5;
  int cap = 768;                                     // stack bytes (multiple of 16)
  struct Frame { int32_t ra, rv; double p, s1, s3, s4, pad; };
  static_assert(sizeof(Frame) == 48, "STACK_f is 48 bytes");
  static const int FRAME = 48;
  enum { B0 = 0, B1 = 1, B2 = 2, B3 = 3, B4 = 4, RA_STOP = -1 };
  struct State { int pc = 0; int sp = 0; double result = 0.0; std::vector<uint8_t> stack; };
  int nf() const { return 3 + 6 * (cap / FRAME); }
  // stack bytes at or above sp are not part of the state (R-22/R-24): reported as 0
  void fields(const State& s, double* f) const {
    f[0] = s.pc; f[1] = s.sp; f[2] = s.result;
    for (int j = 0; j < cap / FRAME; ++j) {
      double* g = f + 3 + 6 * j;
      if ((j + 1) * FRAME <= s.sp) {
        Frame fr;
        std::memcpy(&fr, s.stack.data() + j * FRAME, FRAME);
        g[0] = fr.ra; g[1] = fr.rv; g[2] = fr.p; g[3] = fr.s1; g[4] = fr.s3; g[5] = fr.s4;
      } else {
        for (int k = 0; k < 6; ++k) g[k] = 0.0;
      }
    }
  }
  Frame top(const State& s) const {
    Frame fr;
    std::memcpy(&fr, s.stack.data() + s.sp - FRAME, FRAME);
    return fr;
  }
  void set_top(State& s, const Frame& fr) const { std::memcpy(s.stack.data() + s.sp - FRAME, &fr, FRAME); }
  // push a callee frame; false on stack overflow
  bool call(State& s, int ra, int rv, double p) const {
    if (s.sp + FRAME > cap) return false;
    Frame fr{ra, rv, p, 0.0, 0.0, 0.0, 0.0};
    std::memcpy(s.stack.data() + s.sp, &fr, FRAME);
    s.sp = s.sp + FRAME;
    return true;
  }
  int step(State& s, double& lw, Stream& rs, uint64_t& overflow) const {
    switch (s.pc) {
      case B0:                                        // main: f(p0), result slot
        s.stack.assign(cap, 0);
        s.sp = 0;
        s.result = 0.0;
        if (!call(s, RA_STOP, -1, p0)) { ++overflow; lw = -INFINITY; s.pc = PC_STOP; return 1; }
        s.pc = B1;
        return 0;
      case B1: {                                      // s1 = assume Gamma p p; resample
        Frame fr = top(s);
        fr.s1 = sample_gamma(rs, fr.p, 1.0 / fr.p);
        set_top(s, fr);
        s.pc = B2;
        return 1;
      }
      case B2: {
        Frame fr = top(s);
        const int d = s.sp / FRAME - 1;               // recursion depth of this frame
        if (d < (int)y.size()) lw = lw + normal_logpdf(y[d], fr.s1, sigma);
        if (fr.s1 >= 1.0) {                           // s4 = f(p_rec)
          if (!call(s, B3, s.sp - FRAME + 32, prec)) { ++overflow; lw = -INFINITY; s.pc = PC_STOP; return 1; }
          s.pc = B1;
        } else {                                      // s3 = 8
          fr.s3 = 8.0;
          set_top(s, fr);
          s.pc = B4;
        }
        return 0;
      }
      case B3: {                                      // s3 = s4 + s4
        Frame fr = top(s);
        fr.s3 = fr.s4 + fr.s4;
        set_top(s, fr);
        s.pc = B4;
        return 0;
      }
      default: {                                      // B4: return s3 * s3
        Frame fr = top(s);
        const double t = fr.s3 * fr.s3;
        if (fr.rv < 0) s.result = t;
        else std::memcpy(s.stack.data() + fr.rv, &t, 8);
        s.sp = s.sp - FRAME;
        s.pc = fr.ra == RA_STOP ? PC_STOP : fr.ra;
        return 0;
      }
    }
  }
};

// ---- Weighted geometric, Fig. 2(a) ----------------------
struct GeometricModel {
  double p = 0.5, w = 1.5;
  struct State { int pc = 0; int n = 0; };
  static const int NF = 2;
  void fields(const State& s, double* f) const { f[0] = s.pc; f[1] = s.n; }
  int step(State& s, double& lw, Stream& rs, uint64_t&) const {
    bool x = sample_bernoulli(rs, p);
    s.n = s.n + 1;
    if (x) { lw = lw + std::log(w); s.pc = 0; }
    else { s.pc = PC_STOP; }
    return 1;
  }
};

// ---- State-space model, Eq. (2) / Fig. 4 ------------
struct SsmModel {
  std::vector<double> y;
  double m0 = 0.0, s0 = 100.0, drift = 2.0, q = 1.0, r = 5.0;   // DESIGN.md §R-5 (std devs)
  struct State { int pc = 0; int t = 0; double x = 0; };
  static const int NF = 3;
  void fields(const State& s, double* f) const { f[0] = s.pc; f[1] = s.t; f[2] = s.x; }
  int step(State& s, double& lw, Stream& rs, uint64_t&) const {
    if (s.pc == 0) {
      s.x = sample_normal(rs, m0, s0);
      s.t = 0;
      s.pc = 1;
      return 0;
    }
    s.x = sample_normal(rs, s.x + drift, q);
    lw = lw + normal_logpdf(y[s.t], s.x, r);
    s.t = s.t + 1;
    s.pc = (s.t == (int)y.size()) ? PC_STOP : 1;
    return 1;
  }
};

// ---- Constant weight: weight(log w); resample; ... K times ----------
struct ConstwModel {
  double logw = 1.0986122886681098;   // log 3
  int K = 1;
  struct State { int pc = 0; int k = 0; };
  static const int NF = 2;
  void fields(const State& s, double* f) const { f[0] = s.pc; f[1] = s.k; }
  int step(State& s, double& lw, Stream&, uint64_t&) const {
    lw = lw + logw;
    s.k = s.k + 1;
    s.pc = (s.k == K) ? PC_STOP : 0;
    return 1;
  }
};

// ----------------------------------------------------------------------------
// Exact-integer systematic resampling (reading R1).
//   m = max lw;  q_k = rint(2^62 exp(lw_k - m));  W = sum q (u128);
//   C_k = q_0 + ... + q_k;  u = (2z+1) 2^-54;
//   a_j = min{k : (j + u) W < N C_k}
//       = min{k : (j 2^54 + 2z + 1) W < N 2^54 C_k}   (exact, < 2^180).
// The loop below is the textbook sequential two-pointer sweep.
// ----------------------------------------------------------------------------
struct U256 { uint32_t w[8]; };
U256 mul128(u128 a, u128 b) {
  uint32_t x[4], y[4];
  for (int i = 0; i < 4; ++i) { x[i] = (uint32_t)(a >> (32 * i)); y[i] = (uint32_t)(b >> (32 * i)); }
  uint64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  U256 r;
  for (int i = 0; i < 8; ++i) r.w[i] = 0;
  for (int i = 0; i < 4; ++i) {
    uint64_t carry = 0;
    for (int j = 0; j < 4; ++j) {
      uint64_t cur = (uint64_t)r.w[i + j] + (uint64_t)x[i] * y[j] + carry;
      r.w[i + j] = (uint32_t)cur;
      carry = cur >> 32;
    }
    int k = i + 4;
    while (carry) {
      uint64_t cur = (uint64_t)r.w[k] + carry;
      r.w[k] = (uint32_t)cur;
      carry = cur >> 32;
      ++k;
    }
  }
  (void)acc;
  return r;
}
bool less256(const U256& a, const U256& b) {
  for (int i = 7; i >= 0; --i) {
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  }
  return false;
}
// u128 -> double by truncation to 53 significant bits.
double u128_to_double(u128 x) {
  int bl = 0;
  for (u128 t = x; t; t >>= 1) ++bl;
  int s = bl > 53 ? bl - 53 : 0;
  uint64_t top = (uint64_t)(x >> s);
  return std::ldexp((double)top, s);
}

enum { E_OK = 0, E_INVAL = 1, E_REJECTED = 4, E_NAN = 5 };

struct ResampleOut { double m; u128 W; double logz_inc; uint64_t z; };

// m, W and the log Z increment  logZ += m + log W - 62 ln 2 - log N.
int normalise(const double* lw, uint64_t N, std::vector<uint64_t>& q, ResampleOut& o) {
  double m = -INFINITY;
  for (uint64_t k = 0; k < N; ++k) {
    if (std::isnan(lw[k]) || lw[k] == INFINITY) return E_NAN;
    if (lw[k] > m) m = lw[k];
  }
  o.m = m;
  if (m == -INFINITY) { o.W = 0; o.logz_inc = -INFINITY; return E_REJECTED; }
  q.assign(N, 0);
  u128 W = 0;
  for (uint64_t k = 0; k < N; ++k) {
    if (lw[k] == -INFINITY) { q[k] = 0; continue; }
    double e = std::exp(lw[k] - m);
    q[k] = (uint64_t)std::nearbyint(std::ldexp(e, 62));
    W += q[k];
  }
  o.W = W;
  double lwd = std::log(u128_to_double(W));
  o.logz_inc = m + ((lwd - 62.0 * LN2) - std::log((double)N));
  return E_OK;
}

uint64_t resample_z(uint64_t seed, uint32_t t) {
  Block b = philox4x32_10(0, t, 0, TAG_RESAMPLE, (uint32_t)seed, (uint32_t)(seed >> 32));
  return hq_bits(b.v[0], b.v[1]);
}

void systematic(const std::vector<uint64_t>& q, uint64_t N, u128 W, uint64_t z, uint32_t* anc) {
  const u128 two54 = (u128)1 << 54;
  u128 Nscaled = (u128)N * two54;
  uint64_t k = 0;
  u128 C = q[0];
  for (uint64_t j = 0; j < N; ++j) {
    u128 A = (u128)j * two54 + (u128)(2 * z + 1);
    U256 lhs = mul128(A, W);
    for (;;) {
      U256 rhs = mul128(Nscaled, C);
      if (less256(lhs, rhs)) break;
      ++k;
      C += q[k];
    }
    anc[j] = (uint32_t)k;
  }
}

// Ancestor permutation for in-place resampling (SURVEY §8f
// row f3; the in-place propagation of Murray et al. 2016 that RootPPL does not
// use).  From the sorted ancestors a: every particle k with offspring
// keeps its own slot (c_k = k); the remaining copies -- o_k - 1 of each k, in
// ascending k -- fill the slots of the particles without offspring, in
// ascending slot order.  c is a permutation of a; no slot without offspring
// is a source, so the gather can run in place.
void permute_ancestors(const uint32_t* a, uint64_t N, uint32_t* c) {
  std::vector<uint64_t> o(N, 0);
  for (uint64_t j = 0; j < N; ++j) o[a[j]] += 1;
  std::vector<uint32_t> extras;
  for (uint64_t k = 0; k < N; ++k)
    for (uint64_t e = 1; e < o[k]; ++e) extras.push_back((uint32_t)k);
  uint64_t h = 0;
  for (uint64_t k = 0; k < N; ++k) c[k] = o[k] > 0 ? (uint32_t)k : extras[h++];
}

// ESS-adaptive resampling: with
// integer weights q, ESS = W^2 / sum q^2.  Resample iff tau >= 1 or
// ESS < tau N, tau = a/b, evaluated exactly:  b W^2 < a N sum q^2.
struct U512 { uint64_t w[8]; };
U512 add_mul(U512 acc, u128 x, u128 y) {            // acc += x * y
  U256 p = mul128(x, y);
  uint64_t carry = 0;
  for (int i = 0; i < 8; ++i) {
    uint64_t add = i < 4 ? ((uint64_t)p.w[2 * i] | ((uint64_t)p.w[2 * i + 1] << 32)) : 0;
    u128 cur = (u128)acc.w[i] + add + carry;
    acc.w[i] = (uint64_t)cur;
    carry = (uint64_t)(cur >> 64);
  }
  return acc;
}
U512 mul_small(U512 a, uint64_t m) {
  U512 r{};
  u128 carry = 0;
  for (int i = 0; i < 8; ++i) {
    u128 cur = (u128)a.w[i] * m + carry;
    r.w[i] = (uint64_t)cur;
    carry = cur >> 64;
  }
  return r;
}
bool less512(const U512& a, const U512& b) {
  for (int i = 7; i >= 0; --i) if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  return false;
}
bool ess_resample(const std::vector<uint64_t>& q, u128 W, uint64_t N, uint32_t a, uint32_t b) {
  if (a >= b) return true;                                 // tau >= 1: always (plain Alg. 1)
  U512 Q2{};
  for (uint64_t k = 0; k < q.size(); ++k) Q2 = add_mul(Q2, q[k], q[k]);
  U512 W2{};
  W2 = add_mul(W2, W, W);
  U512 lhs = mul_small(W2, b);
  U512 rhs = mul_small(mul_small(Q2, a), N);
  return less512(lhs, rhs);
}
double ess_value(const std::vector<uint64_t>& q, u128 W) {  // diagnostics only
  long double s2 = 0;
  for (uint64_t v : q) s2 += (long double)v * (long double)v;
  long double w = (long double)W;
  return s2 > 0 ? (double)(w * w / s2) : 0.0;
}

// ----------------------------------------------------------------------------
// Algorithm 1 with the RootPPL loop order:
// propagate all particles to their next checkpoint; stop if all reached
// b_stop (final log Z update, no resample); else resample.
// ----------------------------------------------------------------------------
struct SmcBase {
  virtual ~SmcBase() {}
  virtual int step(int* done) = 0;
  virtual int nfields() const = 0;
  virtual void get_fields(double* out) const = 0;
  uint64_t N = 0, seed = 0;
  uint32_t t = 0;
  double logz = 0.0;
  int status = E_OK;
  bool finished = false;
  uint64_t draws = 0, overflow = 0, resamples = 0, alive_steps = 0, guard = 0;
  uint32_t ess_a = 1, ess_b = 1;        // tau = a / b (>= 1: resample at every checkpoint)
  double last_ess = 0.0;
  bool carry = false;                   // last checkpoint did not resample: lw accumulates
  bool inplace = false;                 // R-21: permuted ancestors (in-place gather)
  std::vector<double> lw;
  std::vector<uint32_t> anc;
  std::vector<uint64_t> last_q;
  ResampleOut last{};
};

inline void set_side_draws(...) {}
inline void set_side_draws(CrbdLRModel& m, uint64_t* d) { m.draws = d; }
inline void set_side_draws(Clads2LRModel& m, uint64_t* d) { m.draws = d; }
inline void set_guard(...) {}
inline void set_guard(Clads2Model& m, uint64_t* g) { m.guard = g; }

// Number of decoded fields: compile-time for most models, run-time (stack size)
// for the PSTATE-stack model.
template <class M> struct NfOf { static int get(const M&) { return M::NF; } };
template <> struct NfOf<StackfModel> { static int get(const StackfModel& m) { return m.nf(); } };

// Adapter: the Alg. 1 loop calls step(); lineage-keyed models need (n, t).
template <class M> struct StepCall {
  static int call(const M& m, typename M::State& s, double& lw, Stream& rs, uint64_t& ovf,
                  uint32_t, uint32_t) { return m.step(s, lw, rs, ovf); }
};
template <> struct StepCall<CrbdLRModel> {
  static int call(const CrbdLRModel& m, CrbdLRModel::State& s, double& lw, Stream& rs,
                  uint64_t& ovf, uint32_t n, uint32_t t) { return m.step_lr(s, lw, rs, ovf, n, t); }
};
template <> struct StepCall<Clads2LRModel> {
  static int call(const Clads2LRModel& m, Clads2LRModel::State& s, double& lw, Stream& rs,
                  uint64_t& ovf, uint32_t n, uint32_t t) { return m.step_lr(s, lw, rs, ovf, n, t); }
};

template <class M>
struct Smc : SmcBase {
  M model;
  std::vector<typename M::State> st, tmp;
  Smc(const M& m, uint64_t n, uint64_t s) : model(m) {
    N = n; seed = s;
    set_side_draws(model, &draws);
    set_guard(model, &guard);
    st.assign(N, typename M::State());
    lw.assign(N, 0.0);
    anc.resize(N);
    for (uint64_t j = 0; j < N; ++j) anc[j] = (uint32_t)j;
  }
  int nfields() const override { return NfOf<M>::get(model); }
  void get_fields(double* out) const override {
    const int nf = NfOf<M>::get(model);
    for (uint64_t n = 0; n < N; ++n) model.fields(st[n], out + n * nf);
  }
  int step(int* done) override {
    if (finished || status != E_OK) { *done = 1; return status; }
    // Propagation (Alg. 1 step 2).  lw holds the weight
    // accumulated since the last resample: it restarts at 0 unless the last
    // checkpoint skipped resampling (R-19).
    for (uint64_t n = 0; n < N; ++n) {
      if (!carry) lw[n] = 0.0;
      if (st[n].pc == PC_STOP) continue;      // b_stop self-loop
      ++alive_steps;
      Stream rs = make_stream(seed, (uint32_t)n, t, TAG_PARTICLE, &draws);
      for (;;) {
        int ckpt = StepCall<M>::call(model, st[n], lw[n], rs, overflow, (uint32_t)n, t);
        if (ckpt || st[n].pc == PC_STOP) break;
      }
    }
    bool alive = false;
    for (uint64_t n = 0; n < N; ++n) if (st[n].pc != PC_STOP) { alive = true; break; }
    // Normalisation and log Z
    int rc = normalise(lw.data(), N, last_q, last);
    if (rc != E_OK) {
      status = rc;
      if (rc == E_REJECTED) logz = -INFINITY;
      finished = true; *done = 1;
      return rc;
    }
    if (!alive) {
      logz += last.logz_inc;
      finished = true; *done = 1; return E_OK;
    }
    last_ess = ess_value(last_q, last.W);
    if (!ess_resample(last_q, last.W, N, ess_a, ess_b)) {      // ESS gate (R-19)
      carry = true;                                            // weights carried over
      ++t;
      *done = 0;
      return E_OK;
    }
    carry = false;
    logz += last.logz_inc;
    // Resampling (Alg. 1 step 3; systematic)
    last.z = resample_z(seed, t);
    systematic(last_q, N, last.W, last.z, anc.data());
    if (inplace) {
      std::vector<uint32_t> sorted(anc);
      permute_ancestors(sorted.data(), N, anc.data());
    }
    tmp.resize(N);
    for (uint64_t j = 0; j < N; ++j) tmp[j] = st[anc[j]];
    st.swap(tmp);
    ++resamples;
    ++t;
    *done = 0;
    return E_OK;
  }
};

Tree parse_tree(const double* d, uint64_t len, bool& ok) {
  // layout: [M, root, (parent, left, right, age) x M]
  Tree T;
  ok = false;
  if (len < 2) return T;
  int M = (int)d[0];
  if (M < 3 || len != (uint64_t)(2 + 4 * M)) return T;
  T.n_nodes = M; T.root = (int)d[1];
  T.parent.resize(M); T.left.resize(M); T.right.resize(M); T.age.resize(M);
  for (int i = 0; i < M; ++i) {
    T.parent[i] = (int)d[2 + 4 * i];
    T.left[i] = (int)d[3 + 4 * i];
    T.right[i] = (int)d[4 + 4 * i];
    T.age[i] = d[5 + 4 * i];
  }
  ok = T.root >= 0 && T.root < M && T.left[T.root] >= 0;
  return T;
}

thread_local std::string g_err;

}  // namespace

// =============================================================================
// C API (ctypes, tests only)
// =============================================================================
extern "C" {

enum { K_CRBD = 1, K_CLADS2 = 2, K_SEIR = 3, K_CRBD_LR = 4, K_CLADS2_LR = 5, K_CRBD_AE = 6,
       K_GEOMETRIC = 10, K_SSM = 11, K_CONSTW = 12, K_FIG3 = 13, K_STACKF = 14 };

const char* oracle_errmsg() { return g_err.c_str(); }

double oracle_crbd_E(double t, double lam, double mu, double rho) { return crbd_E(t, lam, mu, rho); }

void oracle_philox(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  Block b = philox4x32_10(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1]);
  for (int i = 0; i < 4; ++i) out[i] = b.v[i];
}

// Fill out[0..n) with consecutive uniforms of stream (seed, particle, epoch, tag).
void oracle_uniforms(uint64_t seed, uint32_t particle, uint32_t epoch, uint32_t tag,
                     uint64_t n, double* out) {
  Stream s = make_stream(seed, particle, epoch, tag, nullptr);
  for (uint64_t i = 0; i < n; ++i) out[i] = s.uniform();
}

// Draw n variates of distribution `dist` from independent streams: variate i
// uses particle index i (epoch 0, tag 0).  draws_out[i] = uniforms consumed.
// dist: 0 exp(rate) 1 bernoulli(p) 2 uniform(a,b) 3 normal(mu,sigma)
//       4 gamma(k,theta) 5 beta(a,b) 6 binomial(n,p)
int oracle_sample(int dist, const double* prm, uint64_t seed, uint64_t n,
                  double* out, uint32_t* draws_out) {
  for (uint64_t i = 0; i < n; ++i) {
    Stream s = make_stream(seed, (uint32_t)i, 0, TAG_PARTICLE, nullptr);
    double v = 0;
    switch (dist) {
      case 0: v = sample_exp(s, prm[0]); break;
      case 1: v = sample_bernoulli(s, prm[0]) ? 1.0 : 0.0; break;
      case 2: v = sample_uniform(s, prm[0], prm[1]); break;
      case 3: v = sample_normal(s, prm[0], prm[1]); break;
      case 4: v = sample_gamma(s, prm[0], prm[1]); break;
      case 5: v = sample_beta(s, prm[0], prm[1]); break;
      case 6: v = (double)sample_binomial(s, (int64_t)prm[0], prm[1]); break;
      default: g_err = "unknown dist"; return E_INVAL;
    }
    out[i] = v;
    if (draws_out) draws_out[i] = (uint32_t)s.d;
  }
  return E_OK;
}

double oracle_binomial_logpmf(int64_t k, int64_t n, double p) { return binomial_logpmf(k, n, p); }
double oracle_normal_logpdf(double y, double mu, double s) { return normal_logpdf(y, mu, s); }
double oracle_u128_to_double(uint64_t lo, uint64_t hi) {
  return u128_to_double(((u128)hi << 64) | lo);
}

// Resampling alone on caller-supplied log-weights (epoch t, key seed).
// Outputs: anc[N], W (lo, hi), m, logz_inc, z.  Returns status.
int oracle_resample(const double* lw, uint64_t N, uint64_t seed, uint32_t t,
                    uint32_t* anc, uint64_t* W_lohi, double* m_out, double* logz_inc,
                    uint64_t* z_out) {
  if (N == 0 || N > 0xFFFFFFFFull) { g_err = "bad N"; return E_INVAL; }
  std::vector<uint64_t> q;
  ResampleOut o{};
  int rc = normalise(lw, N, q, o);
  if (m_out) *m_out = o.m;
  if (logz_inc) *logz_inc = o.logz_inc;
  if (rc != E_OK) return rc;
  o.z = resample_z(seed, t);
  if (W_lohi) { W_lohi[0] = (uint64_t)o.W; W_lohi[1] = (uint64_t)(o.W >> 64); }
  if (z_out) *z_out = o.z;
  if (anc) systematic(q, N, o.W, o.z, anc);
  return E_OK;
}

// Systematic step alone on caller-supplied integer weights q and resample
// integer z (u = (2z+1) 2^-54): anc[j] = min{k : (j + u) W < N C_k}.
int oracle_systematic(const uint64_t* q, uint64_t N, uint64_t z, uint32_t* anc) {
  std::vector<uint64_t> qq(q, q + N);
  u128 W = 0;
  for (uint64_t k = 0; k < N; ++k) W += qq[k];
  if (W == 0 || z >= (1ull << 53)) return E_INVAL;
  systematic(qq, N, W, z, anc);
  return E_OK;
}

// Quantised weights q_k (for tests).
int oracle_quantize(const double* lw, uint64_t N, uint64_t* q_out) {
  std::vector<uint64_t> q;
  ResampleOut o{};
  int rc = normalise(lw, N, q, o);
  if (rc != E_OK) return rc;
  for (uint64_t k = 0; k < N; ++k) q_out[k] = q[k];
  return E_OK;
}

// Gather of opaque fixed-size states: out[j] = in[anc[j]] (state_bytes each).
void oracle_permute(const uint32_t* a, uint64_t N, uint32_t* c) { permute_ancestors(a, N, c); }

void oracle_gather(const uint8_t* in, uint8_t* out, const uint32_t* anc, uint64_t N,
                   uint64_t state_bytes) {
  for (uint64_t j = 0; j < N; ++j)
    std::memcpy(out + j * state_bytes, in + (uint64_t)anc[j] * state_bytes, state_bytes);
}

void* oracle_smc_create(int kind, const double* data, uint64_t data_len,
                        const double* prm, int n_prm, uint64_t N, uint64_t seed) {
  if (N == 0 || N > 0xFFFFFFFFull) { g_err = "N must be in [1, 2^32)"; return nullptr; }
  auto P = [&](int i, double dflt) { return (prm && i < n_prm) ? prm[i] : dflt; };
  switch (kind) {
    case K_CRBD:
    case K_CRBD_AE: {
      bool ok; Tree T = parse_tree(data, data_len, ok);
      if (!ok) { g_err = "bad tree"; return nullptr; }
      CrbdModel m;
      preorder_left(T, T.root, m.br);
      m.rho = P(0, 1.0); m.lam_fixed = P(1, -1.0); m.mu_fixed = P(2, -1.0);
      m.analytic = kind == K_CRBD_AE;
      return new Smc<CrbdModel>(m, N, seed);
    }
    case K_CLADS2: {
      bool ok; Tree T = parse_tree(data, data_len, ok);
      if (!ok) { g_err = "bad tree"; return nullptr; }
      Clads2Model m;
      int maxpend = 0;
      preorder_smaller(T, T.root, m.br, maxpend, 0);
      if (maxpend > Clads2Model::PEND) { g_err = "pending-rate stack exceeds 6"; return nullptr; }
      int l = T.left[T.root], r = T.right[T.root];
      m.root_first_left = T.ntips(l) <= T.ntips(r);
      m.rho = P(0, 1.0); m.lam0_fixed = P(1, -1.0); m.sigma_fixed = P(2, -1.0);
      m.alpha_fixed = P(3, -1.0); m.eps_fixed = P(4, -1.0);
      m.max_rate = P(5, CLADS2_MAX_RATE);
      return new Smc<Clads2Model>(m, N, seed);
    }
    case K_CRBD_LR: {
      bool ok; Tree T = parse_tree(data, data_len, ok);
      if (!ok) { g_err = "bad tree"; return nullptr; }
      CrbdLRModel m;
      preorder_left(T, T.root, m.br);
      m.rho = P(0, 1.0); m.lam_fixed = P(1, -1.0); m.mu_fixed = P(2, -1.0);
      m.seed = seed;
      return new Smc<CrbdLRModel>(m, N, seed);
    }
    case K_CLADS2_LR: {
      bool ok; Tree T = parse_tree(data, data_len, ok);
      if (!ok) { g_err = "bad tree"; return nullptr; }
      Clads2LRModel m;
      int maxpend = 0;
      preorder_smaller(T, T.root, m.br, maxpend, 0);
      if (maxpend > Clads2Model::PEND) { g_err = "pending-rate stack exceeds 6"; return nullptr; }
      int l = T.left[T.root], r = T.right[T.root];
      m.root_first_left = T.ntips(l) <= T.ntips(r);
      m.rho = P(0, 1.0); m.lam0_fixed = P(1, -1.0); m.sigma_fixed = P(2, -1.0);
      m.alpha_fixed = P(3, -1.0); m.eps_fixed = P(4, -1.0);
      m.max_rate = P(5, CLADS2_MAX_RATE);
      m.seed = seed;
      return new Smc<Clads2LRModel>(m, N, seed);
    }
    case K_SEIR: {
      SeirModel m;
      for (uint64_t i = 0; i < data_len; ++i) m.y.push_back((int64_t)data[i]);
      if (m.y.empty()) { g_err = "empty series"; return nullptr; }
      // params: [lam_h, del_h, gam_h, lam_m, del_m, rho] (any < 0: prior),
      //         [6] n_h (default 7370), [7] initial susceptible mosquitoes (10 n_h),
      //         [8] initial exposed humans (0), [9] initial infectious mosquitoes (0)
      if (n_prm >= 6 && prm[0] >= 0.0) {
        m.fixed = true;
        m.fp = SeirParams{prm[0], prm[1], prm[2], prm[3], prm[4], prm[5]};
      }
      m.nh = (int64_t)P(6, (double)SEIR_NH);
      m.sm0 = (int64_t)P(7, 10.0 * (double)m.nh);
      m.eh0 = (int64_t)P(8, 0.0);
      m.im0 = (int64_t)P(9, 0.0);
      if (m.nh < 1 || m.sm0 < 0 || m.eh0 < 0 || m.im0 < 0 || m.eh0 > m.nh - 1) { g_err = "bad SEIR population"; return nullptr; }
      return new Smc<SeirModel>(m, N, seed);
    }
    case K_GEOMETRIC: {
      GeometricModel m; m.p = P(0, 0.5); m.w = P(1, 1.5);
      return new Smc<GeometricModel>(m, N, seed);
    }
    case K_SSM: {
      SsmModel m;
      for (uint64_t i = 0; i < data_len; ++i) m.y.push_back(data[i]);
      if (m.y.empty()) { g_err = "empty series"; return nullptr; }
      m.m0 = P(0, 0.0); m.s0 = P(1, 100.0); m.drift = P(2, 2.0); m.q = P(3, 1.0); m.r = P(4, 5.0);
      return new Smc<SsmModel>(m, N, seed);
    }
    case K_FIG3: {
      Fig3Model m;
      m.p_loop = P(0, 0.5); m.p3 = P(1, 0.3); m.w1 = P(2, 2.0); m.w2 = P(3, 1.2); m.w3 = P(4, 1.2);
      m.w4 = P(5, 0.5);
      if (!(m.p_loop >= 0 && m.p3 >= 0 && m.p_loop + m.p3 <= 1 && m.w1 > 0 && m.w2 > 0 && m.w3 > 0 && m.w4 > 0)) {
        g_err = "bad Fig. 3 parameters"; return nullptr;
      }
      return new Smc<Fig3Model>(m, N, seed);
    }
    case K_STACKF: {
      StackfModel m;
      for (uint64_t i = 0; i < data_len; ++i) m.y.push_back(data[i]);
      m.p0 = P(0, 2.0); m.prec = P(1, 2.0); m.sigma = P(2, 0.5); m.cap = (int)P(3, 768.0);
      if (!(m.p0 > 0 && m.prec > 0 && m.sigma > 0) || m.cap < 48 || m.cap % 16 || m.cap > 65536) {
        g_err = "bad STACKF parameters"; return nullptr;
      }
      return new Smc<StackfModel>(m, N, seed);
    }
    case K_CONSTW: {
      ConstwModel m; m.logw = P(0, std::log(3.0)); m.K = (int)P(1, 1.0);
      if (m.K < 1) { g_err = "K >= 1"; return nullptr; }
      return new Smc<ConstwModel>(m, N, seed);
    }
    default: g_err = "unknown model kind"; return nullptr;
  }
}

int oracle_smc_step(void* h, int* done) { return ((SmcBase*)h)->step(done); }
// ESS threshold tau = a / b (R-19); a >= b: resample at every checkpoint.
int oracle_smc_set_inplace(void* h, int on) {
  static_cast<SmcBase*>(h)->inplace = on != 0;
  return E_OK;
}

int oracle_smc_set_ess(void* h, uint32_t a, uint32_t b) {
  if (b == 0) return E_INVAL;
  ((SmcBase*)h)->ess_a = a; ((SmcBase*)h)->ess_b = b;
  return E_OK;
}
double oracle_smc_last_ess(void* h) { return ((SmcBase*)h)->last_ess; }
// Exact ESS gate on caller weights (tests): 1 = resample.
int oracle_ess_gate(const double* lw, uint64_t N, uint32_t a, uint32_t b, double* ess) {
  std::vector<uint64_t> q;
  ResampleOut o{};
  int rc = normalise(lw, N, q, o);
  if (rc != E_OK) return -rc;
  if (ess) *ess = ess_value(q, o.W);
  return ess_resample(q, o.W, N, a, b) ? 1 : 0;
}
int oracle_smc_run(void* h) {
  int done = 0, rc = 0;
  while (!done) { rc = oracle_smc_step(h, &done); }
  return rc;
}
double oracle_smc_log_z(void* h) { return ((SmcBase*)h)->logz; }
uint32_t oracle_smc_epoch(void* h) { return ((SmcBase*)h)->t; }
int oracle_smc_nfields(void* h) { return ((SmcBase*)h)->nfields(); }
void oracle_smc_fields(void* h, double* out) { ((SmcBase*)h)->get_fields(out); }
void oracle_smc_lw(void* h, double* out) {
  SmcBase* s = (SmcBase*)h;
  std::memcpy(out, s->lw.data(), s->N * sizeof(double));
}
void oracle_smc_anc(void* h, uint32_t* out) {
  SmcBase* s = (SmcBase*)h;
  std::memcpy(out, s->anc.data(), s->N * sizeof(uint32_t));
}
// stats: [epochs_done, resamples, draws, overflow, alive_particle_steps, status,
//         rate-guard kills (ClaDS2, R-14b)]
void oracle_smc_stats(void* h, uint64_t* out) {
  SmcBase* s = (SmcBase*)h;
  out[0] = s->resamples + (s->finished ? 1 : 0);
  out[1] = s->resamples; out[2] = s->draws; out[3] = s->overflow;
  out[4] = s->alive_steps; out[5] = (uint64_t)s->status; out[6] = s->guard;
}
void oracle_smc_destroy(void* h) { delete (SmcBase*)h; }

// ---- synthetic-input generators (committed scripts call these once) --------
// Yule tree (SURVEY §8d "tree90"): k=2 crown lineages at time 0; while
// k < ntips: wait Exp(k lam0), split lineage floor(u' k) (daughters replace it
// in place and at the end); final Exp(ntips lam0) gap; ages rescaled so the
// crown age is `crown_age`.  Uniforms: tag 2, particle 0, epoch 0.
// Output arrays of size 2*ntips-1: parent, left, right, age; returns #uniforms.
int64_t oracle_gen_yule(uint64_t seed, int ntips, double lam0, double crown_age,
                        int* parent, int* left, int* right, double* age) {
  if (ntips < 2) return -1;
  int M = 2 * ntips - 1;
  Stream s = make_stream(seed, 0, 0, TAG_DATA, nullptr);
  std::vector<double> tsplit(M, 0.0);   // node creation time (forward)
  for (int i = 0; i < M; ++i) { parent[i] = left[i] = right[i] = -1; }
  int next_internal = 1;
  // open lineages: (parent node) ; root = node 0 at time 0
  std::vector<int> lin_parent = {0, 0};
  std::vector<int> lin_side = {0, 1};
  double now = 0.0;
  std::vector<int> pending_child_slot;   // unused
  // we record children lazily: when a lineage ends (split or present) it
  // becomes a node attached to its parent on the recorded side.
  auto attach = [&](int par, int side, int child) {
    parent[child] = par;
    if (side == 0) left[par] = child; else right[par] = child;
  };
  int k = 2;
  while (k < ntips) {
    double u1 = s.uniform();
    double w = -std::log(u1) / ((double)k * lam0);
    now = now + w;
    double u2 = s.uniform();
    int idx = (int)std::floor(u2 * (double)k);
    if (idx >= k) idx = k - 1;
    int v = next_internal++;
    tsplit[v] = now;
    attach(lin_parent[idx], lin_side[idx], v);
    lin_parent[idx] = v; lin_side[idx] = 0;
    lin_parent.push_back(v); lin_side.push_back(1);
    ++k;
  }
  double ug = s.uniform();
  now = now + (-std::log(ug) / ((double)ntips * lam0));
  int tip = next_internal;   // tips follow internal nodes, in list order
  for (int i = 0; i < k; ++i) {
    int v = tip++;
    tsplit[v] = now;
    attach(lin_parent[i], lin_side[i], v);
  }
  double scale = crown_age / now;
  for (int i = 0; i < M; ++i) age[i] = (now - tsplit[i]) * scale;
  age[0] = crown_age;
  for (int i = next_internal; i < M; ++i) age[i] = 0.0;
  return (int64_t)s.d;
}

// Forward simulation of the SEIR model with fixed parameters: y[t] ~
// Bin(z_t, rho) for t = 0..T-1 (tag 2, particle 0).  Returns #uniforms.
int64_t oracle_gen_seir(uint64_t seed, int T, const double* prm, int64_t* y, int64_t* z_out) {
  SeirParams p{prm[0], prm[1], prm[2], prm[3], prm[4], prm[5]};
  SeirCounts c;
  seir_init_counts(c, SEIR_NH, 10 * SEIR_NH, 0, 0);
  Stream s = make_stream(seed, 0, 0, TAG_DATA, nullptr);
  for (int t = 0; t < T; ++t) {
    int64_t z = seir_day(p, c, SEIR_NH, s);
    y[t] = sample_binomial(s, z, p.rho);
    if (z_out) z_out[t] = z;
  }
  return (int64_t)s.d;
}

// Forward simulation of Eq. (2): x0 ~ N(m0, s0); x_t ~ N(x_{t-1}+drift, q);
// y_t ~ N(x_t, r).  prm = (m0, s0, drift, q, r).
int64_t oracle_gen_ssm(uint64_t seed, int T, const double* prm, double* y, double* x_out) {
  Stream s = make_stream(seed, 0, 0, TAG_DATA, nullptr);
  double x = sample_normal(s, prm[0], prm[1]);
  for (int t = 0; t < T; ++t) {
    x = sample_normal(s, x + prm[2], prm[3]);
    y[t] = sample_normal(s, x, prm[4]);
    if (x_out) x_out[t] = x;
  }
  return (int64_t)s.d;
}

}  // extern "C"
