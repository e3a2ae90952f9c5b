// lineage_warp.cuh — warp-independent cooperative propagation for the
// birth-death models under the lineage-keyed side-tree reading (DESIGN.md
// §R-18, §7.1).
//
// Same work as propagate_lr_kernel (lineage.cuh): phase 1 walks each
// particle's observed branch on its own stream and pushes one root task per
// hidden event; phase 2 evaluates the hidden side trees cooperatively (every
// tree node is one Philox block, so nodes may be evaluated in any order);
// phase 3 finishes the particle (-inf if any node was detected, else + ln 2 per
// hidden event).  The difference is the unit of cooperation: each WARP pulls
// its own batch of 32 particles and runs the rounds warp-synchronously —
// counts, fair-share lane assignment, detection flags and pushes go through
// registers, shuffles and per-warp shared memory with __syncwarp only.  No CTA
// barrier sits inside the loop, so a warp stuck on a deep side tree holds back
// nobody, and a round costs a few dozen instructions instead of four CTA
// barriers (ncu, profiles/r02: the CTA rounds were ~40% of the instructions
// and half of the stall samples of the CTA version).
//
// Per round: every owner lane with c pending tasks offers its top
// m = min(c, max(1, 32 / #busy owners)) tasks (LIFO: depth-first per owner, so
// a supercritical tree is detected along one path); lanes are assigned by an
// exclusive scan of m; lanes left over pop the warp's overflow stack.  Owner
// state (task count, detection flag, node count, lw, number of hidden events)
// lives in the owner lane's registers for the whole batch.
#pragma once
#include "lineage.cuh"

namespace smc {

#ifndef SMC_LRW_THREADS
#define SMC_LRW_THREADS 128
#endif
constexpr int kWThreads = SMC_LRW_THREADS;       // CTA = kWThreads / 32 independent warps
constexpr int kWWarps = kWThreads / 32;
constexpr int kWSeg = 256;                       // per-owner LIFO segment (tasks)
#ifndef SMC_LRW_WMAX
#define SMC_LRW_WMAX 32
#endif
constexpr int kWMax = SMC_LRW_WMAX;              // lanes one owner may take in a round
#ifndef SMC_LRW_FASTMAP
#define SMC_LRW_FASTMAP 1
#endif
#ifndef SMC_LRW_OVN_UNIFORM
#define SMC_LRW_OVN_UNIFORM 0   // overflow-pop counters only in rounds with overflow pops: measured slower (46.7 -> 47.3 ms), off
#endif
#ifndef SMC_LRW_BALLOT_SCAN
#define SMC_LRW_BALLOT_SCAN 0   // offsets by bit-sliced ballots (1) or a shuffle scan (0: CRBD 48.1 -> 46.75 ms)
#endif
#ifndef SMC_LRW_BALLOTPUSH
#define SMC_LRW_BALLOTPUSH 0      // ballot-ranked pushes instead of shared atomics: measured slower (CRBD 53.8 -> 57.0, ClaDS2 188 -> 196 ms)
#endif
#ifndef SMC_LRW_SMEM_SLOTS
#define SMC_LRW_SMEM_SLOTS 0       // measured: 4, 8, 12 slots all slower (CRBD 59.3 -> 61.3-62.5 ms)
#endif
constexpr int kSm = SMC_LRW_SMEM_SLOTS;          // bottom slots of every owner segment kept in shared memory
constexpr int kWOvf = 1 << 16;                   // per-warp overflow LIFO (tasks)
constexpr unsigned long long kWSegSlots = 32ull * kWSeg;
constexpr unsigned long long kTasksPerWarp = kWSegSlots + kWOvf;

// fair share max(1, 32 / n) lanes per busy owner (table: no integer division in the round)
__constant__ int c_wshare[33] = {0, 32, 16, 10, 8, 6, 5, 4, 4, 3, 3, 2, 2, 2, 2, 2, 2,
                                 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};

template <class M>
__global__ void __launch_bounds__(kWThreads, M::kLRWMinBlocks) propagate_lrw_kernel(LRArgs a, ModelConst C) {
  __shared__ typename M::Owner s_own[kWWarps][32];   // per-owner constants read by every lane
  __shared__ double2 s_tsk[kWWarps][32 * (kSm > 0 ? kSm : 1)];                    // segment slots < kSm
  __shared__ double s_tlam[kWWarps][M::kHasLam && kSm > 0 ? 32 * kSm : 1];
  __shared__ int s_start[kWWarps][32];               // round: lane where owner o's tasks start
  __shared__ int s_push[kWWarps][32];                // round: slots pushed for owner o
  __shared__ int s_det[kWWarps][32];                 // round: 1 detected, 3 rate guard
  __shared__ int s_ovn[kWWarps][32];                 // round: overflow tasks of owner o evaluated
  __shared__ int s_ovtop[kWWarps];                   // overflow stack top
  __shared__ int s_taskcap;
  __shared__ long long s_key[kWWarps];
  __shared__ unsigned long long s_acc[3][kWWarps];
  const PropArgs& p = a.p;
  if (*(volatile unsigned*)&p.ctrl->done) return;
  constexpr unsigned FULL = 0xffffffffu;
  const unsigned epoch = p.ctrl->epoch;
  const unsigned long long seed = p.ctrl->seed;
  const bool carry = p.ctrl->carry != 0;
  const double rho = C.p[0];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned le_mask = 0xffffffffu >> (31 - lane);   // lanes 0..lane
  const unsigned long long tbase = ((unsigned long long)blockIdx.x * kWWarps + warp) * kTasksPerWarp;
  double2* T_sid = a.t.sid + tbase;
  double* T_lam = M::kHasLam ? a.t.lam + tbase : nullptr;
  unsigned short* T_own = a.t.owner + tbase;
  // this warp's rows of the shared arrays (base addresses computed once)
  typename M::Owner* w_own = s_own[warp];
  int* w_start = s_start[warp];
  int* w_push = s_push[warp];
  int* w_det = s_det[warp];
  int* w_ovn = s_ovn[warp];
  int* w_ovtop = &s_ovtop[warp];
  if (threadIdx.x == 0) s_taskcap = 0;
  // round scratch starts cleared; afterwards every owner clears its own entries
  // when it reads them, and start markers carry the round number
  w_start[lane] = -1;
  w_push[lane] = 0;
  w_det[lane] = 0;
  w_ovn[lane] = 0;
  __syncthreads();
#if !SMC_LRW_FASTMAP
  unsigned stamp = 0;                        // round number of this warp (start markers)
#endif

  double2* w_tsk = s_tsk[warp];
  double* w_tlam = s_tlam[warp];
  // task records: the bottom kSm slots of each owner's segment live in shared
  // memory (small stacks never leave the SM), the rest in this warp's region
  auto put = [&](unsigned slot, double s0, double lam0, unsigned long long id) {
    const double2 v = make_double2(s0, __longlong_as_double((long long)id));
    if (kSm > 0 && slot < kWSegSlots && (int)(slot % kWSeg) < kSm) {
      const int k = (int)(slot / kWSeg) * kSm + (int)(slot % kWSeg);
      w_tsk[k] = v;
      if (M::kHasLam) w_tlam[k] = lam0;
      return;
    }
    T_sid[slot] = v;
    if (M::kHasLam) T_lam[slot] = lam0;
  };
  auto get = [&](unsigned slot, double2& v, double& lam0) {
    if (kSm > 0 && slot < kWSegSlots && (int)(slot % kWSeg) < kSm) {
      const int k = (int)(slot / kWSeg) * kSm + (int)(slot % kWSeg);
      v = w_tsk[k];
      if (M::kHasLam) lam0 = w_tlam[k];
      return;
    }
    v = T_sid[slot];
    if (M::kHasLam) lam0 = T_lam[slot];
  };
  // overflow slot for owner o (-1: the warp's stack is full -> task-cap error)
  auto ovf_slot = [&](int o) -> int {
    const int q = atomicAdd(w_ovtop, 1);
    if (q >= kWOvf) { s_taskcap = 1; return -1; }
    const int slot = (int)kWSegSlots + q;
    T_own[slot] = (unsigned short)o;
    return slot;
  };

  long long key = LLONG_MIN;
  unsigned n_end = 0, n_start = 0, drw = 0, ovf = 0, roots = 0, guard = 0;   // per lane (32-bit: fewer registers)
  bool bad = false;
  unsigned max_rounds = 0, max_nodes = 0;

  for (;;) {
    unsigned batch = 0;
    if (lane == 0) {
      batch = atomicAdd(&p.ctrl->batch, 1u);
      *w_ovtop = 0;
    }
    batch = __shfl_sync(FULL, batch, 0);
    if (batch >= a.n_batches) break;
    const unsigned long long bbase = (unsigned long long)batch * 32;
    const unsigned long long i = bbase + lane;
    const bool valid = i < p.n_local;
    // ---------------- phase 1: the particle's own stream (owner = this lane)
    int c = 0;                       // tasks in this owner's segment
    int dead = 0;                    // 0 alive, 1 detected, 2 node cap, 3 rate guard
    unsigned nodes = 0;
    double lw = (valid && carry) ? p.lw[i] : 0.0;   // R-19 carried weights
    int K = 0;
    bool act = false, alive_end = false;
    __syncwarp();
    if (valid) {
      typename M::State st;
      if (p.lazy) {                              // deferred gather: from the ancestor's slot
        const unsigned long long si = gmap_src(p, i);
        M::load(st, p.src_planes, p.n_local, si);
        relocate<M>(st, p.src_planes, p.planes, p.n_local, si, i);
      } else {
        M::load(st, p.planes, p.n_local, i);
      }
      if (M::pc(st) != kStop) {
        act = true;
        ++n_start;
        Rng r(seed, (uint32_t)(p.shard_base + i), epoch);
        auto push = [&](double s0, double lam0, unsigned kk) {
          int slot;
          if (c < kWSeg) slot = lane * kWSeg + c++;
          else slot = ovf_slot(lane);
          if (slot >= 0) put((unsigned)slot, s0, lam0, root_id(kk));
        };
        if (!M::main_part(st, lw, r, C, w_own[lane], K, push)) dead = 3;   // rate guard
        roots += (unsigned)K;
        drw += 2u * r.blk - (r.has_spare ? 1u : 0u);
        M::store(st, p.planes, p.n_local, i);
      } else if (p.lazy) {
        M::store(st, p.planes, p.n_local, i);    // finished particles move too
      }
      alive_end = M::pc(st) != kStop;
    }
    __syncwarp();
    // ---------------- phase 2: warp-synchronous rounds
    unsigned rounds = 0;
    for (;;) {
      if (dead) c = 0;                                  // a dead owner drops its stack
      const int ov = min(*(volatile int*)w_ovtop, kWOvf);
      const int n_act = __popc(__ballot_sync(FULL, c > 0));
      if (n_act == 0 && ov == 0) break;
      // fair share: a heuristic (no result depends on the schedule, R-18)
      const int W = min(kWMax, c_wshare[n_act]);
      const int m = min(c, W);
#if SMC_LRW_FASTMAP
      // lane offsets: inclusive scan of m (0..32) from six bit-sliced ballots
      // (independent, no shuffle chain); the owner of a lane is the last task
      // range starting at or below it: a bitmask of range starts (one
      // redux.sync) and one shared-memory read of (owner, its count) at that start
#if SMC_LRW_BALLOT_SCAN
      int incl = 0, T = 0;
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        const unsigned bb = __ballot_sync(FULL, (m >> b) & 1);
        incl += __popc(bb & le_mask) << b;
        T += __popc(bb) << b;
      }
      T = min(T, 32);
#else
      int incl = m;                                     // shuffle scan (fewer instructions, longer chain)
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += t;
      }
      const int T = min(__shfl_sync(FULL, incl, 31), 32);
#endif
      const int off = incl - m;
      const int me = max(0, min(m, 32 - off));
      if (me > 0) w_start[off] = (c << 5) | lane;
      const unsigned starts = __reduce_or_sync(FULL, me > 0 ? (1u << off) : 0u);
      __syncwarp();
      bool have = false;
      unsigned slot = 0;
      int ow = 0, s0 = 0;
      if (lane < T) {
        s0 = 31 - __clz(starts & le_mask);             // this lane's range start
        const int sv = w_start[s0];
        have = true;
        ow = sv & 31;
        slot = (unsigned)(ow * kWSeg + ((sv >> 5) - 1 - (lane - s0)));
      } else if (lane - T < ov) {
        have = true;
        slot = (unsigned)kWSegSlots + (unsigned)(ov - 1 - (lane - T));
        ow = (int)T_own[slot];
      }
      c -= me;                                          // pops (the owner's base for pushes)
      const int bd = __shfl_sync(FULL, c | (dead << 16), ow);
      const int base_ow = bd & 0xffff;
      const int dead_ow = bd >> 16;
#else
      int incl = m;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += t;
      }
      const int off = incl - m;
      const int T = min(__shfl_sync(FULL, incl, 31), 32);
      const int me = max(0, min(m, 32 - off));
      ++stamp;
      if (me > 0) w_start[off] = (int)((stamp << 5) | (unsigned)lane);
      __syncwarp();
      const int sv = w_start[lane];
      int o = ((unsigned)sv >> 5) == stamp ? (sv & 31) : -1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {               // owner of lane = last start at or below it
        const int t = __shfl_up_sync(FULL, o, d);
        if (lane >= d) o = max(o, t);
      }
      // lane -> task: own-segment tasks first (lanes [0, T)), then the overflow stack
      const int osrc = max(o, 0);
      const int c_o = __shfl_sync(FULL, c, osrc);
      const int off_o = __shfl_sync(FULL, off, osrc);
      bool have = false;
      unsigned slot = 0;
      int ow = 0;
      if (lane < T) {
        have = true;
        ow = o;
        slot = (unsigned)(o * kWSeg + (c_o - 1 - (lane - off_o)));
      } else if (lane - T < ov) {
        have = true;
        slot = (unsigned)kWSegSlots + (unsigned)(ov - 1 - (lane - T));
        ow = (int)T_own[slot];
      }
      c -= me;                                          // pops (the owner's base for pushes)
      const int base_ow = __shfl_sync(FULL, c, ow);
      const int dead_ow = __shfl_sync(FULL, dead, ow);
#endif
      const bool run = have && dead_ow == 0;
      // read the popped records before any lane pushes: pushes reuse the
      // popped slots (segment: from the owner's base up; overflow: from the
      // new top up)
      double2 rec = make_double2(0.0, 0.0);
      double tl = 0.0;
      if (run) get(slot, rec, tl);
      if (lane == 0) *w_ovtop = ov - min(ov, 32 - T);
      __syncwarp();
#if SMC_LRW_FASTMAP && SMC_LRW_BALLOTPUSH
      // segment lanes (lane < T: contiguous per owner) report births and
      // detections by ballot: a birth's rank among its owner's births gives its
      // push slots, the owner reads its counts from its own lane range — no
      // shared-memory atomics; tasks from the overflow stack keep the atomic
      // path and push to the overflow stack
      int res = -1;
      NodeOut out;
      if (run) {
        const uint32_t n_owner = (uint32_t)(p.shard_base + bbase + ow);
        drw += 2;
        res = M::node(rec.x, tl, (unsigned long long)__double_as_longlong(rec.y), w_own[ow],
                      n_owner, epoch, seed, rho, out);
        if (M::kHasLam && (res == NODE_BIRTH || res == NODE_GUARD)) drw += 2;   // daughters' noise block
      }
      const bool segl = lane < T;
      const unsigned bmask = __ballot_sync(FULL, segl && res == NODE_BIRTH);
      const unsigned dmask = __ballot_sync(FULL, segl && res == NODE_DETECTED);
      const unsigned gmask = __ballot_sync(FULL, segl && res == NODE_GUARD);
      if (segl && res == NODE_BIRTH) {
        const int b = base_ow + 2 * __popc(bmask & (le_mask >> 1) & (0xffffffffu << s0));
        const int s1 = b < kWSeg ? ow * kWSeg + b : ovf_slot(ow);
        const int s2 = b + 1 < kWSeg ? ow * kWSeg + b + 1 : ovf_slot(ow);
        if (s1 >= 0) put((unsigned)s1, out.s2, out.lb, out.idb);
        if (s2 >= 0) put((unsigned)s2, out.s2, out.la, out.ida);   // first daughter on top
      } else if (run && !segl) {                        // a task from the overflow stack
        atomicAdd(&w_ovn[ow], 1);
        if (res == NODE_DETECTED || res == NODE_GUARD) {
          atomicCAS(&w_det[ow], 0, res == NODE_GUARD ? 3 : 1);
        } else if (res == NODE_BIRTH) {
          const int s1 = ovf_slot(ow), s2 = ovf_slot(ow);
          if (s1 >= 0) put((unsigned)s1, out.s2, out.lb, out.idb);
          if (s2 >= 0) put((unsigned)s2, out.s2, out.la, out.ida);
        }
      }
      __syncwarp();
      // owner updates: its lane range [off, off + me) of this round
      const unsigned rmask = me > 0 ? ((me >= 32 ? 0xffffffffu : ((1u << me) - 1u)) << off) : 0u;
      int dc = (dmask & rmask) ? 1 : ((gmask & rmask) ? 3 : 0);
      const int pushed = 2 * __popc(bmask & rmask);
      int ovn = 0;
      if (ov) {                                         // (warp-uniform) overflow tasks this round
        ovn = w_ovn[lane];
        const int dco = w_det[lane];
        w_ovn[lane] = 0;
        w_det[lane] = 0;
        if (!dc) dc = dco;
      }
      if (dead == 0) {
        nodes += (unsigned)(me + ovn);
        if (dc) dead = dc;
        else if (nodes > kSideNodeCap) dead = 2;
      }
#else
      if (run) {
        if (slot >= kWSegSlots) atomicAdd(&w_ovn[ow], 1);
        const uint32_t n_owner = (uint32_t)(p.shard_base + bbase + ow);
        drw += 2;
        NodeOut out;
        const int res = M::node(rec.x, tl, (unsigned long long)__double_as_longlong(rec.y), w_own[ow],
                                n_owner, epoch, seed, rho, out);
        if (M::kHasLam && (res == NODE_BIRTH || res == NODE_GUARD)) drw += 2;   // daughters' noise block
        if (res == NODE_DETECTED || res == NODE_GUARD) {
          atomicCAS(&w_det[ow], 0, res == NODE_GUARD ? 3 : 1);
        } else if (res == NODE_BIRTH) {
          const int b = base_ow + atomicAdd(&w_push[ow], 2);
          const int s1 = b < kWSeg ? ow * kWSeg + b : ovf_slot(ow);
          const int s2 = b + 1 < kWSeg ? ow * kWSeg + b + 1 : ovf_slot(ow);
          if (s1 >= 0) put((unsigned)s1, out.s2, out.lb, out.idb);
          if (s2 >= 0) put((unsigned)s2, out.s2, out.la, out.ida);   // first daughter on top
        }
      }
      __syncwarp();
      // owner updates
#if SMC_LRW_OVN_UNIFORM
      int ovn = 0;
      if (ov) {                                         // (warp-uniform) overflow tasks this round
        ovn = w_ovn[lane];
        w_ovn[lane] = 0;
      }
      const int dc = w_det[lane], pushed = w_push[lane];
#else
      const int ovn = w_ovn[lane], dc = w_det[lane], pushed = w_push[lane];
      w_ovn[lane] = 0;
#endif
      w_det[lane] = 0;
      w_push[lane] = 0;
      if (dead == 0) {
        nodes += (unsigned)(me + ovn);
        if (dc) dead = dc;
        else if (nodes > kSideNodeCap) dead = 2;
      }
#endif
      c = min(c + pushed, kWSeg);
      ++rounds;
      __syncwarp();
    }
    max_rounds = rounds > max_rounds ? rounds : max_rounds;
    max_nodes = nodes > max_nodes ? nodes : max_nodes;
    // ---------------- phase 3: finish the particle
    if (valid) {
      double w = lw;
      if (act) {
        if (dead) {
          w = -INFINITY;
          if (dead == 3) ++guard;
          if (dead == 2) {
            ++ovf;
            atomicMin(&p.ctrl->first_err, (unsigned long long)(p.shard_base + i));
          }
        } else {
          for (int k = 0; k < K; ++k) w = w + kLn2;
        }
      }
      p.lw[i] = w;
      if (alive_end) ++n_end;
      bad |= isnan(w) || w == INFINITY;
      const long long kk = order_key(w);
      key = kk > key ? kk : key;
    }
  }
  // ---------------- epilogue: warp sums, then one set of atomics per CTA
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const long long t = __shfl_xor_sync(FULL, key, d);
    key = t > key ? t : key;
  }
  n_end = __reduce_add_sync(FULL, n_end);
  n_start = __reduce_add_sync(FULL, n_start);
  drw = __reduce_add_sync(FULL, drw);
  ovf = __reduce_add_sync(FULL, ovf);
  roots = __reduce_add_sync(FULL, roots);
  guard = __reduce_add_sync(FULL, guard);
  max_nodes = __reduce_max_sync(FULL, max_nodes);
  bad = __any_sync(FULL, bad);
  if (lane == 0) {
    s_key[warp] = key;
    s_acc[0][warp] = n_end;
    s_acc[1][warp] = n_start;
    s_acc[2][warp] = drw;
    if (ovf) atomicAdd(&p.ctrl->overflow, (unsigned long long)ovf);
    if (guard) atomicAdd(&p.ctrl->guard_kills, (unsigned long long)guard);
    if (roots) atomicAdd(&p.ctrl->side_roots, (unsigned long long)roots);
    atomicMax(&p.ctrl->max_side_nodes, max_nodes);
    atomicMax(&p.ctrl->max_rounds, max_rounds);
  }
  const int any_bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    long long k = s_key[0];
    unsigned long long e = 0, st = 0, dr = 0;
    for (int w = 0; w < kWWarps; ++w) {
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
}

}  // namespace smc
