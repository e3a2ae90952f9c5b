// engine.cu — host engine and C ABI of libsmc (include/smc.h).
//
// The engine owns the SoA particle buffers (double-buffered planes, lw, anc)
// of one or more shards and drives the epoch loop:
//   propagate<M> (all shards) -> all-gather record A (max, alive, flags)
//   -> reduce (tile sums, shard total) -> all-gather record B (shard totals)
//   -> anc_gather (ancestors + fused gather/migration into destination
//      shards) -> barrier -> finalize (log Z, termination, epoch advance)
// Shards are either virtual (several in one process, one GPU) or one per
// process (NCCL or a host all-gather callback for the 16-byte records; CUDA
// IPC peer pointers for the migration stores).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "smc.h"
#include "kernels.cuh"
#include "lineage.cuh"
#include "lineage_warp.cuh"

using namespace smc;

namespace {

thread_local std::string g_last_error = "";

// --------------------------------------------------------------------------
// NCCL, loaded at run time (the process normally already holds torch's copy)
struct Nccl {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (loaded) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { err = std::string("cannot load libnccl.so.2: ") + dlerror(); return false; }
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !AllGather || !AllReduce || !CommDestroy) {
      err = "libnccl.so.2 lacks required symbols";
      return false;
    }
    loaded = true;
    return true;
  }
};
Nccl g_nccl;

struct Shard {
  int id = 0;                      // global shard index (rank for sharded runs)
  unsigned long long base = 0;     // global index of local particle 0
  char* ipc_block = nullptr;       // planes[0], planes[1], anc (one allocation, IPC-exportable)
  uint4* planes[2] = {nullptr, nullptr};
  uint32_t* anc = nullptr;
  double* lw = nullptr;
  u128* tile_sum = nullptr;
  u128* tile_excl = nullptr;
  U192* tile_q2 = nullptr;
  Ctrl* ctrl = nullptr;
  uint32_t* scratch = nullptr;     // in-place resampling (R-21): offs, hole_dst, extra_src, tile_nz[2]
  uint4** d_dst_planes[2] = {nullptr, nullptr};  // device arrays [world]
  uint32_t** d_dst_anc = nullptr;                 // device array [world]
};

enum CommKind { COMM_LOCAL = 0, COMM_NCCL = 1, COMM_CALLBACK = 2 };

}  // namespace

struct smc_ctx {
  int kind = 0;
  bool lineage = false;           // §R-18 lineage-keyed side trees (SMC_FLAG_LINEAGE_RNG)
  bool analytic = false;          // §R-20 CRBD with 2E(t) per hidden event (SMC_FLAG_ANALYTIC_UNDETECTED)
  bool inplace = false;           // §R-21 permuted ancestors, one state buffer (SMC_FLAG_INPLACE)
  int fused_grid = 0;             // > 0: single-shard resampling in one cooperative launch
  int fused_ipt = 0;              // particles per thread of resample_fused_kernel
  size_t fused_smem = 0;
  void** d_call_tab = nullptr;    // smc_resample_device: {state_out, anc} of the current call
  u128* d_blk_sum = nullptr;      // [fused_grid]
  U192* d_blk_q2 = nullptr;       // [fused_grid]
  bool stack_prefix = true;       // §R-22 copy only the used stack prefix (env SMC_NO_STACK_PREFIX=1: off, diagnostics)
  int lr_grid = 0;                // persistent grid of the cooperative kernel
  bool lr_warp = true;            // warp-level cooperative kernel (env SMC_LR_KERNEL=cta: CTA rounds)
  bool lazy = false;              // deferred gather (§7.7): one shard, out of place (env SMC_EAGER_GATHER=1: off)
  int prop_grid = 0;              // resident-CTA grid of propagate_kernel<M> (grid-stride)
  TaskArrays tasks{};
  int planes = 0;                 // 16-byte planes per particle
  uint32_t flags = 0;
  unsigned long long n_per = 0;   // particles per shard
  unsigned long long n_total = 0;
  int world = 1, rank = 0;        // world = number of shards in the run
  int n_local_shards = 1;         // shards held by this handle
  int n_tiles = 0;
  int chunk_tiles = 1, n_chunks = 0;   // reduce_kernel: one warp per chunk of tiles
  int items = kItems;             // particles per thread in a resampling tile
  unsigned long long seed = 0;
  ModelConst mc{};
  double* d_table = nullptr;
  std::vector<double> h_table;
  double* d_logfact = nullptr;    // SEIR: lgamma(k+1) table (model setup, host libm)
  RecA* d_recA = nullptr;         // [2][world]
  RecB* d_recB = nullptr;         // [2][world]
  unsigned ess_a = 1, ess_b = 1;  // ESS threshold (R-19)
  int* d_barrier = nullptr;
  std::vector<Shard> shards;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  CommKind comm = COMM_LOCAL;
  ncclComm_t nccl = nullptr;
  int (*cb_allgather)(const void*, void*, uint64_t, void*) = nullptr;
  void* cb_user = nullptr;
  std::vector<void*> ipc_opened;
  bool ipc_ready = true;
  Ctrl* h_ctrl = nullptr;         // pinned
  unsigned long long enq = 0;     // epochs enqueued since reset
  bool started = false;
  bool timing = false;            // per-phase CUDA-event timing
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t rev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};   // resample-only path
  double ms_kernel[4] = {0, 0, 0, 0};   // max, reduce, anc_gather, finalize (resample-only path)
  double ms_propagate = 0.0, ms_resample = 0.0;
  unsigned long long timed_epochs = 0;
  bool use_graph = true;          // whole run as one graph launch (WHILE conditional node)
  cudaGraphExec_t graph_exec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaStream_t cap_stream = nullptr;
  int status = SMC_OK;
  std::string err;
};

namespace {

int fail(smc_ctx* h, int code, const std::string& msg) {
  if (h) { h->status = code; h->err = msg; }
  g_last_error = msg;
  return code;
}
#define CU(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(h, SMC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

// ---- model setup: traversal tables ------------------------
struct TreeIn {
  int M = 0, root = -1;
  std::vector<int> parent, left, right;
  std::vector<double> age;
  std::vector<int> tips;   // tips below each node
};
bool parse_tree(const double* d, uint64_t len, TreeIn& T, std::string& err) {
  if (!d || len < 2) { err = "tree data missing"; return false; }
  T.M = (int)d[0];
  T.root = (int)d[1];
  if (T.M < 3 || len != (uint64_t)(2 + 4 * T.M) || T.root < 0 || T.root >= T.M) {
    err = "tree data must be [M, root, (parent,left,right,age) x M]";
    return false;
  }
  T.parent.resize(T.M); T.left.resize(T.M); T.right.resize(T.M); T.age.resize(T.M);
  for (int i = 0; i < T.M; ++i) {
    T.parent[i] = (int)d[2 + 4 * i];
    T.left[i] = (int)d[3 + 4 * i];
    T.right[i] = (int)d[4 + 4 * i];
    T.age[i] = d[5 + 4 * i];
    const bool tip = T.left[i] < 0;
    if (tip != (T.right[i] < 0) || T.left[i] >= T.M || T.right[i] >= T.M ||
        T.parent[i] >= T.M || (T.parent[i] < 0) != (i == T.root)) {
      err = "malformed tree node";
      return false;
    }
  }
  if (T.left[T.root] < 0) { err = "root must be internal"; return false; }
  for (int v = 0; v < T.M; ++v)      // child pointers and parent pointers agree
    if (T.left[v] >= 0 && (T.parent[T.left[v]] != v || T.parent[T.right[v]] != v)) {
      err = "tree parent/child pointers disagree";
      return false;
    }
  // tip counts by an explicit post-order (iterative; a cycle stops it at M nodes)
  T.tips.assign(T.M, 0);
  std::vector<int> order, st{T.root};
  while (!st.empty()) {
    if ((int)order.size() >= T.M) { err = "tree is not connected / has cycles"; return false; }
    int v = st.back(); st.pop_back();
    order.push_back(v);
    if (T.left[v] >= 0) { st.push_back(T.left[v]); st.push_back(T.right[v]); }
  }
  if ((int)order.size() != T.M) { err = "tree is not connected / has cycles"; return false; }
  for (int k = T.M - 1; k >= 0; --k) {
    int v = order[k];
    T.tips[v] = T.left[v] < 0 ? 1 : T.tips[T.left[v]] + T.tips[T.right[v]];
  }
  return true;
}
// CRBD: preorder, left child first; rows (t_parent, t_child, internal).
void crbd_table(const TreeIn& T, std::vector<double>& out) {
  std::vector<int> st{T.right[T.root], T.left[T.root]};
  while (!st.empty()) {
    const int c = st.back(); st.pop_back();
    out.push_back(T.age[T.parent[c]]);
    out.push_back(T.age[c]);
    out.push_back(T.left[c] >= 0 ? 1.0 : 0.0);
    if (T.left[c] >= 0) { st.push_back(T.right[c]); st.push_back(T.left[c]); }
  }
}
// ClaDS2: preorder visiting the child with fewer tips first (ties: left);
// rows (t_parent, t_child, internal, first_left at the child).  Returns the
// maximum number of pending sibling rates.
int clads2_table(const TreeIn& T, std::vector<double>& out, bool& root_first_left) {
  auto first_left = [&](int v) { return T.tips[T.left[v]] <= T.tips[T.right[v]]; };
  root_first_left = first_left(T.root);
  // explicit stack of branch children to emit, with the pending depth
  struct Item { int child; int pend; };
  std::vector<Item> st;
  int maxpend = 1;
  auto push_children = [&](int v, int pend) {
    const bool fl = first_left(v);
    const int first = fl ? T.left[v] : T.right[v], second = fl ? T.right[v] : T.left[v];
    // second is pending while the first subtree is traversed
    st.push_back({second, pend});
    st.push_back({first, pend + 1});
    maxpend = std::max(maxpend, pend + 1);
  };
  push_children(T.root, 0);
  while (!st.empty()) {
    Item it = st.back(); st.pop_back();
    const int c = it.child;
    out.push_back(T.age[T.parent[c]]);
    out.push_back(T.age[c]);
    out.push_back(T.left[c] >= 0 ? 1.0 : 0.0);
    out.push_back(T.left[c] >= 0 && first_left(c) ? 1.0 : 0.0);
    if (T.left[c] >= 0) push_children(c, it.pend);
  }
  return maxpend;
}

int setup_model(smc_ctx* h, const smc_model* m) {
  if (!m) return fail(h, SMC_EINVAL, "model is NULL");
  h->kind = m->kind;
  h->flags = m->flags;
  h->analytic = (m->flags & SMC_FLAG_ANALYTIC_UNDETECTED) != 0;
  h->inplace = (m->flags & SMC_FLAG_INPLACE) != 0;
  {
    const char* e = std::getenv("SMC_NO_STACK_PREFIX");
    h->stack_prefix = !(e && e[0] == '1');
  }
  if (h->analytic && m->kind != SMC_CRBD)
    return fail(h, SMC_EINVAL, "SMC_FLAG_ANALYTIC_UNDETECTED applies to SMC_CRBD only");
  h->lineage = !h->analytic && (m->flags & SMC_FLAG_LINEAGE_RNG) &&
               (m->kind == SMC_CRBD || m->kind == SMC_CLADS2);
  for (int i = 0; i < 12; ++i) h->mc.p[i] = 0.0;
  auto P = [&](int i, double dflt) { return (m->params && i < m->n_params) ? m->params[i] : dflt; };
  std::string err;
  switch (m->kind) {
    case SMC_CRBD: {
      TreeIn T;
      if (!parse_tree(m->data, m->data_len, T, err)) return fail(h, SMC_EINVAL, err);
      crbd_table(T, h->h_table);
      h->mc.n = (int)(h->h_table.size() / 3);
      h->mc.p[0] = P(0, 1.0); h->mc.p[1] = P(1, -1.0); h->mc.p[2] = P(2, -1.0);
      h->planes = Crbd::kPlanes;
      break;
    }
    case SMC_CLADS2: {
      TreeIn T;
      if (!parse_tree(m->data, m->data_len, T, err)) return fail(h, SMC_EINVAL, err);
      bool rfl = true;
      const int maxpend = clads2_table(T, h->h_table, rfl);
      if (maxpend > Clads2::kPend)
        return fail(h, SMC_EINVAL, "tree needs more than 6 pending sibling rates");
      h->mc.n = (int)(h->h_table.size() / 4);
      for (int i = 0; i < 5; ++i) h->mc.p[i] = P(i, i == 0 ? 1.0 : -1.0);
      h->mc.p[5] = rfl ? 1.0 : 0.0;
      h->planes = Clads2::kPlanes;
      break;
    }
    case SMC_SEIR: {
      if (!m->data || m->data_len == 0) return fail(h, SMC_EINVAL, "SEIR needs the case series");
      h->h_table.assign(m->data, m->data + m->data_len);
      h->mc.n = (int)m->data_len;
      if (m->n_params >= 6 && m->params[0] >= 0.0) {
        for (int i = 0; i < 6; ++i) h->mc.p[i] = m->params[i];
      } else {
        h->mc.p[0] = -1.0;
      }
      h->mc.p[6] = P(6, 7370.0);
      h->mc.p[7] = P(7, 10.0 * h->mc.p[6]);
      h->mc.p[8] = P(8, 0.0);
      h->mc.p[9] = P(9, 0.0);
      if (h->mc.p[6] < 1 || h->mc.p[7] < 0 || h->mc.p[8] < 0 || h->mc.p[9] < 0 ||
          h->mc.p[8] > h->mc.p[6] - 1 || h->mc.p[7] + h->mc.p[9] > 2e8)
        return fail(h, SMC_EINVAL, "bad SEIR population");
      h->planes = Seir::kPlanes;
      break;
    }
    case SMC_GEOMETRIC:
      h->mc.p[0] = P(0, 0.5); h->mc.p[1] = P(1, 1.5);
      h->planes = Geometric::kPlanes;
      break;
    case SMC_FIG3: {
      const double pl = P(0, 0.5), p3 = P(1, 0.3), w1 = P(2, 2.0), w2 = P(3, 1.2), w3 = P(4, 1.2),
                   w4 = P(5, 0.5);
      if (!(pl >= 0 && p3 >= 0 && pl + p3 <= 1 && w1 > 0 && w2 > 0 && w3 > 0 && w4 > 0))
        return fail(h, SMC_EINVAL, "bad Fig. 3 parameters");
      h->mc.p[0] = pl; h->mc.p[1] = p3;
      h->mc.p[6] = std::log(w1); h->mc.p[7] = std::log(w2); h->mc.p[8] = std::log(w3);
      h->mc.p[9] = std::log(w4);
      h->planes = Fig3::kPlanes;
      break;
    }
    case SMC_STACKF: {
      if (m->data && m->data_len) h->h_table.assign(m->data, m->data + m->data_len);
      h->mc.n = (int)m->data_len;
      const double p0 = P(0, 2.0), prec = P(1, 2.0), sg = P(2, 0.5), cap = P(3, 768.0);
      if (!(p0 > 0 && prec > 0 && sg > 0) || cap < 48 || cap > 65536 || std::fmod(cap, 16.0) != 0.0)
        return fail(h, SMC_EINVAL, "bad STACKF parameters (cap: multiple of 16 in [48, 65536])");
      h->mc.p[0] = p0; h->mc.p[1] = prec; h->mc.p[2] = sg; h->mc.p[3] = cap;
      h->planes = 1 + (int)cap / 16;
      break;
    }
    case SMC_SSM:
      if (!m->data || m->data_len == 0) return fail(h, SMC_EINVAL, "SSM needs observations");
      h->h_table.assign(m->data, m->data + m->data_len);
      h->mc.n = (int)m->data_len;
      h->mc.p[0] = P(0, 0.0); h->mc.p[1] = P(1, 100.0); h->mc.p[2] = P(2, 2.0);
      h->mc.p[3] = P(3, 1.0); h->mc.p[4] = P(4, 5.0);
      h->planes = Ssm::kPlanes;
      break;
    case SMC_CONSTW:
      h->mc.p[0] = P(0, std::log(3.0)); h->mc.p[1] = P(1, 1.0);
      if (h->mc.p[1] < 1) return fail(h, SMC_EINVAL, "CONSTW needs K >= 1");
      h->planes = Constw::kPlanes;
      break;
    case SMC_RESAMPLE_BENCH:
      if (m->state_bytes == 0 || m->state_bytes % 16 || m->state_bytes > 512)
        return fail(h, SMC_EINVAL, "state_bytes must be a multiple of 16 in [16, 512]");
      h->planes = (int)(m->state_bytes / 16);
      break;
    default:
      return fail(h, SMC_EINVAL, "unknown model kind");
  }
  if (m->kind == SMC_CRBD || m->kind == SMC_CLADS2) {
    if (h->mc.n < 2) return fail(h, SMC_EINVAL, "tree has too few branches");
  }
  return SMC_OK;
}

int alloc_shard(smc_ctx* h, Shard& s) {
  const unsigned long long n = h->n_per;
  const size_t plane_bytes = (size_t)h->planes * n * 16;
  const size_t anc_off = (h->inplace ? 1 : 2) * plane_bytes;   // in place: one state buffer
  const size_t block = anc_off + n * sizeof(uint32_t);
  CU(cudaMalloc(&s.ipc_block, block));
  s.planes[0] = (uint4*)s.ipc_block;
  s.planes[1] = h->inplace ? s.planes[0] : (uint4*)(s.ipc_block + plane_bytes);
  s.anc = (uint32_t*)(s.ipc_block + anc_off);
  if (h->inplace) CU(cudaMalloc(&s.scratch, (3 * n + 2 * (size_t)h->n_tiles) * sizeof(uint32_t)));
  CU(cudaMalloc(&s.lw, n * sizeof(double)));
  CU(cudaMalloc(&s.tile_sum, (size_t)h->n_tiles * sizeof(u128)));
  CU(cudaMalloc(&s.tile_excl, (size_t)h->n_tiles * sizeof(u128)));
  CU(cudaMalloc(&s.tile_q2, (size_t)h->n_tiles * sizeof(U192)));
  CU(cudaMalloc(&s.ctrl, sizeof(Ctrl)));
  CU(cudaMalloc(&s.d_dst_planes[0], h->world * sizeof(uint4*)));
  CU(cudaMalloc(&s.d_dst_planes[1], h->world * sizeof(uint4*)));
  CU(cudaMalloc(&s.d_dst_anc, h->world * sizeof(uint32_t*)));
  return SMC_OK;
}

// Destination pointer tables: for virtual shards every shard's buffers are
// local; for sharded runs non-local entries are IPC-opened peer pointers.
int write_dst_tables(smc_ctx* h, const std::vector<uint4*>& p0, const std::vector<uint4*>& p1,
                     const std::vector<uint32_t*>& anc) {
  for (auto& s : h->shards) {
    CU(cudaMemcpy(s.d_dst_planes[0], p0.data(), h->world * sizeof(uint4*), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(s.d_dst_planes[1], p1.data(), h->world * sizeof(uint4*), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(s.d_dst_anc, anc.data(), h->world * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  }
  return SMC_OK;
}

int reset_device(smc_ctx* h) {
  Ctrl c{};
  c.logz = 0.0;
  c.last_inc = 0.0;
  c.first_err = ~0ull;
  c.gmap_id = 1;                        // first epoch: every particle reads its own slot
  c.seed = h->seed;
  c.ess_a = h->ess_a;
  c.ess_b = h->ess_b;
  std::vector<RecA> ra(2 * h->world);
  for (auto& r : ra) { r.key = LLONG_MIN; r.alive = 0; r.flags = 0; }
  CU(cudaMemcpyAsync(h->d_recA, ra.data(), ra.size() * sizeof(RecA), cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemsetAsync(h->d_recB, 0, 2 * h->world * sizeof(RecB), h->stream));
  for (auto& s : h->shards) {
    CU(cudaMemcpyAsync(s.ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream));
    // pc = b0 = 0 and all fields zero; lw = 0; anc = identity
    CU(cudaMemsetAsync(s.planes[0], 0, (size_t)h->planes * h->n_per * 16, h->stream));
    if (h->lazy)   // the first epoch reads the other buffer (deferred gather)
      CU(cudaMemsetAsync(s.planes[1], 0, (size_t)h->planes * h->n_per * 16, h->stream));
    CU(cudaMemsetAsync(s.lw, 0, h->n_per * sizeof(double), h->stream));
  }
  for (auto& s : h->shards) {
    const unsigned g = (unsigned)std::min<unsigned long long>((h->n_per + 255) / 256, 4096ull);
    iota_kernel<<<g, 256, 0, h->stream>>>(s.anc, h->n_per, s.base);
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->stream));
  std::memset(h->h_ctrl, 0, sizeof(Ctrl));
  h->ms_propagate = h->ms_resample = 0.0;
  for (double& v : h->ms_kernel) v = 0.0;
  h->timed_epochs = 0;
  h->enq = 0;
  h->started = false;
  h->status = SMC_OK;
  h->err.clear();
  return SMC_OK;
}

// Fused single-launch resampling (resample_fused_kernel): one shard in this
// process, out of place, and the shard's particles fit the co-resident grid's
// shared memory at 12 B each (q and O_k).  Env SMC_NO_FUSED_RESAMPLE=1 keeps
// the split reduce / anc_gather / finalize path (A/B measurements).
const void* fused_fn(int planes) {
  switch (planes) {
    case 1: return (const void*)resample_fused_kernel<1>;
    case 2: return (const void*)resample_fused_kernel<2>;
    case 4: return (const void*)resample_fused_kernel<4>;
    case 6: return (const void*)resample_fused_kernel<6>;
    case 8: return (const void*)resample_fused_kernel<8>;
    default: return (const void*)resample_fused_kernel<0>;
  }
}
// cudaFuncAttributeMaxDynamicSharedMemorySize is per kernel and process-wide:
// only ever raise it, so a later, smaller handle cannot lower the cap below
// what an earlier handle's launches request.
cudaError_t raise_smem_cap(const void* fn, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, size_t> cap;
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = cap[fn];
  if (smem <= c) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) c = smem;
  return e;
}
int plan_fused(smc_ctx* h) {
  h->fused_grid = 0;
  const char* off = std::getenv("SMC_NO_FUSED_RESAMPLE");
  if ((off && off[0] == '1') || h->world != 1 || h->n_local_shards != 1 || h->inplace)
    return SMC_OK;
  int dev = 0, sms = 0, optin = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int coop = 0;
  CU(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return SMC_OK;
  const void* fn = fused_fn(h->planes);
  const unsigned long long n = h->n_per;
  for (int per_sm = SMC_FUSED_MINB; per_sm >= 1; --per_sm) {
    const unsigned long long g0 = (unsigned long long)sms * per_sm;
    const unsigned long long ipt = std::max(1ull, (n + g0 * kFT - 1) / (g0 * kFT));
    const size_t smem = (size_t)ipt * kFT * 12 + 4;      // q and O_k per particle
    if (smem + 8192 > (size_t)optin) continue;
    CU(raise_smem_cap(fn, smem));
    int nb = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kFT, smem));
    if (nb < per_sm) continue;
    const unsigned long long grid = (n + ipt * kFT - 1) / (ipt * kFT);
    if (grid > (unsigned long long)kMaxFusedGrid) continue;
    h->fused_grid = (int)grid;
    h->fused_ipt = (int)ipt;
    h->fused_smem = smem;
    CU(cudaMalloc(&h->d_blk_sum, grid * sizeof(u128)));
    CU(cudaMalloc(&h->d_blk_q2, grid * sizeof(U192)));
    return SMC_OK;
  }
  return SMC_OK;
}

int common_init(smc_ctx* h, const smc_model* m, unsigned long long n_per, int world, int rank,
                int n_local_shards, unsigned long long seed) {
  int rc = setup_model(h, m);
  if (rc) return rc;
  if (n_per == 0) return fail(h, SMC_EINVAL, "n_particles must be >= 1");
  const unsigned long long total = n_per * (unsigned long long)world;
  if (total >= (1ull << 32) || total / world != n_per)
    return fail(h, SMC_EINVAL, "total particles must be < 2^32");
  int dev_count = 0;
  cudaError_t e = cudaGetDeviceCount(&dev_count);
  if (e != cudaSuccess || dev_count == 0)
    return fail(h, SMC_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  h->n_per = n_per;
  h->n_total = total;
  h->world = world;
  h->rank = rank;
  h->n_local_shards = n_local_shards;
  h->seed = seed;
  h->items = n_per <= kSmallN ? kItemsSmall : kItems;
  h->n_tiles = (int)((n_per + (unsigned long long)kThreads * h->items - 1) / ((unsigned long long)kThreads * h->items));
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int target = sms * 3 * (kThreads / 32);      // 3 resident reduce CTAs per SM (85-register cap)
    h->chunk_tiles = std::max(1, (h->n_tiles + target - 1) / target);
    h->n_chunks = (h->n_tiles + h->chunk_tiles - 1) / h->chunk_tiles;
  }
  CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;
  if (!h->h_table.empty()) {
    CU(cudaMalloc(&h->d_table, h->h_table.size() * sizeof(double)));
    CU(cudaMemcpy(h->d_table, h->h_table.data(), h->h_table.size() * sizeof(double),
                  cudaMemcpyHostToDevice));
  }
  h->mc.table = h->d_table;
  h->mc.flags = (int)h->flags;
  h->mc.logfact = nullptr;
  h->mc.n_logfact = 0;
  if (h->kind == SMC_SEIR) {
    // log-factorials for every integer the binomial code can see (populations
    // up to 2^18; larger arguments fall back to the device lgamma)
    const long long nlf = 1 << 18;
    std::vector<double> lf(nlf);
    for (long long k = 0; k < nlf; ++k) lf[k] = std::lgamma((double)k + 1.0);
    CU(cudaMalloc(&h->d_logfact, nlf * sizeof(double)));
    CU(cudaMemcpy(h->d_logfact, lf.data(), nlf * sizeof(double), cudaMemcpyHostToDevice));
    h->mc.logfact = h->d_logfact;
    h->mc.n_logfact = nlf;
  }
  CU(cudaMalloc(&h->d_recA, 2 * world * sizeof(RecA)));
  CU(cudaMalloc(&h->d_recB, 2 * world * sizeof(RecB)));
  CU(cudaMalloc(&h->d_barrier, sizeof(int)));
  CU(cudaMallocHost(&h->h_ctrl, sizeof(Ctrl)));
  if (h->lineage) {
    const char* ek = std::getenv("SMC_LR_KERNEL");
    h->lr_warp = !(ek && std::strcmp(ek, "cta") == 0);
    int per_sm = 0;
    if (h->lr_warp) {
      if (h->kind == SMC_CRBD)
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, propagate_lrw_kernel<CrbdLR>, kWThreads, 0));
      else
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, propagate_lrw_kernel<Clads2LR>, kWThreads, 0));
    } else if (h->kind == SMC_CRBD) {
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, propagate_lr_kernel<CrbdLR>, kLRThreads, 0));
    } else {
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, propagate_lr_kernel<Clads2LR>, kLRThreads, 0));
    }
    int dev = 0, sms = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned long long per_batch = h->lr_warp ? 32ull * kWWarps : (unsigned long long)kOwners;
    const unsigned long long batches = (n_per + per_batch - 1) / per_batch;
    h->lr_grid = (int)std::min<unsigned long long>(batches, (unsigned long long)std::max(1, per_sm) * sms);
    h->tasks.cap = h->lr_warp ? (unsigned)(kWWarps * kTasksPerWarp) : kTasksPerCta;
    const size_t nt = (size_t)h->lr_grid * h->tasks.cap;
    CU(cudaMalloc(&h->tasks.sid, nt * sizeof(double2)));
    if (h->kind == SMC_CLADS2) CU(cudaMalloc(&h->tasks.lam, nt * sizeof(double)));
    CU(cudaMalloc(&h->tasks.owner, nt * sizeof(unsigned short)));
  }
  if (h->inplace && world > 1)
    return fail(h, SMC_EINVAL, "SMC_FLAG_INPLACE needs a single shard (no cross-shard hole matching yet)");
  rc = plan_fused(h);
  if (rc) return rc;
  {
    // deferred gather: the resampling step writes ancestors only and the next
    // propagation reads every state from its ancestor's slot (one shard,
    // out-of-place runs of the models; the CTA cooperative kernel and the
    // resampler-only handles keep the materialised gather)
    // (measured: pays from 4 planes up — SEIR 85.6 -> 81.0 ms/sweep; CRBD's 2
    // planes neutral, Fig. 3's single plane 10% slower — SMC_DEFERRED_GATHER=1
    // forces it on for any model, SMC_EAGER_GATHER=1 off)
    const char* eg = std::getenv("SMC_EAGER_GATHER");
    const char* dg = std::getenv("SMC_DEFERRED_GATHER");
    const bool want = (dg && dg[0] == '1') || h->planes >= 4;
    h->lazy = want && world == 1 && n_local_shards == 1 && !h->inplace && h->kind != SMC_RESAMPLE_BENCH &&
              (!h->lineage || h->lr_warp) && h->stack_prefix && !(eg && eg[0] == '1');
  }
  h->shards.resize(n_local_shards);
  for (int i = 0; i < n_local_shards; ++i) {
    Shard& s = h->shards[i];
    s.id = n_local_shards == world ? i : rank;
    s.base = (unsigned long long)s.id * n_per;
    rc = alloc_shard(h, s);
    if (rc) return rc;
  }
  return SMC_OK;
}

// ---- collectives ------------------------------------------------------------
int allgather_rec(smc_ctx* h, void* d_arr, size_t rec_bytes) {
  // d_arr = [world] records of rec_bytes; this rank filled slot `rank`.
  if (h->comm == COMM_LOCAL) return SMC_OK;   // shards share the array
  if (h->comm == COMM_NCCL) {
    char* base = (char*)d_arr;
    ncclResult_t r = g_nccl.AllGather(base + h->rank * rec_bytes, base, rec_bytes, ncclUint8, h->nccl,
                                      h->stream);
    if (r != ncclSuccess) return fail(h, SMC_ENCCL, "ncclAllGather failed");
    return SMC_OK;
  }
  std::vector<char> send(rec_bytes), recv(rec_bytes * h->world);
  CU(cudaMemcpyAsync(send.data(), (char*)d_arr + h->rank * rec_bytes, rec_bytes, cudaMemcpyDeviceToHost,
                     h->stream));
  CU(cudaStreamSynchronize(h->stream));
  if (h->cb_allgather(send.data(), recv.data(), rec_bytes, h->cb_user) != 0)
    return fail(h, SMC_ENCCL, "allgather callback failed");
  CU(cudaMemcpyAsync(d_arr, recv.data(), recv.size(), cudaMemcpyHostToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return SMC_OK;
}
int barrier(smc_ctx* h) {
  if (h->comm == COMM_LOCAL) return SMC_OK;
  if (h->comm == COMM_NCCL) {
    ncclResult_t r = g_nccl.AllReduce(h->d_barrier, h->d_barrier, 1, ncclInt32, ncclSum, h->nccl, h->stream);
    if (r != ncclSuccess) return fail(h, SMC_ENCCL, "ncclAllReduce (barrier) failed");
    return SMC_OK;
  }
  CU(cudaStreamSynchronize(h->stream));
  int one = 1;
  std::vector<int> all(h->world);
  if (h->cb_allgather(&one, all.data(), sizeof(int), h->cb_user) != 0)
    return fail(h, SMC_ENCCL, "barrier callback failed");
  return SMC_OK;
}

// ---- launches -----------------------------------------------------------------
void set_prop_io(smc_ctx* h, Shard& s, int cur, PropArgs& a) {
  a.planes = s.planes[cur];
  a.lazy = h->lazy ? 1 : 0;
  a.src_planes = h->lazy ? s.planes[cur ^ 1] : s.planes[cur];   // previous epoch's buffer
  a.gmap = s.anc;
}
template <class M>
void launch_prop(smc_ctx* h, Shard& s, int cur) {
  PropArgs a;
  set_prop_io(h, s, cur, a);
  a.lw = s.lw;
  a.n_local = h->n_per;
  a.shard_base = s.base;
  a.recA = h->d_recA;
  a.world = h->world;
  a.rank = s.id;
  a.ctrl = s.ctrl;
  if (!h->prop_grid) {
    // light models: one wave of resident CTAs (the kernel grid-strides), so the
    // epilogue's same-address atomics run once per CTA; uneven models: one CTA
    // per 256 particles.  Occupancy query only, nothing enqueued (safe during
    // graph capture)
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, propagate_kernel<M>, kPThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned long long need = (h->n_per + kPThreads - 1) / kPThreads;
    h->prop_grid = M::kOneWave
        ? (int)std::min<unsigned long long>(need, (unsigned long long)std::max(1, per_sm * sms))
        : (int)need;
  }
  propagate_kernel<M><<<(unsigned)h->prop_grid, kPThreads, 0, h->stream>>>(a, h->mc);
}
template <class M>
void launch_prop_lr(smc_ctx* h, Shard& s, int cur) {
  LRArgs a;
  set_prop_io(h, s, cur, a.p);
  a.p.lw = s.lw;
  a.p.n_local = h->n_per;
  a.p.shard_base = s.base;
  a.p.recA = h->d_recA;
  a.p.world = h->world;
  a.p.rank = s.id;
  a.p.ctrl = s.ctrl;
  a.t = h->tasks;
  if (h->lr_warp) {
    a.n_batches = (unsigned)((h->n_per + 31) / 32);
    propagate_lrw_kernel<M><<<h->lr_grid, kWThreads, 0, h->stream>>>(a, h->mc);
    return;
  }
  a.n_batches = (unsigned)((h->n_per + kOwners - 1) / kOwners);
  propagate_lr_kernel<M><<<h->lr_grid, kLRThreads, 0, h->stream>>>(a, h->mc);
}
void launch_propagate(smc_ctx* h, Shard& s, int cur) {
  if (h->lineage) {
    if (h->kind == SMC_CRBD) launch_prop_lr<CrbdLR>(h, s, cur);
    else launch_prop_lr<Clads2LR>(h, s, cur);
    return;
  }
  switch (h->kind) {
    case SMC_CRBD:
      if (h->analytic) launch_prop<CrbdAE>(h, s, cur);
      else launch_prop<Crbd>(h, s, cur);
      break;
    case SMC_CLADS2: launch_prop<Clads2>(h, s, cur); break;
    case SMC_SEIR: launch_prop<Seir>(h, s, cur); break;
    case SMC_GEOMETRIC: launch_prop<Geometric>(h, s, cur); break;
    case SMC_FIG3: launch_prop<Fig3>(h, s, cur); break;
    case SMC_STACKF: launch_prop<Stackf>(h, s, cur); break;
    case SMC_SSM: launch_prop<Ssm>(h, s, cur); break;
    case SMC_CONSTW: launch_prop<Constw>(h, s, cur); break;
    default: break;
  }
}
ResArgs res_args(smc_ctx* h, Shard& s, const double* lw, const uint4* src, int dst_par) {
  ResArgs a;
  a.lw = lw;
  a.n_local = h->n_per;
  a.shard_base = s.base;
  a.n_total = h->n_total;
  a.world = h->world;
  a.rank = s.id;
  a.recA = h->d_recA;
  a.recB = h->d_recB;
  a.tile_sum = s.tile_sum;
  a.tile_excl = s.tile_excl;
  a.tile_q2 = s.tile_q2;
  a.n_tiles = h->n_tiles;
  a.chunk_tiles = h->chunk_tiles;
  a.n_chunks = h->n_chunks;
  a.src_planes = src;
  a.planes = h->planes;
  a.dst_planes = s.d_dst_planes[dst_par];
  a.dst_anc = s.d_dst_anc;
  a.ctrl = s.ctrl;
  const unsigned long long n = h->n_per;
  a.offs = s.scratch;
  a.hole_dst = s.scratch ? s.scratch + n : nullptr;
  a.extra_src = s.scratch ? s.scratch + 2 * n : nullptr;
  a.tile_nz = s.scratch ? s.scratch + 3 * n : nullptr;
  a.tile_nz_excl = s.scratch ? s.scratch + 3 * n + h->n_tiles : nullptr;
  a.stk0 = a.stk_n = a.stk_per = a.sp_word = 0;
  a.lazy = h->lazy ? 1 : 0;
  if (h->kind == SMC_CLADS2 && h->stack_prefix) {   // R-22: pending-rate stack, planes 2..4, sp = P5.z
    a.stk0 = 2; a.stk_n = 3; a.stk_per = 2; a.sp_word = 22;
  }
  if (h->kind == SMC_STACKF && h->stack_prefix) {   // R-24: byte stack, planes 1.., sp (bytes) = P0.y
    a.stk0 = 1; a.stk_n = h->planes - 1; a.stk_per = 16; a.sp_word = 1;
  }
  return a;
}
template <int IT>
void launch_anc_gather_it(smc_ctx* h, const ResArgs& a) {
  const unsigned grid = (unsigned)h->n_tiles;
  switch (h->planes) {
    case 1: anc_gather_kernel<1, IT><<<grid, kThreads, 0, h->stream>>>(a); break;
    case 2: anc_gather_kernel<2, IT><<<grid, kThreads, 0, h->stream>>>(a); break;
    case 4: anc_gather_kernel<4, IT><<<grid, kThreads, 0, h->stream>>>(a); break;
    case 6: anc_gather_kernel<6, IT><<<grid, kThreads, 0, h->stream>>>(a); break;
    case 8: anc_gather_kernel<8, IT><<<grid, kThreads, 0, h->stream>>>(a); break;
    default: anc_gather_kernel<0, IT><<<grid, kThreads, 0, h->stream>>>(a); break;
  }
}
void launch_anc_gather(smc_ctx* h, const ResArgs& a) {
  if (h->items == kItemsSmall) launch_anc_gather_it<kItemsSmall>(h, a);
  else launch_anc_gather_it<kItems>(h, a);
}
// in-place chain (R-21): offspring, permute, fill holes
void launch_inplace(smc_ctx* h, const ResArgs& a) {
  const unsigned grid = (unsigned)h->n_tiles;
  if (h->items == kItemsSmall) {
    offspring_kernel<kItemsSmall><<<grid, kThreads, 0, h->stream>>>(a);
    permute_kernel<kItemsSmall><<<grid, kThreads, 0, h->stream>>>(a);
  } else {
    offspring_kernel<kItems><<<grid, kThreads, 0, h->stream>>>(a);
    permute_kernel<kItems><<<grid, kThreads, 0, h->stream>>>(a);
  }
  const unsigned fgrid = (unsigned)std::min<unsigned long long>((h->n_per + kThreads - 1) / kThreads, 148ull * 8);
  switch (h->planes) {
    case 1: fill_holes_kernel<1><<<fgrid, kThreads, 0, h->stream>>>(a); break;
    case 2: fill_holes_kernel<2><<<fgrid, kThreads, 0, h->stream>>>(a); break;
    case 4: fill_holes_kernel<4><<<fgrid, kThreads, 0, h->stream>>>(a); break;
    case 6: fill_holes_kernel<6><<<fgrid, kThreads, 0, h->stream>>>(a); break;
    case 8: fill_holes_kernel<8><<<fgrid, kThreads, 0, h->stream>>>(a); break;
    default: fill_holes_kernel<0><<<fgrid, kThreads, 0, h->stream>>>(a); break;
  }
}
// ancestors + state gather: the out-of-place fused kernel or the in-place chain
void launch_resample_tail(smc_ctx* h, const ResArgs& a) {
  if (h->inplace) launch_inplace(h, a);
  else launch_anc_gather(h, a);
}
void launch_reduce(smc_ctx* h, const ResArgs& a) {
  const unsigned grid = (unsigned)((h->n_chunks + kThreads / 32 - 1) / (kThreads / 32));   // a warp per chunk
  if (h->items == kItemsSmall) reduce_kernel<kItemsSmall><<<grid, kThreads, 0, h->stream>>>(a);
  else reduce_kernel<kItems><<<grid, kThreads, 0, h->stream>>>(a);
}
FinArgs fin_args(smc_ctx* h, Shard& s) {
  FinArgs f;
  f.recA = h->d_recA;
  f.recB = h->d_recB;
  f.world = h->world;
  f.rank = s.id;
  f.n_total = h->n_total;
  f.strict = (h->flags & SMC_FLAG_STRICT) ? 1 : 0;
  f.ctrl = s.ctrl;
  return f;
}
int launch_fused(smc_ctx* h, Shard& s, const ResArgs& a) {
  FusedArgs f;
  f.blk_sum = h->d_blk_sum;
  f.blk_q2 = h->d_blk_q2;
  f.ipt = h->fused_ipt;
  f.fin = fin_args(h, s);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)h->fused_grid);
  cfg.blockDim = dim3(kFT);
  cfg.dynamicSmemBytes = h->fused_smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;        // co-residency for the grid barrier
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* args[] = {(void*)&a, (void*)&f};
  CU(cudaLaunchKernelExC(&cfg, fused_fn(h->planes), args));
  return SMC_OK;
}
void launch_finalize(smc_ctx* h, Shard& s) {
  finalize_kernel<<<1, 32, 0, h->stream>>>(fin_args(h, s));
}

// One epoch for all local shards (no host synchronisation unless the comm
// is host-staged).  The host's parity `enq` equals the device epoch as long
// as no shard has finished; after the end every kernel is a no-op.
int enqueue_epoch(smc_ctx* h) {
  const int cur = (int)(h->enq & 1);
  const size_t rec = 16;
  if (h->timing) CU(cudaEventRecord(h->ev[0], h->stream));
  for (auto& s : h->shards) launch_propagate(h, s, cur);
  CU(cudaGetLastError());
  if (h->timing) CU(cudaEventRecord(h->ev[1], h->stream));
  int rc = allgather_rec(h, h->d_recA + cur * h->world, rec);
  if (rc) return rc;
  if (h->fused_grid > 0) {               // single shard: one launch for the whole resampling step
    Shard& s = h->shards[0];
    rc = launch_fused(h, s, res_args(h, s, s.lw, s.planes[cur], cur ^ 1));
    if (rc) return rc;
    CU(cudaGetLastError());
    if (h->timing) CU(cudaEventRecord(h->ev[2], h->stream));
    h->enq++;
    return SMC_OK;
  }
  for (auto& s : h->shards) {
    launch_reduce(h, res_args(h, s, s.lw, s.planes[cur], cur ^ 1));
  }
  CU(cudaGetLastError());
  rc = allgather_rec(h, h->d_recB + cur * h->world, sizeof(RecB));
  if (rc) return rc;
  for (auto& s : h->shards) launch_resample_tail(h, res_args(h, s, s.lw, s.planes[cur], cur ^ 1));
  CU(cudaGetLastError());
  rc = barrier(h);
  if (rc) return rc;
  for (auto& s : h->shards) launch_finalize(h, s);
  CU(cudaGetLastError());
  if (h->timing) CU(cudaEventRecord(h->ev[2], h->stream));
  h->enq++;
  return SMC_OK;
}

int collect_timing(smc_ctx* h) {
  if (!h->timing) return SMC_OK;
  float a = 0.f, b = 0.f;
  CU(cudaEventElapsedTime(&a, h->ev[0], h->ev[1]));
  CU(cudaEventElapsedTime(&b, h->ev[1], h->ev[2]));
  h->ms_propagate += a;
  h->ms_resample += b;
  h->timed_epochs++;
  return SMC_OK;
}

// One CUDA graph for a whole sweep: WHILE(!done) { epoch (parity 0); epoch
// (parity 1); set condition }.  Kernel arguments are fixed at capture (buffer
// pointers, parity); epoch, seed and all per-run state live in device memory.
int build_graph(smc_ctx* h) {
  if (h->graph_exec) return SMC_OK;
  if (!h->cap_stream) CU(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  CU(cudaGraphCreate(&h->graph, 0));
  cudaGraphConditionalHandle hdl;
  CU(cudaGraphConditionalHandleCreate(&hdl, h->graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = hdl;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CU(cudaGraphAddNode(&node, h->graph, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaStream_t keep = h->stream;
  const unsigned long long keep_enq = h->enq;
  h->stream = h->cap_stream;
  CU(cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  int rc = SMC_OK;
  for (int par = 0; par < 2 && rc == SMC_OK; ++par) {
    h->enq = (unsigned long long)par;
    rc = enqueue_epoch(h);
  }
  set_condition_kernel<<<1, 32, 0, h->stream>>>(hdl, h->shards[0].ctrl, 0xFFFFFFF0u);
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(h->stream, &captured);
  h->stream = keep;
  h->enq = keep_enq;
  if (rc) return rc;
  if (e != cudaSuccess) return fail(h, SMC_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  CU(cudaGraphInstantiate(&h->graph_exec, h->graph, 0));
  return SMC_OK;
}

void drop_graph(smc_ctx* h) {
  if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
  if (h->graph) cudaGraphDestroy(h->graph);
  h->graph_exec = nullptr;
  h->graph = nullptr;
}

int read_ctrl(smc_ctx* h) {
  CU(cudaMemcpyAsync(h->h_ctrl, h->shards[0].ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return SMC_OK;
}

int status_of(const Ctrl& c) {
  switch (c.status) {
    case ST_OK: return SMC_OK;
    case ST_REJECTED: return SMC_EREJECTED;
    case ST_NAN: return SMC_ENAN;
    case ST_OVERFLOW: return SMC_EOVERFLOW;
    default: return SMC_ECUDA;
  }
}

int check_ready(smc_ctx* h) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  if (h->kind == SMC_RESAMPLE_BENCH) return fail(h, SMC_ESTATE, "RESAMPLE_BENCH handles only resample");
  if (!h->ipc_ready) return fail(h, SMC_ESTATE, "smc_ipc_import has not been called");
  return SMC_OK;
}

// Decoded observable state.
int nfields_of(int kind, int planes = 0) {
  switch (kind) {
    case SMC_STACKF: return 3 + 6 * (((planes - 1) * 16) / 48);
    case SMC_FIG3: return 3;
    case SMC_CRBD: return 4;
    case SMC_CLADS2: return 13;
    case SMC_SEIR: return 15;
    case SMC_GEOMETRIC: return 2;
    case SMC_SSM: return 3;
    case SMC_CONSTW: return 2;
    default: return 0;
  }
}
void decode(int kind, const uint32_t* w, double* f, int planes = 0) {
  // w: the particle's planes concatenated (4 words per plane)
  auto d = [&](int word) { double x; std::memcpy(&x, w + word, 8); return x; };
  auto i = [&](int word) { return (double)(int32_t)w[word]; };
  switch (kind) {
    case SMC_CRBD:
      f[0] = i(4); f[1] = i(5); f[2] = d(0); f[3] = d(2); break;
    case SMC_CLADS2:   // stack entries at or above sp are not state (R-22): 0
      f[0] = i(20); f[1] = i(21); f[2] = i(22); f[3] = d(0); f[4] = d(2); f[5] = d(4); f[6] = d(6);
      for (int k = 0; k < 6; ++k) f[7 + k] = k < (int)w[22] ? d(8 + 2 * k) : 0.0;
      break;
    case SMC_SEIR:
      f[0] = i(20); f[1] = i(19); f[2] = d(0); f[3] = d(2); f[4] = d(4); f[5] = d(6); f[6] = d(8);
      f[7] = d(10);
      for (int k = 0; k < 4; ++k) f[8 + k] = i(12 + k);
      for (int k = 0; k < 3; ++k) f[12 + k] = i(16 + k);
      break;
    case SMC_GEOMETRIC: f[0] = i(0); f[1] = i(1); break;
    case SMC_FIG3: f[0] = i(0); f[1] = i(1); f[2] = i(2); break;
    case SMC_STACKF: {   // stack bytes at or above sp are not state (R-22/R-24): 0
      f[0] = i(0); f[1] = i(1); f[2] = d(2);
      const int sp = (int)w[1], nfr = ((planes - 1) * 16) / 48;
      for (int j = 0; j < nfr; ++j) {
        double* g = f + 3 + 6 * j;
        const int b = 4 + 12 * j;   // first word of frame j (stack starts at plane 1 = word 4)
        if ((j + 1) * 48 <= sp) {
          g[0] = i(b); g[1] = i(b + 1); g[2] = d(b + 2); g[3] = d(b + 4); g[4] = d(b + 6); g[5] = d(b + 8);
        } else {
          for (int k = 0; k < 6; ++k) g[k] = 0.0;
        }
      }
      break;
    }
    case SMC_SSM: f[0] = i(2); f[1] = i(3); f[2] = d(0); break;
    case SMC_CONSTW: f[0] = i(0); f[1] = i(1); break;
  }
}

smc_ctx* finish_create(smc_ctx* h, int rc) {
  if (rc == SMC_OK) return h;
  g_last_error = h->err;
  smc_destroy(h);
  return nullptr;
}

// Draw-rate ceiling of propagation: every lane draws D
// Exp(rate) variates from its own Philox stream (hq conversion, fp64 log and
// division: the minimal work of one uniform consumed by a sampler), with no
// divergence, no memory traffic and full occupancy.
__global__ void __launch_bounds__(256) draw_peak_kernel(unsigned draws, double* out) {
  const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
  Rng r(0x5EEDull, gid, 0u);
  // the minimal work of one consumed Exp uniform as the kernels implement it:
  // Philox half-block + hq + log_u + a multiply by the precomputed 1/rate
  double acc = 0.0;
  const double irate = 1.0 / (1.0 + 1e-3 * (double)(threadIdx.x & 7));
  for (unsigned d = 0; d < draws; ++d) acc += -log_u(r.uniform()) * irate;
  out[gid] = acc;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int smc_draw_peak(uint32_t draws_per_thread, double* draws_per_s) {
  smc_ctx* h = nullptr;
  if (!draws_per_s || draws_per_thread == 0) return fail(h, SMC_EINVAL, "bad argument");
  int dev = 0, sms = 0, per_sm = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, draw_peak_kernel, 256, 0));
  const unsigned grid = (unsigned)(sms * std::max(per_sm, 1));
  double* out = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CU(cudaMalloc(&out, (size_t)grid * 256 * sizeof(double)));
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {           // first launch warms up
    CU(cudaEventRecord(e0, st));
    draw_peak_kernel<<<grid, 256, 0, st>>>(draws_per_thread, out);
    CU(cudaEventRecord(e1, st));
    CU(cudaEventSynchronize(e1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    if (rep) best = std::min(best, ms);
  }
  CU(cudaGetLastError());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  cudaStreamDestroy(st);
  *draws_per_s = (double)grid * 256.0 * (double)draws_per_thread / (best * 1e-3);
  return SMC_OK;
}

int smc_abi_version(void) { return SMC_ABI_VERSION; }

smc_handle smc_create(const smc_model* model, uint64_t n_particles, uint64_t seed) {
  return smc_create_virtual(model, n_particles, seed, 1);
}

smc_handle smc_create_virtual(const smc_model* model, uint64_t n_per_shard, uint64_t seed,
                              int32_t n_shards) {
  smc_ctx* h = new smc_ctx();
  if (n_shards < 1 || n_shards > 64) return finish_create(h, fail(h, SMC_EINVAL, "n_shards in [1, 64]"));
  int rc = common_init(h, model, n_per_shard, n_shards, 0, n_shards, seed);
  if (rc) return finish_create(h, rc);
  h->comm = COMM_LOCAL;
  std::vector<uint4*> p0, p1;
  std::vector<uint32_t*> an;
  for (auto& s : h->shards) { p0.push_back(s.planes[0]); p1.push_back(s.planes[1]); an.push_back(s.anc); }
  rc = write_dst_tables(h, p0, p1, an);
  if (rc) return finish_create(h, rc);
  rc = reset_device(h);
  return finish_create(h, rc);
}

int smc_get_nccl_id(void* out128) {
  std::string err;
  if (!out128) return fail(nullptr, SMC_EINVAL, "out is NULL");
  if (!g_nccl.load(err)) return fail(nullptr, SMC_ENCCL, err);
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return fail(nullptr, SMC_ENCCL, "ncclGetUniqueId failed");
  std::memcpy(out128, &id, sizeof(id));
  return SMC_OK;
}

smc_handle smc_create_sharded(const smc_model* model, uint64_t n_per_rank, uint64_t seed,
                              int32_t rank, int32_t world, const smc_comm* comm) {
  smc_ctx* h = new smc_ctx();
  if (world < 1 || rank < 0 || rank >= world || !comm)
    return finish_create(h, fail(h, SMC_EINVAL, "bad rank/world/comm"));
  int rc = common_init(h, model, n_per_rank, world, rank, 1, seed);
  if (rc) return finish_create(h, rc);
  if (comm->nccl_id) {
    std::string err;
    if (!g_nccl.load(err)) return finish_create(h, fail(h, SMC_ENCCL, err));
    ncclUniqueId id;
    std::memcpy(&id, comm->nccl_id, sizeof(id));
    if (g_nccl.CommInitRank(&h->nccl, world, id, rank) != ncclSuccess)
      return finish_create(h, fail(h, SMC_ENCCL, "ncclCommInitRank failed"));
    h->comm = COMM_NCCL;
  } else if (comm->allgather) {
    h->cb_allgather = comm->allgather;
    h->cb_user = comm->user;
    h->comm = COMM_CALLBACK;
  } else {
    return finish_create(h, fail(h, SMC_EINVAL, "comm needs nccl_id or allgather"));
  }
  h->ipc_ready = world == 1;
  if (world == 1) {
    Shard& s = h->shards[0];
    rc = write_dst_tables(h, {s.planes[0]}, {s.planes[1]}, {s.anc});
    if (rc) return finish_create(h, rc);
  }
  rc = reset_device(h);
  return finish_create(h, rc);
}

uint64_t smc_ipc_blob_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int smc_ipc_export(smc_handle h, void* out) {
  if (!h || !out) return fail(h, SMC_EINVAL, "NULL argument");
  cudaIpcMemHandle_t mh;
  CU(cudaIpcGetMemHandle(&mh, h->shards[0].ipc_block));
  std::memcpy(out, &mh, sizeof(mh));
  return SMC_OK;
}

int smc_ipc_import(smc_handle h, const void* blobs) {
  if (!h || !blobs) return fail(h, SMC_EINVAL, "NULL argument");
  const size_t plane_bytes = (size_t)h->planes * h->n_per * 16;
  std::vector<uint4*> p0(h->world), p1(h->world);
  std::vector<uint32_t*> an(h->world);
  for (int g = 0; g < h->world; ++g) {
    char* base;
    if (g == h->rank) {
      base = h->shards[0].ipc_block;
    } else {
      cudaIpcMemHandle_t mh;
      std::memcpy(&mh, (const char*)blobs + g * sizeof(mh), sizeof(mh));
      void* p = nullptr;
      CU(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
      h->ipc_opened.push_back(p);
      base = (char*)p;
    }
    p0[g] = (uint4*)base;
    p1[g] = (uint4*)(base + plane_bytes);
    an[g] = (uint32_t*)(base + 2 * plane_bytes);
  }
  int rc = write_dst_tables(h, p0, p1, an);
  if (rc) return rc;
  h->ipc_ready = true;
  return SMC_OK;
}

void smc_destroy(smc_handle h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  for (auto& s : h->shards) {
    cudaFree(s.ipc_block); cudaFree(s.lw); cudaFree(s.tile_sum); cudaFree(s.tile_excl); cudaFree(s.tile_q2);
    cudaFree(s.ctrl); cudaFree(s.d_dst_planes[0]); cudaFree(s.d_dst_planes[1]); cudaFree(s.d_dst_anc);
    cudaFree(s.scratch);
  }
  cudaFree(h->d_table); cudaFree(h->d_logfact); cudaFree(h->d_recA); cudaFree(h->d_recB); cudaFree(h->d_barrier);
  cudaFree(h->d_blk_sum); cudaFree(h->d_blk_q2); cudaFree(h->d_call_tab);
  cudaFree(h->tasks.sid); cudaFree(h->tasks.lam); cudaFree(h->tasks.owner);
  if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
  if (h->graph) cudaGraphDestroy(h->graph);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->h_ctrl) cudaFreeHost(h->h_ctrl);
  for (auto& e : h->ev) if (e) cudaEventDestroy(e);
  for (auto& e : h->rev) if (e) cudaEventDestroy(e);
  if (h->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(h->nccl);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int smc_set_stream(smc_handle h, void* s) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  CU(cudaStreamSynchronize(h->stream));
  if (s) {
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = (cudaStream_t)s;
    h->own_stream = false;
  } else if (!h->own_stream) {
    CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  return SMC_OK;
}

int smc_set_data(smc_handle h, const double* data, uint64_t data_len) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  if (h->kind == SMC_RESAMPLE_BENCH || h->kind == SMC_GEOMETRIC || h->kind == SMC_CONSTW || h->kind == SMC_FIG3)
    return fail(h, SMC_ESTATE, "model has no data");
  // rebuild the device table exactly as setup_model does, same shape required
  smc_model m{};
  m.kind = h->kind;
  m.data = data;
  m.data_len = data_len;
  m.flags = h->flags;
  std::vector<double> old = h->h_table;
  const int old_n = h->mc.n;
  double saved_p[12];
  std::memcpy(saved_p, h->mc.p, sizeof(saved_p));
  std::vector<double> prm(saved_p, saved_p + 12);
  m.params = prm.data();
  m.n_params = 0;                       // keep the handle's parameters
  h->h_table.clear();
  int rc = setup_model(h, &m);
  const double derived_p5 = h->mc.p[5];          // ClaDS2: root child order of the NEW tree
  std::memcpy(h->mc.p, saved_p, sizeof(saved_p));
  if (h->kind == SMC_CLADS2 && rc == SMC_OK && derived_p5 != saved_p[5]) {
    // the root child order is a kernel argument captured by value in the
    // whole-run graph: recapture it (stale ModelConst)
    h->mc.p[5] = derived_p5;
    drop_graph(h);
  }
  if (rc == SMC_OK && (h->mc.n != old_n || h->h_table.size() != old.size()))
    rc = fail(h, SMC_EINVAL, "new data must have the same shape");
  if (rc != SMC_OK) {
    h->h_table = old;
    h->mc.n = old_n;
    return rc;
  }
  h->mc.table = h->d_table;
  CU(cudaMemcpyAsync(h->d_table, h->h_table.data(), h->h_table.size() * sizeof(double),
                     cudaMemcpyHostToDevice, h->stream));
  return SMC_OK;
}

int smc_set_ess_threshold(smc_handle h, uint32_t a, uint32_t b) {
  if (!h || b == 0) return fail(h, SMC_EINVAL, "threshold a/b needs b > 0");
  h->ess_a = a;
  h->ess_b = b;
  for (auto& s : h->shards) {
    CU(cudaMemcpyAsync(&s.ctrl->ess_a, &h->ess_a, sizeof(unsigned), cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(&s.ctrl->ess_b, &h->ess_b, sizeof(unsigned), cudaMemcpyHostToDevice, h->stream));
  }
  CU(cudaStreamSynchronize(h->stream));
  return SMC_OK;
}

int smc_set_graph(smc_handle h, int32_t on) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  h->use_graph = on != 0;
  return SMC_OK;
}

int smc_set_timing(smc_handle h, int32_t on) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  if (on && !h->ev[0]) {
    for (auto& e : h->ev) CU(cudaEventCreate(&e));
    for (auto& e : h->rev) CU(cudaEventCreate(&e));
  }
  h->timing = on != 0;
  return SMC_OK;
}

int smc_reset(smc_handle h, uint64_t seed) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  h->seed = seed;
  return reset_device(h);
}

int smc_step(smc_handle h, int32_t* done) {
  int rc = check_ready(h);
  if (rc) return rc;
  if (h->h_ctrl->done) { if (done) *done = 1; return status_of(*h->h_ctrl); }
  h->started = true;
  rc = enqueue_epoch(h);
  if (rc) return rc;
  rc = read_ctrl(h);
  if (rc) return rc;
  rc = collect_timing(h);
  if (rc) return rc;
  if (done) *done = (int32_t)h->h_ctrl->done;
  return status_of(*h->h_ctrl);
}

int smc_run(smc_handle h) {
  int rc = check_ready(h);
  if (rc) return rc;
  if (h->comm == COMM_NCCL && !h->timing) {
    // one process per GPU with NCCL records: NCCL calls stay out of the WHILE
    // conditional graph.  The host enqueues kBatch epochs at a
    // time and reads the device flag once per batch; epochs enqueued after the
    // end are device no-ops, and every rank sees the same global `done`, so all
    // ranks enqueue the same collectives.
    constexpr int kBatch = 8;
    h->started = true;
    while (!h->h_ctrl->done) {
      for (int k = 0; k < kBatch; ++k) {
        rc = enqueue_epoch(h);
        if (rc) return rc;
      }
      rc = read_ctrl(h);
      if (rc) return rc;
    }
    h->enq = h->h_ctrl->epochs;
    return status_of(*h->h_ctrl);
  }
  if (h->use_graph && !h->timing && h->comm != COMM_CALLBACK && !h->h_ctrl->done && (h->enq & 1)) {
    // the graph body is captured as {even epoch, odd epoch}: after an odd
    // number of smc_step calls take one host step to return to even parity
    int32_t done = 0;
    rc = smc_step(h, &done);
    if (rc || done) return rc;
  }
  if (h->use_graph && !h->timing && h->comm != COMM_CALLBACK && !h->h_ctrl->done) {
    // device-side epoch loop: one graph launch, one synchronisation
    rc = build_graph(h);
    if (rc) return rc;
    h->started = true;
    CU(cudaGraphLaunch(h->graph_exec, h->stream));
    rc = read_ctrl(h);
    if (rc) return rc;
    h->enq = h->h_ctrl->epochs;
    return status_of(*h->h_ctrl);
  }
  int32_t done = 0;
  while (!done) {
    rc = smc_step(h, &done);
    if (rc) return rc;
  }
  return SMC_OK;
}

double smc_log_z(smc_handle h) {
  if (!h) return NAN;
  if (!h->started || read_ctrl(h)) return NAN;
  return h->h_ctrl->logz;
}

int smc_nfields(smc_handle h) { return h ? nfields_of(h->kind, h->planes) : 0; }

int smc_ancestors(smc_handle h, uint32_t* out, uint64_t n) {
  if (!h || !out || n != h->n_per * h->shards.size()) return fail(h, SMC_EINVAL, "bad output size");
  CU(cudaStreamSynchronize(h->stream));
  for (size_t i = 0; i < h->shards.size(); ++i)
    CU(cudaMemcpy(out + i * h->n_per, h->shards[i].anc, h->n_per * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return SMC_OK;
}

int smc_log_weights(smc_handle h, double* out, uint64_t n) {
  if (!h || !out || n != h->n_per * h->shards.size()) return fail(h, SMC_EINVAL, "bad output size");
  CU(cudaStreamSynchronize(h->stream));
  for (size_t i = 0; i < h->shards.size(); ++i)
    CU(cudaMemcpy(out + i * h->n_per, h->shards[i].lw, h->n_per * sizeof(double), cudaMemcpyDeviceToHost));
  return SMC_OK;
}

static int current_parity(smc_ctx* h) {
  if (h->kind == SMC_RESAMPLE_BENCH) {
    if (h->stream) cudaStreamSynchronize(h->stream);
    return (int)(h->enq & 1);
  }
  if (read_ctrl(h)) return -1;
  // every non-final epoch swaps buffers (resample or, under R-19, an identity
  // copy) and advances ctrl->epoch; the final epoch does neither
  return (int)(h->h_ctrl->epoch & 1);
}

// The buffer holding the current (post-resample) states of shard s.  Deferred
// gather: after a resampling epoch they are the previous buffer seen through
// the ancestors; materialise them into the buffer of parity `par` (the next
// propagation's output, free until then).
static int view_buffer(smc_ctx* h, Shard& s, int par, const uint4** out) {
  *out = s.planes[par];
  if (!h->lazy || !h->started || h->h_ctrl->done) return SMC_OK;
  if (h->h_ctrl->gmap_id) {
    *out = s.planes[par ^ 1];
    return SMC_OK;
  }
  const unsigned g = (unsigned)std::min<unsigned long long>((h->n_per + 255) / 256, 4096ull);
  gather_view_kernel<<<g, 256, 0, h->stream>>>(s.planes[par ^ 1], s.planes[par], s.anc, h->n_per, h->planes,
                                                 s.base);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->stream));
  return SMC_OK;
}

int smc_state(smc_handle h, void* out, uint64_t bytes) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  const uint64_t per = (uint64_t)h->planes * 16 * h->n_per;
  if (!out || bytes != per * h->shards.size()) return fail(h, SMC_EINVAL, "bad output size");
  const int par = current_parity(h);
  if (par < 0) return h->status;
  for (size_t i = 0; i < h->shards.size(); ++i) {
    const uint4* src = nullptr;
    int rc = view_buffer(h, h->shards[i], par, &src);
    if (rc) return rc;
    CU(cudaMemcpy((char*)out + i * per, src, per, cudaMemcpyDeviceToHost));
  }
  return SMC_OK;
}

int smc_fields(smc_handle h, double* out, uint64_t n_doubles) {
  if (!h) return fail(h, SMC_EINVAL, "NULL handle");
  const int F = nfields_of(h->kind, h->planes);
  const uint64_t nl = h->n_per * h->shards.size();
  if (!F || !out || n_doubles != nl * F) return fail(h, SMC_EINVAL, "bad output size");
  const uint64_t per = (uint64_t)h->planes * 16 * h->n_per;
  std::vector<uint32_t> raw(per / 4);
  std::vector<uint32_t> w(h->planes * 4);
  const int par = current_parity(h);
  if (par < 0) return h->status;
  for (size_t si = 0; si < h->shards.size(); ++si) {
    const uint4* src = nullptr;
    int rc = view_buffer(h, h->shards[si], par, &src);
    if (rc) return rc;
    CU(cudaMemcpy(raw.data(), src, per, cudaMemcpyDeviceToHost));
    for (uint64_t k = 0; k < h->n_per; ++k) {
      for (int p = 0; p < h->planes; ++p)
        for (int q = 0; q < 4; ++q) w[4 * p + q] = raw[4 * (p * h->n_per + k) + q];
      decode(h->kind, w.data(), out + (si * h->n_per + k) * F, h->planes);
    }
  }
  return SMC_OK;
}

int smc_stats(smc_handle h, smc_stats_t* out) {
  if (!h || !out) return fail(h, SMC_EINVAL, "NULL argument");
  std::memset(out, 0, sizeof(*out));
  out->n_total = h->n_total;
  out->n_local = h->n_per * h->shards.size();
  out->rank = h->rank;
  out->world = h->comm == COMM_LOCAL ? 1 : h->world;
  out->shards = (int32_t)h->shards.size();
  out->state_bytes = (uint32_t)h->planes * 16;
  out->first_error_particle = -1;
  out->status = h->status;
  out->deferred_gather = h->lazy ? 1u : 0u;
  out->ms_propagate = h->ms_propagate;
  out->ms_resample = h->ms_resample;
  out->timed_epochs = h->timed_epochs;
  for (int k = 0; k < 4; ++k) out->ms_kernel[k] = h->ms_kernel[k];
  if (h->stream && cudaStreamSynchronize(h->stream) == cudaSuccess) {
    unsigned long long alive = 0, ovf = 0, fe = ~0ull, drw = 0, roots = 0, dist = 0, grd = 0, stk = 0;
    unsigned mr = 0, mn = 0;
    for (auto& s : h->shards) {
      Ctrl c;
      if (cudaMemcpy(&c, s.ctrl, sizeof(c), cudaMemcpyDeviceToHost) != cudaSuccess) break;
      alive += c.alive_steps; ovf += c.overflow; fe = std::min(fe, c.first_err); drw += c.draws;
      roots += c.side_roots; mr = std::max(mr, c.max_rounds); mn = std::max(mn, c.max_side_nodes);
      dist += c.distinct; grd += c.guard_kills; stk += c.stack_planes;
      out->epochs = c.epochs; out->resamples = c.resamples; out->done = c.done;
      if (c.status && !out->status) out->status = status_of(c);
    }
    out->alive_particle_steps = alive;
    out->overflow = ovf;
    out->draws = drw;
    out->side_roots = roots;
    out->distinct = dist;
    out->max_rounds = mr;
    out->max_side_nodes = mn;
    out->guard_kills = grd;
    out->stack_planes = stk;
    out->first_error_particle = fe == ~0ull ? -1 : (int64_t)fe;
  }
  return SMC_OK;
}

const char* smc_errmsg(smc_handle h) {
  if (h) return h->err.c_str();
  return g_last_error.c_str();
}

// ---- resampler alone --------------------------------------------------------
int smc_resample_device(smc_handle h, const double* d_lw, const void* d_state_in, void* d_state_out,
                        uint32_t* d_anc, uint32_t epoch, double* logz_inc) {
  if (!h || h->kind != SMC_RESAMPLE_BENCH || h->shards.size() != 1 || h->world != 1)
    return fail(h, SMC_ESTATE, "smc_resample_device needs a single-shard RESAMPLE_BENCH handle");
  if (h->inplace && !d_state_out) d_state_out = const_cast<void*>(d_state_in);
  if (!d_lw || !d_state_in || !d_state_out || !d_anc) return fail(h, SMC_EINVAL, "NULL buffer");
  if (h->inplace && d_state_out != d_state_in)
    return fail(h, SMC_EINVAL, "SMC_FLAG_INPLACE: d_state_out must be NULL or d_state_in");
  if (((uintptr_t)d_lw | (uintptr_t)d_state_in | (uintptr_t)d_state_out) & 15)
    return fail(h, SMC_EINVAL, "device buffers must be 16-byte aligned");
  Shard& s = h->shards[0];
  // this call's destinations go through the handle's per-call pointer table
  // (the shard's own destination tables stay untouched); pageable
  // host sources are consumed before cudaMemcpyAsync returns
  if (!h->d_call_tab) CU(cudaMalloc(&h->d_call_tab, 2 * sizeof(void*)));
  void* tab[2] = {d_state_out, d_anc};
  CU(cudaMemcpyAsync(h->d_call_tab, tab, sizeof(tab), cudaMemcpyHostToDevice, h->stream));
  prep_resample_kernel<<<1, 32, 0, h->stream>>>(s.ctrl, h->d_recA, h->d_recB, 1, 0, epoch);
  const unsigned mgrid = (unsigned)std::min<unsigned long long>((h->n_per + kThreads - 1) / kThreads, 148ull * 8);
  if (h->timing) CU(cudaEventRecord(h->rev[0], h->stream));
  max_kernel<<<mgrid, kThreads, 0, h->stream>>>(d_lw, h->n_per, h->d_recA, 1, 0, s.ctrl);
  if (h->timing) CU(cudaEventRecord(h->rev[1], h->stream));
  ResArgs a = res_args(h, s, d_lw, (const uint4*)d_state_in, 1);
  a.dst_planes = reinterpret_cast<uint4* const*>(h->d_call_tab);
  a.dst_anc = reinterpret_cast<uint32_t* const*>(h->d_call_tab + 1);
  if (h->fused_grid > 0) {
    // one cooperative launch: quantise + sum, grid barrier, ancestors + gather,
    // log Z (timed in the anc_gather slot; reduce and finalize slots stay 0)
    if (h->timing) CU(cudaEventRecord(h->rev[2], h->stream));
    int rc = launch_fused(h, s, a);
    if (rc) return rc;
    if (h->timing) CU(cudaEventRecord(h->rev[3], h->stream));
    if (h->timing) CU(cudaEventRecord(h->rev[4], h->stream));
  } else {
    launch_reduce(h, a);
    if (h->timing) CU(cudaEventRecord(h->rev[2], h->stream));
    launch_resample_tail(h, a);
    if (h->timing) CU(cudaEventRecord(h->rev[3], h->stream));
    launch_finalize(h, s);
    if (h->timing) CU(cudaEventRecord(h->rev[4], h->stream));
  }
  CU(cudaGetLastError());
  h->started = true;
  if (h->timing) {
    CU(cudaEventSynchronize(h->rev[4]));
    for (int k = 0; k < 4; ++k) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, h->rev[k], h->rev[k + 1]));
      h->ms_kernel[k] += ms;
    }
  }
  if (logz_inc) {
    CU(cudaMemcpyAsync(h->h_ctrl, s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    *logz_inc = h->h_ctrl->last_inc;
    if (h->h_ctrl->status) return fail(h, status_of(*h->h_ctrl), "resampling failed (NaN or all -inf)");
  }
  return SMC_OK;
}

int smc_resample_host(smc_handle h, const double* lw, const void* state_in, void* state_out,
                      uint32_t* anc, uint32_t epoch, double* logz_inc) {
  if (!h || h->kind != SMC_RESAMPLE_BENCH) return fail(h, SMC_ESTATE, "needs a RESAMPLE_BENCH handle");
  Shard& s = h->shards[0];
  const size_t sb = (size_t)h->planes * 16 * h->n_per;
  CU(cudaMemcpyAsync(s.lw, lw, h->n_per * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(s.planes[0], state_in, sb, cudaMemcpyHostToDevice, h->stream));
  double inc = 0.0;
  int rc = smc_resample_device(h, s.lw, s.planes[0], s.planes[1], s.anc, epoch, &inc);
  if (rc) return rc;
  CU(cudaMemcpyAsync(anc, s.anc, h->n_per * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaMemcpyAsync(state_out, s.planes[1], sb, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  if (logz_inc) *logz_inc = inc;
  return SMC_OK;
}

// Host-side exact planner (same integer arithmetic as Grid::count_below).
static bool plan_below(unsigned long long j, u128 C, u128 W, unsigned long long z2p1, u128 Nsc) {
  // (j 2^54 + 2z + 1) W < N 2^54 C  in 256-bit
  auto mul = [](u128 a, u128 b, unsigned long long r[4]) {
    const unsigned long long a0 = (unsigned long long)a, a1 = (unsigned long long)(a >> 64);
    const unsigned long long b0 = (unsigned long long)b, b1 = (unsigned long long)(b >> 64);
    const u128 p00 = (u128)a0 * b0, p01 = (u128)a0 * b1, p10 = (u128)a1 * b0, p11 = (u128)a1 * b1;
    r[0] = (unsigned long long)p00;
    u128 mid = (p00 >> 64) + (unsigned long long)p01 + (unsigned long long)p10;
    r[1] = (unsigned long long)mid;
    u128 hi = (mid >> 64) + (p01 >> 64) + (p10 >> 64) + (unsigned long long)p11;
    r[2] = (unsigned long long)hi;
    r[3] = (unsigned long long)(hi >> 64) + (unsigned long long)(p11 >> 64);
  };
  unsigned long long l[4], r[4];
  mul(((u128)j << 54) + z2p1, W, l);
  mul(Nsc, C, r);
  for (int i = 3; i >= 0; --i)
    if (l[i] != r[i]) return l[i] < r[i];
  return false;
}
static unsigned long long plan_count(u128 C, u128 W, unsigned long long z2p1, unsigned long long N) {
  const u128 Nsc = (u128)N << 54;
  unsigned long long lo = 0, hi = N;          // smallest j in [0, N] with !below(j)
  while (lo < hi) {
    const unsigned long long mid = lo + (hi - lo) / 2;
    if (plan_below(mid, C, W, z2p1, Nsc)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

int smc_plan_ranges(const uint64_t* w_lohi, int32_t world, uint64_t n_per, uint64_t z,
                    uint64_t* out) {
  if (!w_lohi || !out || world < 1 || n_per == 0 || z >= (1ull << 53))
    return fail(nullptr, SMC_EINVAL, "bad planner arguments");
  const unsigned long long N = n_per * (unsigned long long)world;
  u128 W = 0;
  for (int g = 0; g < world; ++g) W += ((u128)w_lohi[2 * g + 1] << 64) | w_lohi[2 * g];
  if (W == 0) return fail(nullptr, SMC_EREJECTED, "total weight is zero");
  u128 P = 0;
  for (int g = 0; g <= world; ++g) {
    out[g] = plan_count(P, W, 2 * z + 1, N);
    if (g < world) P += ((u128)w_lohi[2 * g + 1] << 64) | w_lohi[2 * g];
  }
  return SMC_OK;
}

int smc_load(smc_handle h, const double* lw, const void* state, int32_t device_ptrs) {
  if (!h || !lw || !state) return fail(h, SMC_EINVAL, "NULL argument");
  if (h->kind != SMC_RESAMPLE_BENCH) return fail(h, SMC_ESTATE, "smc_load needs a RESAMPLE_BENCH handle");
  const size_t per = (size_t)h->planes * 16 * h->n_per;
  const int cur = (int)(h->enq & 1);
  const cudaMemcpyKind kind = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  for (size_t i = 0; i < h->shards.size(); ++i) {
    CU(cudaMemcpyAsync(h->shards[i].lw, lw + i * h->n_per, h->n_per * sizeof(double), kind, h->stream));
    CU(cudaMemcpyAsync(h->shards[i].planes[cur], (const char*)state + i * per, per, kind, h->stream));
  }
  CU(cudaStreamSynchronize(h->stream));
  return SMC_OK;
}

int smc_resample_step(smc_handle h, uint32_t epoch) {
  if (!h || h->kind != SMC_RESAMPLE_BENCH) return fail(h, SMC_ESTATE, "needs a RESAMPLE_BENCH handle");
  if (!h->ipc_ready) return fail(h, SMC_ESTATE, "smc_ipc_import has not been called");
  const int cur = (int)(h->enq & 1);
  const unsigned par = epoch & 1;
  for (auto& s : h->shards) {
    prep_resample_kernel<<<1, 32, 0, h->stream>>>(s.ctrl, h->d_recA, h->d_recB, h->world, s.id, epoch);
    const unsigned mgrid = (unsigned)std::min<unsigned long long>((h->n_per + kThreads - 1) / kThreads, 148ull * 8);
    max_kernel<<<mgrid, kThreads, 0, h->stream>>>(s.lw, h->n_per, h->d_recA, h->world, s.id, s.ctrl);
  }
  CU(cudaGetLastError());
  int rc = allgather_rec(h, h->d_recA + par * h->world, 16);
  if (rc) return rc;
  for (auto& s : h->shards) launch_reduce(h, res_args(h, s, s.lw, s.planes[cur], cur ^ 1));
  rc = allgather_rec(h, h->d_recB + par * h->world, sizeof(RecB));
  if (rc) return rc;
  for (auto& s : h->shards) launch_resample_tail(h, res_args(h, s, s.lw, s.planes[cur], cur ^ 1));
  rc = barrier(h);
  if (rc) return rc;
  for (auto& s : h->shards) launch_finalize(h, s);
  CU(cudaGetLastError());
  h->enq++;
  h->started = true;
  return SMC_OK;
}

int smc_resample_grid(smc_handle h, int32_t* grid_out) {
  if (!h || !grid_out) return fail(h, SMC_EINVAL, "NULL argument");
  *grid_out = h->fused_grid;
  return SMC_OK;
}

int smc_last_distinct(smc_handle h, uint64_t* out) {
  if (!h || !out) return fail(h, SMC_EINVAL, "NULL argument");
  CU(cudaStreamSynchronize(h->stream));
  unsigned long long d = 0;
  for (auto& sh : h->shards) {
    Ctrl c;
    CU(cudaMemcpy(&c, sh.ctrl, sizeof(c), cudaMemcpyDeviceToHost));
    d += c.distinct;
  }
  *out = d;
  return SMC_OK;
}

}  // extern "C"
