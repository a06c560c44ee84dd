// executor.cpp — device executor for BE / MBE / DPOP plans.
//
// Alg. 3 re-designed for one B200: the original tables go to the
// device in ONE batched copy and are re-laid-out there;
// every (mini-)bucket is one fused aggregate+project kernel (BK) whose
// messages stay device-resident and are freed once consumed; the
// value phase is a single-warp kernel walking the forward
// order over the argmin tables.  Row-sharded buckets call the
// all-gather hook only when a consumer needs a whole message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "common.h"
#include "executor.h"
#include "bk_fast.h"
#include "bk_stream.h"
#include "kernels.h"

namespace gbe {

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) GBE_FAIL(GBE_E_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// hooks

static void *(*g_alloc)(size_t, void *, void *) = nullptr;
static void (*g_free)(void *, void *) = nullptr;
static void *g_alloc_u = nullptr;
static int (*g_ag)(const void *, void *, size_t, void *, void *) = nullptr;
static void *g_ag_u = nullptr;
static TableHook g_hook = nullptr;
static void *g_hook_u = nullptr;

void set_table_hook(TableHook fn, void *u) {
  g_hook = fn;
  g_hook_u = u;
}

void set_allocator(void *(*a)(size_t, void *, void *), void (*f)(void *, void *), void *u) {
  g_alloc = a;
  g_free = f;
  g_alloc_u = u;
}
static bool g_ag_graph = false;  // the hook only enqueues stream work (capturable)
void set_allgather(int (*ag)(const void *, void *, size_t, void *, void *), void *u) {
  g_ag = ag;
  g_ag_u = u;
  g_ag_graph = false;
}
void set_allgather_capturable(int (*ag)(const void *, void *, size_t, void *, void *), void *u) {
  set_allgather(ag, u);
  g_ag_graph = ag != nullptr;
}

static void *dalloc(size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~size_t(255);  // slack for vector tails
  void *p = nullptr;
  if (g_alloc) {
    p = g_alloc(bytes, (void *)s, g_alloc_u);
    if (!p) GBE_FAIL(GBE_E_BUDGET, "allocator hook failed for %zu bytes", bytes);
    return p;
  }
  cudaError_t e = cudaMallocAsync(&p, bytes, s);
  if (e != cudaSuccess) GBE_FAIL(e == cudaErrorMemoryAllocation ? GBE_E_BUDGET : GBE_E_CUDA,
                                 "device allocation of %zu bytes: %s", bytes, cudaGetErrorString(e));
  return p;
}
static void dfree(void *p, cudaStream_t s) {
  if (!p) return;
  if (g_free) {
    g_free(p, g_alloc_u);
    return;
  }
  cudaFreeAsync(p, s);
}

// ---------------------------------------------------------------------------
// per-plan device state

struct DevPlan {
  int device = 0, num_sms = 148;
  std::vector<gbe_bucket_desc> h_desc;
  std::vector<BkLaunchInfo> launch;
  std::vector<FastDesc> h_fast;
  // direct-store descriptors of the tiled kernel (an autotuning candidate
  // for the hot int32 shape: no staging buffers, more ring stages)
  std::vector<FastDesc> h_fds;
  std::vector<BkfLaunch> fl_ds;
  std::vector<char> use_ds;
  FastDesc *d_fds = nullptr;
  std::vector<BkfLaunch> fl;
  std::vector<char> use_fast;
  std::vector<StreamDesc> h_stream;  // streaming kernel (bk_stream.cu) descriptors
  std::vector<BksLaunch> sl;
  std::vector<char> use_stream;
  StreamDesc *d_stream = nullptr;
  // the streaming kernel's staged mode (per-warp TMA double buffers): its
  // own descriptors (smaller warp-tiles); use_stage picks it for a task
  std::vector<StreamDesc> h_stage;
  std::vector<BksLaunch> sl3;
  std::vector<char> use_stage;
  StreamDesc *d_stage = nullptr;
  // a second streaming descriptor with warp-tiles of at most half the rows
  // (an autotuning candidate: C5 x77 1.36 -> 1.10 ms, C4-d4 x27 0.91 -> 0.71
  // ms, while x91 / x80 lose with it); use_half picks it for a task
  std::vector<StreamDesc> h_half;
  std::vector<BksLaunch> slh;
  std::vector<char> use_half;
  StreamDesc *d_half = nullptr;
  // the streaming launch of task ti with the descriptor its choice names
  cudaError_t stream_launch(size_t ti, const InPtrs &in, void *out, uint8_t *arg, int64_t lo, int64_t hi,
                            cudaStream_t st) const {
    if (use_stage[ti]) return bks_launch(d_stage + ti, sl3[ti], in, out, arg, lo, hi, st);
    if (use_half[ti]) return bks_launch(d_half + ti, slh[ti], in, out, arg, lo, hi, st);
    return bks_launch(d_stream + ti, sl[ti], in, out, arg, lo, hi, st);
  }
  // autotuning (exec option "autotune", kernel auto): a task with more than
  // one candidate launch -- the tiled kernel, the streaming kernel with and
  // without its L2 prefetch -- runs candidate p mod nc on tuning solve p
  // (eager, CUDA events around each launch; solves 0..nc-1 pay lazy module
  // loading and are not scored, solves nc..2nc-1 are); then each task keeps
  // its fastest candidate (3 % margin over its default) and the graph is
  // captured with the final choice
  struct Cand {
    int variant;  // 1 tiled, 2 streaming
    bool pf;      // streaming: L2 prefetch of the next tile's slices
    bool stage;   // streaming: staged mode
    bool half;    // streaming: the half-tile descriptor
    bool ds = false;  // tiled: direct stores
  };
  std::vector<std::vector<Cand>> cands;  // [task]: candidate 0 = the default choice
  std::vector<std::vector<float>> t_cand;
  int tune_nc = 0;      // max candidates over the tuned tasks
  int tune_phase = -1;  // -1: no tuning; 0..2*tune_nc-1: the next tuning solve; 2*tune_nc: done
  std::vector<cudaEvent_t> tune_ev;
  // pre-aggregation of small inputs (DESIGN.md §5 "input merging"): merge mi
  // sums some inputs of task merges[mi].task into one table, a d = 1 bucket
  struct Merge {
    int32_t task = -1;
    gbe_bucket_desc h{};
    BkLaunchInfo li{};
    bool stream = false;  // run by the streaming kernel (else bk_generic)
    StreamDesc sd{};
    BksLaunch sl{};
    std::vector<int32_t> src;  // task input indices (canonical member positions)
    size_t bytes = 0;
  };
  std::vector<Merge> merges;
  std::vector<std::vector<int32_t>> task_merges;  // per task: its merges
  std::vector<std::vector<int32_t>> in_map;       // per task input: member index, or -(1 + merge)
  gbe_bucket_desc *d_mdesc = nullptr;
  StreamDesc *d_mstream = nullptr;  // streaming-kernel descriptors of the merges
  // "retain":"host" (§8(f) row 2, argmin spill): each bucket runs in row
  // chunks whose argmins land in a 2-slot device ring and stream to mapped
  // pinned host memory on a copy stream while the next chunk computes (the
  // host/device concurrency of Fig. 8); the value phase reads them
  // in place (zero-copy)
  struct Chunk {
    int64_t lo = 0, hi = 0;
    int fidx = -1;        // index into h_cfast / cfl (tiled kernel), -1: generic
    bool stream = false;  // streaming kernel over [lo, hi)
    int sidx = -1;        // its descriptor: index into h_cstream
    BksLaunch sl{};
    BkLaunchInfo li{};
    // out-of-core plans ("spill"): staging-slot layout of this chunk
    size_t out_off = 0, arg_off = 0;
    struct HostIn {
      int j;            // task input (after merging)
      int32_t src;      // producing task (a host message)
      int64_t lo, n;    // element range of that message the chunk reads
      size_t off;       // byte offset in the slot (16-byte phase of lo * el added at use)
    };
    std::vector<HostIn> hin;
  };
  // "spill" (out-of-core, §8(f) row 2): host messages in pinned host memory,
  // two device staging slots, an H2D stream beside the D2H copy stream
  char *h_msg = nullptr;
  std::vector<size_t> msg_off;
  char *d_slot = nullptr;
  cudaStream_t h2d_stream = nullptr;
  cudaEvent_t h_ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> done_ev;  // per host-message task: its last chunk copied out
  std::vector<std::vector<Chunk>> chunks;
  std::vector<FastDesc> h_cfast;
  std::vector<BkfLaunch> cfl;
  FastDesc *d_cfast = nullptr;
  // the streaming kernel's descriptor depends on the row range (warp-tile
  // length, tile order): one per chunk
  std::vector<StreamDesc> h_cstream;
  StreamDesc *d_cstream = nullptr;
  uint8_t *h_harg = nullptr, *d_harg = nullptr;  // pinned mapped host argmins and their device alias
  std::vector<size_t> harg_off;
  uint8_t *d_ring = nullptr;
  int64_t ring = 0;                               // bytes per ring slot
  cudaStream_t cp_stream = nullptr;
  cudaEvent_t k_ev[2] = {nullptr, nullptr}, c_ev[2] = {nullptr, nullptr};
  FastDesc *d_fast = nullptr;
  gbe_bucket_desc *d_desc = nullptr;
  int64_t *d_off = nullptr;
  int32_t *d_poff = nullptr, *d_prad = nullptr, *d_pstride = nullptr;
  void *h_raw = nullptr;  // pinned copy of the declared-order tables
  size_t raw_bytes = 0;
  void *d_resident = nullptr;  // resident raw tables (resident_inputs)
  bool resident = false;
  cudaStream_t cap_stream = nullptr;  // CUDA-graph capture
  std::vector<cudaStream_t> side;     // capture branches (concurrent subtrees)
  std::vector<cudaEvent_t> tev;       // capture-internal task completion events
  // static memory plans (exact / MBE mode): every large buffer of a run at a
  // fixed offset of one arena allocation, reused by consecutive runs
  struct Arena {
    bool planned = false;
    size_t bytes = 0, off_raw = 0, off_sorted = 0;
    std::vector<size_t> off_out, off_full, off_arg, off_merge, off_cnt;
    // UTIL-phase DAG: deps[t] = tasks that must finish before task t starts
    // (its producers and the last users of arena ranges it overwrites)
    std::vector<std::vector<int32_t>> deps;
    void *mem = nullptr;
    bool busy = false, hook = false;
    void *vprog = nullptr;  // cached value-phase program (device)
    cudaGraphExec_t exec = nullptr;  // captured UTIL phase
    int runs = 0;
    bool no_graph = false;  // capture failed (W > 1): eager enqueue
    void *d_opt = nullptr, *d_cp = nullptr, *d_ccp = nullptr, *h_opt = nullptr;
    int32_t *d_assign = nullptr;
    std::vector<cudaEvent_t> ev;
    int vsteps = 0;
    size_t b_steps = 0, b_mems = 0;
    std::vector<char> vsharded;
  } arena[2];
  ~DevPlan() {
    for (auto &a : arena) {
      if (a.vprog) cudaFree(a.vprog);
      if (a.exec) cudaGraphExecDestroy(a.exec);
      cudaFree(a.d_opt);
      cudaFree(a.d_cp);
      cudaFree(a.d_ccp);
      cudaFree(a.d_assign);
      if (a.h_opt) cudaFreeHost(a.h_opt);
      for (auto e : a.ev) cudaEventDestroy(e);
    }
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto st : side) cudaStreamDestroy(st);
    for (auto e : tev) cudaEventDestroy(e);
    for (auto &a : arena)
      if (a.mem) {
        if (a.hook && g_free) g_free(a.mem, g_alloc_u);
        else cudaFree(a.mem);
      }
    cudaFree(d_desc);
    cudaFree(d_mdesc);
    cudaFree(d_mstream);
    cudaFree(d_cfast);
    cudaFree(d_cstream);
    cudaFree(d_ring);
    if (h_harg) cudaFreeHost(h_harg);
    if (h_msg) cudaFreeHost(h_msg);
    cudaFree(d_slot);
    if (h2d_stream) cudaStreamDestroy(h2d_stream);
    for (auto e : h_ev) if (e) cudaEventDestroy(e);
    for (auto e : done_ev) if (e) cudaEventDestroy(e);
    if (cp_stream) cudaStreamDestroy(cp_stream);
    for (auto e : k_ev) if (e) cudaEventDestroy(e);
    for (auto e : tune_ev) cudaEventDestroy(e);
    for (auto e : c_ev) if (e) cudaEventDestroy(e);
    cudaFree(d_fast);
    cudaFree(d_fds);
    cudaFree(d_stream);
    cudaFree(d_stage);
    cudaFree(d_half);
    cudaFree(d_off);
    cudaFree(d_poff);
    cudaFree(d_prad);
    cudaFree(d_pstride);
    cudaFree(d_resident);
    if (h_raw) cudaFreeHost(h_raw);
  }
};

// First-fit offsets for the run's buffers in the exact order run_util
// allocates and frees them (DESIGN.md §5 "memory plan").
namespace {
struct FreeList {
  std::vector<std::pair<size_t, size_t>> iv{{0, SIZE_MAX}};  // [start, end)
  size_t top = 0;
  size_t alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    for (size_t i = 0; i < iv.size(); i++)
      if (iv[i].second - iv[i].first >= bytes) {
        size_t o = iv[i].first;
        iv[i].first += bytes;
        if (iv[i].first == iv[i].second) iv.erase(iv.begin() + i);
        top = std::max(top, o + bytes);
        return o;
      }
    return SIZE_MAX;
  }
  void release(size_t o, size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    auto it = std::lower_bound(iv.begin(), iv.end(), std::make_pair(o, size_t(0)));
    it = iv.insert(it, {o, o + bytes});
    size_t i = it - iv.begin();
    if (i + 1 < iv.size() && iv[i].second == iv[i + 1].first) {
      iv[i].second = iv[i + 1].second;
      iv.erase(iv.begin() + i + 1);
    }
    if (i > 0 && iv[i - 1].second == iv[i].first) {
      iv[i - 1].second = iv[i].second;
      iv.erase(iv.begin() + i);
    }
  }
};
}  // namespace

static void plan_arena(const Plan &P, DevPlan *D, bool mbe_mode) {
  const Problem &p = *P.prob;
  const size_t el = p.elem();
  const int W = P.ex.world_size;
  const size_t nt = P.tasks.size();
  FreeList fl;
  DevPlan::Arena &A = D->arena[mbe_mode ? 1 : 0];
  A.off_out.assign(nt, SIZE_MAX);
  A.off_full.assign(nt, SIZE_MAX);
  A.off_arg.assign(nt, SIZE_MAX);
  size_t raw = D->raw_bytes;
  A.off_raw = fl.alloc(raw);
  A.off_sorted = fl.alloc(raw);
  fl.release(A.off_raw, raw);  // raw tables are dead after the relayout
  // sum-product plans have no argmin (no VALUE phase, A18)
  const bool want_arg = ((!mbe_mode && P.ex.retain >= 1) || P.ex.retain >= 2) && !P.ex.host_args && !P.ex.sumprod;
  std::vector<size_t> out_b(nt, 0), full_b(nt, 0);
  // ranges[t]: the arena ranges task t writes; a later task overwriting any of
  // them must wait for t and for t's consumer (the only reader of t's output)
  std::vector<std::vector<std::pair<size_t, size_t>>> ranges(nt);
  auto put = [&](size_t ti, size_t o, size_t b) {
    ranges[ti].push_back({o, o + std::max<size_t>((b + 255) & ~size_t(255), 256)});
  };
  A.off_merge.assign(D->merges.size(), SIZE_MAX);
  A.off_cnt.assign(nt, SIZE_MAX);
  std::vector<size_t> cnt_b(nt, 0);
  for (size_t ti = 0; ti < nt; ti++) {
    const Task &t = P.tasks[ti];
    const Shard &sh = t.shard;
    int64_t local = sh.on ? sh.hi - sh.lo : t.rows;
    int64_t cap = sh.on ? sh.per * sh.block_rows : t.rows;
    for (int32_t mi : D->task_merges[ti]) {  // live only while task ti runs
      A.off_merge[mi] = fl.alloc(D->merges[mi].bytes);
      put(ti, A.off_merge[mi], D->merges[mi].bytes);
    }
    if (!t.host) {  // (a host message of an out-of-core plan has no device range)
      out_b[ti] = el * (size_t)cap;
      A.off_out[ti] = fl.alloc(out_b[ti]);
      put(ti, A.off_out[ti], out_b[ti]);
    }
    if (P.ex.count) {  // (min, count) semiring: a float64 count per row
      cnt_b[ti] = 8 * (size_t)cap;
      A.off_cnt[ti] = fl.alloc(cnt_b[ti]);
      put(ti, A.off_cnt[ti], cnt_b[ti]);
    }
    if (want_arg) {
      A.off_arg[ti] = fl.alloc((size_t)std::max<int64_t>(local, 1));
      put(ti, A.off_arg[ti], (size_t)std::max<int64_t>(local, 1));
    }
    if (sh.on && sh.gather) {
      full_b[ti] = out_b[ti] * W;
      A.off_full[ti] = fl.alloc(full_b[ti]);
      put(ti, A.off_full[ti], full_b[ti]);
      fl.release(A.off_out[ti], out_b[ti]);
      out_b[ti] = 0;
    }
    for (int32_t mi : D->task_merges[ti]) fl.release(A.off_merge[mi], D->merges[mi].bytes);
    if ((!mbe_mode || P.ex.retain == 0) && P.ex.retain < 2)
      for (auto &m : t.members)
        if (m.kind == 1) {
          if (out_b[m.index]) fl.release(A.off_out[m.index], out_b[m.index]);
          if (full_b[m.index]) fl.release(A.off_full[m.index], full_b[m.index]);
          if (cnt_b[m.index]) fl.release(A.off_cnt[m.index], cnt_b[m.index]);
          out_b[m.index] = full_b[m.index] = cnt_b[m.index] = 0;
        }
  }
  A.bytes = std::max<size_t>(fl.top, 256);
  // the DAG of the UTIL phase (sibling subtrees are independent)
  A.deps.assign(nt, {});
  for (size_t ti = 0; ti < nt; ti++) {
    std::vector<int32_t> &dp = A.deps[ti];
    for (auto &m : P.tasks[ti].members)
      if (m.kind == 1) dp.push_back(m.index);
    for (size_t k = 0; k < ti; k++) {
      bool hit = false;
      for (auto &a : ranges[ti])
        for (auto &b : ranges[k])
          if (a.first < b.second && b.first < a.second) hit = true;
      if (!hit) continue;
      dp.push_back((int32_t)k);
      int32_t c = P.tasks[k].consumer;
      if (c >= 0 && (size_t)c < ti) dp.push_back(c);
    }
    std::sort(dp.begin(), dp.end());
    dp.erase(std::unique(dp.begin(), dp.end()), dp.end());
  }
  // transitive reduction: drop an edge k -> t when another predecessor of t
  // already descends from k (fewer cross-branch waits in the graph)
  {
    const size_t words = (nt + 63) / 64;
    std::vector<uint64_t> anc(nt * words, 0);  // anc[t] = all ancestors of t
    for (size_t ti = 0; ti < nt; ti++) {
      uint64_t *a = &anc[ti * words];
      for (int32_t k : A.deps[ti]) {
        a[k >> 6] |= 1ull << (k & 63);
        const uint64_t *b = &anc[(size_t)k * words];
        for (size_t w = 0; w < words; w++) a[w] |= b[w];
      }
      std::vector<int32_t> keep;
      for (int32_t k : A.deps[ti]) {
        bool implied = false;
        for (int32_t k2 : A.deps[ti])
          if (k2 != k && (anc[(size_t)k2 * words + (k >> 6)] >> (k & 63) & 1)) implied = true;
        if (!implied) keep.push_back(k);
      }
      A.deps[ti].swap(keep);
    }
  }
  A.planned = true;
}

// Input merging (pre-aggregation): inside a large bucket, inputs that lack
// the same group digits of the tiled kernel (same "class", bk_fast.cu) are
// each re-loaded per register block; the small ones are summed ONCE into one
// table over the union of their scopes — a d = 1 bucket (out = the sum of its
// members, the minimum over a single value being the identity) — and the
// bucket reads that table instead.  Small class-0 inputs (neither group
// digit) fold into the merged table of another class when one exists: the
// fold adds no per-cell loads.  Sums are the same ones Alg. 1 line 3 forms
// (P:204-205); for int32 with the clamp of A9 they are bit-identical, for
// f64 the summation order changes (canonical order note).
static void plan_merges(const Plan &P, DevPlan *D, size_t ti, gbe_bucket_desc &h, bool noinf) {
  static const bool off = std::getenv("GBE_NO_MERGE") != nullptr;  // A/B knob
  const Task &t = P.tasks[ti];
  const int k = h.ninputs, m = h.nsep, d = h.d;
  auto &map = D->in_map[ti];
  map.resize(k);
  for (int j = 0; j < k; j++) map[j] = j;
  if (off || P.ex.kernel == 0 || k < 2) return;
  const int64_t C = (t.shard.hi - t.shard.lo) * d;
  static const int min_log2 = [] {  // GBE_MERGE_MIN_LOG2: tuning knob
    const char *e = std::getenv("GBE_MERGE_MIN_LOG2");
    return e ? std::atoi(e) : 27;
  }();
  // small buckets: the extra launches cost more than they save, unless the
  // merge removes many inputs (checked once the sets are known, below)
  if (C < (int64_t(1) << std::min(22, min_log2))) return;
  const bool big_enough = C >= (int64_t(1) << min_log2);
  FastDesc *F = new FastDesc();
  BkfLaunch L;
  const bool ok = bkf_build(h, t.shard.lo, t.shard.hi, D->num_sms, *F, L, noinf);
  delete F;
  if (!ok) return;
  auto has = [&](int j, int p) { return h.stride[j][p] != 0; };
  auto union_cells = [&](const std::vector<int> &js) {
    int64_t c = d;
    for (int p = 0; p < m; p++)
      for (int j : js)
        if (has(j, p)) {
          c *= h.radix[p];
          break;
        }
    return c;
  };
  static const int cap_log2 = [] {  // GBE_MERGE_CAP_LOG2: tuning knob
    const char *e = std::getenv("GBE_MERGE_CAP_LOG2");
    return e ? std::atoi(e) : 26;
  }();
  static const int cap_div = [] {  // GBE_MERGE_CAP_DIV: tuning knob (merged table <= C / div)
    const char *e = std::getenv("GBE_MERGE_CAP_DIV");
    return e ? std::max(1, std::atoi(e)) : 128;
  }();
  const int64_t small = C / 64, cap = std::min<int64_t>(C / cap_div, int64_t(1) << cap_log2);
  std::vector<int> cand[4];
  for (int j = 0; j < k; j++) {
    if (h.shift[j] != 0) continue;
    if (t.members[j].kind == 1 && P.tasks[t.members[j].index].host) continue;  // staged per chunk
    if (union_cells({j}) > small) continue;
    const int cls = (has(j, L.g1) ? 1 : 0) + (L.g2 >= 0 && has(j, L.g2) ? 2 : 0);
    cand[cls].push_back(j);
  }
  if (!cand[0].empty()) {  // fold class 0 into the class whose union stays smallest
    int best = -1;
    int64_t bestc = INT64_MAX;
    for (int c = 1; c < 4; c++) {
      if (cand[c].empty()) continue;
      std::vector<int> u = cand[c];
      u.insert(u.end(), cand[0].begin(), cand[0].end());
      const int64_t uc = union_cells(u);
      if (uc <= cap && uc < bestc) {
        bestc = uc;
        best = c;
      }
    }
    if (best > 0) {
      cand[best].insert(cand[best].end(), cand[0].begin(), cand[0].end());
      std::sort(cand[best].begin(), cand[best].end());
      cand[0].clear();
    }
  }
  // a class whose whole candidate set unions past the cap still merges its
  // largest subset that fits: members taken smallest first while the union
  // stays <= cap (C4-d4's x3: 6 class-0 inputs whose full union is 8x the
  // cap; the 5 smallest fit)
  std::vector<std::vector<int>> sets;
  for (int c = 0; c < 4; c++) {
    if (cand[c].size() < 2) continue;
    if (union_cells(cand[c]) <= cap) {
      sets.push_back(cand[c]);
      continue;
    }
    std::vector<int> byc = cand[c];
    std::stable_sort(byc.begin(), byc.end(), [&](int a, int b) { return union_cells({a}) < union_cells({b}); });
    std::vector<int> sub;
    for (int j : byc) {
      sub.push_back(j);
      if (union_cells(sub) > cap) sub.pop_back();
    }
    std::sort(sub.begin(), sub.end());  // canonical member order inside the merged table
    if (sub.size() >= 2) sets.push_back(sub);
  }
  if (sets.empty()) return;
  size_t removed = 0;
  for (auto &st : sets) removed += st.size() - 1;
  if (!big_enough && removed < 4) return;
  std::vector<char> merged(k, 0);
  for (auto &st : sets)
    for (int j : st) merged[j] = 1;
  gbe_bucket_desc h2 = h;
  std::memset(h2.stride, 0, sizeof(h2.stride));
  std::memset(h2.shift, 0, sizeof(h2.shift));
  map.clear();
  int n2 = 0;
  for (int j = 0; j < k; j++)
    if (!merged[j]) {
      for (int p = 0; p < m; p++) h2.stride[n2][p] = h.stride[j][p];
      h2.shift[n2] = h.shift[j];
      map.push_back(j);
      n2++;
    }
  const size_t el = h.semiring == GBE_MINSUM_I32 ? 4 : 8;
  for (auto &st : sets) {
    std::vector<int> U;  // union scope, ascending output position (lexicographic layout)
    for (int p = 0; p < m; p++)
      for (int j : st)
        if (has(j, p)) {
          U.push_back(p);
          break;
        }

    DevPlan::Merge M;
    M.task = (int32_t)ti;
    M.src.assign(st.begin(), st.end());
    gbe_bucket_desc &hm = M.h;
    std::memset(&hm, 0, sizeof(hm));
    hm.semiring = h.semiring == GBE_MINSUM_I32 ? GBE_MINSUM_I32 : GBE_MINSUM_F64;
    hm.nsep = (int32_t)U.size() + 1;  // U, then the eliminated variable as a plain digit
    hm.d = 1;
    hm.ninputs = (int32_t)st.size();
    hm.rows = 1;
    for (size_t q = 0; q < U.size(); q++) {
      hm.radix[q] = h.radix[U[q]];
      hm.rows *= h.radix[U[q]];
    }
    hm.radix[U.size()] = d;
    hm.rows *= d;
    for (size_t i = 0; i < st.size(); i++) {
      for (size_t q = 0; q < U.size(); q++) hm.stride[i][q] = h.stride[st[i]][U[q]];
      hm.stride[i][U.size()] = 1;
    }
    M.li = bk_plan_launch(hm, 0, hm.rows, BK_GENERIC, D->num_sms);
    // the sum (a d = 1 bucket) streams: tiles of the trailing digits, vector
    // loads, several rows per lane (bk_generic measured 0.8 TB/s on C4's
    // largest merges); GBE_MERGE_GENERIC: A/B knob
    static const bool mg = std::getenv("GBE_MERGE_GENERIC") != nullptr;
    M.stream = !mg && bks_build(hm, 0, hm.rows, D->num_sms, M.sd, M.sl);
    M.bytes = el * (size_t)hm.rows;
    // the bucket reads the merged table with its own mixed-radix strides
    int64_t st_ = d;
    for (int q = (int)U.size() - 1; q >= 0; q--) {
      h2.stride[n2][U[q]] = st_;
      st_ *= h.radix[U[q]];
    }
    map.push_back(-(1 + (int32_t)D->merges.size()));
    D->task_merges[ti].push_back((int32_t)D->merges.size());
    D->merges.push_back(std::move(M));
    n2++;
  }
  h2.ninputs = n2;
  h = h2;
}

// Tiled (register-blocked, TMA ring) vs streaming kernel for a bucket both
// can run.  GBE_KERNEL_POLICY=tiled|stream forces one (A/B knob).
static int kernel_policy() {
  static const int pol = [] {
    const char *e = std::getenv("GBE_KERNEL_POLICY");
    if (!e) return -1;
    return std::strcmp(e, "stream") == 0 ? 1 : (std::strcmp(e, "tiled") == 0 ? 0 : -1);
  }();
  return pol;
}
static bool prefer_stream(const gbe_bucket_desc &h, const BkfLaunch &fl) {
  const int pol = kernel_policy();
  if (pol >= 0) return pol == 1;
  // without timings: float64 buckets stream (C5: 17.5 vs 21.1 ms), int32
  // buckets take the register-blocked tiled kernel (C4: 28.3 vs 45.4 ms)
  (void)fl;
  return h.semiring != GBE_MINSUM_I32;
}

// Out-of-core chunks (planner.cpp plan_spill): every task runs in chunks of
// t.chunk_rows rows; a chunk's slot holds its output rows when the message
// lives on the host, its argmins (streamed to host memory), and the slices of
// its host-resident inputs (copied in on the H2D stream while the previous
// chunk computes: Fig. 8).
static void plan_spill_chunks(const Plan &P, DevPlan *D, bool noinf) {
  const size_t el = P.prob->elem();
  const size_t nt = P.tasks.size();
  D->chunks.assign(nt, {});
  D->harg_off.assign(nt, 0);
  D->msg_off.assign(nt, SIZE_MAX);
  size_t aoff = 0, moff = 0;
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  for (size_t ti = 0; ti < nt; ti++) {
    const Task &t = P.tasks[ti];
    D->harg_off[ti] = aoff;
    aoff += (size_t)std::max<int64_t>(t.rows, 1);
    if (t.host) {
      D->msg_off[ti] = moff;
      moff += up(el * (size_t)t.rows);
    }
    int64_t blocks = 1;
    for (int q = 0; q < t.chunk_digits; q++) blocks *= t.desc.radix[q];
    const int64_t brows = t.rows / blocks;
    for (int64_t b0 = 0; b0 < blocks; b0 += t.chunk_blocks) {
      const int64_t b1 = std::min(blocks, b0 + t.chunk_blocks);
      DevPlan::Chunk c;
      c.lo = b0 * brows;
      c.hi = b1 * brows;
      size_t off = 0;
      if (t.host) {
        c.out_off = off;
        off += up(el * (size_t)(c.hi - c.lo));
      }
      c.arg_off = off;
      off += up((size_t)(c.hi - c.lo));
      const std::vector<int32_t> &map = D->in_map[ti];
      for (size_t j = 0; j < map.size(); j++) {
        if (map[j] < 0) continue;  // a merged table (device)
        const Member &m = t.members[map[j]];
        if (m.kind != 1 || !P.tasks[m.index].host) continue;
        const SpillChunk r = spill_chunk_input(P, ti, t.chunk_digits, b0, b1, map[j]);
        c.hin.push_back({(int)j, m.index, r.lo, r.n, off});
        off += up(el * (size_t)r.n + 64);
      }
      if ((int64_t)off > P.slot_bytes)
        GBE_FAIL(GBE_E_INTERNAL, "spill chunk of x%d needs %zu bytes > slot %lld", t.var, off,
                 (long long)P.slot_bytes);
      FastDesc F;
      BkfLaunch L;
      StreamDesc Sd;
      if (D->use_fast[ti] && bkf_build(D->h_desc[ti], c.lo, c.hi, D->num_sms, F, L, noinf)) {
        c.fidx = (int)D->h_cfast.size();
        D->h_cfast.push_back(F);
        D->cfl.push_back(L);
      } else if (D->use_stream[ti] && bks_build(D->h_desc[ti], c.lo, c.hi, D->num_sms, Sd, c.sl)) {
        c.stream = true;
        c.sidx = (int)D->h_cstream.size();
        D->h_cstream.push_back(Sd);
      } else {
        c.li = bk_plan_launch(D->h_desc[ti], c.lo, c.hi, BK_GENERIC, D->num_sms);
      }
      D->chunks[ti].push_back(std::move(c));
    }
  }
  if (P.ex.host_args) {
    CK(cudaHostAlloc((void **)&D->h_harg, std::max<size_t>(aoff, 1), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void **)&D->d_harg, D->h_harg, 0));
  }
  if (moff) CK(cudaHostAlloc((void **)&D->h_msg, moff, cudaHostAllocDefault));
  CK(cudaMalloc(&D->d_slot, 2 * (size_t)P.slot_bytes));
  CK(cudaMalloc(&D->d_cfast, sizeof(FastDesc) * std::max<size_t>(D->h_cfast.size(), 1)));
  if (!D->h_cfast.empty())
    CK(cudaMemcpy(D->d_cfast, D->h_cfast.data(), sizeof(FastDesc) * D->h_cfast.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_cstream, sizeof(StreamDesc) * std::max<size_t>(D->h_cstream.size(), 1)));
  if (!D->h_cstream.empty())
    CK(cudaMemcpy(D->d_cstream, D->h_cstream.data(), sizeof(StreamDesc) * D->h_cstream.size(),
                  cudaMemcpyHostToDevice));
  CK(cudaStreamCreateWithFlags(&D->cp_stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&D->h2d_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; i++) {
    CK(cudaEventCreateWithFlags(&D->k_ev[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&D->c_ev[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&D->h_ev[i], cudaEventDisableTiming));
  }
  D->done_ev.assign(nt, nullptr);
  for (size_t ti = 0; ti < nt; ti++)
    if (P.tasks[ti].host) CK(cudaEventCreateWithFlags(&D->done_ev[ti], cudaEventDisableTiming));
}

static DevPlan *dev_plan(gbe_plan *gp) {
  if (gp->dev) return (DevPlan *)gp->dev;
  const Plan &P = *gp->plan;
  const Problem &p = *P.prob;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    GBE_FAIL(GBE_E_CUDA, "no CUDA device: libgbe has no CPU fallback");
  if (P.ex.device >= ndev) GBE_FAIL(GBE_E_INVALID, "device %d not present (%d devices)", P.ex.device, ndev);
  CK(cudaSetDevice(P.ex.device));
  auto *D = new DevPlan();
  D->device = P.ex.device;
  CK(cudaDeviceGetAttribute(&D->num_sms, cudaDevAttrMultiProcessorCount, D->device));
  // infinity-free int32 problems take the packed-key kernels: no entry is INF,
  // so no table is, and every cell sum stays below (maxsum << 3) + 7 < 2^32
  static const bool nf_off = std::getenv("GBE_NO_NF") != nullptr;  // A/B knob
  const bool noinf = !nf_off && !p.is_f64() && !P.ex.sumprod && !p.has_inf && p.maxsum < (int64_t(1) << 29) - 1;
  // descriptors with the per-rank input shifts (row-sharded messages kept local)
  D->h_desc.resize(P.tasks.size());
  D->launch.resize(P.tasks.size());
  D->h_fast.resize(P.tasks.size());
  D->h_fds.resize(P.tasks.size());
  D->fl_ds.resize(P.tasks.size());
  D->use_ds.assign(P.tasks.size(), 0);
  D->fl.resize(P.tasks.size());
  D->use_fast.assign(P.tasks.size(), 0);
  D->h_stream.resize(P.tasks.size());
  D->sl.resize(P.tasks.size());
  D->use_stream.assign(P.tasks.size(), 0);
  D->h_stage.resize(P.tasks.size());
  D->sl3.resize(P.tasks.size());
  D->use_stage.assign(P.tasks.size(), 0);
  D->h_half.resize(P.tasks.size());
  D->slh.resize(P.tasks.size());
  D->use_half.assign(P.tasks.size(), 0);
  D->cands.assign(P.tasks.size(), {});
  D->t_cand.assign(P.tasks.size(), {});
  D->tune_nc = 0;
  D->task_merges.assign(P.tasks.size(), {});
  D->in_map.assign(P.tasks.size(), {});
  for (size_t ti = 0; ti < P.tasks.size(); ti++) {
    const Task &t = P.tasks[ti];
    gbe_bucket_desc h = t.desc;
    for (int j = 0; j < h.ninputs; j++) {
      h.shift[j] = 0;
      const Member &m = t.members[j];
      if (m.kind == 1) {
        const Task &src = P.tasks[m.index];
        if (src.shard.on && !src.shard.gather) h.shift[j] = src.shard.lo;
      }
    }
    if (P.ex.count) {  // counting plans: bk_count (generic tiling), inputs as declared
      D->in_map[ti].resize(h.ninputs);
      for (int j = 0; j < h.ninputs; j++) D->in_map[ti][j] = j;
    } else {
      plan_merges(P, D, ti, h, noinf);
    }
    D->h_desc[ti] = h;
    D->launch[ti] = bk_plan_launch(h, t.shard.lo, t.shard.hi, P.ex.kernel, D->num_sms);
    // kernel variant: tiled TMA (1), streaming (2), generic (0)
    const int want = P.ex.kernel;  // -1 auto
    const bool fast_ok = (want == -1 || want == 1) && !P.ex.count &&
                         bkf_build(h, t.shard.lo, t.shard.hi, D->num_sms, D->h_fast[ti], D->fl[ti], noinf);
    const bool stream_ok = (want == -1 || want == 2) && !P.ex.count &&
                           bks_build(h, t.shard.lo, t.shard.hi, D->num_sms, D->h_stream[ti], D->sl[ti]);
    // staged mode (GBE_STREAM_STAGE: unset/0 never -- measured 2-4x slower
    // on C5 and C4-d4; 1 the default wherever it fits; 2 an
    // autotuning candidate)
    static const int stage_env = [] {
      const char *e = std::getenv("GBE_STREAM_STAGE");
      return e ? std::atoi(e) : 0;
    }();
    const bool stage_ok = stream_ok && stage_env != 0 && !P.ex.host_args && !P.ex.spill &&
                          bks_build(h, t.shard.lo, t.shard.hi, D->num_sms, D->h_stage[ti], D->sl3[ti], true);
    if (fast_ok && (!stream_ok || !prefer_stream(h, D->fl[ti])) && !(stage_ok && stage_env == 1)) {
      D->use_fast[ti] = 1;
      D->launch[ti].variant = 1;
    } else if (stream_ok) {
      D->use_stream[ti] = 1;
      D->use_stage[ti] = stage_ok && stage_env == 1;
      D->launch[ti].variant = 2;
    }
    // autotuning candidates: the default first, then the other variant and
    // the streaming kernel with its L2 prefetch flipped (unless forced)
    const bool tune = want == -1 && P.ex.autotune && kernel_policy() < 0 && !P.ex.host_args && !P.ex.spill;
    if (tune && (fast_ok || stream_ok)) {
      static const bool pf_forced = std::getenv("GBE_STREAM_PF") != nullptr;
      auto &cs = D->cands[ti];
      const bool pf = D->sl[ti].pf, pf_alt = stream_ok && D->sl[ti].pf_ok && !pf_forced;
      if (D->use_fast[ti]) cs.push_back({1, false, false, false});
      if (D->use_stage[ti]) cs.push_back({2, false, true, false});
      if (stream_ok) cs.push_back({2, pf, false, false});
      if (fast_ok && !D->use_fast[ti]) cs.push_back({1, false, false, false});
      if (pf_alt) cs.push_back({2, !pf, false, false});
      if (stage_ok && !D->use_stage[ti]) cs.push_back({2, false, true, false});
      // direct-store tiled descriptor (hot int32 shape; GBE_FAST_DS=0: off)
      static const bool ds_off = [] {
        const char *e = std::getenv("GBE_FAST_DS");
        return e && std::atoi(e) == 0;
      }();
      if (fast_ok && !ds_off && bkf_build(h, t.shard.lo, t.shard.hi, D->num_sms, D->h_fds[ti], D->fl_ds[ti], noinf, true))
        cs.push_back({1, false, false, false, true});
      // half-tile streaming descriptor (when it really has shorter tiles)
      static const bool half_off = [] {
        const char *e = std::getenv("GBE_STREAM_HALF");
        return e && std::atoi(e) == 0;
      }();
      if (stream_ok && !half_off && D->h_stream[ti].PL >= 64 &&
          bks_build(h, t.shard.lo, t.shard.hi, D->num_sms, D->h_half[ti], D->slh[ti], false,
                    D->h_stream[ti].PL / 2) &&
          D->h_half[ti].PL < D->h_stream[ti].PL) {
        const bool hp = D->slh[ti].pf;
        cs.push_back({2, hp, false, true});
        if (D->slh[ti].pf_ok && !pf_forced) cs.push_back({2, !hp, false, true});
      }
      if (cs.size() < 2) cs.clear();
      if (!cs.empty()) {
        D->tune_phase = 0;
        D->tune_nc = std::max(D->tune_nc, (int)cs.size());
        D->t_cand[ti].assign(cs.size(), 0.f);
      }
    }
  }
  if (P.ex.spill) {
    plan_spill_chunks(P, D, noinf);
  } else if (P.ex.host_args) {  // row chunks per task, host argmin layout, ring, copy stream
    D->chunks.assign(P.tasks.size(), {});
    D->harg_off.assign(P.tasks.size(), 0);
    size_t off = 0;
    for (size_t ti = 0; ti < P.tasks.size(); ti++) {
      const Task &t = P.tasks[ti];
      D->harg_off[ti] = off;
      off += (size_t)std::max<int64_t>(t.rows, 1);
      int64_t step = std::max<int64_t>(1, std::min<int64_t>(t.rows, P.ex.host_arg_chunk));
      if (D->use_fast[ti]) {
        const int64_t PL = D->h_fast[ti].hot.PL;
        step = std::max<int64_t>(PL, step / PL * PL);
      }
      for (int64_t lo = 0; lo < t.rows; lo += step) {
        DevPlan::Chunk c;
        c.lo = lo;
        c.hi = std::min<int64_t>(t.rows, lo + step);
        FastDesc F;
        BkfLaunch L;
        StreamDesc Sd;
        if (D->use_fast[ti] && bkf_build(D->h_desc[ti], c.lo, c.hi, D->num_sms, F, L, noinf)) {
          c.fidx = (int)D->h_cfast.size();
          D->h_cfast.push_back(F);
          D->cfl.push_back(L);
        } else if (D->use_stream[ti] && bks_build(D->h_desc[ti], c.lo, c.hi, D->num_sms, Sd, c.sl)) {
          c.stream = true;
          c.sidx = (int)D->h_cstream.size();
          D->h_cstream.push_back(Sd);
        } else {
          c.li = bk_plan_launch(D->h_desc[ti], c.lo, c.hi, BK_GENERIC, D->num_sms);
        }
        D->ring = std::max<int64_t>(D->ring, c.hi - c.lo);
        D->chunks[ti].push_back(c);
      }
    }
    CK(cudaHostAlloc((void **)&D->h_harg, std::max<size_t>(off, 1), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void **)&D->d_harg, D->h_harg, 0));
    CK(cudaMalloc(&D->d_ring, 2 * (size_t)std::max<int64_t>(D->ring, 1)));
    CK(cudaMalloc(&D->d_cfast, sizeof(FastDesc) * std::max<size_t>(D->h_cfast.size(), 1)));
    if (!D->h_cfast.empty())
      CK(cudaMemcpy(D->d_cfast, D->h_cfast.data(), sizeof(FastDesc) * D->h_cfast.size(), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&D->d_cstream, sizeof(StreamDesc) * std::max<size_t>(D->h_cstream.size(), 1)));
    if (!D->h_cstream.empty())
      CK(cudaMemcpy(D->d_cstream, D->h_cstream.data(), sizeof(StreamDesc) * D->h_cstream.size(),
                    cudaMemcpyHostToDevice));
    CK(cudaStreamCreateWithFlags(&D->cp_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++) {
      CK(cudaEventCreateWithFlags(&D->k_ev[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&D->c_ev[i], cudaEventDisableTiming));
    }
  }
  CK(cudaMalloc(&D->d_stream, sizeof(StreamDesc) * std::max<size_t>(P.tasks.size(), 1)));
  if (!P.tasks.empty())
    CK(cudaMemcpy(D->d_stream, D->h_stream.data(), sizeof(StreamDesc) * P.tasks.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_half, sizeof(StreamDesc) * std::max<size_t>(P.tasks.size(), 1)));
  if (!P.tasks.empty())
    CK(cudaMemcpy(D->d_half, D->h_half.data(), sizeof(StreamDesc) * P.tasks.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_stage, sizeof(StreamDesc) * std::max<size_t>(P.tasks.size(), 1)));
  if (!P.tasks.empty())
    CK(cudaMemcpy(D->d_stage, D->h_stage.data(), sizeof(StreamDesc) * P.tasks.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_fds, sizeof(FastDesc) * std::max<size_t>(P.tasks.size(), 1)));
  if (!P.tasks.empty())
    CK(cudaMemcpy(D->d_fds, D->h_fds.data(), sizeof(FastDesc) * P.tasks.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_fast, sizeof(FastDesc) * std::max<size_t>(P.tasks.size(), 1)));
  if (!P.tasks.empty())
    CK(cudaMemcpy(D->d_fast, D->h_fast.data(), sizeof(FastDesc) * P.tasks.size(), cudaMemcpyHostToDevice));
  size_t nt = std::max<size_t>(P.tasks.size(), 1);
  CK(cudaMalloc(&D->d_mdesc, sizeof(gbe_bucket_desc) * std::max<size_t>(D->merges.size(), 1)));
  for (size_t mi = 0; mi < D->merges.size(); mi++)
    CK(cudaMemcpy(D->d_mdesc + mi, &D->merges[mi].h, sizeof(gbe_bucket_desc), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_mstream, sizeof(StreamDesc) * std::max<size_t>(D->merges.size(), 1)));
  for (size_t mi = 0; mi < D->merges.size(); mi++)
    CK(cudaMemcpy(D->d_mstream + mi, &D->merges[mi].sd, sizeof(StreamDesc), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_desc, sizeof(gbe_bucket_desc) * nt));
  if (!P.tasks.empty())
    CK(cudaMemcpy(D->d_desc, D->h_desc.data(), sizeof(gbe_bucket_desc) * P.tasks.size(), cudaMemcpyHostToDevice));
  // relayout metadata
  std::vector<int32_t> poff(p.nf + 1, 0), prad;
  for (int f = 0; f < p.nf; f++) poff[f + 1] = poff[f] + p.arity[f];
  prad.resize(std::max<int32_t>(poff[p.nf], 1));
  for (int f = 0; f < p.nf; f++) {
    std::vector<int32_t> sc(p.scope(f), p.scope(f) + p.arity[f]);
    std::sort(sc.begin(), sc.end(), [&](int a, int b) { return P.pos[a] < P.pos[b]; });
    for (int q = 0; q < p.arity[f]; q++) prad[poff[f] + q] = p.dom[sc[q]];
  }
  std::vector<int32_t> pstr = P.perm_strides;
  pstr.resize(std::max<size_t>(pstr.size(), 1));
  CK(cudaMalloc(&D->d_off, sizeof(int64_t) * (p.nf + 1)));
  CK(cudaMemcpy(D->d_off, p.table_off.data(), sizeof(int64_t) * (p.nf + 1), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_poff, sizeof(int32_t) * (p.nf + 1)));
  CK(cudaMemcpy(D->d_poff, poff.data(), sizeof(int32_t) * (p.nf + 1), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_prad, sizeof(int32_t) * prad.size()));
  CK(cudaMemcpy(D->d_prad, prad.data(), sizeof(int32_t) * prad.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&D->d_pstride, sizeof(int32_t) * pstr.size()));
  CK(cudaMemcpy(D->d_pstride, pstr.data(), sizeof(int32_t) * pstr.size(), cudaMemcpyHostToDevice));
  // pinned host staging of the inputs (the H2D of every solve reads this)
  D->raw_bytes = p.elem() * (size_t)p.table_off[p.nf];
  CK(cudaMallocHost(&D->h_raw, std::max<size_t>(D->raw_bytes, 16)));
  if (D->raw_bytes)
    std::memcpy(D->h_raw, p.is_f64() ? (const void *)p.fcost.data() : (const void *)p.icost.data(), D->raw_bytes);
  // stream-ordered pool: keep freed memory reserved between solves
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, D->device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  gp->dev = D;
  return D;
}

void dev_plan_free(void *d) { delete (DevPlan *)d; }

// ---------------------------------------------------------------------------
// a run: device-resident messages / argmins of one UTIL phase

struct RunImpl {
  gbe_plan *gp = nullptr;
  DevPlan *D = nullptr;
  cudaStream_t stream = nullptr;
  bool mbe = false;
  void *d_raw = nullptr, *d_sorted = nullptr;
  char *base = nullptr;         // arena of this run
  DevPlan::Arena *A = nullptr;  // its layout
  bool arena_own = false;       // base allocated for this run (cached arena busy)
  std::vector<void *> out, full;
  std::vector<uint8_t *> arg;
  std::vector<cudaEvent_t> ev;
  std::vector<float> ms, merge_ms;  // per task: total (merges + bucket) and merges only
  void *d_opt = nullptr;
  int32_t *d_assign = nullptr, *d_gbuf = nullptr;
  gbe_value optimum{};
  double count = 0.0;           // counting plans: number of optimal / consistent solutions
  bool util_done = false;
  bool shared_scalars = false;  // d_opt / d_assign belong to the arena (graph path)
  bool args_written = false;    // the bucket kernels wrote argmin tables (byte accounting)
  bool replayed = false;        // this UTIL phase was a CUDA-graph replay
  bool tuned = false;           // this solve was an autotuning solve
  ~RunImpl() { release(); }
  void release() {
    if (!D) return;
    cudaSetDevice(D->device);
    cudaStreamSynchronize(stream);  // the arena may be handed to the next run
    out.clear();
    full.clear();
    arg.clear();
    if (base) {
      if (arena_own) dfree(base, stream);
      else A->busy = false;
      base = nullptr;
    }
    if (!shared_scalars) {
      dfree(d_opt, stream);
      dfree(d_assign, stream);
    }
    dfree(d_gbuf, stream);
    d_raw = d_sorted = d_opt = nullptr;
    d_assign = d_gbuf = nullptr;
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    cudaStreamSynchronize(stream);
  }
  const void *msg_ptr(int ti) const { return full[ti] ? full[ti] : out[ti]; }
  const void *member_ptr(const Member &m) const {
    const Problem &p = *gp->plan->prob;
    if (m.kind == 0) return (const char *)d_sorted + p.elem() * p.table_off[m.index];
    return msg_ptr(m.index);
  }
};

static gbe_value read_value(const Problem &p, const void *host) {
  gbe_value v{0, 0, 0.0};
  if (p.is_f64()) {
    v.f = *(const double *)host;
    v.is_inf = std::isinf(v.f) ? 1 : 0;
  } else {
    v.i = *(const int32_t *)host;
    v.is_inf = v.i >= kInfI32 ? 1 : 0;
  }
  return v;
}

// UTIL / elimination phase (Alg. 1 lines 1-5, Alg. 2 lines 1-7)
static void run_util(RunImpl &R) {
  gbe_plan *gp = R.gp;
  const Plan &P = *gp->plan;
  const Problem &p = *P.prob;
  DevPlan *D = R.D;
  cudaStream_t s = R.stream;
  const size_t el = p.elem();
  const int W = P.ex.world_size;
  const size_t nt = P.tasks.size();

  // pre-flight memory budget: plan estimate vs what the device has
  // (once: later runs reuse the plan's arena)
  if (!D->arena[R.mbe ? 1 : 0].mem) {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    uint64_t reserved = 0, used = 0;
    cudaMemPool_t pool;
    if (!g_alloc && cudaDeviceGetDefaultMemPool(&pool, D->device) == cudaSuccess) {
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    int64_t avail = (int64_t)fr + (int64_t)(reserved - used);
    if (P.peak_bytes > avail) {
      const Task *big = &P.tasks[0];
      for (auto &t : P.tasks)
        if (t.rows > big->rows) big = &t;
      GBE_FAIL(GBE_E_BUDGET, "bucket x%d: %.3g rows; plan needs %.3g bytes > %.3g available on device %d",
               big->var, (double)big->rows, (double)P.peak_bytes, (double)avail, D->device);
    }
  }

  R.out.assign(nt, nullptr);
  R.full.assign(nt, nullptr);
  R.arg.assign(nt, nullptr);
  {
    DevPlan::Arena &A = D->arena[R.mbe ? 1 : 0];
    if (!A.planned) plan_arena(P, D, R.mbe);
    R.A = &A;
    if (!A.busy) {
      if (!A.mem) {
        A.hook = g_alloc != nullptr;
        A.mem = A.hook ? g_alloc(A.bytes, (void *)s, g_alloc_u) : nullptr;
        if (!A.hook) {
          cudaError_t e = cudaMalloc(&A.mem, A.bytes);
          if (e != cudaSuccess)
            GBE_FAIL(GBE_E_BUDGET, "device arena of %.3g bytes: %s", (double)A.bytes, cudaGetErrorString(e));
        }
        if (!A.mem) GBE_FAIL(GBE_E_BUDGET, "device arena of %.3g bytes", (double)A.bytes);
      }
      A.busy = true;
      R.base = (char *)A.mem;
    } else {
      R.base = (char *)dalloc(A.bytes, s);
      R.arena_own = true;
    }
  }
  // ---- host pass: buffer addresses and launch inputs.  With an arena these
  // are the same for every run of the plan, which is what makes the device
  // pass below replayable as a CUDA graph.
  if (P.ex.resident_inputs) {
    if (!D->resident) {
      D->d_resident = nullptr;
      CK(cudaMalloc(&D->d_resident, std::max<size_t>(D->raw_bytes, 16)));
      CK(cudaMemcpy(D->d_resident, D->h_raw, D->raw_bytes, cudaMemcpyHostToDevice));
      D->resident = true;
    }
    R.d_raw = D->d_resident;
  } else {
    R.d_raw = R.base + R.A->off_raw;
  }
  R.d_sorted = R.base + R.A->off_sorted;
  const bool want_arg = ((!R.mbe && P.ex.retain >= 1) || P.ex.retain >= 2) && !P.ex.sumprod;
  const bool host_args = P.ex.host_args;
  std::vector<InPtrs> ins(nt), mins(D->merges.size());
  std::vector<void *> gathered_src(nt, nullptr);
  for (size_t ti = 0; ti < nt; ti++) {
    const Task &t = P.tasks[ti];
    R.out[ti] = t.host ? (void *)(D->h_msg + D->msg_off[ti]) : (void *)(R.base + R.A->off_out[ti]);
    if (host_args) R.arg[ti] = D->d_harg + D->harg_off[ti];
    else if (want_arg) R.arg[ti] = (uint8_t *)(R.base + R.A->off_arg[ti]);
    const std::vector<int32_t> &map = D->in_map[ti];
    for (size_t j = 0; j < map.size(); j++)
      ins[ti].p[j] = map[j] >= 0 ? R.member_ptr(t.members[map[j]]) : R.base + R.A->off_merge[-(map[j] + 1)];
    for (int32_t mi : D->task_merges[ti])
      for (size_t q = 0; q < D->merges[mi].src.size(); q++)
        mins[mi].p[q] = R.member_ptr(t.members[D->merges[mi].src[q]]);
    if (t.shard.on && t.shard.gather) {
      gathered_src[ti] = R.out[ti];
      R.full[ti] = R.base + R.A->off_full[ti];
      R.out[ti] = nullptr;
    }
    // consumed messages are dead (BE/DPOP; MBE keeps them for its value phase, A7)
    if ((!R.mbe || P.ex.retain == 0) && P.ex.retain < 2)
      for (auto &m : t.members)
        if (m.kind == 1) R.out[m.index] = R.full[m.index] = nullptr;
  }
  std::vector<const void *> cptrs;
  for (auto &m : P.constants) cptrs.push_back(R.member_ptr(m));
  // counting plans: count tables of the members / constants (nullptr for an
  // original function: every entry counts 1)
  auto cnt_ptr = [&](const Member &m) -> const void * {
    return (P.ex.count && m.kind == 1) ? (const void *)(R.base + R.A->off_cnt[m.index]) : nullptr;
  };
  std::vector<const void *> ccptrs;
  for (auto &m : P.constants) ccptrs.push_back(cnt_ptr(m));
  std::vector<InPtrs> cins(P.ex.count ? nt : 0);
  for (size_t ti = 0; ti < cins.size(); ti++)
    for (int j = 0; j < P.tasks[ti].desc.ninputs; j++) cins[ti].p[j] = cnt_ptr(P.tasks[ti].members[j]);

  DevPlan::Arena &A = *R.A;
  // a table hook inspects every bucket on the host: serial, no graph, and an
  // argmin scratch buffer when the plan does not retain argmins
  const TableHook hook = g_hook;
  void *const hook_u = g_hook_u;
  // W > 1: the UTIL phase is still one CUDA graph when the all-gather is the
  // built-in NCCL one (it only enqueues work on the stream; a Python hook
  // that stages through the host cannot be captured)
  // autotuning solve: eager, candidates forced to one variant, timed
  const bool tuning = D->tune_phase >= 0 && D->tune_phase < 2 * D->tune_nc;
  if (tuning) {
    while (D->tune_ev.size() < 2 * nt) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      D->tune_ev.push_back(e);
    }
    for (size_t ti = 0; ti < nt; ti++)
      if (!D->cands[ti].empty()) {
        const int ci = D->tune_phase % D->tune_nc;
        const DevPlan::Cand c = D->cands[ti][ci < (int)D->cands[ti].size() ? ci : 0];
        D->use_fast[ti] = c.variant == 1;
        D->use_stream[ti] = c.variant == 2;
        D->use_stage[ti] = c.stage;
        D->use_half[ti] = c.half;
        D->use_ds[ti] = c.ds;
        (c.half ? D->slh[ti] : D->sl[ti]).pf = c.pf;
      }
  }
  const bool graph = P.ex.graph && (W == 1 || g_ag_graph) && !g_alloc && !R.arena_own && !P.ex.host_args &&
                     !P.ex.spill && !hook && !tuning;
  uint8_t *hook_arg = nullptr;
  if (hook && !want_arg && !host_args && !P.ex.sumprod) {
    int64_t mx = 1;
    for (auto &t : P.tasks) mx = std::max<int64_t>(mx, t.shard.hi - t.shard.lo);
    hook_arg = (uint8_t *)dalloc((size_t)mx, s);
  }
  struct HookArgFree {
    uint8_t *p;
    cudaStream_t s;
    ~HookArgFree() {
      if (p) {
        cudaStreamSynchronize(s);
        dfree(p, s);
      }
    }
  } hook_arg_free{hook_arg, s};
  R.args_written = want_arg || host_args || hook_arg != nullptr;
  if (graph) {  // persistent per-arena scalars, pinned result slot, events
    if (!A.d_opt) {
      CK(cudaMalloc(&A.d_opt, 16));
      CK(cudaMalloc(&A.d_assign, sizeof(int32_t) * std::max(p.n, 1)));
      CK(cudaMalloc(&A.d_cp, sizeof(void *) * std::max<size_t>(cptrs.size(), 1)));
      if (!cptrs.empty())
        CK(cudaMemcpy(A.d_cp, cptrs.data(), sizeof(void *) * cptrs.size(), cudaMemcpyHostToDevice));
      CK(cudaMalloc(&A.d_ccp, sizeof(void *) * std::max<size_t>(ccptrs.size(), 1)));
      if (!ccptrs.empty())
        CK(cudaMemcpy(A.d_ccp, ccptrs.data(), sizeof(void *) * ccptrs.size(), cudaMemcpyHostToDevice));
      CK(cudaMallocHost(&A.h_opt, 16));
    }
    if (P.ex.timing && A.ev.empty()) {
      A.ev.resize(3 * nt);
      for (auto &e : A.ev) CK(cudaEventCreate(&e));
    }
    R.d_opt = A.d_opt;
    R.d_assign = A.d_assign;
    R.shared_scalars = true;
  } else {
    R.d_opt = dalloc(16, s);
    R.d_assign = (int32_t *)dalloc(sizeof(int32_t) * std::max(p.n, 1), s);
    if (P.ex.timing) {
      R.ev.resize(3 * nt);
      for (auto &e : R.ev) CK(cudaEventCreate(&e));
    }
  }
  std::vector<cudaEvent_t> &ev = graph ? A.ev : R.ev;
  void *d_cp = graph ? A.d_cp : nullptr;
  void *d_ccp = graph ? A.d_ccp : nullptr;
  alignas(16) unsigned char hopt_local[16] = {0};
  unsigned char *hopt = graph ? (unsigned char *)A.h_opt : hopt_local;

  // ---- device pass: one batched H2D, relayout, one BK per bucket, constants
  auto enqueue = [&](cudaStream_t st, bool capturing) {
    // inside a capture a timing event must be an external event-record node
    auto rec = [&](cudaEvent_t e) {
      CK(capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st));
    };
    if (!P.ex.resident_inputs)
      CK(cudaMemcpyAsync(R.d_raw, D->h_raw, D->raw_bytes, cudaMemcpyHostToDevice, st));
    CK(relayout_launch(R.d_raw, R.d_sorted, (int)el, p.nf, D->d_off, D->d_poff, D->d_prad,
                       D->d_pstride, st));
    // concurrent subtrees: inside a capture (and without per-launch timing)
    // each task runs on a branch that waits only on its DAG predecessors;
    // otherwise the tasks run in creation order on `st`
    const bool dag = capturing && P.ex.concurrent && !P.ex.timing && nt > 1;
    std::vector<int> last_on;   // last task enqueued on each branch
    std::vector<int> branch_of(nt, -1);
    if (dag) {
      static const size_t kBranches = [] {
        const char *e = std::getenv("GBE_BRANCHES");
        return (size_t)std::max(1, e ? std::atoi(e) : 16);
      }();
      while (D->side.size() < kBranches) {
        cudaStream_t b;
        CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
        D->side.push_back(b);
      }
      while (D->tev.size() < nt + 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        D->tev.push_back(e);
      }
      CK(cudaEventRecord(D->tev[nt], st));  // fork after the relayout
      last_on.assign(D->side.size(), -2);   // -2: branch not forked yet
    }
    size_t rr = 0;
    int64_t ring_n = 0;  // argmin chunks streamed so far (host_args)
    // collectives must run in the same order on every rank: inside the DAG
    // each all-gathering task also waits for the previous one
    int last_gather = -1;
    for (size_t ti = 0; ti < nt; ti++) {
      const Task &t = P.tasks[ti];
      const Shard &sh = t.shard;
      cudaStream_t st0 = st;
      if (dag) {
        const std::vector<int32_t> &dp = A.deps[ti];
        int b = -1;  // continue the branch whose last task is a predecessor
        for (size_t q = 0; q < last_on.size() && b < 0; q++)
          if (last_on[q] >= 0 && std::binary_search(dp.begin(), dp.end(), last_on[q])) b = (int)q;
        if (b < 0) b = (int)(rr++ % last_on.size());
        st = D->side[b];
        if (last_on[b] == -2) CK(cudaStreamWaitEvent(st, D->tev[nt], 0));
        for (int32_t k : dp)
          if (branch_of[k] != b) CK(cudaStreamWaitEvent(st, D->tev[k], 0));
        if (gathered_src[ti] && last_gather >= 0 && branch_of[last_gather] != b)
          CK(cudaStreamWaitEvent(st, D->tev[last_gather], 0));
        last_on[b] = (int)ti;
        branch_of[ti] = b;
      }
      void *out = gathered_src[ti] ? gathered_src[ti]
                  : t.host            ? (void *)(D->h_msg + D->msg_off[ti])
                                      : (void *)(R.base + R.A->off_out[ti]);
      uint8_t *argp = want_arg && !host_args ? (uint8_t *)(R.base + R.A->off_arg[ti]) : hook_arg;
      if (P.ex.timing) rec(ev[3 * ti]);
      for (int32_t mi : D->task_merges[ti]) {
        const DevPlan::Merge &M = D->merges[mi];
        if (M.stream)
          CK(bks_launch(D->d_mstream + mi, M.sl, mins[mi], R.base + R.A->off_merge[mi], nullptr, 0, M.h.rows, st));
        else
          CK(bk_launch(M.h, D->d_mdesc + mi, mins[mi], R.base + R.A->off_merge[mi], nullptr, 0, M.h.rows, M.li, st));
        static const bool sync_m = std::getenv("GBE_SYNC_EACH") != nullptr;  // debugging knob
        if (sync_m && !capturing) {
          cudaError_t e = cudaStreamSynchronize(st);
          if (e != cudaSuccess)
            GBE_FAIL(GBE_E_CUDA, "merge %d of task %zu (rows %lld, k %d): %s", mi, ti, (long long)M.h.rows,
                     M.h.ninputs, cudaGetErrorString(e));
        }
      }
      if (P.ex.timing) rec(ev[3 * ti + 1]);  // merges done
      if (P.ex.spill) {  // out-of-core: chunks through the two staging slots
        bool waited = false;
        for (const DevPlan::Chunk &c : D->chunks[ti]) {
          const int slot = ring_n & 1;
          char *sb = D->d_slot + (size_t)slot * P.slot_bytes;
          InPtrs in = ins[ti];
          if (!c.hin.empty()) {  // H2D of the host-resident input slices
            if (!waited) {
              for (const auto &hi : c.hin) CK(cudaStreamWaitEvent(D->h2d_stream, D->done_ev[hi.src], 0));
              waited = true;
            }
            if (ring_n >= 2) {  // the slot's previous chunk: inputs read, outputs / argmins copied out
              CK(cudaStreamWaitEvent(D->h2d_stream, D->k_ev[slot], 0));
              CK(cudaStreamWaitEvent(D->h2d_stream, D->c_ev[slot], 0));
            }
            for (const auto &hi : c.hin) {
              // the slice keeps the 16-byte phase it has in the full table, so
              // the kernel's aligned (TMA / vector) reads see the same layout
              const size_t ph = (size_t)(hi.lo * (int64_t)el) & 15;
              char *dst = sb + hi.off + ph;
              CK(cudaMemcpyAsync(dst, D->h_msg + D->msg_off[hi.src] + (size_t)hi.lo * el, (size_t)hi.n * el,
                                 cudaMemcpyHostToDevice, D->h2d_stream));
              in.p[hi.j] = (const void *)((uintptr_t)dst - (uintptr_t)hi.lo * el);
            }
            CK(cudaEventRecord(D->h_ev[slot], D->h2d_stream));
            CK(cudaStreamWaitEvent(st, D->h_ev[slot], 0));
          }
          if (ring_n >= 2) CK(cudaStreamWaitEvent(st, D->c_ev[slot], 0));  // slot outputs copied out
          void *oc = t.host ? (void *)(sb + c.out_off) : (void *)((char *)out + (size_t)c.lo * el);
          uint8_t *ra = host_args ? (uint8_t *)(sb + c.arg_off) : nullptr;
          if (c.fidx >= 0)
            CK(bkf_launch(D->d_cfast + c.fidx, D->cfl[c.fidx], in, oc, ra, c.lo, st));
          else if (c.stream)
            CK(bks_launch(D->d_cstream + c.sidx, c.sl, in, oc, ra, c.lo, c.hi, st));
          else
            CK(bk_launch(D->h_desc[ti], D->d_desc + ti, in, oc, ra, c.lo, c.hi, c.li, st));
          CK(cudaEventRecord(D->k_ev[slot], st));
          CK(cudaStreamWaitEvent(D->cp_stream, D->k_ev[slot], 0));
          if (t.host)
            CK(cudaMemcpyAsync(D->h_msg + D->msg_off[ti] + (size_t)c.lo * el, oc, (size_t)(c.hi - c.lo) * el,
                               cudaMemcpyDeviceToHost, D->cp_stream));
          if (ra)
            CK(cudaMemcpyAsync(D->h_harg + D->harg_off[ti] + c.lo, ra, (size_t)(c.hi - c.lo),
                               cudaMemcpyDeviceToHost, D->cp_stream));
          CK(cudaEventRecord(D->c_ev[slot], D->cp_stream));
          ring_n++;
        }
        if (t.host) CK(cudaEventRecord(D->done_ev[ti], D->cp_stream));
      } else if (host_args) {  // row chunks; argmins through the device ring to host memory
        for (const DevPlan::Chunk &c : D->chunks[ti]) {
          const int slot = ring_n & 1;
          if (ring_n >= 2) CK(cudaStreamWaitEvent(st, D->c_ev[slot], 0));  // slot copied out
          uint8_t *ra = D->d_ring + (size_t)slot * D->ring;
          void *oc = (char *)out + (size_t)(c.lo - sh.lo) * el;
          if (c.fidx >= 0)
            CK(bkf_launch(D->d_cfast + c.fidx, D->cfl[c.fidx], ins[ti], oc, ra, c.lo, st));
          else if (c.stream)
            CK(bks_launch(D->d_cstream + c.sidx, c.sl, ins[ti], oc, ra, c.lo, c.hi, st));
          else
            CK(bk_launch(D->h_desc[ti], D->d_desc + ti, ins[ti], oc, ra, c.lo, c.hi, c.li, st));
          CK(cudaEventRecord(D->k_ev[slot], st));
          CK(cudaStreamWaitEvent(D->cp_stream, D->k_ev[slot], 0));
          CK(cudaMemcpyAsync(D->h_harg + D->harg_off[ti] + (c.lo - sh.lo), ra, (size_t)(c.hi - c.lo),
                             cudaMemcpyDeviceToHost, D->cp_stream));
          CK(cudaEventRecord(D->c_ev[slot], D->cp_stream));
          ring_n++;
        }
      } else if (tuning && !D->cands[ti].empty()) {
        CK(cudaEventRecord(D->tune_ev[2 * ti], st));
        if (D->use_fast[ti])
          CK(D->use_ds[ti] ? bkf_launch(D->d_fds + ti, D->fl_ds[ti], ins[ti], out, argp, sh.lo, st)
                           : bkf_launch(D->d_fast + ti, D->fl[ti], ins[ti], out, argp, sh.lo, st));
        else
          CK(D->stream_launch(ti, ins[ti], out, argp, sh.lo, sh.hi, st));
        CK(cudaEventRecord(D->tune_ev[2 * ti + 1], st));
      } else if (P.ex.count)
        CK(bk_count_launch(D->h_desc[ti], D->d_desc + ti, ins[ti], cins[ti], out,
                           (double *)(R.base + R.A->off_cnt[ti]), argp, sh.lo, sh.hi, P.ex.count == 2, st));
      else if (D->use_fast[ti])
        CK(D->use_ds[ti] ? bkf_launch(D->d_fds + ti, D->fl_ds[ti], ins[ti], out, argp, sh.lo, st)
                         : bkf_launch(D->d_fast + ti, D->fl[ti], ins[ti], out, argp, sh.lo, st));
      else if (D->use_stream[ti])
        CK(D->stream_launch(ti, ins[ti], out, argp, sh.lo, sh.hi, st));
      else
        CK(bk_launch(D->h_desc[ti], D->d_desc + ti, ins[ti], out, argp, sh.lo, sh.hi, D->launch[ti], st));
      if (P.ex.timing) rec(ev[3 * ti + 2]);
      if (hook) {
        CK(cudaStreamSynchronize(st));
        const uint8_t *ha = host_args ? nullptr : argp;
        if (hook((int32_t)ti, out, ha, sh.lo, sh.hi - sh.lo, (void *)st, hook_u) != 0)
          GBE_FAIL(GBE_E_INTERNAL, "table hook failed on task %zu (x%d)", ti, t.var);
      }
      static const bool sync_each = std::getenv("GBE_SYNC_EACH") != nullptr;  // debugging knob
      if (sync_each && !capturing) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess)
          GBE_FAIL(GBE_E_CUDA, "task %zu (x%d, %zu merges, fast=%d nst=%d PL=%d k=%d): %s", ti, t.var,
                   D->task_merges[ti].size(), (int)D->use_fast[ti], D->h_fast[ti].hot.nstages,
                   D->h_fast[ti].hot.PL, D->h_fast[ti].hot.k, cudaGetErrorString(e));
      }
      if (gathered_src[ti]) {
        if (!g_ag) GBE_FAIL(GBE_E_COMM, "bucket x%d is row-sharded but no all-gather hook is set", t.var);
        size_t bytes = el * (size_t)(sh.per * sh.block_rows);
        if (g_ag(gathered_src[ti], R.base + R.A->off_full[ti], bytes, (void *)st, g_ag_u) != 0)
          GBE_FAIL(GBE_E_COMM, "all-gather of the message of x%d failed", t.var);
      }
      if (gathered_src[ti]) last_gather = (int)ti;
      if (dag) {
        CK(cudaEventRecord(D->tev[ti], st));
        st = st0;
      }
    }
    if (host_args || P.ex.spill)  // every argmin / message chunk is in host memory before the value phase
      for (int i = 0; i < 2 && i < ring_n; i++) CK(cudaStreamWaitEvent(st, D->c_ev[i], 0));
    if (dag)  // join every branch before the constants
      for (size_t q = 0; q < last_on.size(); q++)
        if (last_on[q] >= 0) CK(cudaStreamWaitEvent(st, D->tev[last_on[q]], 0));
    // optimum / lower bound = sum of the constants
    void *cp = d_cp;
    if (!graph) {
      cp = dalloc(sizeof(void *) * std::max<size_t>(cptrs.size(), 1), st);
      if (!cptrs.empty())
        CK(cudaMemcpyAsync(cp, cptrs.data(), sizeof(void *) * cptrs.size(), cudaMemcpyHostToDevice, st));
    }
    CK(value_launch(p.is_f64(), nullptr, 0, 0, nullptr, nullptr, R.d_assign, nullptr, -1, W,
                    (const void *const *)cp, (int)cptrs.size(), R.d_opt, st));
    if (P.ex.count) {  // number of solutions: product of the constants' counts (d_opt + 8)
      void *ccp = d_ccp;
      if (!graph) {
        ccp = dalloc(sizeof(void *) * std::max<size_t>(ccptrs.size(), 1), st);
        if (!ccptrs.empty())
          CK(cudaMemcpyAsync(ccp, ccptrs.data(), sizeof(void *) * ccptrs.size(), cudaMemcpyHostToDevice, st));
      }
      CK(count_total_launch(p.is_f64(), (const void *const *)cp, (const double *const *)ccp, (int)cptrs.size(),
                            P.ex.count == 2, R.d_opt, (double *)((char *)R.d_opt + 8), st));
      if (!graph) dfree(ccp, st);
    }
    CK(cudaMemcpyAsync(hopt, R.d_opt, P.ex.count ? 16 : el, cudaMemcpyDeviceToHost, st));
    if (!graph) dfree(cp, st);
  };

  bool replayed = false;
  if (graph && A.runs > 0 && !A.no_graph) {  // the first run warms up (kernel attributes), later runs replay
    if (!A.exec) {
      if (!D->cap_stream) CK(cudaStreamCreateWithFlags(&D->cap_stream, cudaStreamNonBlocking));
      cudaGraph_t g = nullptr;
      try {
        CK(cudaStreamBeginCapture(D->cap_stream, cudaStreamCaptureModeThreadLocal));
        try {
          enqueue(D->cap_stream, true);
        } catch (...) {
          cudaStreamEndCapture(D->cap_stream, &g);
          if (g) cudaGraphDestroy(g);
          g = nullptr;
          throw;
        }
        CK(cudaStreamEndCapture(D->cap_stream, &g));
        CK(cudaGraphInstantiate(&A.exec, g, 0));
        CK(cudaGraphDestroy(g));
      } catch (const Error &) {
        // a row-sharded plan whose collective cannot be captured runs eagerly
        // (the collectives then go through the hook stream by stream)
        if (W == 1) throw;
        cudaGetLastError();
        A.exec = nullptr;
        A.no_graph = true;
      }
    }
    if (A.exec) {
      CK(cudaGraphLaunch(A.exec, s));
      replayed = true;
    }
  }
  if (!replayed) enqueue(s, false);
  R.replayed = replayed;
  R.tuned = tuning;
  if (graph) A.runs++;
  CK(cudaStreamSynchronize(s));
  R.optimum = read_value(p, hopt);
  if (tuning) {  // this solve's candidate times; after both rounds keep each task's fastest
    const int ci = D->tune_phase % D->tune_nc;
    for (size_t ti = 0; ti < nt; ti++)
      if (!D->cands[ti].empty() && ci < (int)D->cands[ti].size()) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, D->tune_ev[2 * ti], D->tune_ev[2 * ti + 1]));
        // the first round pays lazy module loading: keep the second
        if (D->tune_phase >= D->tune_nc) D->t_cand[ti][ci] = ms;
      }
    if (++D->tune_phase == 2 * D->tune_nc) {
      for (auto &a : D->arena) a.runs = std::max(a.runs, 1);  // every kernel has run: capture next
      for (size_t ti = 0; ti < nt; ti++) {
        const auto &cs = D->cands[ti];
        if (cs.empty()) continue;
        size_t best = 0;  // the default unless another candidate is >= 3 % faster
        for (size_t c = 1; c < cs.size(); c++)
          if (D->t_cand[ti][c] < 0.97f * D->t_cand[ti][0] && D->t_cand[ti][c] < D->t_cand[ti][best]) best = c;
        D->use_fast[ti] = cs[best].variant == 1;
        D->use_stream[ti] = cs[best].variant == 2;
        D->use_stage[ti] = cs[best].stage;
        D->use_half[ti] = cs[best].half;
        D->use_ds[ti] = cs[best].ds;
        (cs[best].half ? D->slh[ti] : D->sl[ti]).pf = cs[best].pf;
        D->launch[ti].variant = cs[best].variant;
      }
    }
  }
  if (P.ex.count) std::memcpy(&R.count, hopt + 8, sizeof(double));
  if (P.ex.timing) {
    R.ms.assign(nt, 0.f);
    R.merge_ms.assign(nt, 0.f);
    for (size_t ti = 0; ti < nt; ti++) {
      CK(cudaEventElapsedTime(&R.ms[ti], ev[3 * ti], ev[3 * ti + 2]));
      CK(cudaEventElapsedTime(&R.merge_ms[ti], ev[3 * ti], ev[3 * ti + 1]));
    }
  }
  R.util_done = true;
}

struct VProg {
  VStep *steps;
  VMember *mems;
  VTerm *terms;
};

// launch the value kernel over the program, exchanging sharded lookups
static void run_value_steps(RunImpl &R, const VProg &pg, int nsteps, const std::vector<char> &sharded,
                            int32_t *assign_out) {
  const Plan &P = *R.gp->plan;
  const Problem &p = *P.prob;
  cudaStream_t s = R.stream;
  const int W = P.ex.world_size;
  if (W > 1 && !R.d_gbuf) R.d_gbuf = (int32_t *)dalloc(sizeof(int32_t) * W, s);
  // segments end at row-sharded steps: the owner's lookup is exchanged
  int s0 = 0, gvar = -1;
  for (int i = 0; i < nsteps; i++) {
    if (!(W > 1 && sharded[i])) continue;
    CK(value_launch(p.is_f64(), pg.steps, s0, i + 1, pg.mems, pg.terms, R.d_assign, R.d_gbuf, gvar,
                    W, nullptr, -1, nullptr, s));
    if (!g_ag) GBE_FAIL(GBE_E_COMM, "sharded value phase needs the all-gather hook");
    int var = P.order[i];
    if (g_ag(R.d_assign + var, R.d_gbuf, sizeof(int32_t), (void *)s, g_ag_u) != 0)
      GBE_FAIL(GBE_E_COMM, "all-gather of the value of x%d failed", var);
    gvar = var;
    s0 = i + 1;
  }
  CK(value_launch(p.is_f64(), pg.steps, s0, nsteps, pg.mems, pg.terms, R.d_assign, R.d_gbuf, gvar, W,
                  nullptr, -1, nullptr, s));
  CK(cudaMemcpyAsync(assign_out, R.d_assign, sizeof(int32_t) * p.n, cudaMemcpyDeviceToHost, s));
}

static void run_value_program(RunImpl &R, void *buf, int nsteps, const std::vector<char> &sharded,
                              int32_t *assign_out) {
  DevPlan::Arena *A = R.A;
  VProg pg{(VStep *)buf, (VMember *)((char *)buf + A->b_steps),
           (VTerm *)((char *)buf + A->b_steps + A->b_mems)};
  run_value_steps(R, pg, nsteps, sharded, assign_out);
  CK(cudaStreamSynchronize(R.stream));
}

// VALUE / assignment phase (Alg. 1 lines 6-7)
static void run_value(RunImpl &R, int32_t *assign_out) {
  const Plan &P = *R.gp->plan;
  const Problem &p = *P.prob;
  cudaStream_t s = R.stream;
  // the program depends only on the plan and the arena addresses: a run on
  // the plan's cached arena reuses the device copy built by the first run
  DevPlan::Arena *A = R.arena_own ? nullptr : R.A;
  if (A && A->vprog) {
    run_value_program(R, A->vprog, A->vsteps, A->vsharded, assign_out);
    return;
  }
  std::vector<VStep> steps;
  std::vector<VMember> mems;
  std::vector<VTerm> terms;
  std::vector<char> sharded;
  for (int i = 0; i < p.n; i++) {
    int x = P.order[i];
    VStep st{};
    st.var = x;
    st.d = p.dom[x];
    if (!R.mbe) {
      int ti = P.var_task[x];
      const Task &t = P.tasks[ti];
      if (!R.arg[ti]) GBE_FAIL(GBE_E_INTERNAL, "argmin table of x%d not retained", x);
      st.kind = 0;
      st.term_off = (int64_t)terms.size();
      st.nterm = (int32_t)t.sep.size();
      int64_t rs = 1;
      std::vector<VTerm> tt(t.sep.size());
      for (int q = (int)t.sep.size() - 1; q >= 0; q--) {
        tt[q] = VTerm{t.sep[q], 0, rs};
        rs *= p.dom[t.sep[q]];
      }
      terms.insert(terms.end(), tt.begin(), tt.end());
      st.lo = t.shard.lo;
      st.hi = t.shard.hi;
      st.ptr = R.arg[ti];
      sharded.push_back(t.shard.on ? 1 : 0);
    } else {
      st.kind = 1;
      st.mem_off = (int64_t)mems.size();
      st.nmem = (int32_t)P.bucket[x].size();
      for (auto &m : P.bucket[x]) {
        VMember vm{};
        vm.ptr = R.member_ptr(m);
        vm.term_off = (int64_t)terms.size();
        // member scope ascending by position, x last: strides
        std::vector<int32_t> sc;
        if (m.kind == 0) {
          sc.assign(p.scope(m.index), p.scope(m.index) + p.arity[m.index]);
          std::sort(sc.begin(), sc.end(), [&](int a, int b) { return P.pos[a] < P.pos[b]; });
        } else {
          sc = P.tasks[m.index].sep;
        }
        int64_t st2 = 1;
        std::vector<VTerm> tt;
        for (int q = (int)sc.size() - 1; q >= 0; q--) {
          if (sc[q] != x) tt.push_back(VTerm{sc[q], 0, st2});
          st2 *= p.dom[sc[q]];
        }
        vm.nterm = (int32_t)tt.size();
        terms.insert(terms.end(), tt.begin(), tt.end());
        mems.push_back(vm);
      }
      sharded.push_back(0);
    }
    steps.push_back(st);
  }
  size_t b_steps = sizeof(VStep) * std::max<size_t>(steps.size(), 1);
  size_t b_mems = sizeof(VMember) * std::max<size_t>(mems.size(), 1);
  size_t b_terms = sizeof(VTerm) * std::max<size_t>(terms.size(), 1);
  char *buf = nullptr;
  if (A) {
    CK(cudaMalloc(&buf, b_steps + b_mems + b_terms));
  } else {
    buf = (char *)dalloc(b_steps + b_mems + b_terms, s);
  }
  VStep *d_steps = (VStep *)buf;
  VMember *d_mems = (VMember *)(buf + b_steps);
  VTerm *d_terms = (VTerm *)(buf + b_steps + b_mems);
  if (!steps.empty()) CK(cudaMemcpyAsync(d_steps, steps.data(), sizeof(VStep) * steps.size(), cudaMemcpyHostToDevice, s));
  if (!mems.empty()) CK(cudaMemcpyAsync(d_mems, mems.data(), sizeof(VMember) * mems.size(), cudaMemcpyHostToDevice, s));
  if (!terms.empty()) CK(cudaMemcpyAsync(d_terms, terms.data(), sizeof(VTerm) * terms.size(), cudaMemcpyHostToDevice, s));
  if (A) {
    A->vprog = buf;
    A->vsteps = (int)steps.size();
    A->vsharded = sharded;
    A->b_steps = b_steps;
    A->b_mems = b_mems;
  }
  VProg prog{d_steps, d_mems, d_terms};
  run_value_steps(R, prog, (int)steps.size(), sharded, assign_out);
  if (!A) dfree(buf, s);
  CK(cudaStreamSynchronize(s));
}

static std::string stats_json(const RunImpl &R) {
  const Plan &P = *R.gp->plan;
  const Problem &p = *P.prob;
  std::ostringstream o;
  // kernel launches of one UTIL phase: relayout, one per bucket, one per
  // input merge, constants (+ the count product of counting plans)
  const size_t util_launches = 2 + P.tasks.size() + R.D->merges.size() + (P.ex.count ? 1 : 0);
  o << "{\"total_cells\":" << P.total_cells << ",\"total_bytes\":" << P.total_bytes
    << ",\"merges\":" << R.D->merges.size() << ",\"util_launches\":" << util_launches
    << ",\"graph_replay\":" << (R.replayed ? "true" : "false") << ",\"autotune_solve\":" << (R.tuned ? "true" : "false")
    << ",\"tasks\":[";
  for (size_t ti = 0; ti < P.tasks.size(); ti++) {
    const Task &t = P.tasks[ti];
    int64_t local = t.shard.hi - t.shard.lo;
    int64_t frac_in = t.rows ? (int64_t)((double)t.in_cells * local / t.rows) : 0;
    // algorithmic bytes: inputs read once, output written once, and one
    // argmin byte per row only when the kernel wrote argmins
    int64_t bytes = (int64_t)p.elem() * (frac_in + local) + (R.args_written ? local : 0);
    if (P.ex.count) {  // + the float64 count tables read (messages) and written
      int64_t msg = 0;
      for (auto &m : t.members)
        if (m.kind == 1) msg += P.tasks[m.index].rows;
      bytes += 8 * ((t.rows ? (int64_t)((double)msg * local / t.rows) : 0) + local);
    }
    o << (ti ? "," : "") << "{\"var\":" << t.var << ",\"mb\":" << t.mb << ",\"rows\":" << local
      << ",\"d\":" << t.d << ",\"k\":" << t.desc.ninputs << ",\"cells\":" << local * t.d
      << ",\"bytes\":" << bytes << ",\"variant\":" << R.D->launch[ti].variant
      << ",\"k_eff\":" << R.D->h_desc[ti].ninputs << ",\"merges\":" << R.D->task_merges[ti].size()
      << ",\"staged\":" << (R.D->use_stream[ti] && R.D->use_stage[ti] ? "true" : "false")
      << ",\"half_tiles\":" << (R.D->use_stream[ti] && R.D->use_half[ti] ? "true" : "false");
    if (R.D->use_fast[ti]) {
      const FastHot &fh = (R.D->use_ds[ti] ? R.D->h_fds[ti] : R.D->h_fast[ti]).hot;
      o << ",\"tile_rows\":" << fh.PL << ",\"stages\":" << fh.nstages << ",\"staging_bufs\":" << fh.nout
        << ",\"direct_stores\":" << (R.D->use_ds[ti] ? "true" : "false")
        << ",\"groups\":" << R.D->fl[ti].NG << ",\"classes\":[" << fh.cls_off[1] - fh.cls_off[0] << ","
        << fh.cls_off[2] - fh.cls_off[1] << "," << fh.cls_off[3] - fh.cls_off[2] << "," << fh.cls_off[4] - fh.cls_off[3]
        << "],\"g\":[" << R.D->fl[ti].g1 << "," << R.D->fl[ti].g2 << "],\"slen\":[";
      for (int q = 0; q < fh.k; q++) o << (q ? "," : "") << fh.slen[q];
      o << "],\"in_scope\":[";  // per class-ordered input: the output digits it has
      const gbe_bucket_desc &hd = R.D->h_desc[ti];
      for (int q = 0; q < fh.k; q++) {
        o << (q ? "," : "") << "\"";
        for (int pp = 0; pp < hd.nsep; pp++) o << (hd.stride[fh.in_idx[q]][pp] ? 'X' : '.');
        o << "\"";
      }
      o << "]";
    }
    if (!R.D->use_fast[ti]) {  // post-merge inputs of the other variants
      const gbe_bucket_desc &hd = R.D->h_desc[ti];
      o << ",\"in_scope\":[";
      for (int q = 0; q < hd.ninputs; q++) {
        o << (q ? "," : "") << "\"";
        for (int pp = 0; pp < hd.nsep; pp++) o << (hd.stride[q][pp] ? 'X' : '.');
        o << "\"";
      }
      o << "]";
    }
    o
      << ",\"ms\":" << (ti < R.ms.size() ? R.ms[ti] : -1.0f)
      << ",\"merge_ms\":" << (ti < R.merge_ms.size() ? R.merge_ms[ti] : -1.0f) << "}";
  }
  o << "]}";
  return o.str();
}

static void copy_stats(const RunImpl &R, char *buf, size_t cap) {
  if (!buf || cap == 0) return;
  std::string s = stats_json(R);
  size_t n = std::min(cap - 1, s.size());
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}

// ---------------------------------------------------------------------------
// entry points used by capi.cpp

RunImpl *run_create(gbe_plan *gp, void *stream, bool mbe) {
  auto *R = new RunImpl();
  R->gp = gp;
  try {
    R->D = dev_plan(gp);
    CK(cudaSetDevice(R->D->device));
    R->stream = (cudaStream_t)stream;
    R->mbe = mbe;
    run_util(*R);
  } catch (...) {
    delete R;
    throw;
  }
  return R;
}

void run_destroy(RunImpl *R) { delete R; }

gbe_value run_optimum(const RunImpl *R) { return R->optimum; }

void run_value_phase(RunImpl *R, int32_t *assign_out) {
  if (R->gp->plan->ex.sumprod) GBE_FAIL(GBE_E_INVALID, "a sum-product run has no VALUE phase");
  CK(cudaSetDevice(R->D->device));
  run_value(*R, assign_out);
}

void run_stats(const RunImpl *R, char *buf, size_t cap) { copy_stats(*R, buf, cap); }

void run_table(const RunImpl *R, int32_t t, void *host_out, uint8_t *host_arg) {
  const Plan &P = *R->gp->plan;
  if (t < 0 || t >= (int)P.tasks.size()) GBE_FAIL(GBE_E_INVALID, "table %d out of range", t);
  const Task &T = P.tasks[t];
  int64_t local = T.shard.hi - T.shard.lo;
  CK(cudaSetDevice(R->D->device));
  if (host_out) {
    const void *src = R->out[t] ? R->out[t] : R->full[t];
    if (T.host) {  // out-of-core plan: the message is in pinned host memory
      CK(cudaStreamSynchronize(R->stream));
      std::memcpy(host_out, R->D->h_msg + R->D->msg_off[t], P.prob->elem() * local);
      src = nullptr;
    } else if (!src) GBE_FAIL(GBE_E_INVALID, "table %d not retained (plan needs \"retain\":\"all\")", t);
    if (src) {
      if (R->full[t] && !R->out[t])  // gathered: this rank's rows start at lo
        src = (const char *)src + P.prob->elem() * T.shard.lo;
      CK(cudaMemcpyAsync(host_out, src, P.prob->elem() * local, cudaMemcpyDeviceToHost, R->stream));
    }
  }
  if (host_arg && P.ex.sumprod) {  // sum-product tables have no argmin
    std::memset(host_arg, 0, (size_t)local);
  } else if (host_arg && P.ex.host_args) {  // argmins already in (pinned) host memory
    CK(cudaStreamSynchronize(R->stream));
    std::memcpy(host_arg, R->D->h_harg + R->D->harg_off[t], (size_t)local);
  } else if (host_arg) {
    if (!R->arg[t]) GBE_FAIL(GBE_E_INVALID, "argmin table %d not retained", t);
    CK(cudaMemcpyAsync(host_arg, R->arg[t], local, cudaMemcpyDeviceToHost, R->stream));
  }
  CK(cudaStreamSynchronize(R->stream));
}

void run_count(const RunImpl *R, double *count, void *) {
  if (!R->gp->plan->ex.count) GBE_FAIL(GBE_E_INVALID, "run of a plan without \"count\"");
  *count = R->count;
}

void run_count_table(const RunImpl *R, int32_t t, double *host_out) {
  const Plan &P = *R->gp->plan;
  if (!P.ex.count) GBE_FAIL(GBE_E_INVALID, "run of a plan without \"count\"");
  if (t < 0 || (size_t)t >= P.tasks.size()) GBE_FAIL(GBE_E_INVALID, "table %d out of range", t);
  if (P.ex.retain < 2) GBE_FAIL(GBE_E_INVALID, "count tables need \"retain\":\"all\"");
  const Task &T = P.tasks[t];
  CK(cudaMemcpy(host_out, R->base + R->A->off_cnt[t], 8 * (size_t)T.rows, cudaMemcpyDeviceToHost));
}

void solve(gbe_plan *gp, void *stream, bool mbe, gbe_value *opt, gbe_value *upper,
           int32_t *assign_out, char *stats, size_t cap) {
  RunImpl *R = run_create(gp, stream, mbe);
  try {
    if (opt) *opt = R->optimum;
    // value-only solves (no assignment requested, e.g. "retain":"none" on the
    // exact 20x20 grid whose argmins would need 1.27 TB) skip the value phase
    if (assign_out || upper) {
      if (gp->plan->ex.retain < 1)
        GBE_FAIL(GBE_E_INVALID, "an assignment needs the argmin tables / retained messages (plan has \"retain\":\"none\")");
      std::vector<int32_t> a(std::max(gp->plan->prob->n, 1));
      run_value(*R, a.data());
      if (assign_out) std::memcpy(assign_out, a.data(), sizeof(int32_t) * gp->plan->prob->n);
      if (upper) *upper = problem_evaluate(*gp->plan->prob, a.data());
    }
    copy_stats(*R, stats, cap);
  } catch (...) {
    delete R;
    throw;
  }
  delete R;
}

// the variant the bare primitive runs: the same rule as a plan's buckets
// (tiled when it fits, unless the policy prefers streaming; else streaming;
// the generic kernel only for descriptors neither takes)
int bucket_kernel_variant(const gbe_bucket_desc *h, int64_t row_begin, int64_t row_end) {
  if (row_end <= row_begin) return 0;
  FastDesc *F = new FastDesc();
  BkfLaunch fl;
  const bool fast = bkf_build(*h, row_begin, row_end, 148, *F, fl);
  delete F;
  StreamDesc *Sd = new StreamDesc();
  BksLaunch sl;
  const bool stream = bks_build(*h, row_begin, row_end, 148, *Sd, sl);
  delete Sd;
  if (fast && (!stream || !prefer_stream(*h, fl))) return 1;
  return stream ? 2 : 0;
}

// the bare hot primitive
void bucket_kernel(const gbe_bucket_desc *h, const void *const *dev_inputs, void *dev_out,
                   uint8_t *dev_arg, int64_t row_begin, int64_t row_end, void *stream, int variant) {
  if (variant < -1 || variant > 3) GBE_FAIL(GBE_E_INVALID, "variant must be -1, 0, 1, 2 or 3");
  if (!h) GBE_FAIL(GBE_E_INVALID, "null descriptor");
  if (h->semiring != GBE_MINSUM_I32 && h->semiring != GBE_MINSUM_F64 && h->semiring != GBE_SUMPROD_F64)
    GBE_FAIL(GBE_E_INVALID, "bad semiring");
  if (h->nsep < 0 || h->nsep > GBE_MAX_SEP || h->ninputs < 0 || h->ninputs > GBE_MAX_INPUTS)
    GBE_FAIL(GBE_E_INVALID, "nsep/ninputs out of range");
  if (h->d < 1 || h->d > GBE_MAX_DOMAIN) GBE_FAIL(GBE_E_INVALID, "d=%d outside [1,%d]", h->d, GBE_MAX_DOMAIN);
  int64_t rows = 1;
  for (int q = 0; q < h->nsep; q++) {
    if (h->radix[q] < 1) GBE_FAIL(GBE_E_INVALID, "radix[%d] < 1", q);
    rows *= h->radix[q];
  }
  if (rows != h->rows) GBE_FAIL(GBE_E_INVALID, "rows (%lld) != prod(radix) (%lld)", (long long)h->rows, (long long)rows);
  if (row_begin < 0 || row_end > rows || row_begin > row_end) GBE_FAIL(GBE_E_INVALID, "bad row range");
  if (h->ninputs && !dev_inputs) GBE_FAIL(GBE_E_INVALID, "null inputs");
  if (row_end > row_begin && !dev_out) GBE_FAIL(GBE_E_INVALID, "null output");
  int dev = 0, nsm = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t s = (cudaStream_t)stream;
  InPtrs in{};
  for (int j = 0; j < h->ninputs; j++) in.p[j] = dev_inputs[j];
  const int var = variant >= 0 ? variant : bucket_kernel_variant(h, row_begin, row_end);
  if (var == 3) {  // streaming, staged mode
    StreamDesc *Sd = new StreamDesc();
    BksLaunch sl;
    const bool ok = bks_build(*h, row_begin, row_end, nsm, *Sd, sl, true);
    if (ok) {
      StreamDesc *d_s = (StreamDesc *)dalloc(sizeof(StreamDesc), s);
      cudaError_t e = cudaMemcpyAsync(d_s, Sd, sizeof(StreamDesc), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = bks_launch(d_s, sl, in, dev_out, dev_arg, row_begin, row_end, s);
      dfree(d_s, s);
      delete Sd;
      CK(e);
      return;
    }
    delete Sd;
    GBE_FAIL(GBE_E_INVALID, "the staged streaming kernel does not fit this descriptor");
  }
  if (var == 2) {  // streaming
    StreamDesc *Sd = new StreamDesc();
    BksLaunch sl;
    const bool ok = bks_build(*h, row_begin, row_end, nsm, *Sd, sl);
    if (ok) {
      StreamDesc *d_s = (StreamDesc *)dalloc(sizeof(StreamDesc), s);
      cudaError_t e = cudaMemcpyAsync(d_s, Sd, sizeof(StreamDesc), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = bks_launch(d_s, sl, in, dev_out, dev_arg, row_begin, row_end, s);
      dfree(d_s, s);
      delete Sd;
      CK(e);
      return;
    }
    delete Sd;
    if (variant == 2) GBE_FAIL(GBE_E_INVALID, "the streaming kernel does not fit this descriptor");
  }
  if (var == 1) {  // tiled TMA
    FastDesc *F = new FastDesc();
    BkfLaunch fl;
    const bool ok = bkf_build(*h, row_begin, row_end, nsm, *F, fl);
    if (ok) {
      FastDesc *d_f = (FastDesc *)dalloc(sizeof(FastDesc), s);
      cudaError_t e = cudaMemcpyAsync(d_f, F, sizeof(FastDesc), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = bkf_launch(d_f, fl, in, dev_out, dev_arg, row_begin, s);
      dfree(d_f, s);
      delete F;
      CK(e);
      return;
    }
    delete F;
    if (variant == 1) GBE_FAIL(GBE_E_INVALID, "the tiled kernel does not fit this descriptor");
  }
  gbe_bucket_desc *d_desc = (gbe_bucket_desc *)dalloc(sizeof(gbe_bucket_desc), s);
  cudaError_t e = cudaMemcpyAsync(d_desc, h, sizeof(gbe_bucket_desc), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    BkLaunchInfo li = bk_plan_launch(*h, row_begin, row_end, -1, nsm);
    e = bk_launch(*h, d_desc, in, dev_out, dev_arg, row_begin, row_end, li, s);
  }
  dfree(d_desc, s);
  CK(e);
}

}  // namespace gbe
