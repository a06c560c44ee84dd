// planner.cpp — host planner: primal graph, orderings, induced width,
// (mini-)bucket construction, canonical layouts, stride maps, row-shard plan.
//
// Alg. 3 lines 1-4 and §6.2 re-designed: the whole
// symbolic elimination is planned once, so the device loop only launches
// kernels.  Readings: A1 (bucket of the latest-ordered variable), A2 (scopes
// ascending by order position, eliminated variable last = stride 1), A3
// (min-fill ties), A5/A6 (i-bound = generated arity, greedy first-fit).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <sstream>

#include "bk_fast.h"
#include "common.h"

namespace gbe {

// ---------------------------------------------------------------------------
// graph structure

std::vector<std::vector<char>> primal_adjacency(const Problem &p) {
  std::vector<std::vector<char>> adj(p.n, std::vector<char>(p.n, 0));
  for (int f = 0; f < p.nf; f++) {
    const int32_t *sc = p.scope(f);
    for (int a = 0; a < p.arity[f]; a++)
      for (int b = a + 1; b < p.arity[f]; b++) adj[sc[a]][sc[b]] = adj[sc[b]][sc[a]] = 1;
  }
  return adj;
}

namespace {
// bitset adjacency for the O(n^3)-ish greedy heuristics
struct Bits {
  int n, w;
  std::vector<uint64_t> b;
  Bits(int n_) : n(n_), w((n_ + 63) / 64), b((size_t)n_ * ((n_ + 63) / 64), 0) {}
  uint64_t *row(int v) { return b.data() + (size_t)v * w; }
  bool get(int u, int v) const { return (b[(size_t)u * w + v / 64] >> (v % 64)) & 1; }
  void set(int u, int v) { b[(size_t)u * w + v / 64] |= 1ull << (v % 64); }
};
}  // namespace

// greedy min-fill: key (fill-in edges, current degree, id), first eliminated
// variable = last in the ordering (A3)
void order_minfill(const Problem &p, std::vector<int32_t> &order) {
  int n = p.n;
  Bits g(n);
  auto adj = primal_adjacency(p);
  for (int u = 0; u < n; u++)
    for (int v = 0; v < n; v++)
      if (adj[u][v]) g.set(u, v);
  std::vector<char> alive(n, 1);
  order.assign(n, -1);
  std::vector<int> nb;
  for (int step = 0; step < n; step++) {
    int best = -1;
    long long bfill = 0, bdeg = 0;
    for (int v = 0; v < n; v++) {
      if (!alive[v]) continue;
      nb.clear();
      for (int u = 0; u < n; u++)
        if (alive[u] && g.get(v, u)) nb.push_back(u);
      long long fill = 0;
      for (size_t a = 0; a < nb.size(); a++)
        for (size_t c = a + 1; c < nb.size(); c++)
          if (!g.get(nb[a], nb[c])) fill++;
      long long deg = (long long)nb.size();
      if (best < 0 || fill < bfill || (fill == bfill && deg < bdeg)) {
        best = v;
        bfill = fill;
        bdeg = deg;
      }
    }
    nb.clear();
    for (int u = 0; u < n; u++)
      if (alive[u] && g.get(best, u)) nb.push_back(u);
    for (int a : nb)
      for (int c : nb)
        if (a != c) g.set(a, c);
    alive[best] = 0;
    order[n - 1 - step] = best;
  }
}

// x_i before x_j iff |N(x_i)| < |N(x_j)|, ties by id (stable sort)
void order_degree(const Problem &p, std::vector<int32_t> &order) {
  auto adj = primal_adjacency(p);
  std::vector<int> deg(p.n, 0);
  for (int v = 0; v < p.n; v++)
    for (int u = 0; u < p.n; u++) deg[v] += adj[v][u];
  order.resize(p.n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return deg[a] < deg[b]; });
}

// Definition
int32_t induced_width(const Problem &p, const std::vector<int32_t> &order) {
  int n = p.n;
  Bits g(n);
  auto adj = primal_adjacency(p);
  for (int u = 0; u < n; u++)
    for (int v = 0; v < n; v++)
      if (adj[u][v]) g.set(u, v);
  std::vector<int> pos(n);
  for (int i = 0; i < n; i++) pos[order[i]] = i;
  int32_t w = 0;
  std::vector<int> prev;
  for (int i = n - 1; i >= 0; i--) {
    int v = order[i];
    prev.clear();
    for (int u = 0; u < n; u++)
      if (g.get(v, u) && pos[u] < i) prev.push_back(u);
    w = std::max<int32_t>(w, (int32_t)prev.size());
    for (int a : prev)
      for (int c : prev)
        if (a != c) g.set(a, c);
  }
  return w;
}

// ---------------------------------------------------------------------------
// plan

namespace {

int64_t mul_sat(int64_t a, int64_t b) {
  if (a != 0 && b > (int64_t(1) << 62) / a) return int64_t(1) << 62;
  return a * b;
}

}  // namespace

// Out-of-core plan (the chunked host<->device pipeline of
// Fig. 8, generalised to messages): the largest messages move to
// pinned host memory until the device peak plus two staging slots fits
// budget_bytes.  Every task then runs in row chunks = runs of whole blocks of
// its leading output digits: inside one block every input's slice is ONE
// contiguous range (an input's scope is a subsequence of sep + x in the same
// order, so the block's fixed digits are its most significant ones), and a
// chunk's slice of input j is [base_j(first block), base_j(last block) +
// span_j).  A chunk's staging = its output rows (host message) + argmins +
// the slices of its host-resident inputs, within one slot.
namespace {
// element range of input j over the blocks [b0, b1) of the c leading output
// digits: the run splits into aligned pieces (a prefix of digits fixed, the
// rest free); a piece's offsets span [base, base + sum of its free digits'
// strides * (radix - 1)], plus the in-block extent of the trailing digits
SpillChunk spill_span(const gbe_bucket_desc &h, int j, int c, int64_t b0, int64_t b1) {
  int64_t span = h.d;
  for (int p = c; p < h.nsep; p++) span += h.stride[j][p] * (h.radix[p] - 1);
  auto base = [&](int64_t b) {
    int64_t o = 0;
    for (int p = c - 1; p >= 0; p--) {
      o += h.stride[j][p] * (b % h.radix[p]);
      b /= h.radix[p];
    }
    return o;
  };
  int64_t mn = INT64_MAX, mx = INT64_MIN;
  int64_t lo = b0;
  while (lo < b1) {
    int k = 0;  // free trailing prefix digits of the piece starting at lo
    int64_t size = 1, ext = 0;
    while (k < c) {
      const int p = c - 1 - k;
      const int64_t nsize = size * h.radix[p];
      if (lo % nsize != 0 || lo + nsize > b1) break;
      ext += h.stride[j][p] * (h.radix[p] - 1);
      size = nsize;
      k++;
    }
    const int64_t o = base(lo);
    mn = std::min(mn, o);
    mx = std::max(mx, o + ext);
    lo += size;
  }
  if (mn > mx) return {0, 0};
  return {mn, mx - mn + span};
}
}  // namespace

int64_t spill_chunk_bytes(const Plan &P, size_t ti, int c, int64_t b0, int64_t b1) {
  const Task &t = P.tasks[ti];
  const int64_t el = (int64_t)P.prob->elem();
  int64_t blocks = 1;
  for (int q = 0; q < c; q++) blocks *= t.desc.radix[q];
  const int64_t rows = (b1 - b0) * (t.rows / std::max<int64_t>(blocks, 1));
  int64_t b = ((t.host ? el * rows : 0) + 255) / 256 * 256 + (rows + 255) / 256 * 256;
  for (int j = 0; j < t.desc.ninputs; j++) {
    const Member &m = t.members[j];
    if (m.kind != 1 || !P.tasks[m.index].host) continue;
    b += (el * spill_span(t.desc, j, c, b0, b1).n + 64 + 255) / 256 * 256;
  }
  return b;
}

SpillChunk spill_chunk_input(const Plan &P, size_t ti, int c, int64_t b0, int64_t b1, int j) {
  return spill_span(P.tasks[ti].desc, j, c, b0, b1);
}

static void plan_spill(Plan &P) {
  const Problem &p = *P.prob;
  const int64_t el = (int64_t)p.elem();
  const size_t nt = P.tasks.size();
  const int64_t B = P.ex.budget_bytes;
  const int64_t S = P.ex.stage_bytes > 0 ? P.ex.stage_bytes
                                          : std::min<int64_t>(std::max<int64_t>(B / 4, int64_t(1) << 24),
                                                              int64_t(4) << 30);
  P.slot_bytes = S / 2 / 256 * 256;
  auto dev_peak = [&]() {  // executor allocation sequence with host messages off the device
    int64_t live = 2 * el * p.table_off[p.nf], peak = live;
    for (size_t ti = 0; ti < nt; ti++) {
      const Task &t = P.tasks[ti];
      live += t.host ? 0 : el * t.rows;
      peak = std::max(peak, live);
      if (P.ex.retain < 2)
        for (auto &m : t.members)
          if (m.kind == 1 && !P.tasks[m.index].host) live -= el * P.tasks[m.index].rows;
    }
    return peak;
  };
  std::vector<size_t> by_size(nt);
  for (size_t i = 0; i < nt; i++) by_size[i] = i;
  std::stable_sort(by_size.begin(), by_size.end(),
                   [&](size_t a, size_t b) { return P.tasks[a].rows > P.tasks[b].rows; });
  size_t next = 0;
  while (dev_peak() + S > B && next < nt) P.tasks[by_size[next++]].host = true;
  P.host_bytes = 0;
  for (auto &t : P.tasks)
    if (t.host) P.host_bytes += el * t.rows;
  P.peak_bytes = dev_peak() + S;
  // chunks: the fewest leading digits whose blocks each fit a slot, then the
  // largest power-of-two run of consecutive blocks for which every chunk fits
  constexpr int64_t kMaxChunks = int64_t(1) << 20;
  for (size_t ti = 0; ti < nt; ti++) {
    Task &t = P.tasks[ti];
    auto fits = [&](int c, int64_t blocks, int64_t per) {
      if ((blocks + per - 1) / per > kMaxChunks) return false;
      for (int64_t b0 = 0; b0 < blocks; b0 += per)
        if (spill_chunk_bytes(P, ti, c, b0, std::min(blocks, b0 + per)) > P.slot_bytes) return false;
      return true;
    };
    int c = 0;
    int64_t blocks = 1;
    while (c < t.desc.nsep && blocks <= kMaxChunks && !fits(c, blocks, 1)) blocks *= t.desc.radix[c++];
    if (!fits(c, blocks, 1)) {
      P.peak_bytes = INT64_MAX / 2;  // even the smallest chunks exceed a slot: over budget
      return;
    }
    int64_t per = 1;
    while (per < blocks && fits(c, blocks, std::min(blocks, 2 * per))) per = std::min(blocks, 2 * per);
    t.chunk_digits = c;
    t.chunk_blocks = per;
    t.chunk_rows = per * (t.rows / blocks);
  }
}

std::unique_ptr<Plan> make_plan(std::shared_ptr<const Problem> pp, const int32_t *order_in,
                                int32_t ibound, const ExecOptions &ex) {
  const Problem &p = *pp;
  auto plan = std::make_unique<Plan>();
  plan->prob = pp;
  plan->ibound = ibound;
  plan->ex = ex;
  if (ex.sumprod) {
    if (!p.is_f64()) GBE_FAIL(GBE_E_INVALID, "semiring sumprod needs a float64 (-log) problem");
    if (ibound >= 0) GBE_FAIL(GBE_E_INVALID, "semiring sumprod: exact BE only (ibound < 0)");
    if (plan->ex.retain == 1) plan->ex.retain = 0;  // no value phase: argmins are never read
  }
  if (ex.host_args) {
    if (ibound >= 0) GBE_FAIL(GBE_E_INVALID, "retain host: exact BE / DPOP only (ibound < 0)");
    if (ex.world_size != 1) GBE_FAIL(GBE_E_INVALID, "retain host: single-rank plans only");
    if (ex.sumprod || ex.count) GBE_FAIL(GBE_E_INVALID, "retain host: min-sum plans only");
  }
  if (ex.spill) {
    if (ibound >= 0) GBE_FAIL(GBE_E_INVALID, "spill: exact BE / DPOP only (ibound < 0)");
    if (ex.world_size != 1) GBE_FAIL(GBE_E_INVALID, "spill: single-rank plans only");
    if (ex.count) GBE_FAIL(GBE_E_INVALID, "spill: not with count");
    if (ex.budget_bytes <= 0) GBE_FAIL(GBE_E_INVALID, "spill needs budget_bytes > 0");
    // argmins of an out-of-core plan always stream to host memory
    plan->ex.host_args = ex.retain >= 1 && !ex.sumprod;
  }
  if (ex.count) {
    if (ex.sumprod) GBE_FAIL(GBE_E_INVALID, "count and semiring sumprod are exclusive");
    if (ibound >= 0) GBE_FAIL(GBE_E_INVALID, "count: exact BE only (ibound < 0)");
    if (ex.world_size != 1) GBE_FAIL(GBE_E_INVALID, "count: single-rank plans only");
  }
  int n = p.n;
  if (ex.world_size < 1 || ex.rank < 0 || ex.rank >= ex.world_size)
    GBE_FAIL(GBE_E_INVALID, "bad world_size/rank (%d/%d)", ex.world_size, ex.rank);
  plan->order.assign(order_in, order_in + n);
  plan->pos.assign(n, -1);
  for (int i = 0; i < n; i++) {
    int v = plan->order[i];
    if (v < 0 || v >= n || plan->pos[v] >= 0) GBE_FAIL(GBE_E_INVALID, "order is not a permutation (entry %d)", i);
    plan->pos[v] = i;
  }
  const auto &pos = plan->pos;
  plan->width = induced_width(p, plan->order);

  // relayout of the originals: sorted scope (ascending position), eliminated
  // (latest) variable last; perm_strides[f][q] = stride in the DECLARED table
  // of the q-th sorted scope variable
  plan->sorted_off.assign(p.nf + 1, 0);
  for (int f = 0; f < p.nf; f++) plan->sorted_off[f + 1] = p.table_off[f + 1];
  std::vector<std::vector<int32_t>> sorted_scope(p.nf);
  plan->perm_strides.clear();
  for (int f = 0; f < p.nf; f++) {
    const int32_t *sc = p.scope(f);
    std::vector<int32_t> s(sc, sc + p.arity[f]);
    std::vector<int64_t> decl_stride(p.arity[f]);
    int64_t st = 1;
    for (int a = p.arity[f] - 1; a >= 0; a--) {
      decl_stride[a] = st;
      st *= p.dom[sc[a]];
    }
    std::vector<int> idx(p.arity[f]);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return pos[sc[a]] < pos[sc[b]]; });
    for (int a = 0; a < p.arity[f]; a++) {
      s[a] = sc[idx[a]];
      plan->perm_strides.push_back((int32_t)decl_stride[idx[a]]);
    }
    sorted_scope[f] = s;
  }

  // bucket membership (A1): latest-ordered scope variable
  plan->bucket.assign(n, {});
  for (int f = 0; f < p.nf; f++) {
    if (p.arity[f] == 0) {
      plan->constants.push_back({0, f});
      continue;
    }
    plan->bucket[sorted_scope[f].back()].push_back({0, f});
  }

  std::vector<std::vector<Member>> pending = plan->bucket;  // grows with messages
  auto scope_of = [&](const Member &m) -> const std::vector<int32_t> & {
    return m.kind == 0 ? sorted_scope[m.index] : plan->tasks[m.index].sep;
  };
  auto cells_of = [&](const Member &m) -> int64_t {
    if (m.kind == 0) return p.table_off[m.index + 1] - p.table_off[m.index];
    return plan->tasks[m.index].rows;
  };

  plan->var_task.assign(n, -1);
  std::vector<char> inU(n, 0);
  for (int i = n - 1; i >= 0; i--) {
    int x = plan->order[i];
    const std::vector<Member> &B = pending[x];
    plan->bucket[x] = B;  // canonical B_x (originals, then messages by creation)
    int nm = (int)B.size();
    std::vector<int> mb_of(nm, 0);
    int nmb = 1;
    if (ibound >= 0 && nm > 0) {
      // A6: members by descending arity (stable), first fit with |U| <= i+1
      std::vector<int> ordm(nm);
      std::iota(ordm.begin(), ordm.end(), 0);
      std::stable_sort(ordm.begin(), ordm.end(), [&](int a, int b) {
        return scope_of(B[a]).size() > scope_of(B[b]).size();
      });
      std::vector<std::vector<char>> sets;
      std::vector<int> sizes;
      for (int a : ordm) {
        const auto &sc = scope_of(B[a]);
        if ((int)sc.size() > ibound + 1)
          GBE_FAIL(GBE_E_INVALID, "i-bound %d below a member of arity %zu in the bucket of x%d",
                   ibound, sc.size(), x);
        int placed = -1;
        for (int b = 0; b < (int)sets.size() && placed < 0; b++) {
          int extra = 0;
          for (int v : sc) extra += !sets[b][v];
          if (sizes[b] + extra <= ibound + 1) placed = b;
        }
        if (placed < 0) {
          placed = (int)sets.size();
          sets.emplace_back(n, 0);
          sizes.push_back(0);
        }
        for (int v : sc)
          if (!sets[placed][v]) {
            sets[placed][v] = 1;
            sizes[placed]++;
          }
        mb_of[a] = placed;
      }
      nmb = (int)sets.size();
    }
    for (int b = 0; b < nmb; b++) {
      Task t;
      t.var = x;
      t.mb = b;
      t.d = p.dom[x];
      for (int k = 0; k < nm; k++)
        if (mb_of[k] == b) t.members.push_back(B[k]);
      if ((int)t.members.size() > GBE_MAX_INPUTS)
        GBE_FAIL(GBE_E_INVALID, "bucket of x%d has %zu inputs (> %d)", x, t.members.size(), GBE_MAX_INPUTS);
      std::fill(inU.begin(), inU.end(), 0);
      for (auto &m : t.members)
        for (int v : scope_of(m)) inU[v] = 1;
      for (int v = 0; v < n; v++)
        if (inU[v] && v != x) t.sep.push_back(v);
      std::sort(t.sep.begin(), t.sep.end(), [&](int a, int c) { return pos[a] < pos[c]; });
      if ((int)t.sep.size() > GBE_MAX_SEP)
        GBE_FAIL(GBE_E_BUDGET, "bucket x%d: separator of %zu variables (> %d)", x, t.sep.size(), GBE_MAX_SEP);
      t.rows = 1;
      for (int v : t.sep) t.rows = mul_sat(t.rows, p.dom[v]);
      if (t.rows >= (int64_t(1) << 62) / 256)
        GBE_FAIL(GBE_E_BUDGET, "bucket x%d: %.3g rows exceed addressable memory", x, (double)t.rows);
      t.dest = t.sep.empty() ? -1 : t.sep.back();
      // descriptor: radices + stride maps (Eq. P:673-697 as per-input strides)
      gbe_bucket_desc &D = t.desc;
      D.semiring = ex.sumprod ? GBE_SUMPROD_F64 : p.sr;
      D.nsep = (int32_t)t.sep.size();
      D.d = t.d;
      D.ninputs = (int32_t)t.members.size();
      D.rows = t.rows;
      for (int q = 0; q < D.nsep; q++) D.radix[q] = p.dom[t.sep[q]];
      t.in_cells = 0;
      for (int j = 0; j < D.ninputs; j++) {
        const auto &sc = scope_of(t.members[j]);
        // member tables are ascending by position with x last
        int64_t st = 1;
        std::vector<int64_t> stv(n, 0);
        for (int a = (int)sc.size() - 1; a >= 0; a--) {
          stv[sc[a]] = st;
          st *= p.dom[sc[a]];
        }
        if (sc.empty() || sc.back() != x) GBE_FAIL(GBE_E_INTERNAL, "member of x%d does not end with x", x);
        for (int q = 0; q < D.nsep; q++) D.stride[j][q] = stv[t.sep[q]];
        D.shift[j] = 0;
        t.in_cells += cells_of(t.members[j]);
        if (t.members[j].kind == 1) plan->tasks[t.members[j].index].consumer = (int)plan->tasks.size();
      }
      int h = 0;
      for (auto &m : t.members)
        if (m.kind == 1) h = std::max(h, plan->tasks[m.index].height + 1);
      t.height = h;
      int tid = (int)plan->tasks.size();
      if (plan->var_task[x] < 0) plan->var_task[x] = tid;
      plan->tasks.push_back(t);
      if (t.dest >= 0)
        pending[t.dest].push_back({1, tid});
      else
        plan->constants.push_back({1, tid});
    }
  }

  // totals: algorithmic bytes = inputs once + output + the
  // argmin byte when the solve writes argmins (BE / DPOP with retained
  // argmins, MBE with retained messages, host argmins; never sum-product)
  const int64_t el = (int64_t)p.elem();
  const bool args = !ex.sumprod && ((ibound < 0 && ex.retain >= 1) || ex.retain >= 2 || ex.host_args);
  plan->total_cells = 0;
  plan->total_bytes = 0;
  for (auto &t : plan->tasks) {
    plan->total_cells += t.rows * t.d;
    plan->total_bytes += el * t.in_cells + el * t.rows + (args ? t.rows : 0);
  }

  // row-shard plan: only tasks with >= shard_min_rows rows.
  // Key = the leading output digits; the default key is the shortest prefix
  // with >= 8*W blocks (>= ~90 % balance).  Then, walking from the root side,
  // a producer adopts its consumer's key whenever the consumer's key variables
  // are also the leading variables of the producer's separator (same blocks),
  // so messages along a chain of big buckets never need an all-gather.
  const int W = ex.world_size;
  const int nt = (int)plan->tasks.size();
  std::vector<int> kd(nt, 0);
  auto blocks_of = [&](const Task &t, int k) {
    int64_t b = 1;
    for (int q = 0; q < k; q++) b *= p.dom[t.sep[q]];
    return b;
  };
  for (int ti = 0; ti < nt; ti++) {
    Task &t = plan->tasks[ti];
    if (W <= 1 || t.rows < ex.shard_min_rows || t.sep.empty()) continue;
    int k = 0;
    while (k < (int)t.sep.size() && blocks_of(t, k) < 8LL * W) k++;  // >= ~90 % balance
    if (blocks_of(t, k) < W) continue;
    kd[ti] = k;
  }
  for (int ti = nt - 1; ti >= 0; ti--) {
    const Task &t = plan->tasks[ti];
    if (!kd[ti]) continue;
    for (auto &m : t.members) {
      if (m.kind != 1 || !kd[m.index]) continue;
      const Task &pr = plan->tasks[m.index];
      if (kd[ti] > (int)pr.sep.size()) continue;
      bool same = true;
      for (int q = 0; same && q < kd[ti]; q++) same = pr.sep[q] == t.sep[q];
      if (same) kd[m.index] = kd[ti];
    }
  }
  for (int ti = 0; ti < nt; ti++) {
    Task &t = plan->tasks[ti];
    Shard &s = t.shard;
    s = Shard{};
    s.lo = 0;
    s.hi = t.rows;
    if (!kd[ti]) continue;
    int64_t blocks = blocks_of(t, kd[ti]);
    s.on = true;
    s.key_digits = kd[ti];
    s.blocks = blocks;
    s.block_rows = t.rows / blocks;
    s.per = (blocks + W - 1) / W;
    int64_t b0 = std::min<int64_t>((int64_t)ex.rank * s.per, blocks);
    int64_t b1 = std::min<int64_t>(b0 + s.per, blocks);
    s.lo = b0 * s.block_rows;
    s.hi = b1 * s.block_rows;
  }
  // a sharded message can stay sharded only if its consumer is sharded on
  // the same key variables (then the consumer's rows need exactly the local
  // block range); otherwise it is all-gathered after it is produced
  for (size_t ti = 0; ti < plan->tasks.size(); ti++) {
    Task &t = plan->tasks[ti];
    if (!t.shard.on) continue;
    bool keep = false;
    if (t.consumer >= 0) {
      const Task &c = plan->tasks[t.consumer];
      if (c.shard.on && c.shard.key_digits <= (int)t.sep.size()) {
        keep = c.shard.key_digits == t.shard.key_digits;
        for (int q = 0; keep && q < c.shard.key_digits; q++) keep = c.sep[q] == t.sep[q];
      }
    }
    t.shard.gather = !keep || ibound >= 0;  // MBE value phase reads whole messages
  }

  // device memory estimate (executor allocation sequence)
  int64_t live = 0, peak = 0;
  live += 2 * el * p.table_off[p.nf];
  std::vector<int64_t> msg_bytes(plan->tasks.size(), 0);
  for (size_t ti = 0; ti < plan->tasks.size(); ti++) {
    const Task &t = plan->tasks[ti];
    int64_t local = t.shard.on ? (t.shard.hi - t.shard.lo) : t.rows;
    int64_t full = t.shard.on && t.shard.gather ? t.shard.per * t.shard.block_rows * W : 0;
    msg_bytes[ti] = el * (local + full);
    const bool want_arg = ((ibound < 0 && plan->ex.retain >= 1) || plan->ex.retain >= 2) && !plan->ex.host_args;
    live += msg_bytes[ti] + (want_arg ? local : 0);  // message + argmin
    peak = std::max(peak, live);
    if (plan->ex.retain < 2 && (ibound < 0 || plan->ex.retain == 0))
      for (auto &m : t.members)
        if (m.kind == 1) live -= msg_bytes[m.index];
  }
  if (plan->ex.host_args) {  // + the two device chunk buffers the argmins stream through
    int64_t big = 0;
    for (auto &t : plan->tasks) big = std::max(big, t.rows);
    peak += 2 * std::min(big, plan->ex.host_arg_chunk);
  }
  plan->peak_bytes = peak;
  if (ex.spill) {
    plan_spill(*plan);
    peak = plan->peak_bytes;
  }
  if (ex.budget_bytes > 0 && peak > ex.budget_bytes) {
    // name the largest bucket
    const Task *big = &plan->tasks[0];
    for (auto &t : plan->tasks)
      if (t.rows > big->rows) big = &t;
    GBE_FAIL(GBE_E_BUDGET, "bucket x%d: %.3g rows; plan needs %.3g bytes > budget %.3g", big->var,
             (double)big->rows, (double)peak, (double)ex.budget_bytes);
  }
  return plan;
}

std::string plan_json(const Plan &plan) {
  std::ostringstream o;
  o << "{\"n\":" << plan.prob->n << ",\"ibound\":" << plan.ibound << ",\"width\":" << plan.width
    << ",\"total_cells\":" << plan.total_cells << ",\"total_bytes\":" << plan.total_bytes
    << ",\"peak_bytes\":" << plan.peak_bytes << ",\"world_size\":" << plan.ex.world_size
    << ",\"rank\":" << plan.ex.rank << ",\"spill\":" << (plan.ex.spill ? "true" : "false")
    << ",\"host_bytes\":" << plan.host_bytes << ",\"slot_bytes\":" << plan.slot_bytes << ",\"order\":[";
  for (size_t i = 0; i < plan.order.size(); i++) o << (i ? "," : "") << plan.order[i];
  o << "],\"constants\":[";
  for (size_t i = 0; i < plan.constants.size(); i++)
    o << (i ? "," : "") << "[" << plan.constants[i].kind << "," << plan.constants[i].index << "]";
  o << "],\"tables\":[";
  for (size_t ti = 0; ti < plan.tasks.size(); ti++) {
    const Task &t = plan.tasks[ti];
    o << (ti ? "," : "") << "{\"var\":" << t.var << ",\"mb\":" << t.mb << ",\"rows\":" << t.rows
      << ",\"d\":" << t.d << ",\"dest\":" << t.dest << ",\"consumer\":" << t.consumer
      << ",\"height\":" << t.height << ",\"in_cells\":" << t.in_cells << ",\"sep\":[";
    for (size_t q = 0; q < t.sep.size(); q++) o << (q ? "," : "") << t.sep[q];
    o << "],\"members\":[";
    for (size_t k = 0; k < t.members.size(); k++)
      o << (k ? "," : "") << "[" << t.members[k].kind << "," << t.members[k].index << "]";
    o << "],\"shard\":{\"on\":" << (t.shard.on ? "true" : "false") << ",\"key_digits\":"
      << t.shard.key_digits << ",\"blocks\":" << t.shard.blocks << ",\"per\":" << t.shard.per
      << ",\"lo\":" << t.shard.lo << ",\"hi\":" << t.shard.hi
      << ",\"gather\":" << (t.shard.gather ? "true" : "false") << "}";
    if (plan.ex.spill)
      o << ",\"host\":" << (t.host ? "true" : "false") << ",\"chunk_rows\":" << t.chunk_rows
        << ",\"chunk_digits\":" << t.chunk_digits;
    {
      FastDesc *F = new FastDesc();
      BkfLaunch L;
      bool ok = plan.ex.kernel != 0 && bkf_build(t.desc, t.shard.lo, t.shard.hi, 148, *F, L);
      o << ",\"kernel\":{\"variant\":" << (ok ? 1 : 0);
      if (ok) {
        const FastHot &f = F->hot;
        o << ",\"PL\":" << f.PL << ",\"R\":" << f.R << ",\"Pmid\":" << f.Pmid << ",\"nH\":" << f.nH
          << ",\"classes\":[" << f.cls_off[1] - f.cls_off[0] << "," << f.cls_off[2] - f.cls_off[1] << ","
          << f.cls_off[3] - f.cls_off[2] << "," << f.cls_off[4] - f.cls_off[3] << "],\"rs\":[" << f.rs1
          << "," << f.rs2 << "],\"stage_bytes\":" << f.stage_bytes << ",\"smem\":" << L.smem
          << ",\"grid\":" << L.grid << ",\"slen\":[";
        for (int q = 0; q < f.k; q++) o << (q ? "," : "") << f.slen[q];
        o << "]";
      }
      o << "}}";
      delete F;
    }
  }
  o << "]}";
  return o.str();
}

}  // namespace gbe
