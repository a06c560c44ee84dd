// common.h — internal types of libgbe (not part of the C ABI).
//
// Citations: P:n = PAPER.md line n (arXiv 1608.05288).  Readings A1..A17:
// DESIGN.md §3.  This file and everything under csrc/ is product code: it
// never includes or links anything from oracle/.
#pragma once

#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gbe.h"

namespace gbe {

constexpr int32_t kInfI32 = GBE_INF_I32;

// ---------------------------------------------------------------------------
// errors: thread-local last error + status propagation

void set_error(const std::string &msg);
const char *last_error();

struct Error {
  gbe_status status;
  std::string msg;
};

#define GBE_FAIL(st, ...)                                   \
  do {                                                      \
    char _gbe_buf[512];                                     \
    std::snprintf(_gbe_buf, sizeof(_gbe_buf), __VA_ARGS__); \
    throw ::gbe::Error{st, _gbe_buf};                       \
  } while (0)

// ---------------------------------------------------------------------------
// problem: <X, D, C>, functions in declared scope order

struct Problem {
  int32_t n = 0, nf = 0;
  gbe_semiring sr = GBE_MINSUM_I32;
  std::vector<int32_t> dom;       // [n]
  std::vector<int32_t> arity;     // [nf]
  std::vector<int64_t> scope_off; // [nf+1]
  std::vector<int32_t> scopes;
  std::vector<int64_t> table_off; // [nf+1]
  std::vector<int32_t> icost;     // int32 semiring
  std::vector<double> fcost;      // f64 semiring
  bool has_inf = false;           // int32: some entry is INF (A9)
  int64_t maxsum = 0;             // int32: sum of the largest finite entries (< 2^30, A9)
  bool is_f64() const { return sr == GBE_MINSUM_F64; }
  size_t elem() const { return is_f64() ? 8 : 4; }
  const int32_t *scope(int f) const { return scopes.data() + scope_off[f]; }
};

// ---------------------------------------------------------------------------
// minimal JSON (flat objects of numbers / strings / bools)

struct Json {
  std::map<std::string, std::string> kv; // raw scalar text (strings unquoted)
  static Json parse(const char *text);   // throws Error{GBE_E_INVALID}
  bool has(const std::string &k) const { return kv.count(k) != 0; }
  int64_t i(const std::string &k, int64_t def) const;
  double f(const std::string &k, double def) const;
  std::string s(const std::string &k, const std::string &def) const;
  bool b(const std::string &k, bool def) const;
};

// ---------------------------------------------------------------------------
// plan: ordering, (mini-)bucket tasks, layouts, stride maps, shard plan

struct Member {
  int32_t kind;  // 0 original function, 1 message (task index)
  int32_t index;
};

// Row sharding of one task's output over the ranks: the rows
// split into `blocks` blocks of `block_rows` rows (a block = one value of the
// `key_digits` most significant output digits); rank r owns blocks
// [r*per, min((r+1)*per, blocks)).
struct Shard {
  bool on = false;
  int32_t key_digits = 0;
  int64_t blocks = 1, block_rows = 0, per = 0;
  int64_t lo = 0, hi = 0;   // this rank's row range
  bool gather = false;      // the consumer needs the whole message
};

struct Task {                  // one (mini-)bucket: Alg. 1 line 3 / Alg. 2 line 5
  int32_t var = -1, mb = 0;    // eliminated variable, mini-bucket index
  int32_t dest = -1;           // bucket variable receiving the message (-1 const)
  int32_t consumer = -1;       // task consuming the message (-1 = constant)
  std::vector<Member> members; // canonical order (originals, then messages)
  std::vector<int32_t> sep;    // output scope, ascending order position
  int64_t rows = 1;
  int32_t d = 1;
  int32_t height = 0;          // longest chain of producers below (DPOP levels)
  gbe_bucket_desc desc{};      // radices + per-input stride maps (shift = 0)
  int64_t in_cells = 0;        // sum of input table sizes
  Shard shard;
  // out-of-core plans ("spill"): the message lives in
  // pinned host memory; the task runs in row chunks of `chunk_rows` rows
  // (whole blocks of its leading output digits), each chunk's host-resident
  // input slices staged into a device slot (Fig. 8)
  bool host = false;
  int32_t chunk_digits = 0;    // chunk = chunk_blocks consecutive blocks of these leading digits
  int64_t chunk_blocks = 1, chunk_rows = 0;
};

struct ExecOptions {
  int device = 0;
  int64_t budget_bytes = -1;   // <0: device memory at plan time
  int world_size = 1, rank = 0;
  int64_t shard_min_rows = 1ll << 24;
  int retain = 1;              // 0 none, 1 args, 2 all
  bool timing = false;
  int kernel = -1;             // -1 auto, else force a kernel variant (0 generic, 1 tiled, 2 streaming)
  bool autotune = true;        // auto: time tiled vs streaming per bucket on the first solves
  bool resident_inputs = false; // keep the uploaded originals on the device between solves
  bool graph = true;            // replay the UTIL phase as a CUDA graph (1 GPU, cached arena)
  bool concurrent = true;       // the graph is the task DAG: sibling subtrees overlap
  bool sumprod = false;         // sum-product semiring (-log Z), f64 exact BE only
  int count = 0;                // (min, count) semiring: 0 off, 1 optimal, 2 consistent solutions
  bool host_args = false;       // argmin tables in pinned host memory, streamed out chunk by chunk
  int64_t host_arg_chunk = int64_t(1) << 28;  // rows per streamed chunk (device ring buffer bytes)
  bool spill = false;           // out-of-core: messages beyond budget_bytes live in host memory
  int64_t stage_bytes = 0;      // spill: device staging (two slots); 0 = budget / 4, clamped
};

struct Plan {
  std::shared_ptr<const Problem> prob;
  std::vector<int32_t> order, pos;
  int32_t ibound = -1;
  int32_t width = 0;
  std::vector<Task> tasks;                     // creation order
  std::vector<std::vector<Member>> bucket;     // canonical B_x per variable
  std::vector<int32_t> var_task;               // BE: the task of each variable
  std::vector<Member> constants;               // originals of arity 0, then root messages
  std::vector<int32_t> perm_strides;           // relayout: per original, per sorted pos
  std::vector<int64_t> sorted_off;             // relayout
  int64_t total_cells = 0;                     // sum over tasks of rows*d
  int64_t total_bytes = 0;                     // algorithmic bytes
  int64_t peak_bytes = 0;                      // estimated device peak
  int64_t host_bytes = 0;                      // spill: pinned host bytes of the host messages
  int64_t slot_bytes = 0;                      // spill: bytes of each of the two device staging slots
  ExecOptions ex;
};

// planner.cpp
std::vector<std::vector<char>> primal_adjacency(const Problem &p);
void order_minfill(const Problem &p, std::vector<int32_t> &order);
void order_degree(const Problem &p, std::vector<int32_t> &order);
int32_t induced_width(const Problem &p, const std::vector<int32_t> &order);
std::unique_ptr<Plan> make_plan(std::shared_ptr<const Problem> p, const int32_t *order,
                                int32_t ibound, const ExecOptions &ex);
std::string plan_json(const Plan &plan);
// out-of-core plans: device staging bytes of task ti's chunk over blocks
// [b0, b1) of its c leading output digits, and input j's element range there
struct SpillChunk {
  int64_t lo = 0, n = 0;
};
int64_t spill_chunk_bytes(const Plan &P, size_t ti, int c, int64_t b0, int64_t b1);
SpillChunk spill_chunk_input(const Plan &P, size_t ti, int c, int64_t b0, int64_t b1, int j);

// problem.cpp
std::shared_ptr<Problem> problem_create(int32_t n, const int32_t *dom, int32_t nf,
                                        const int32_t *arity, const int32_t *scopes,
                                        gbe_semiring sr, const void *costs);
std::shared_ptr<Problem> problem_load_wcsp(const char *path);
std::shared_ptr<Problem> problem_load_uai(const char *model, const char *evid);
std::shared_ptr<Problem> problem_generate(const char *json);
gbe_value problem_evaluate(const Problem &p, const int32_t *assign);

}  // namespace gbe

// opaque handles of the C ABI
struct gbe_problem {
  std::shared_ptr<gbe::Problem> p;
};
struct gbe_plan {
  std::unique_ptr<gbe::Plan> plan;
  void *dev = nullptr;  // executor state (executor.cpp)
};
