// capi.cpp — the extern "C" boundary declared in include/gbe.h.  Each entry
// converts C++ exceptions into a gbe_status + thread-local message.
#include <cstring>
#include <new>

#include "common.h"
#include "executor.h"

using namespace gbe;

namespace {
template <typename F>
gbe_status guard(F &&f) {
  try {
    f();
    set_error("");
    return GBE_OK;
  } catch (const Error &e) {
    set_error(e.msg);
    return e.status;
  } catch (const std::bad_alloc &) {
    set_error("host out of memory");
    return GBE_E_BUDGET;
  } catch (const std::exception &e) {
    set_error(e.what());
    return GBE_E_INTERNAL;
  } catch (...) {
    set_error("unknown error");
    return GBE_E_INTERNAL;
  }
}

ExecOptions parse_exec(const char *json) {
  ExecOptions ex;
  Json j = Json::parse(json);
  ex.device = (int)j.i("device", 0);
  ex.budget_bytes = j.i("budget_bytes", -1);
  ex.world_size = (int)j.i("world_size", 1);
  ex.rank = (int)j.i("rank", 0);
  ex.shard_min_rows = j.i("shard_min_rows", ex.shard_min_rows);
  std::string r = j.s("retain", "args");
  if (r == "none") ex.retain = 0;
  else if (r == "args") ex.retain = 1;
  else if (r == "all") ex.retain = 2;
  else if (r == "host") ex.retain = 1, ex.host_args = true;
  else GBE_FAIL(GBE_E_INVALID, "retain must be none|args|all|host");
  ex.host_arg_chunk = j.i("host_arg_chunk", ex.host_arg_chunk);
  if (ex.host_arg_chunk < 1) GBE_FAIL(GBE_E_INVALID, "host_arg_chunk must be >= 1");
  ex.spill = j.b("spill", false);
  ex.stage_bytes = j.i("stage_bytes", 0);
  if (ex.stage_bytes < 0) GBE_FAIL(GBE_E_INVALID, "stage_bytes must be >= 0");
  ex.timing = j.b("timing", false);
  ex.kernel = (int)j.i("kernel", -1);
  if (ex.kernel < -1 || ex.kernel > 2) GBE_FAIL(GBE_E_INVALID, "kernel must be -1 (auto), 0, 1 or 2");
  ex.autotune = j.b("autotune", true);
  ex.resident_inputs = j.b("resident_inputs", false);
  ex.graph = j.b("graph", true);
  ex.concurrent = j.b("concurrent", true);
  std::string sr = j.s("semiring", "minsum");
  if (sr == "sumprod") ex.sumprod = true;
  else if (sr != "minsum") GBE_FAIL(GBE_E_INVALID, "semiring must be minsum|sumprod");
  std::string c = j.s("count", "none");
  if (c == "optimal") ex.count = 1;
  else if (c == "consistent") ex.count = 2;
  else if (c != "none") GBE_FAIL(GBE_E_INVALID, "count must be none|optimal|consistent");
  return ex;
}

void copy_str(const std::string &s, char *buf, size_t cap) {
  if (!buf || cap == 0) return;
  if (s.size() + 1 > cap) GBE_FAIL(GBE_E_INVALID, "buffer too small (%zu bytes needed)", s.size() + 1);
  std::memcpy(buf, s.c_str(), s.size() + 1);
}
}  // namespace

extern "C" {

gbe_status gbe_problem_create(int32_t n, const int32_t *dom, int32_t nf, const int32_t *arity,
                              const int32_t *scopes, gbe_semiring sr, const void *costs,
                              gbe_problem **out) {
  return guard([&] {
    if (!out) GBE_FAIL(GBE_E_INVALID, "null out");
    auto *h = new gbe_problem{problem_create(n, dom, nf, arity, scopes, sr, costs)};
    *out = h;
  });
}

gbe_status gbe_problem_load_wcsp(const char *path, gbe_problem **out) {
  return guard([&] {
    if (!out) GBE_FAIL(GBE_E_INVALID, "null out");
    *out = new gbe_problem{problem_load_wcsp(path)};
  });
}

gbe_status gbe_problem_load_uai(const char *model, const char *evid, gbe_problem **out) {
  return guard([&] {
    if (!out) GBE_FAIL(GBE_E_INVALID, "null out");
    *out = new gbe_problem{problem_load_uai(model, evid)};
  });
}

gbe_status gbe_generate(const char *json_cfg, gbe_problem **out) {
  return guard([&] {
    if (!out) GBE_FAIL(GBE_E_INVALID, "null out");
    *out = new gbe_problem{problem_generate(json_cfg)};
  });
}

gbe_status gbe_problem_info(const gbe_problem *p, int32_t *n, int32_t *nf, gbe_semiring *sr) {
  return guard([&] {
    if (!p) GBE_FAIL(GBE_E_INVALID, "null problem");
    if (n) *n = p->p->n;
    if (nf) *nf = p->p->nf;
    if (sr) *sr = p->p->sr;
  });
}

void gbe_problem_destroy(gbe_problem *p) { delete p; }

gbe_status gbe_evaluate(const gbe_problem *p, const int32_t *assign, gbe_value *out) {
  return guard([&] {
    if (!p || !assign || !out) GBE_FAIL(GBE_E_INVALID, "null argument");
    *out = problem_evaluate(*p->p, assign);
  });
}

gbe_status gbe_order(const gbe_problem *p, gbe_order_kind kind, const int32_t *given,
                     int32_t *order_out, int32_t *width_out) {
  return guard([&] {
    if (!p || !order_out) GBE_FAIL(GBE_E_INVALID, "null argument");
    std::vector<int32_t> o;
    if (kind == GBE_ORDER_MINFILL) order_minfill(*p->p, o);
    else if (kind == GBE_ORDER_PAPER_DEGREE) order_degree(*p->p, o);
    else if (kind == GBE_ORDER_GIVEN) {
      if (!given) GBE_FAIL(GBE_E_INVALID, "GBE_ORDER_GIVEN needs `given`");
      o.assign(given, given + p->p->n);
      std::vector<char> seen(p->p->n, 0);
      for (int v : o) {
        if (v < 0 || v >= p->p->n || seen[v]) GBE_FAIL(GBE_E_INVALID, "given order is not a permutation");
        seen[v] = 1;
      }
    } else
      GBE_FAIL(GBE_E_INVALID, "unknown ordering kind %d", (int)kind);
    std::memcpy(order_out, o.data(), sizeof(int32_t) * o.size());
    if (width_out) *width_out = induced_width(*p->p, o);
  });
}

gbe_status gbe_pseudotree(const gbe_problem *p, const int32_t *order, int32_t *parent_out,
                          int32_t *sep_size_out) {
  return guard([&] {
    if (!p || !order || !parent_out) GBE_FAIL(GBE_E_INVALID, "null argument");
    ExecOptions ex;
    auto plan = make_plan(p->p, order, -1, ex);
    for (int v = 0; v < p->p->n; v++) {
      const Task &t = plan->tasks[plan->var_task[v]];
      parent_out[v] = t.dest;
      if (sep_size_out) sep_size_out[v] = (int32_t)t.sep.size();
    }
  });
}

gbe_status gbe_plan_create(const gbe_problem *p, const int32_t *order, int32_t ibound,
                           const char *json_exec, gbe_plan **out) {
  return guard([&] {
    if (!p || !order || !out) GBE_FAIL(GBE_E_INVALID, "null argument");
    ExecOptions ex = parse_exec(json_exec);
    auto *h = new gbe_plan();
    try {
      h->plan = make_plan(p->p, order, ibound < 0 ? -1 : ibound, ex);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

gbe_status gbe_plan_info(const gbe_plan *plan, char *buf, size_t cap) {
  return guard([&] {
    if (!plan) GBE_FAIL(GBE_E_INVALID, "null plan");
    copy_str(plan_json(*plan->plan), buf, cap);
  });
}

void gbe_plan_destroy(gbe_plan *plan) {
  if (!plan) return;
  if (plan->dev) dev_plan_free(plan->dev);
  delete plan;
}

gbe_status gbe_solve_be(gbe_plan *plan, void *stream, gbe_value *opt, int32_t *assign_out,
                        char *stats_json, size_t cap) {
  return guard([&] {
    if (!plan) GBE_FAIL(GBE_E_INVALID, "null plan");
    if (plan->plan->ibound >= 0) GBE_FAIL(GBE_E_INVALID, "plan was built for MBE (i-bound %d)", plan->plan->ibound);
    if (plan->plan->ex.sumprod && assign_out)
      GBE_FAIL(GBE_E_INVALID, "a sum-product plan has no assignment (pass assign_out = NULL)");
    solve(plan, stream, false, opt, nullptr, assign_out, stats_json, cap);
  });
}

gbe_status gbe_solve_count(gbe_plan *plan, void *stream, gbe_value *opt, double *count) {
  return guard([&] {
    if (!plan || !count) GBE_FAIL(GBE_E_INVALID, "null argument");
    if (!plan->plan->ex.count) GBE_FAIL(GBE_E_INVALID, "plan was not built with \"count\"");
    RunImpl *R = run_create(plan, stream, false);
    try {
      if (opt) *opt = run_optimum(R);
      run_count(R, count, nullptr);
    } catch (...) {
      run_destroy(R);
      throw;
    }
    run_destroy(R);
  });
}

gbe_status gbe_run_count(const gbe_run *run, double *count) {
  return guard([&] {
    if (!run || !count) GBE_FAIL(GBE_E_INVALID, "null argument");
    run_count(run->impl, count, nullptr);
  });
}

gbe_status gbe_run_count_table(const gbe_run *run, int32_t t, double *host_out) {
  return guard([&] {
    if (!run || !host_out) GBE_FAIL(GBE_E_INVALID, "null argument");
    run_count_table(run->impl, t, host_out);
  });
}

gbe_status gbe_solve_mbe(gbe_plan *plan, void *stream, gbe_value *lower, gbe_value *upper,
                         int32_t *assign_out, char *stats_json, size_t cap) {
  return guard([&] {
    if (!plan) GBE_FAIL(GBE_E_INVALID, "null plan");
    solve(plan, stream, true, lower, upper, assign_out, stats_json, cap);
  });
}

gbe_status gbe_dpop_util(gbe_plan *plan, void *stream, gbe_run **run_out, gbe_value *root_util) {
  return guard([&] {
    if (!plan || !run_out) GBE_FAIL(GBE_E_INVALID, "null argument");
    auto *r = new gbe_run();
    try {
      // an MBE plan gives ADPOP: UTIL messages = mini-bucket functions
      r->impl = run_create(plan, stream, plan->plan->ibound >= 0);
    } catch (...) {
      delete r;
      throw;
    }
    if (root_util) *root_util = run_optimum(r->impl);
    *run_out = r;
  });
}

gbe_status gbe_dpop_value(gbe_run *run, int32_t *assign_out) {
  return guard([&] {
    if (!run || !assign_out) GBE_FAIL(GBE_E_INVALID, "null argument");
    run_value_phase(run->impl, assign_out);
  });
}

gbe_status gbe_run_stats(const gbe_run *run, char *buf, size_t cap) {
  return guard([&] {
    if (!run) GBE_FAIL(GBE_E_INVALID, "null run");
    run_stats(run->impl, buf, cap);
  });
}

gbe_status gbe_run_table(const gbe_run *run, int32_t t, void *host_out, uint8_t *host_arg) {
  return guard([&] {
    if (!run) GBE_FAIL(GBE_E_INVALID, "null run");
    run_table(run->impl, t, host_out, host_arg);
  });
}

void gbe_run_destroy(gbe_run *run) {
  if (!run) return;
  run_destroy(run->impl);
  delete run;
}

gbe_status gbe_bucket_kernel(const void *desc, const void *const *dev_inputs, void *dev_out,
                             uint8_t *dev_arg, int64_t row_begin, int64_t row_end, void *stream) {
  return guard([&] {
    bucket_kernel((const gbe_bucket_desc *)desc, dev_inputs, dev_out, dev_arg, row_begin, row_end,
                  stream);
  });
}

gbe_status gbe_bucket_kernel_ex(const void *desc, const void *const *dev_inputs, void *dev_out,
                                uint8_t *dev_arg, int64_t row_begin, int64_t row_end, void *stream,
                                int32_t variant) {
  return guard([&] {
    bucket_kernel((const gbe_bucket_desc *)desc, dev_inputs, dev_out, dev_arg, row_begin, row_end,
                  stream, variant);
  });
}

int32_t gbe_bucket_kernel_variant(const void *desc, int64_t row_begin, int64_t row_end) {
  if (!desc) return -1;
  const gbe_bucket_desc *h = (const gbe_bucket_desc *)desc;
  if (h->nsep < 0 || h->nsep > GBE_MAX_SEP || h->ninputs < 0 || h->ninputs > GBE_MAX_INPUTS) return -1;
  return bucket_kernel_variant(h, row_begin, row_end);
}

gbe_status gbe_set_allocator(void *(*alloc_fn)(size_t, void *, void *),
                             void (*free_fn)(void *, void *), void *u) {
  return guard([&] {
    if ((alloc_fn == nullptr) != (free_fn == nullptr))
      GBE_FAIL(GBE_E_INVALID, "set both allocator functions or neither");
    set_allocator(alloc_fn, free_fn, u);
  });
}

gbe_status gbe_set_allgather(int (*ag)(const void *, void *, size_t, void *, void *), void *u) {
  return guard([&] { set_allgather(ag, u); });
}

gbe_status gbe_set_table_hook(int (*fn)(int32_t, const void *, const uint8_t *, int64_t, int64_t, void *, void *),
                              void *u) {
  return guard([&] { set_table_hook(fn, u); });
}

gbe_status gbe_comm_nccl_id(void *id128) {
  return guard([&] {
    if (!id128) GBE_FAIL(GBE_E_INVALID, "null id");
    comm_nccl_id(id128);
  });
}

gbe_status gbe_comm_nccl_init(const void *id128, int32_t nranks, int32_t rank, int32_t device) {
  return guard([&] {
    if (!id128) GBE_FAIL(GBE_E_INVALID, "null id");
    comm_nccl_init(id128, nranks, rank, device);
  });
}

gbe_status gbe_comm_finalize(void) {
  return guard([&] { comm_finalize(); });
}

const char *gbe_last_error(void) { return last_error(); }

const char *gbe_version(void) { return "gbe-b200 0.1 (sm_100a)"; }

}  // extern "C"
