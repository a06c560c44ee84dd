// executor.h — device executor entry points (executor.cpp).
#pragma once
#include "common.h"

namespace gbe {

struct RunImpl;

void set_allocator(void *(*a)(size_t, void *, void *), void (*f)(void *, void *), void *u);
void set_allgather(int (*ag)(const void *, void *, size_t, void *, void *), void *u);
// an all-gather that only enqueues stream work (built-in NCCL): the UTIL
// phase of a row-sharded plan can then be captured as a CUDA graph
void set_allgather_capturable(int (*ag)(const void *, void *, size_t, void *, void *), void *u);
using TableHook = int (*)(int32_t, const void *, const uint8_t *, int64_t, int64_t, void *, void *);
void set_table_hook(TableHook fn, void *u);
void dev_plan_free(void *d);
void comm_nccl_id(void *id128);
void comm_nccl_init(const void *id128, int nranks, int rank, int device);
void comm_finalize();

RunImpl *run_create(gbe_plan *gp, void *stream, bool mbe);
void run_destroy(RunImpl *R);
gbe_value run_optimum(const RunImpl *R);
void run_value_phase(RunImpl *R, int32_t *assign_out);
void run_stats(const RunImpl *R, char *buf, size_t cap);
void run_table(const RunImpl *R, int32_t t, void *host_out, uint8_t *host_arg);
void run_count(const RunImpl *R, double *count, void *unused);
void run_count_table(const RunImpl *R, int32_t t, double *host_out);

void solve(gbe_plan *gp, void *stream, bool mbe, gbe_value *opt, gbe_value *upper,
           int32_t *assign_out, char *stats, size_t cap);
int bucket_kernel_variant(const gbe_bucket_desc *h, int64_t row_begin, int64_t row_end);
void bucket_kernel(const gbe_bucket_desc *h, const void *const *dev_inputs, void *dev_out,
                   uint8_t *dev_arg, int64_t row_begin, int64_t row_end, void *stream, int variant = -1);

}  // namespace gbe

struct gbe_run {
  gbe::RunImpl *impl = nullptr;
};
