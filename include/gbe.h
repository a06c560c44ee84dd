/* gbe.h — C ABI of the B200 bucket-elimination library (libgbe.so).
 *
 * The library computes the (mini-)bucket / UTIL-message tables of Bucket
 * Elimination, Mini-Bucket Elimination and DPOP on an NVIDIA B200 (sm_100a)
 * with hand-written CUDA kernels.  Citations: P:n = line n of PAPER.md
 * (arXiv 1608.05288, Fioretto, Pontelli, Yeoh, Dechter), S:n = line n of
 * SPEC.md.  Readings of ambiguous passages (A1..A17) are listed in DESIGN.md.
 *
 * Conventions (all calls):
 *   - Every call returns a gbe_status; on failure gbe_last_error() returns a
 *     thread-local message (e.g. "bucket x17: 3.49e9 rows > budget").  No
 *     partial results are written on failure unless stated.
 *   - The caller owns every host array passed in or out; outputs are
 *     caller-allocated with the documented sizes.  The library copies what it
 *     keeps.  Opaque handles are freed only by the matching *_destroy.
 *   - `stream` is a cudaStream_t cast to void* (NULL = legacy default stream).
 *   - Variables are 0..n-1.  An ordering lists the variables from the first
 *     (root side, lowest priority) to the last; BE eliminates from
 *     order[n-1] down to order[0] (Alg. 1).
 *   - Tables are flat, lexicographic, first scope variable most significant
 *     (bucket-table).  Original functions are given in their
 *     declared scope order; every table the library produces has its scope
 *     sorted by ascending order position (root side most significant, A2).
 *   - Integer costs: int32 with infinity = GBE_INF_I32 = 2^30 ("R+ u {inf}",
 *     P:118); every aggregation clamps at infinity (A9).  Float64 costs are
 *     IEEE doubles (MPE stored as -log p, A10), +inf = forbidden.
 *   - Infeasible instances are not errors: the optimum is returned with
 *     is_inf = 1.
 */
#ifndef GBE_H
#define GBE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GBE_INF_I32 (1 << 30)
#define GBE_MAX_SEP 40    /* output-scope variables of one bucket            */
#define GBE_MAX_INPUTS 32 /* input tables of one (mini-)bucket               */
#define GBE_MAX_DOMAIN 256 /* argmins are stored as uint8                    */

typedef enum {
  GBE_OK = 0,
  GBE_E_INVALID = 1, /* bad argument, i-bound below a member arity */
  GBE_E_PARSE = 2,   /* file parse error; message carries the line */
  GBE_E_BUDGET = 3,  /* plan exceeds the memory budget; names the bucket */
  GBE_E_CUDA = 4,    /* CUDA runtime / kernel failure, or no device */
  GBE_E_COMM = 5,    /* collective hook failed */
  GBE_E_INTERNAL = 6
} gbe_status;

/* Semiring of the aggregate/eliminate operators.
 * MPE is solved as min-sum over -log p in float64 (A10).  GBE_SUMPROD_F64
 * (buckets and plans only; problems hold GBE_MINSUM_F64 costs): the same
 * aggregation of -log values, eliminated by -log sum_v exp(-s_v) — the
 * sum/product semiring of P:210, giving -log Z (partition function, P(E);
 * SURVEY §8(f) row 3, the paper's future work P:1631).  No argmin. */
typedef enum { GBE_MINSUM_I32 = 0, GBE_MINSUM_F64 = 1, GBE_SUMPROD_F64 = 2 } gbe_semiring;

typedef enum {
  GBE_ORDER_MINFILL = 0,      /* greedy min-fill, ties (fill, degree, id) (A3) */
  GBE_ORDER_PAPER_DEGREE = 1, /* x_i < x_j iff |N(x_i)| < |N(x_j)|, ties by id */
  GBE_ORDER_GIVEN = 2         /* `given` is validated and copied */
} gbe_order_kind;

/* A cost value: is_inf = 1 means infinity; i holds int32-semiring values,
 * f holds float64 ones (the other field is 0). */
typedef struct {
  int32_t is_inf;
  int64_t i;
  double f;
} gbe_value;

typedef struct gbe_problem gbe_problem; /* immutable after creation     */
typedef struct gbe_plan gbe_plan;       /* ordering, (mini-)buckets, layouts,
                                           stride maps, shard plan            */
typedef struct gbe_run gbe_run;         /* device-resident UTIL messages/argmins */

/* ---------------------------------------------------------------------
 * Problems: WCSP <X,D,C>, DCOP = WCSP + identity agent map
 * (P:416-417), belief network CPTs for MPE.
 * ------------------------------------------------------------------- */

/* n variables with domain sizes dom[n] (1 <= dom <= GBE_MAX_DOMAIN); nf
 * functions, function f has arity[f] variables listed consecutively in
 * `scopes` (declared order) and prod(dom over its scope) consecutive costs in
 * `costs` (int32 for GBE_MINSUM_I32, double for GBE_MINSUM_F64).
 * Errors: GBE_E_INVALID (bad ids, duplicate scope variable, negative cost,
 * sum of the largest finite entries >= 2^30 for int32). */
gbe_status gbe_problem_create(int32_t n, const int32_t *dom, int32_t nf,
                              const int32_t *arity, const int32_t *scopes,
                              gbe_semiring sr, const void *costs, gbe_problem **out);

/* WCSP text format: `name n maxdom nf ub`, n domain sizes, then per
 * function `arity vars... default ntuples` and ntuples lines `vals... cost`;
 * costs >= ub are infinity.  GBE_E_PARSE with the line number on error. */
gbe_status gbe_problem_load_wcsp(const char *path, gbe_problem **out);

/* UAI BAYES/MARKOV model; tables are probabilities, stored as
 * -log p (p = 0 -> +inf).  `evid` (NULL ok): `count var val ...`; evidence
 * variables are conditioned by slicing; out-of-domain evidence ->
 * GBE_E_INVALID. */
gbe_status gbe_problem_load_uai(const char *model, const char *evid, gbe_problem **out);

/* Synthetic instances (§8.1) from a JSON
 * object, e.g. {"topology":"scalefree","n":200,"d":3,"p2":0,"seed":5}.
 * topology: "random" (n,d,edges,mode), "scalefree" (n,d), "grid"
 * (rows,cols,d), "bn" (n,dmin,dmax,maxpar,window), "network" (n,dmin,dmax,
 * nf,amin,amax,cmax).  Uses the shared seeded generator module gen/. */
gbe_status gbe_generate(const char *json_cfg, gbe_problem **out);

/* sizes of a problem */
gbe_status gbe_problem_info(const gbe_problem *p, int32_t *n, int32_t *nf,
                            gbe_semiring *sr);

void gbe_problem_destroy(gbe_problem *p);

/* Cost of a complete assignment assign[n] (Eq. 1); MPE: sum of -log p. */
gbe_status gbe_evaluate(const gbe_problem *p, const int32_t *assign, gbe_value *out);

/* ---------------------------------------------------------------------
 * Structure: ordering / induced width, pseudo-tree
 * ------------------------------------------------------------------- */

/* order_out[n] receives the ordering; width_out (NULL ok) its induced width. */
gbe_status gbe_order(const gbe_problem *p, gbe_order_kind kind, const int32_t *given,
                     int32_t *order_out, int32_t *width_out);

/* Pseudo-tree of `order` = its elimination tree (A14): parent_out[v] is the
 * latest-ordered variable of v's UTIL-message scope (-1 for a root), and
 * sep_size_out[v] (NULL ok) = |sep(v)|.  Every primal edge joins an ancestor
 * and a descendant. */
gbe_status gbe_pseudotree(const gbe_problem *p, const int32_t *order,
                          int32_t *parent_out, int32_t *sep_size_out);

/* ---------------------------------------------------------------------
 * Plans and solves
 * ------------------------------------------------------------------- */

/* Plan BE (ibound < 0) or MBE(ibound) (Alg. 2; i-bound = maximum arity of a
 * generated function, |mini-bucket scope union| <= ibound + 1, reading A5;
 * greedy first-fit partition, reading A6).  json_exec (NULL ok):
 *   {"device":0, "budget_bytes":N, "world_size":W, "rank":r,
 *    "shard_min_rows":N, "retain":"none"|"args"|"all"|"host", "timing":true,
 *    "kernel":-1|0|1|2, "autotune":true, "resident_inputs":false, "graph":true, "concurrent":true,
 *    "semiring":"minsum"|"sumprod", "count":"none"|"optimal"|"consistent",
 *    "host_arg_chunk":N, "spill":false, "stage_bytes":N}
 * "retain":"all" keeps every table on the device for gbe_run_table().
 * "spill":true (exact BE / DPOP, one rank, no "count"; needs "budget_bytes"
 * > 0; else GBE_E_INVALID) makes an out-of-core plan (SURVEY §8(f) row 2,
 * the chunked host<->device pipeline of Fig. 8): while the
 * device peak plus the staging budget ("stage_bytes", default budget / 4
 * clamped to [16 MB, 4 GB]; two slots of half of it) exceeds the budget, the
 * largest remaining message moves to pinned host memory; every bucket then
 * runs in row chunks (runs of whole blocks of its leading output digits)
 * whose host-resident input slices are copied into a slot on an H2D stream
 * while a D2H stream copies the previous chunk's rows and argmins out.
 * Argmins go to host memory ("retain":"args"), or nowhere ("none").
 * gbe_run_table() reads host messages from host memory.  A budget no
 * chunking meets is GBE_E_BUDGET naming the largest bucket.  Eager (no
 * CUDA-graph replay).
 * "retain":"host" (exact BE / DPOP, one rank, min-sum; else GBE_E_INVALID)
 * puts the argmin tables in pinned host memory: buckets run in row chunks of
 * "host_arg_chunk" rows (default 2^28) whose argmins stream out through a
 * 2-slot device ring while the next chunk computes (Fig. 8); the
 * value phase reads them in place.  No CUDA-graph replay for such plans.
 * "kernel" forces the generic (0), tiled TMA (1) or streaming (2) bucket
 * kernel where the bucket fits it (-1 = auto: tiled for int32, streaming for
 * float64 and for domains d > 5).  With "autotune" (auto only) the first two
 * solves of a plan time the tiled and the streaming kernel on every bucket
 * both can run and each bucket keeps the faster one from then on (the
 * results are the same up to the f64 summation order, reading A10).
 * "resident_inputs" keeps the uploaded tables on the device between solves.
 * "graph" replays the UTIL phase as a CUDA graph from the second solve on
 * (1 GPU); "concurrent" makes that graph the task DAG (a bucket waits only on
 * its producers and on earlier users of the arena ranges it reuses), so
 * sibling subtrees run concurrently.  "timing" serialises the
 * buckets (per-launch events).
 * "semiring":"sumprod" (float64 problems, ibound < 0 only, else
 * GBE_E_INVALID): every bucket eliminates by -log sum exp(-.), so
 * gbe_solve_be's opt is -log Z; there is no assignment (assign_out must be
 * NULL, gbe_dpop_value fails) and argmin tables read back as zeros.
 * "count" (exact BE on one rank only, not with sumprod, else GBE_E_INVALID):
 * solution counting, the (min, count) semiring:
 * every table also carries a float64 count table (8 bytes per row), the
 * number of completions of the eliminated variables attaining its value;
 * "optimal" counts the optimal assignments, "consistent" the assignments of
 * finite cost (every finite cost read as 0: opt is then 0 or INF).  Counts
 * are exact integers below 2^53.  Read with gbe_solve_count / gbe_run_count.
 * Errors: GBE_E_INVALID (bad order, i-bound < member arity - 1),
 * GBE_E_BUDGET (names the bucket and its rows). */
gbe_status gbe_plan_create(const gbe_problem *p, const int32_t *order, int32_t ibound,
                           const char *json_exec, gbe_plan **out);

/* Plan description as JSON into buf[cap] (tables: var, mini-bucket, sep,
 * rows, inputs, dest, shard range; totals: cells, algorithmic bytes). */
gbe_status gbe_plan_info(const gbe_plan *plan, char *buf, size_t cap);

void gbe_plan_destroy(gbe_plan *plan);

/* Exact BE (Alg. 1 / Alg. 3 with no partition): uploads the original tables
 * (one batched H2D), runs one bucket kernel per bucket with device-resident
 * messages, then the value phase; blocks until done.  opt = optimum,
 * assign_out[n] = the assignment (smallest-index tie-break, A8); assign_out
 * NULL = value-only solve (no value phase; allowed with "retain":"none").  stats_json
 * (NULL ok) receives per-bucket timings when the plan has "timing":true. */
gbe_status gbe_solve_be(gbe_plan *plan, void *stream, gbe_value *opt, int32_t *assign_out,
                        char *stats_json, size_t cap);

/* Solution counting ("as a byproduct ... BE can compute the number
 * of consistent solutions"), plan built with "count": runs the UTIL phase
 * in the (min, count) semiring and returns opt (optimum; 0 / INF for
 * "consistent") and *count = number of optimal / consistent solutions (the
 * product over connected components; 0 if infeasible).  Caller-owned
 * outputs; GBE_E_INVALID for a plan without "count". */
gbe_status gbe_solve_count(gbe_plan *plan, void *stream, gbe_value *opt, double *count);

/* MBE(i) (Alg. 2): lower = sum of constants; upper = evaluate(assignment);
 * the value phase minimises the sum of all mini-bucket functions (A7), so the
 * messages are retained until it runs.  upper = assign_out = NULL gives the
 * lower bound only; with "retain":"none" messages are then freed once
 * consumed (e.g. the 20x20 grid at i = 18, whose messages total ~0.5 TB). */
gbe_status gbe_solve_mbe(gbe_plan *plan, void *stream, gbe_value *lower, gbe_value *upper,
                         int32_t *assign_out, char *stats_json, size_t cap);

/* DPOP UTIL phase on the plan's pseudo-tree: UTIL messages are the
 * bucket functions (Thm 1).  The run keeps the argmin tables for
 * the VALUE phase.  root_util = optimum.  With an MBE plan (ibound >= 0) this
 * is ADPOP: the messages are the mini-bucket functions, root_util
 * is the lower bound, and the VALUE phase minimises over all mini-bucket
 * functions of each variable (A7). */
gbe_status gbe_dpop_util(gbe_plan *plan, void *stream, gbe_run **run_out,
                         gbe_value *root_util);
/* DPOP VALUE phase: assign_out[n]. */
gbe_status gbe_dpop_value(gbe_run *run, int32_t *assign_out);
/* statistics of a run as JSON (per-bucket kernel ms, cells, bytes) */
gbe_status gbe_run_stats(const gbe_run *run, char *buf, size_t cap);
/* copy table t (creation order, as in gbe_plan_info) to host; needs
 * "retain":"all".  host_out: rows * (4 or 8) bytes; host_arg: rows bytes
 * (either may be NULL).  Only rows owned by this rank are written. */
gbe_status gbe_run_table(const gbe_run *run, int32_t t, void *host_out, uint8_t *host_arg);
/* counting runs (plan with "count"): number of optimal / consistent
 * solutions, and the count table of table t (host_out: rows doubles; needs
 * "retain":"all"; GBE_E_INVALID otherwise) */
gbe_status gbe_run_count(const gbe_run *run, double *count);
gbe_status gbe_run_count_table(const gbe_run *run, int32_t t, double *host_out);
void gbe_run_destroy(gbe_run *run);

/* ---------------------------------------------------------------------
 * The hot primitive: one (mini-)bucket, Alg. 1 line 3 / Alg. 2 line 5.
 * out[r - row_begin] = min_v ⊕_j T_j[off_j(r) + v],  arg = first minimiser,
 * where off_j(r) = sum_p digit_p(r) * stride[j][p] - shift[j] and digit_p(r)
 * is the mixed-radix decomposition of r over radix[0..nsep) (radix[0] most
 * significant).  This restates the index map Eq. with strides
 * precomputed per input (the "mul/div/mod" vectors) and fuses Gpu::
 * Aggregate (Proc. 4) with Gpu::Eliminate (Proc. 5):
 * the d^{|sep|+1} aggregated table is never materialised.
 * ------------------------------------------------------------------- */
typedef struct gbe_bucket_desc {
  int32_t semiring;              /* gbe_semiring                                  */
  int32_t nsep;                  /* output scope size m (0 = one output row)      */
  int32_t d;                     /* domain size of the eliminated variable         */
  int32_t ninputs;               /* k, 0 <= k <= GBE_MAX_INPUTS                    */
  int64_t rows;                  /* prod(radix) = R                               */
  int32_t radix[GBE_MAX_SEP];    /* output digit radices, [0] most significant     */
  int64_t stride[GBE_MAX_INPUTS][GBE_MAX_SEP]; /* element stride of output digit p
                                    in input j; 0 if the variable is absent.  The
                                    eliminated variable has stride 1 in every input */
  int64_t shift[GBE_MAX_INPUTS]; /* subtracted from every offset of input j (row-
                                    sharded inputs: first local element)           */
} gbe_bucket_desc;

/* With semiring GBE_SUMPROD_F64: out = -log sum_v exp(-s_v) (m - log sum_v
 * exp(m - s_v), m = min_v s_v; +inf rows stay +inf) and arg = 0.
 * desc: HOST pointer; dev_inputs[k]: device pointers to int32 or double tables;
 * the tiled variant reads inputs in whole 16-byte-aligned granules (TMA bulk
 * copies), i.e. up to 15 bytes before the first and after the last element
 * it needs: every granule that holds an element of an input must lie in
 * readable device memory (true for any table inside a cudaMalloc / pool
 * allocation, whose sizes are rounded to >= 256 bytes);
 * dev_out: device array of (row_end - row_begin) int32/double; dev_arg: device
 * uint8 array of the same length or NULL.  Asynchronous on `stream`.
 * Errors: GBE_E_INVALID (sizes, d > 256, k > GBE_MAX_INPUTS), GBE_E_CUDA. */
gbe_status gbe_bucket_kernel(const void *desc, const void *const *dev_inputs, void *dev_out,
                             uint8_t *dev_arg, int64_t row_begin, int64_t row_end,
                             void *stream);

/* The same with the kernel variant chosen by the caller: -1 auto (as
 * gbe_bucket_kernel), 0 generic, 1 tiled TMA, 2 streaming, 3 streaming in
 * its staged mode (per-warp TMA double buffers; d = 2..5, min-sum, every
 * input's warp-tile slice one dense range; it reads inputs in 16-byte
 * granules like the tiled variant); GBE_E_INVALID if the descriptor does not
 * fit the requested variant. */
gbe_status gbe_bucket_kernel_ex(const void *desc, const void *const *dev_inputs, void *dev_out,
                                uint8_t *dev_arg, int64_t row_begin, int64_t row_end, void *stream,
                                int32_t variant);

/* Which kernel variant gbe_bucket_kernel would run for this descriptor and
 * row range: 0 = generic (per-row decode), 1 = tiled TMA + register-blocked,
 * 2 = streaming (lanes over the eliminated domain).  Returns
 * -1 for an invalid descriptor. */
int32_t gbe_bucket_kernel_variant(const void *desc, int64_t row_begin, int64_t row_end);

/* ---------------------------------------------------------------------
 * Hooks
 * ------------------------------------------------------------------- */
/* Device memory: alloc(bytes, stream, u) / free(ptr, u).  Default:
 * cudaMallocAsync / cudaFreeAsync on the solve stream. NULL restores it. */
gbe_status gbe_set_allocator(void *(*alloc_fn)(size_t, void *stream, void *u),
                             void (*free_fn)(void *, void *u), void *u);

/* All-gather of a row-sharded message among the plan's world_size ranks:
 * every rank contributes `bytes` from `send` and receives world_size * bytes
 * into `recv` (rank-major).  Return 0 on success.  Needed only when a plan has
 * world_size > 1.  NULL removes the hook. */
gbe_status gbe_set_allgather(int (*ag)(const void *send, void *recv, size_t bytes,
                                       void *stream, void *u),
                             void *u);

/* Table inspection (checksums, parity tests, streaming tables to the host):
 * fn is called on the host after each (mini-)bucket of a solve / UTIL phase
 * has been computed on this rank and before its message can be freed, with
 * task = creation index (gbe_plan_info order), dev_out = its `rows` local
 * output rows (first global row row_begin) and dev_arg = their argmins (the
 * executor computes them into a scratch buffer when the plan does not retain
 * argmins; NULL for sum-product plans).  The pointers are valid only during
 * the call; `stream` (cudaStream_t) has completed the bucket.  While a hook
 * is installed solves run the buckets in creation order without a CUDA
 * graph.  A non-zero return aborts the solve with GBE_E_INTERNAL.  NULL
 * removes the hook. */
gbe_status gbe_set_table_hook(int (*fn)(int32_t task, const void *dev_out, const uint8_t *dev_arg,
                                        int64_t row_begin, int64_t rows, void *stream, void *u),
                              void *u);

/* Built-in NCCL transport for the all-gather (NVLink 5 / NVSwitch), loaded
 * with dlopen("libnccl.so.2").  Rank 0 calls gbe_comm_nccl_id(id[128]) and
 * shares the 128 bytes with the other ranks (e.g. over torch.distributed);
 * every rank then calls gbe_comm_nccl_init(id, nranks, rank, device), which
 * installs the all-gather hook.  gbe_comm_finalize() destroys the
 * communicator and removes the hook.  GBE_E_COMM if NCCL is unavailable. */
gbe_status gbe_comm_nccl_id(void *id128);
gbe_status gbe_comm_nccl_init(const void *id128, int32_t nranks, int32_t rank, int32_t device);
gbe_status gbe_comm_finalize(void);

/* Thread-local message of the last failing call ("" if none). */
const char *gbe_last_error(void);

/* Library version string. */
const char *gbe_version(void);

#ifdef __cplusplus
}
#endif
#endif
