/* oracle.h — plain, slow, obviously-correct CPU oracle for the bucket
 * (UTIL-message) computation of BE / MBE / DPOP.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1608_05288_b200/) never includes, links or calls it, and
 * it shares no code with the product (not even headers); the only common
 * module is gen/ (seeded input generators, no method arithmetic).
 *
 * Every function cites the PAPER.md passage it restates (P:n = line n of
 * /root/reference/PAPER.md).  Readings of ambiguous passages are the A1..A17
 * readings listed in DESIGN.md §3.
 *
 * Conventions:
 *   - An ordering `order` lists the variables from first (root side, lowest
 *     priority) to last; BE eliminates from order[n-1] down to
 *     order[0] (Alg. 1).
 *   - Integer costs: INF = 2^30, every addition clamps min(a+b, INF) (A9).
 *   - Float64 costs: IEEE double, members summed in canonical order (A10).
 *   - Tables: lexicographic rows, first scope variable most significant
 *     (P:553-554); bucket-function scopes sorted by ascending order
 *     position, so the root-side variable is most significant (A2).
 *   - Argmin ties go to the smallest value index (A8).
 *
 * parity pinned: see tests/test_oracle_pins.py (brute force, Example 1-4
 * structure, the §6.3 index example, closed forms, invariants).
 */
#ifndef GBE_ORACLE_H
#define GBE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_INF_I32 (1 << 30)

typedef struct or_problem {
  int32_t n, nf, is_f64;
  const int32_t *dom;       /* [n]     */
  const int32_t *arity;     /* [nf]    */
  const int64_t *scope_off; /* [nf+1]  */
  const int32_t *scopes;    /* declared scope order */
  const int64_t *table_off; /* [nf+1]  */
  const int32_t *icost;     /* int32 costs (INF = 2^30) or NULL */
  const double *fcost;      /* f64 costs or NULL */
} or_problem;

/* ---- graph structure ------------------------------------ */
/* adjacency of the primal graph, n*n bytes */
void or_primal_graph(const or_problem *p, unsigned char *adj);
/* induced width of `order` (Definition) */
int32_t or_induced_width(const or_problem *p, const int32_t *order);
/* greedy min-fill elimination ordering, ties (fill, degree, id) (A3) */
void or_minfill_order(const or_problem *p, int32_t *order);
/* paper heuristic x_i < x_j iff |N(x_i)| < |N(x_j)|, ties by id (A3) */
void or_degree_order(const or_problem *p, int32_t *order);
/* elimination-tree pseudo-tree: parent[v] = latest-ordered variable of the
 * UTIL message scope of v, -1 for roots (A14) */
void or_elim_tree(const or_problem *p, const int32_t *order, int32_t *parent);

/* ---- one (mini-)bucket, Alg. 1 line 3 / Alg. 2 line 5 ---------------- */
/* Computes rows [row_begin, row_end) of pi_{-x}( sum of members ) (P:218,
 * P:279; aggregation P:204-205, elimination P:207).
 *   x          eliminated variable
 *   nmem       number of members; member k has arity mar[k], scope
 *              mscope[moff[k] .. moff[k]+mar[k]) (its own table order) and
 *              table itab[k] / ftab[k]
 *   sep        output scope (nsep variables, most significant first)
 *   out_i/out_f, arg   outputs indexed by (row - row_begin)
 * Each row is decoded into an explicit tuple and re-ranked per member. */
void or_bucket_rows(const int32_t *dom, int32_t n, int32_t is_f64, int32_t x,
                    int32_t nmem, const int32_t *mar, const int64_t *moff,
                    const int32_t *mscope, const int32_t *const *itab,
                    const double *const *ftab, int32_t nsep, const int32_t *sep,
                    int64_t row_begin, int64_t row_end, int32_t *out_i,
                    double *out_f, uint8_t *arg, int32_t nthreads);

/* Sum-product variant of the bucket (the
 * sum/product semiring of P:210): out = -log sum_v exp(-sum_k f_k), written
 * as m - log sum_v exp(m - s_v) with m = min_v s_v; f64 only, no argmin. */
/* aggregation only, for selected rows: sums[q*d + v] (tests: near-ties, A10) */
void or_bucket_row_sums(const int32_t *dom, int32_t n, int32_t is_f64, int32_t x,
                        int32_t nmem, const int32_t *mar, const int64_t *moff,
                        const int32_t *mscope, const int32_t *const *itab,
                        const double *const *ftab, int32_t nsep, const int32_t *sep,
                        int64_t nrows, const int64_t *rows, int64_t *sums_i, double *sums_f);
void or_bucket_rows_sp(const int32_t *dom, int32_t n, int32_t x, int32_t nmem,
                       const int32_t *mar, const int64_t *moff, const int32_t *mscope,
                       const double *const *ftab, int32_t nsep, const int32_t *sep,
                       int64_t row_begin, int64_t row_end, double *out_f, int32_t nthreads);

/* Counting variant of the bucket: the (min,
 * count) semiring.  ctab[k] = member k's count table (NULL: an original,
 * every entry 1).  out = min_v s_v (arg = first minimiser), out_c = sum of
 * prod_k count_k over the v attaining it (0 if the minimum is infinite).
 * consistent = 1 reads every finite member entry as cost 0, so out_c counts
 * the consistent completions. */
void or_bucket_rows_cnt(const int32_t *dom, int32_t n, int32_t is_f64, int32_t x,
                        int32_t nmem, const int32_t *mar, const int64_t *moff,
                        const int32_t *mscope, const int32_t *const *itab,
                        const double *const *ftab, const double *const *ctab,
                        int32_t consistent, int32_t nsep, const int32_t *sep,
                        int64_t row_begin, int64_t row_end, int32_t *out_i,
                        double *out_f, double *out_c, uint8_t *arg, int32_t nthreads);

/* ---- whole solve: BE (ibound < 0) or MBE(ibound) (Alg. 1, Alg. 2) ----- */
typedef struct or_run or_run;
/* keep_tables: 1 keeps every (mini-)bucket table and argmin for inspection
 * and runs the forward (value assignment) pass; 0 frees each message once
 * consumed (digests are still recorded) and skips the forward pass. */
or_run *or_solve(const or_problem *p, const int32_t *order, int32_t ibound,
                 int32_t keep_tables, int32_t nthreads);
/* Exact BE in the sum-product semiring (f64 problems; NULL otherwise): the
 * value is -log Z, Z = sum over all assignments of prod exp(-f) (the
 * partition function; a belief network with evidence as 0/INF unary
 * functions gives -log P(E)).  No forward pass (no assignment); argmin
 * tables are all zero. */
or_run *or_solve_sumprod(const or_problem *p, const int32_t *order, int32_t keep_tables,
                         int32_t nthreads);
/* Exact BE in the (min, count) semiring:
 * consistent = 0 counts the optimal assignments (value = the optimum),
 * consistent = 1 the assignments of finite cost (value 0, or INF when there
 * is none).  Counts are doubles (exact integers below 2^53). */
or_run *or_solve_count(const or_problem *p, const int32_t *order, int32_t consistent,
                       int32_t keep_tables, int32_t nthreads);
/* number of optimal / consistent solutions of a counting run */
double or_run_count(const or_run *r);
/* count table of table t (counting runs, kept tables); 0 if unavailable */
int32_t or_run_table_count(const or_run *r, int32_t t, double *out_c);
/* 0 ok; 1 invalid i-bound (a member cannot fit, A5/A6); 2 out of memory */
int32_t or_run_status(const or_run *r);
int32_t or_run_ntables(const or_run *r);
/* meta of table t (creation order: x from last to first, mini-buckets in
 * creation order): eliminated var, mini-bucket index, |sep|, rows,
 * destination bucket variable (-1 = constant), number of members */
void or_run_table_meta(const or_run *r, int32_t t, int32_t *var, int32_t *mb,
                       int32_t *nsep, int64_t *rows, int32_t *dest, int32_t *nmem);
void or_run_table_sep(const or_run *r, int32_t t, int32_t *sep);
/* members of table t: kind (0 original function, 1 message) and index */
void or_run_table_members(const or_run *r, int32_t t, int32_t *kind, int32_t *index);
/* 0 if the table was freed (keep_tables = 0) */
int32_t or_run_table_out(const or_run *r, int32_t t, int32_t *out_i, double *out_f,
                         uint8_t *arg);
/* FNV-1a 64 over the output bytes, then over the argmin bytes */
uint64_t or_run_table_digest(const or_run *r, int32_t t);
/* optimum = sum of constants; BE: exact; MBE: lower bound */
int64_t or_run_value_i(const or_run *r);
double or_run_value_f(const or_run *r);
/* forward pass result (keep_tables = 1 only); returns 0 if not computed */
int32_t or_run_assignment(const or_run *r, int32_t *assign);
/* evaluate(assignment): MBE upper bound */
int64_t or_run_upper_i(const or_run *r);
double or_run_upper_f(const or_run *r);
void or_run_free(or_run *r);

/* ---- cost of a complete assignment (Eq. 1) ---------- */
int64_t or_evaluate_i(const or_problem *p, const int32_t *assign);
double or_evaluate_f(const or_problem *p, const int32_t *assign);

/* FNV-1a 64 of a byte range, seeded with h (use 0xcbf29ce484222325) */
uint64_t or_fnv1a(uint64_t h, const void *data, int64_t nbytes);
/* position-keyed sum checksum (parallel; see oracle.c) and the digest kind
 * or_solve records: 0 FNV-1a (default), 1 mixsum(out,1) + mixsum(arg,2) */
uint64_t or_mixsum(const void *data, int32_t elem, int64_t n, uint64_t salt, int32_t nthreads);
void or_set_digest_kind(int32_t kind);

#ifdef __cplusplus
}
#endif
#endif
