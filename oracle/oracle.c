/* oracle.c — plain CPU oracle for BE / MBE / DPOP bucket tables.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Deliberately naive: every output
 * row is decoded into an explicit tuple and every member function is
 * re-ranked from that tuple.  No blocking, no incremental index arithmetic,
 * no fusion beyond what Alg. 1 line 3 states.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* small helpers                                                       */

static int64_t add_i(int64_t a, int64_t b) { /* A9: clamp after every add */
  int64_t s = a + b;
  return s < OR_INF_I32 ? s : OR_INF_I32;
}

uint64_t or_fnv1a(uint64_t h, const void *data, int64_t nbytes) {
  const unsigned char *b = (const unsigned char *)data;
  for (int64_t i = 0; i < nbytes; i++) {
    h ^= b[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* Position-keyed checksum of a table (not method arithmetic): element i with
 * bits x (zero-extended: u8 argmin, uint32 view of an int32, f64 bits) maps
 * to z = mix(i * 0x9E3779B97F4A7C15 + x + salt * 0xD1B54A32D192ED03) with
 * mix(z) = ((z ^ z>>31) * 0xBF58476D1CE4E5B9) ^ (... >> 29); the digest is
 * the sum of z mod 2^64.  Unlike FNV-1a it is a sum, so it parallelises
 * (tables of 1e10 cells) and a GPU-side test can form it with plain torch
 * ops.  elem = 1, 4 or 8 bytes. */
uint64_t or_mixsum(const void *data, int32_t elem, int64_t n, uint64_t salt, int32_t nthreads) {
  uint64_t h = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for reduction(+ : h) schedule(static) num_threads(nthreads)
#endif
  for (int64_t i = 0; i < n; i++) {
    uint64_t x;
    if (elem == 1)
      x = ((const uint8_t *)data)[i];
    else if (elem == 4)
      x = ((const uint32_t *)data)[i];
    else
      x = ((const uint64_t *)data)[i];
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ULL + x + salt * 0xD1B54A32D192ED03ULL;
    z = (z ^ (z >> 31)) * 0xBF58476D1CE4E5B9ULL;
    z = z ^ (z >> 29);
    h += z;
  }
  return h;
}

/* which digest or_solve records per table: 0 FNV-1a over (out bytes, arg
 * bytes) (default); 1 or_mixsum(out, salt 1) + or_mixsum(arg, salt 2) */
static int g_digest_kind = 0;
void or_set_digest_kind(int32_t kind) { g_digest_kind = kind; }

static int32_t *position_of(const int32_t *order, int32_t n) {
  int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  for (int i = 0; i < n; i++) pos[order[i]] = i;
  return pos;
}

/* ------------------------------------------------------------------ */
/* primal graph, induced width, orderings      */

/* {x,y} is an edge iff some function has both in its scope */
void or_primal_graph(const or_problem *p, unsigned char *adj) {
  int n = p->n;
  memset(adj, 0, (size_t)n * n);
  for (int f = 0; f < p->nf; f++) {
    const int32_t *s = p->scopes + p->scope_off[f];
    for (int a = 0; a < p->arity[f]; a++)
      for (int b = 0; b < p->arity[f]; b++)
        if (s[a] != s[b]) adj[(size_t)s[a] * n + s[b]] = 1;
  }
}

/* Definition (Induced Graph, Induced Width): process nodes in
 * descending order of priority (last to first), connect each node's
 * preceding neighbours pairwise; the width of a node is its number of
 * preceding neighbours; w* is the maximum. */
int32_t or_induced_width(const or_problem *p, const int32_t *order) {
  int n = p->n;
  unsigned char *adj = (unsigned char *)malloc((size_t)n * n + 1);
  or_primal_graph(p, adj);
  int32_t *pos = position_of(order, n);
  int32_t *prev = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  int32_t w = 0;
  for (int i = n - 1; i >= 0; i--) {
    int v = order[i], np = 0;
    for (int u = 0; u < n; u++)
      if (adj[(size_t)v * n + u] && pos[u] < i) prev[np++] = u;
    if (np > w) w = np;
    for (int a = 0; a < np; a++)
      for (int b = 0; b < np; b++)
        if (a != b) adj[(size_t)prev[a] * n + prev[b]] = 1;
  }
  free(adj);
  free(pos);
  free(prev);
  return w;
}

/* Greedy min-fill (reading A3): repeatedly eliminate the remaining variable
 * with the fewest fill-in edges among its remaining neighbours, ties by
 * fewest remaining neighbours, then smallest id.  The first eliminated
 * variable is the LAST of the ordering. */
void or_minfill_order(const or_problem *p, int32_t *order) {
  int n = p->n;
  unsigned char *adj = (unsigned char *)malloc((size_t)n * n + 1);
  or_primal_graph(p, adj);
  unsigned char *gone = (unsigned char *)calloc(n ? n : 1, 1);
  int32_t *nb = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  for (int step = 0; step < n; step++) {
    int best = -1;
    int64_t bfill = 0, bdeg = 0;
    for (int v = 0; v < n; v++) {
      if (gone[v]) continue;
      int k = 0;
      for (int u = 0; u < n; u++)
        if (!gone[u] && adj[(size_t)v * n + u]) nb[k++] = u;
      int64_t fill = 0;
      for (int a = 0; a < k; a++)
        for (int b = a + 1; b < k; b++)
          if (!adj[(size_t)nb[a] * n + nb[b]]) fill++;
      if (best < 0 || fill < bfill || (fill == bfill && k < bdeg)) {
        best = v;
        bfill = fill;
        bdeg = k;
      }
    }
    int k = 0;
    for (int u = 0; u < n; u++)
      if (!gone[u] && adj[(size_t)best * n + u]) nb[k++] = u;
    for (int a = 0; a < k; a++)
      for (int b = 0; b < k; b++)
        if (a != b) adj[(size_t)nb[a] * n + nb[b]] = 1;
    gone[best] = 1;
    order[n - 1 - step] = best;
  }
  free(adj);
  free(gone);
  free(nb);
}

/* x_i precedes x_j iff |N(x_i)| < |N(x_j)|; ties by id (A3).
 * Insertion sort keeps it obviously stable. */
void or_degree_order(const or_problem *p, int32_t *order) {
  int n = p->n;
  unsigned char *adj = (unsigned char *)malloc((size_t)n * n + 1);
  or_primal_graph(p, adj);
  int32_t *deg = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
  for (int v = 0; v < n; v++)
    for (int u = 0; u < n; u++) deg[v] += adj[(size_t)v * n + u];
  for (int i = 0; i < n; i++) {
    int v = i, j = i;
    while (j > 0 && deg[order[j - 1]] > deg[v]) {
      order[j] = order[j - 1];
      j--;
    }
    order[j] = v;
  }
  free(adj);
  free(deg);
}

/* ------------------------------------------------------------------ */
/* one (mini-)bucket: Alg. 1 line 3 / Alg. 2 line 5                    */

void or_bucket_rows(const int32_t *dom, int32_t n, int32_t is_f64, int32_t x,
                    int32_t nmem, const int32_t *mar, const int64_t *moff,
                    const int32_t *mscope, const int32_t *const *itab,
                    const double *const *ftab, int32_t nsep, const int32_t *sep,
                    int64_t row_begin, int64_t row_end, int32_t *out_i,
                    double *out_f, uint8_t *arg, int32_t nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    int32_t *a = (int32_t *)calloc(n ? n : 1, sizeof(int32_t)); /* the tuple */
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t row = row_begin; row < row_end; row++) {
      /* decode the row into the tuple theta over sep (lexicographic rank,
       * first variable most significant: P:553-554) */
      int64_t r = row;
      for (int q = nsep - 1; q >= 0; q--) {
        a[sep[q]] = (int32_t)(r % dom[sep[q]]);
        r /= dom[sep[q]];
      }
      int64_t best_i = 0;
      double best_f = 0.0;
      int best_v = 0;
      for (int v = 0; v < dom[x]; v++) {
        a[x] = v;
        /* aggregation: sum of every member at theta.v */
        int64_t s_i = 0;
        double s_f = 0.0;
        for (int k = 0; k < nmem; k++) {
          const int32_t *sc = mscope + moff[k];
          int64_t idx = 0; /* re-rank theta.v in the member's own order */
          for (int q = 0; q < mar[k]; q++) idx = idx * dom[sc[q]] + a[sc[q]];
          if (is_f64)
            s_f = s_f + ftab[k][idx];
          else
            s_i = add_i(s_i, itab[k][idx]);
        }
        /* elimination: min over x, smallest index on ties (A8) */
        if (is_f64) {
          if (v == 0 || s_f < best_f) {
            best_f = s_f;
            best_v = v;
          }
        } else {
          if (v == 0 || s_i < best_i) {
            best_i = s_i;
            best_v = v;
          }
        }
      }
      if (is_f64)
        out_f[row - row_begin] = best_f;
      else
        out_i[row - row_begin] = (int32_t)best_i;
      if (arg) arg[row - row_begin] = (uint8_t)best_v;
    }
    free(a);
  }
}

/* The aggregation step alone (Alg. 1 line 3 before the projection,
 * P:204-205) for selected rows: sums[q*d + v] = sum_k f_k(theta_q . v) for
 * theta_q = the row rows[q] of the output scope sep (int: clamped adds, A9;
 * f64: IEEE adds in member order).  Used by the tests to decide whether two
 * argmin choices of a row are a near-tie (reading A10); same decode and
 * re-rank as or_bucket_rows. */
void or_bucket_row_sums(const int32_t *dom, int32_t n, int32_t is_f64, int32_t x,
                        int32_t nmem, const int32_t *mar, const int64_t *moff,
                        const int32_t *mscope, const int32_t *const *itab,
                        const double *const *ftab, int32_t nsep, const int32_t *sep,
                        int64_t nrows, const int64_t *rows, int64_t *sums_i, double *sums_f) {
  int32_t *a = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
  const int d = dom[x];
  for (int64_t q = 0; q < nrows; q++) {
    int64_t r = rows[q];
    for (int p = nsep - 1; p >= 0; p--) {
      a[sep[p]] = (int32_t)(r % dom[sep[p]]);
      r /= dom[sep[p]];
    }
    for (int v = 0; v < d; v++) {
      a[x] = v;
      int64_t s_i = 0;
      double s_f = 0.0;
      for (int k = 0; k < nmem; k++) {
        const int32_t *sc = mscope + moff[k];
        int64_t idx = 0;
        for (int p = 0; p < mar[k]; p++) idx = idx * dom[sc[p]] + a[sc[p]];
        if (is_f64)
          s_f = s_f + ftab[k][idx];
        else
          s_i = add_i(s_i, itab[k][idx]);
      }
      if (is_f64)
        sums_f[q * d + v] = s_f;
      else
        sums_i[q * d + v] = s_i;
    }
  }
  free(a);
}

/* Sum-product bucket (the paper's future work):
 * the same aggregation as or_bucket_rows (the members' -log
 * values are added, i.e. the factors multiplied), but the elimination sums x
 * out instead of minimising (the sum/product semiring P:210 names):
 *     out[theta] = -log sum_v exp(-s_v),   s_v = sum_k f_k(theta.v).
 * Written as the textbook log-sum-exp: with m = min_v s_v (if m = +inf the
 * row is +inf), out = m - log sum_v exp(m - s_v).  f64 only; no argmin. */
void or_bucket_rows_sp(const int32_t *dom, int32_t n, int32_t x, int32_t nmem,
                       const int32_t *mar, const int64_t *moff, const int32_t *mscope,
                       const double *const *ftab, int32_t nsep, const int32_t *sep,
                       int64_t row_begin, int64_t row_end, double *out_f, int32_t nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    int32_t *a = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
    double *s = (double *)malloc(sizeof(double) * (dom[x] ? dom[x] : 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t row = row_begin; row < row_end; row++) {
      int64_t r = row;
      for (int q = nsep - 1; q >= 0; q--) {
        a[sep[q]] = (int32_t)(r % dom[sep[q]]);
        r /= dom[sep[q]];
      }
      for (int v = 0; v < dom[x]; v++) {
        a[x] = v;
        s[v] = 0.0;
        for (int k = 0; k < nmem; k++) {
          const int32_t *sc = mscope + moff[k];
          int64_t idx = 0;
          for (int q = 0; q < mar[k]; q++) idx = idx * dom[sc[q]] + a[sc[q]];
          s[v] = s[v] + ftab[k][idx];
        }
      }
      double m = INFINITY;
      for (int v = 0; v < dom[x]; v++)
        if (s[v] < m) m = s[v];
      double o = INFINITY;
      if (m < INFINITY) {
        double z = 0.0;
        for (int v = 0; v < dom[x]; v++) z += exp(m - s[v]);
        o = m - log(z);
      }
      out_f[row - row_begin] = o;
    }
    free(s);
    free(a);
  }
}

/* Counting bucket ("as a byproduct ... BE can
 * compute the number of consistent solutions").  The (min, count)
 * semiring: every member carries a count table beside its cost table
 * (ctab[k] == NULL for an original function: every entry counts 1).  For
 * theta.v the cost s_v is the sum of or_bucket_rows and c_v = prod_k
 * count_k(theta.v) (doubles, member order).  The row keeps
 *     out   = min_v s_v                     (first minimiser in arg, A8)
 *     count = sum over v = 0..d-1 with s_v == out of c_v
 * and count = 0 when the minimum is infinite (no finite completion).
 * consistent = 1 reads every finite member entry as cost 0: s_v is then 0
 * or infinite and count is the number of consistent completions. */
void or_bucket_rows_cnt(const int32_t *dom, int32_t n, int32_t is_f64, int32_t x,
                        int32_t nmem, const int32_t *mar, const int64_t *moff,
                        const int32_t *mscope, const int32_t *const *itab,
                        const double *const *ftab, const double *const *ctab,
                        int32_t consistent, int32_t nsep, const int32_t *sep,
                        int64_t row_begin, int64_t row_end, int32_t *out_i,
                        double *out_f, double *out_c, uint8_t *arg, int32_t nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    int32_t *a = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
    int64_t *si = (int64_t *)malloc(sizeof(int64_t) * (dom[x] ? dom[x] : 1));
    double *sf = (double *)malloc(sizeof(double) * (dom[x] ? dom[x] : 1));
    double *c = (double *)malloc(sizeof(double) * (dom[x] ? dom[x] : 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t row = row_begin; row < row_end; row++) {
      int64_t r = row;
      for (int q = nsep - 1; q >= 0; q--) {
        a[sep[q]] = (int32_t)(r % dom[sep[q]]);
        r /= dom[sep[q]];
      }
      for (int v = 0; v < dom[x]; v++) {
        a[x] = v;
        si[v] = 0;
        sf[v] = 0.0;
        c[v] = 1.0;
        for (int k = 0; k < nmem; k++) {
          const int32_t *sc = mscope + moff[k];
          int64_t idx = 0;
          for (int q = 0; q < mar[k]; q++) idx = idx * dom[sc[q]] + a[sc[q]];
          if (is_f64) {
            double f = ftab[k][idx];
            if (consistent && f < INFINITY) f = 0.0;
            sf[v] = sf[v] + f;
          } else {
            int32_t f = itab[k][idx];
            if (consistent && f < OR_INF_I32) f = 0;
            si[v] = add_i(si[v], f);
          }
          if (ctab[k]) c[v] = c[v] * ctab[k][idx];
        }
      }
      int best_v = 0;
      for (int v = 1; v < dom[x]; v++)
        if (is_f64 ? sf[v] < sf[best_v] : si[v] < si[best_v]) best_v = v;
      const int inf = is_f64 ? !(sf[best_v] < INFINITY) : si[best_v] >= OR_INF_I32;
      double cnt = 0.0;
      if (!inf)
        for (int v = 0; v < dom[x]; v++)
          if (is_f64 ? sf[v] == sf[best_v] : si[v] == si[best_v]) cnt = cnt + c[v];
      if (is_f64)
        out_f[row - row_begin] = sf[best_v];
      else
        out_i[row - row_begin] = (int32_t)si[best_v];
      out_c[row - row_begin] = cnt;
      if (arg) arg[row - row_begin] = (uint8_t)best_v;
    }
    free(c);
    free(sf);
    free(si);
    free(a);
  }
}

/* ------------------------------------------------------------------ */
/* whole solve: Alg. 1 (BE) / Alg. 2 (MBE)                              */

typedef struct {
  int32_t kind; /* 0 original, 1 message (table index) */
  int32_t index;
} member;

typedef struct {
  int32_t var, mb, nsep, dest, nmem;
  int32_t *sep;
  member *mem;
  int64_t rows;
  int32_t *out_i;
  double *out_f;
  double *out_c; /* counting mode: completions attaining out */
  uint8_t *arg;
  uint64_t digest;
} otable;

typedef struct {
  int32_t n, cap;
  member *m;
} mlist;

struct or_run {
  int32_t status, is_f64, n;
  int32_t ntab, cap;
  otable *tab;
  int64_t value_i, upper_i;
  double value_f, upper_f;
  int32_t have_assign;
  int32_t *assign;
  double count; /* counting mode: number of optimal (or consistent) solutions */
};

static void ml_push(mlist *l, int32_t kind, int32_t index) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 8;
    l->m = (member *)realloc(l->m, sizeof(member) * l->cap);
  }
  l->m[l->n].kind = kind;
  l->m[l->n].index = index;
  l->n++;
}

/* scope and table of a member */
static int32_t mem_arity(const or_problem *p, const or_run *r, member m) {
  return m.kind == 0 ? p->arity[m.index] : r->tab[m.index].nsep;
}
static const int32_t *mem_scope(const or_problem *p, const or_run *r, member m) {
  return m.kind == 0 ? p->scopes + p->scope_off[m.index] : r->tab[m.index].sep;
}
static const int32_t *mem_itab(const or_problem *p, const or_run *r, member m) {
  return m.kind == 0 ? p->icost + p->table_off[m.index] : r->tab[m.index].out_i;
}
static const double *mem_ftab(const or_problem *p, const or_run *r, member m) {
  return m.kind == 0 ? p->fcost + p->table_off[m.index] : r->tab[m.index].out_f;
}

static int cmp_pos_ctx_n;
static const int32_t *cmp_pos_ctx;
static int cmp_by_pos(const void *a, const void *b) {
  int32_t x = cmp_pos_ctx[*(const int32_t *)a], y = cmp_pos_ctx[*(const int32_t *)b];
  return (x > y) - (x < y);
}

static or_run *or_solve_impl(const or_problem *p, const int32_t *order, int32_t ibound,
                             int32_t keep_tables, int32_t nthreads, int32_t mode) {
  /* mode: 0 min-sum, 1 sum-product, 2 count optimal, 3 count consistent */
  const int sumprod = mode == 1, counting = mode >= 2;
  int n = p->n;
  or_run *r = (or_run *)calloc(1, sizeof(or_run));
  r->is_f64 = p->is_f64;
  r->n = n;
  r->assign = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
  int32_t *pos = position_of(order, n);
  mlist *bucket = (mlist *)calloc(n ? n : 1, sizeof(mlist));
  mlist constants = {0};

  /* Bucket membership (reading A1, Example 3 P:250): a function goes
   * to the bucket of its latest-ordered scope variable.  Originals enter in
   * function-index order. */
  for (int f = 0; f < p->nf; f++) {
    if (p->arity[f] == 0) {
      ml_push(&constants, 0, f);
      continue;
    }
    const int32_t *s = p->scopes + p->scope_off[f];
    int v = s[0];
    for (int a = 1; a < p->arity[f]; a++)
      if (pos[s[a]] > pos[v]) v = s[a];
    ml_push(&bucket[v], 0, f);
  }

  unsigned char *inU = (unsigned char *)calloc(n ? n : 1, 1);
  int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));

  /* Variable elimination phase: i = n downto 1 (Alg. 1 line 1) */
  for (int i = n - 1; i >= 0 && r->status == 0; i--) {
    int x = order[i];
    mlist *B = &bucket[x];
    /* mini-bucket partition (Alg. 2 line 3; readings A5, A6).  BE: one
     * mini-bucket holding the whole bucket. */
    int nm = B->n;
    int32_t *mb_of = (int32_t *)malloc(sizeof(int32_t) * (nm ? nm : 1));
    int nmb = 0;
    if (ibound < 0 || nm == 0) {
      for (int k = 0; k < nm; k++) mb_of[k] = 0;
      nmb = 1;
    } else {
      /* members by descending arity, stable in the canonical order */
      int32_t *ordm = (int32_t *)malloc(sizeof(int32_t) * nm);
      for (int k = 0; k < nm; k++) ordm[k] = k;
      for (int a = 1; a < nm; a++) { /* stable insertion sort */
        int v = ordm[a], b = a;
        while (b > 0 && mem_arity(p, r, B->m[ordm[b - 1]]) < mem_arity(p, r, B->m[v])) {
          ordm[b] = ordm[b - 1];
          b--;
        }
        ordm[b] = v;
      }
      unsigned char **mbset = (unsigned char **)malloc(sizeof(unsigned char *) * nm);
      int32_t *mbsize = (int32_t *)malloc(sizeof(int32_t) * nm);
      for (int a = 0; a < nm; a++) {
        member m = B->m[ordm[a]];
        int ar = mem_arity(p, r, m);
        const int32_t *sc = mem_scope(p, r, m);
        if (ar > ibound + 1) {
          r->status = 1; /* cannot satisfy |union| <= i+1 */
          break;
        }
        int placed = -1;
        for (int b = 0; b < nmb && placed < 0; b++) {
          int extra = 0;
          for (int q = 0; q < ar; q++)
            if (!mbset[b][sc[q]]) extra++;
          if (mbsize[b] + extra <= ibound + 1) placed = b;
        }
        if (placed < 0) {
          placed = nmb++;
          mbset[placed] = (unsigned char *)calloc(n, 1);
          mbsize[placed] = 0;
        }
        for (int q = 0; q < ar; q++)
          if (!mbset[placed][sc[q]]) {
            mbset[placed][sc[q]] = 1;
            mbsize[placed]++;
          }
        mb_of[ordm[a]] = placed;
      }
      for (int b = 0; b < nmb; b++) free(mbset[b]);
      free(mbset);
      free(mbsize);
      free(ordm);
      if (r->status) {
        free(mb_of);
        break;
      }
    }

    for (int b = 0; b < nmb; b++) {
      /* members of mini-bucket b, canonical order */
      int cnt = 0;
      for (int k = 0; k < nm; k++) cnt += (mb_of[k] == b);
      otable t;
      memset(&t, 0, sizeof(t));
      t.var = x;
      t.mb = b;
      t.nmem = cnt;
      t.mem = (member *)malloc(sizeof(member) * (cnt ? cnt : 1));
      cnt = 0;
      for (int k = 0; k < nm; k++)
        if (mb_of[k] == b) t.mem[cnt++] = B->m[k];
      /* scope union U, sep = U \ {x} sorted by ascending position (A2) */
      memset(inU, 0, n);
      for (int k = 0; k < t.nmem; k++) {
        int ar = mem_arity(p, r, t.mem[k]);
        const int32_t *sc = mem_scope(p, r, t.mem[k]);
        for (int q = 0; q < ar; q++) inU[sc[q]] = 1;
      }
      int ns = 0;
      for (int v = 0; v < n; v++)
        if (inU[v] && v != x) tmp[ns++] = v;
      cmp_pos_ctx = pos;
      cmp_pos_ctx_n = n;
      qsort(tmp, ns, sizeof(int32_t), cmp_by_pos);
      t.nsep = ns;
      t.sep = (int32_t *)malloc(sizeof(int32_t) * (ns ? ns : 1));
      memcpy(t.sep, tmp, sizeof(int32_t) * ns);
      t.rows = 1;
      for (int q = 0; q < ns; q++) t.rows *= p->dom[t.sep[q]];
      t.dest = ns ? t.sep[ns - 1] : -1;
      if (p->is_f64)
        t.out_f = (double *)malloc(sizeof(double) * t.rows);
      else
        t.out_i = (int32_t *)malloc(sizeof(int32_t) * t.rows);
      t.arg = (uint8_t *)malloc(t.rows);
      if ((p->is_f64 ? (void *)t.out_f : (void *)t.out_i) == NULL || t.arg == NULL) {
        r->status = 2;
        free(t.out_f);
        free(t.out_i);
        free(t.arg);
        free(t.sep);
        free(t.mem);
        break;
      }
      /* member descriptors */
      int32_t *mar = (int32_t *)malloc(sizeof(int32_t) * (t.nmem ? t.nmem : 1));
      int64_t *moff = (int64_t *)malloc(sizeof(int64_t) * (t.nmem ? t.nmem : 1));
      int64_t tot = 0;
      for (int k = 0; k < t.nmem; k++) {
        mar[k] = mem_arity(p, r, t.mem[k]);
        moff[k] = tot;
        tot += mar[k];
      }
      int32_t *msc = (int32_t *)malloc(sizeof(int32_t) * (tot ? tot : 1));
      const int32_t **it = (const int32_t **)malloc(sizeof(void *) * (t.nmem ? t.nmem : 1));
      const double **ft = (const double **)malloc(sizeof(void *) * (t.nmem ? t.nmem : 1));
      for (int k = 0; k < t.nmem; k++) {
        memcpy(msc + moff[k], mem_scope(p, r, t.mem[k]), sizeof(int32_t) * mar[k]);
        it[k] = p->is_f64 ? NULL : mem_itab(p, r, t.mem[k]);
        ft[k] = p->is_f64 ? mem_ftab(p, r, t.mem[k]) : NULL;
      }
      if (counting) {
        const double **ct = (const double **)malloc(sizeof(void *) * (t.nmem ? t.nmem : 1));
        for (int k = 0; k < t.nmem; k++) ct[k] = t.mem[k].kind == 1 ? r->tab[t.mem[k].index].out_c : NULL;
        t.out_c = (double *)malloc(sizeof(double) * t.rows);
        or_bucket_rows_cnt(p->dom, n, p->is_f64, x, t.nmem, mar, moff, msc, it, ft, ct, mode == 3,
                           t.nsep, t.sep, 0, t.rows, t.out_i, t.out_f, t.out_c, t.arg, nthreads);
        free(ct);
      } else if (sumprod) {
        or_bucket_rows_sp(p->dom, n, x, t.nmem, mar, moff, msc, ft, t.nsep, t.sep, 0, t.rows,
                          t.out_f, nthreads);
        memset(t.arg, 0, t.rows); /* no argmin in the sum-product semiring */
      } else {
        or_bucket_rows(p->dom, n, p->is_f64, x, t.nmem, mar, moff, msc, it, ft, t.nsep,
                       t.sep, 0, t.rows, t.out_i, t.out_f, t.arg, nthreads);
      }
      free(mar);
      free(moff);
      free(msc);
      free(it);
      free(ft);
      if (g_digest_kind == 1) {
        t.digest = or_mixsum(p->is_f64 ? (const void *)t.out_f : (const void *)t.out_i, p->is_f64 ? 8 : 4,
                             t.rows, 1, nthreads) +
                   or_mixsum(t.arg, 1, t.rows, 2, nthreads);
      } else {
        uint64_t h = 0xcbf29ce484222325ULL;
        if (p->is_f64)
          h = or_fnv1a(h, t.out_f, t.rows * (int64_t)sizeof(double));
        else
          h = or_fnv1a(h, t.out_i, t.rows * (int64_t)sizeof(int32_t));
        t.digest = or_fnv1a(h, t.arg, t.rows);
      }
      if (!keep_tables) {
        free(t.arg);
        t.arg = NULL;
      }
      /* append the table, route the message (Alg. 1 line 5 / Alg. 2 line 6) */
      if (r->ntab == r->cap) {
        r->cap = r->cap ? 2 * r->cap : 64;
        r->tab = (otable *)realloc(r->tab, sizeof(otable) * r->cap);
      }
      r->tab[r->ntab] = t;
      if (t.dest >= 0)
        ml_push(&bucket[t.dest], 1, r->ntab);
      else
        ml_push(&constants, 1, r->ntab);
      r->ntab++;
    }
    free(mb_of);
    /* messages consumed by this bucket are no longer needed (keep = 0) */
    if (!keep_tables && r->status == 0)
      for (int k = 0; k < nm; k++)
        if (B->m[k].kind == 1) {
          otable *c = &r->tab[B->m[k].index];
          free(c->out_i);
          free(c->out_f);
          free(c->out_c);
          c->out_i = NULL;
          c->out_f = NULL;
          c->out_c = NULL;
        }
  }

  if (r->status == 0) {
    /* optimum (BE) / lower bound (MBE) = sum of the constants, originals
     * first then messages in creation order (reading A11) */
    int64_t vi = 0;
    double vf = 0.0;
    for (int k = 0; k < constants.n; k++) {
      member m = constants.m[k];
      if (p->is_f64)
        vf = vf + mem_ftab(p, r, m)[0];
      else
        vi = add_i(vi, mem_itab(p, r, m)[0]);
    }
    r->value_i = vi;
    r->value_f = vf;
    if (counting) {
      /* counting: the components' counts multiply (P:639-640 for the costs);
       * an original constant is one assignment of no variable (count 1) */
      if (mode == 3) { /* consistent: every finite constant reads as 0 */
        int inf = 0;
        for (int k = 0; k < constants.n; k++) {
          member m = constants.m[k];
          if (p->is_f64 ? !(mem_ftab(p, r, m)[0] < INFINITY) : mem_itab(p, r, m)[0] >= OR_INF_I32) inf = 1;
        }
        r->value_i = inf ? OR_INF_I32 : 0;
        r->value_f = inf ? INFINITY : 0.0;
      }
      double cnt = 1.0;
      for (int k = 0; k < constants.n; k++)
        if (constants.m[k].kind == 1) cnt = cnt * r->tab[constants.m[k].index].out_c[0];
      const int inf = p->is_f64 ? !(r->value_f < INFINITY) : r->value_i >= OR_INF_I32;
      r->count = inf ? 0.0 : cnt;
    }

    /* Value assignment phase (Alg. 1 lines 6-7; MBE: Example 4,
     * P:341, reading A7): for x = first..last pick the value minimising the
     * sum of ALL functions of B_x (canonical order) given earlier values. */
    if (keep_tables && !sumprod && mode != 3) {
      int32_t *a = r->assign;
      for (int i = 0; i < n; i++) {
        int x = order[i];
        mlist *B = &bucket[x];
        int64_t best_i = 0;
        double best_f = 0.0;
        int best_v = 0;
        for (int v = 0; v < p->dom[x]; v++) {
          a[x] = v;
          int64_t s_i = 0;
          double s_f = 0.0;
          for (int k = 0; k < B->n; k++) {
            int ar = mem_arity(p, r, B->m[k]);
            const int32_t *sc = mem_scope(p, r, B->m[k]);
            int64_t idx = 0;
            for (int q = 0; q < ar; q++) idx = idx * p->dom[sc[q]] + a[sc[q]];
            if (p->is_f64)
              s_f = s_f + mem_ftab(p, r, B->m[k])[idx];
            else
              s_i = add_i(s_i, mem_itab(p, r, B->m[k])[idx]);
          }
          if (p->is_f64 ? (v == 0 || s_f < best_f) : (v == 0 || s_i < best_i)) {
            best_i = s_i;
            best_f = s_f;
            best_v = v;
          }
        }
        a[x] = best_v;
      }
      r->have_assign = 1;
      if (p->is_f64)
        r->upper_f = or_evaluate_f(p, a);
      else
        r->upper_i = or_evaluate_i(p, a);
    }
  }

  for (int v = 0; v < n; v++) free(bucket[v].m);
  free(bucket);
  free(constants.m);
  free(inU);
  free(tmp);
  free(pos);
  return r;
}

int32_t or_run_status(const or_run *r) { return r->status; }
int32_t or_run_ntables(const or_run *r) { return r->ntab; }

void or_run_table_meta(const or_run *r, int32_t t, int32_t *var, int32_t *mb,
                       int32_t *nsep, int64_t *rows, int32_t *dest, int32_t *nmem) {
  const otable *x = &r->tab[t];
  *var = x->var;
  *mb = x->mb;
  *nsep = x->nsep;
  *rows = x->rows;
  *dest = x->dest;
  *nmem = x->nmem;
}

void or_run_table_sep(const or_run *r, int32_t t, int32_t *sep) {
  memcpy(sep, r->tab[t].sep, sizeof(int32_t) * r->tab[t].nsep);
}

void or_run_table_members(const or_run *r, int32_t t, int32_t *kind, int32_t *index) {
  for (int k = 0; k < r->tab[t].nmem; k++) {
    kind[k] = r->tab[t].mem[k].kind;
    index[k] = r->tab[t].mem[k].index;
  }
}

int32_t or_run_table_out(const or_run *r, int32_t t, int32_t *out_i, double *out_f,
                         uint8_t *arg) {
  const otable *x = &r->tab[t];
  if ((r->is_f64 ? (void *)x->out_f : (void *)x->out_i) == NULL || x->arg == NULL) return 0;
  if (out_i && x->out_i) memcpy(out_i, x->out_i, sizeof(int32_t) * x->rows);
  if (out_f && x->out_f) memcpy(out_f, x->out_f, sizeof(double) * x->rows);
  if (arg) memcpy(arg, x->arg, x->rows);
  return 1;
}

uint64_t or_run_table_digest(const or_run *r, int32_t t) { return r->tab[t].digest; }
int64_t or_run_value_i(const or_run *r) { return r->value_i; }
double or_run_value_f(const or_run *r) { return r->value_f; }
int64_t or_run_upper_i(const or_run *r) { return r->upper_i; }
double or_run_upper_f(const or_run *r) { return r->upper_f; }

int32_t or_run_assignment(const or_run *r, int32_t *assign) {
  if (!r->have_assign) return 0;
  memcpy(assign, r->assign, sizeof(int32_t) * r->n);
  return 1;
}

void or_run_free(or_run *r) {
  if (!r) return;
  for (int t = 0; t < r->ntab; t++) {
    free(r->tab[t].sep);
    free(r->tab[t].mem);
    free(r->tab[t].out_i);
    free(r->tab[t].out_f);
    free(r->tab[t].out_c);
    free(r->tab[t].arg);
  }
  free(r->tab);
  free(r->assign);
  free(r);
}

/* elimination tree (A14): a symbolic run of Alg. 1 on scopes only */
void or_elim_tree(const or_problem *p, const int32_t *order, int32_t *parent) {
  int n = p->n;
  int32_t *pos = position_of(order, n);
  unsigned char *inB = (unsigned char *)calloc((size_t)n * n + 1, 1); /* bucket scope unions */
  for (int f = 0; f < p->nf; f++) {
    const int32_t *s = p->scopes + p->scope_off[f];
    if (p->arity[f] == 0) continue;
    int v = s[0];
    for (int a = 1; a < p->arity[f]; a++)
      if (pos[s[a]] > pos[v]) v = s[a];
    for (int a = 0; a < p->arity[f]; a++) inB[(size_t)v * n + s[a]] = 1;
  }
  for (int i = n - 1; i >= 0; i--) {
    int x = order[i], dest = -1;
    for (int u = 0; u < n; u++)
      if (u != x && inB[(size_t)x * n + u] && (dest < 0 || pos[u] > pos[dest])) dest = u;
    parent[x] = dest;
    if (dest >= 0)
      for (int u = 0; u < n; u++)
        if (u != x && inB[(size_t)x * n + u]) inB[(size_t)dest * n + u] = 1;
  }
  free(pos);
  free(inB);
}

/* cost of a complete assignment: sum over all functions (Eq. 1) */
int64_t or_evaluate_i(const or_problem *p, const int32_t *assign) {
  int64_t s = 0;
  for (int f = 0; f < p->nf; f++) {
    const int32_t *sc = p->scopes + p->scope_off[f];
    int64_t idx = 0;
    for (int q = 0; q < p->arity[f]; q++) idx = idx * p->dom[sc[q]] + assign[sc[q]];
    s = add_i(s, p->icost[p->table_off[f] + idx]);
  }
  return s;
}

double or_evaluate_f(const or_problem *p, const int32_t *assign) {
  double s = 0.0;
  for (int f = 0; f < p->nf; f++) {
    const int32_t *sc = p->scopes + p->scope_off[f];
    int64_t idx = 0;
    for (int q = 0; q < p->arity[f]; q++) idx = idx * p->dom[sc[q]] + assign[sc[q]];
    s = s + p->fcost[p->table_off[f] + idx];
  }
  return s;
}

or_run *or_solve(const or_problem *p, const int32_t *order, int32_t ibound,
                 int32_t keep_tables, int32_t nthreads) {
  return or_solve_impl(p, order, ibound, keep_tables, nthreads, 0);
}

or_run *or_solve_count(const or_problem *p, const int32_t *order, int32_t consistent,
                       int32_t keep_tables, int32_t nthreads) {
  return or_solve_impl(p, order, -1, keep_tables, nthreads, consistent ? 3 : 2);
}

double or_run_count(const or_run *r) { return r->count; }

int32_t or_run_table_count(const or_run *r, int32_t t, double *out_c) {
  if (!r->tab[t].out_c) return 0;
  memcpy(out_c, r->tab[t].out_c, sizeof(double) * r->tab[t].rows);
  return 1;
}

or_run *or_solve_sumprod(const or_problem *p, const int32_t *order, int32_t keep_tables,
                         int32_t nthreads) {
  if (!p->is_f64) return NULL;
  return or_solve_impl(p, order, -1, keep_tables, nthreads, 1);
}
