/* gen.c — seeded synthetic instance generators (see gen.h).
 * No method arithmetic lives here: only graph drawing and cost sampling. */
#include "gen.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

uint64_t gen_splitmix64(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* unbiased integer in [0, n) by rejection */
static uint64_t rand_below(uint64_t *s, uint64_t n) {
  uint64_t lim = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = gen_splitmix64(s);
  } while (x >= lim);
  return x % n;
}

/* uniform double in (0, 1] */
static double rand_unit_open0(uint64_t *s) {
  return ((gen_splitmix64(s) >> 11) + 1) * 0x1.0p-53;
}

static uint64_t mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t s = seed ^ (0xD1B54A32D192ED03ULL * (stream + 1));
  gen_splitmix64(&s);
  return s;
}

/* ------------------------------------------------------------------ */
/* instance assembly                                                   */

typedef struct {
  int32_t nf, cap;
  int32_t *arity;
  int32_t **scope;
} fn_list;

static void fl_push(fn_list *fl, int32_t arity, const int32_t *vars) {
  if (fl->nf == fl->cap) {
    fl->cap = fl->cap ? 2 * fl->cap : 64;
    fl->arity = (int32_t *)realloc(fl->arity, sizeof(int32_t) * fl->cap);
    fl->scope = (int32_t **)realloc(fl->scope, sizeof(int32_t *) * fl->cap);
  }
  fl->arity[fl->nf] = arity;
  fl->scope[fl->nf] = (int32_t *)malloc(sizeof(int32_t) * (arity ? arity : 1));
  memcpy(fl->scope[fl->nf], vars, sizeof(int32_t) * arity);
  fl->nf++;
}

static void fl_free(fn_list *fl) {
  for (int i = 0; i < fl->nf; i++) free(fl->scope[i]);
  free(fl->arity);
  free(fl->scope);
}

/* Allocate an instance with structure from fl; tables are left for the
 * caller to fill. */
static gen_instance *assemble(int32_t n, const int32_t *dom, const fn_list *fl,
                              int is_f64) {
  gen_instance *g = (gen_instance *)calloc(1, sizeof(gen_instance));
  g->n = n;
  g->nf = fl->nf;
  g->is_f64 = is_f64;
  g->dom = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  memcpy(g->dom, dom, sizeof(int32_t) * n);
  g->arity = (int32_t *)malloc(sizeof(int32_t) * (fl->nf ? fl->nf : 1));
  g->scope_off = (int64_t *)malloc(sizeof(int64_t) * (fl->nf + 1));
  g->table_off = (int64_t *)malloc(sizeof(int64_t) * (fl->nf + 1));
  int64_t so = 0, to = 0;
  for (int i = 0; i < fl->nf; i++) {
    g->arity[i] = fl->arity[i];
    g->scope_off[i] = so;
    g->table_off[i] = to;
    so += fl->arity[i];
    int64_t cells = 1;
    for (int a = 0; a < fl->arity[i]; a++) cells *= dom[fl->scope[i][a]];
    to += cells;
  }
  g->scope_off[fl->nf] = so;
  g->table_off[fl->nf] = to;
  g->scopes = (int32_t *)malloc(sizeof(int32_t) * (so ? so : 1));
  for (int i = 0; i < fl->nf; i++)
    memcpy(g->scopes + g->scope_off[i], fl->scope[i], sizeof(int32_t) * fl->arity[i]);
  if (is_f64)
    g->fcost = (double *)malloc(sizeof(double) * (to ? to : 1));
  else
    g->icost = (int32_t *)malloc(sizeof(int32_t) * (to ? to : 1));
  return g;
}

/* Integer costs uniform in [0, cmax]; exactly floor(p2*cells) cells set to
 * GEN_INF_I32, chosen uniformly (partial Fisher-Yates). P:928. */
static void fill_int_tables(gen_instance *g, int32_t cmax, double p2, uint64_t *rs) {
  for (int f = 0; f < g->nf; f++) {
    int64_t a = g->table_off[f], b = g->table_off[f + 1], cells = b - a;
    int32_t *t = g->icost + a;
    for (int64_t c = 0; c < cells; c++) t[c] = (int32_t)rand_below(rs, (uint64_t)cmax + 1);
    int64_t ninf = (int64_t)floor(p2 * (double)cells);
    if (ninf > 0) {
      int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * cells);
      for (int64_t c = 0; c < cells; c++) idx[c] = c;
      for (int64_t c = 0; c < ninf; c++) {
        int64_t j = c + (int64_t)rand_below(rs, (uint64_t)(cells - c));
        int64_t tmp = idx[c];
        idx[c] = idx[j];
        idx[j] = tmp;
        t[idx[c]] = GEN_INF_I32;
      }
      free(idx);
    }
  }
}

static void fill_f64_tables(gen_instance *g, double fmax, double p2, uint64_t *rs) {
  for (int f = 0; f < g->nf; f++) {
    int64_t a = g->table_off[f], b = g->table_off[f + 1], cells = b - a;
    double *t = g->fcost + a;
    for (int64_t c = 0; c < cells; c++) t[c] = (rand_unit_open0(rs) - 0x1.0p-53) * fmax;
    int64_t ninf = (int64_t)floor(p2 * (double)cells);
    if (ninf > 0) {
      int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * cells);
      for (int64_t c = 0; c < cells; c++) idx[c] = c;
      for (int64_t c = 0; c < ninf; c++) {
        int64_t j = c + (int64_t)rand_below(rs, (uint64_t)(cells - c));
        int64_t tmp = idx[c];
        idx[c] = idx[j];
        idx[j] = tmp;
        t[idx[c]] = INFINITY;
      }
      free(idx);
    }
  }
}

/* ------------------------------------------------------------------ */
/* graphs                                                              */

static int connected(int32_t n, const unsigned char *adj) {
  if (n <= 1) return 1;
  int32_t *stack = (int32_t *)malloc(sizeof(int32_t) * n);
  unsigned char *seen = (unsigned char *)calloc(n, 1);
  int top = 0, cnt = 1;
  stack[top++] = 0;
  seen[0] = 1;
  while (top) {
    int u = stack[--top];
    for (int v = 0; v < n; v++)
      if (adj[(size_t)u * n + v] && !seen[v]) {
        seen[v] = 1;
        cnt++;
        stack[top++] = v;
      }
  }
  free(stack);
  free(seen);
  return cnt == n;
}

/* Edge set -> binary functions, edges in lexicographic (u<v) order, declared
 * scope (u, v). */
static gen_instance *from_adjacency(int32_t n, int32_t d, const unsigned char *adj,
                                    double p2, uint64_t *rs) {
  fn_list fl = {0};
  for (int u = 0; u < n; u++)
    for (int v = u + 1; v < n; v++)
      if (adj[(size_t)u * n + v]) {
        int32_t sc[2] = {u, v};
        fl_push(&fl, 2, sc);
      }
  int32_t *dom = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  for (int i = 0; i < n; i++) dom[i] = d;
  gen_instance *g = assemble(n, dom, &fl, 0);
  fill_int_tables(g, 100, p2, rs);
  free(dom);
  fl_free(&fl);
  return g;
}

gen_instance *gen_random_graph(int32_t n, int32_t d, int64_t nedges, int32_t mode,
                               double p2, uint64_t seed) {
  if (n < 1 || d < 1) return NULL;
  int64_t maxe = (int64_t)n * (n - 1) / 2;
  if (nedges > maxe) nedges = maxe;
  if (nedges < n - 1) return NULL; /* cannot be connected */
  unsigned char *adj = (unsigned char *)malloc((size_t)n * n);
  for (int attempt = 0; attempt < 1000; attempt++) {
    uint64_t rs = mix_seed(seed, (uint64_t)attempt);
    memset(adj, 0, (size_t)n * n);
    int64_t have = 0;
    if (mode == 1 && n >= 2) {
      /* uniform labelled spanning tree from a uniform Pruefer sequence */
      int32_t *pr = (int32_t *)malloc(sizeof(int32_t) * (n > 2 ? n - 2 : 1));
      int32_t *deg = (int32_t *)malloc(sizeof(int32_t) * n);
      for (int i = 0; i < n - 2; i++) pr[i] = (int32_t)rand_below(&rs, (uint64_t)n);
      for (int i = 0; i < n; i++) deg[i] = 1;
      for (int i = 0; i < n - 2; i++) deg[pr[i]]++;
      for (int i = 0; i < n - 2; i++) {
        int leaf = 0;
        while (deg[leaf] != 1) leaf++;
        int u = leaf, v = pr[i];
        adj[(size_t)u * n + v] = adj[(size_t)v * n + u] = 1;
        deg[u]--;
        deg[v]--;
      }
      int u = -1, v = -1;
      for (int i = 0; i < n; i++)
        if (deg[i] == 1) {
          if (u < 0) u = i; else v = i;
        }
      adj[(size_t)u * n + v] = adj[(size_t)v * n + u] = 1;
      have = n - 1;
      free(pr);
      free(deg);
    }
    while (have < nedges) {
      int u = (int)rand_below(&rs, (uint64_t)n), v = (int)rand_below(&rs, (uint64_t)n);
      if (u == v || adj[(size_t)u * n + v]) continue;
      adj[(size_t)u * n + v] = adj[(size_t)v * n + u] = 1;
      have++;
    }
    if (connected(n, adj)) {
      gen_instance *g = from_adjacency(n, d, adj, p2, &rs);
      free(adj);
      return g;
    }
  }
  free(adj);
  return NULL;
}

gen_instance *gen_scalefree(int32_t n, int32_t d, double p2, uint64_t seed) {
  if (n < 2 || d < 1) return NULL;
  uint64_t rs = mix_seed(seed, 0);
  unsigned char *adj = (unsigned char *)calloc((size_t)n * n, 1);
  /* endpoint list: each edge contributes both endpoints -> sampling an entry
   * uniformly picks a node with probability proportional to its degree */
  int64_t cap = 2 * (2 * (int64_t)n + 2), ne = 0;
  int32_t *ends = (int32_t *)malloc(sizeof(int32_t) * cap);
  adj[0 * n + 1] = adj[1 * n + 0] = 1;
  ends[ne++] = 0;
  ends[ne++] = 1;
  for (int t = 2; t < n; t++) {
    int a = ends[rand_below(&rs, (uint64_t)ne)];
    int b;
    do {
      b = ends[rand_below(&rs, (uint64_t)ne)];
    } while (b == a);
    adj[(size_t)t * n + a] = adj[(size_t)a * n + t] = 1;
    adj[(size_t)t * n + b] = adj[(size_t)b * n + t] = 1;
    ends[ne++] = t;
    ends[ne++] = a;
    ends[ne++] = t;
    ends[ne++] = b;
  }
  gen_instance *g = from_adjacency(n, d, adj, p2, &rs);
  free(adj);
  free(ends);
  return g;
}

gen_instance *gen_grid(int32_t rows, int32_t cols, int32_t d, double p2, uint64_t seed) {
  if (rows < 1 || cols < 1 || d < 1) return NULL;
  uint64_t rs = mix_seed(seed, 0);
  int32_t n = rows * cols;
  fn_list fl = {0};
  for (int r = 0; r < rows; r++)
    for (int c = 0; c < cols; c++) {
      int v = r * cols + c;
      if (c + 1 < cols) {
        int32_t sc[2] = {v, v + 1};
        fl_push(&fl, 2, sc);
      }
      if (r + 1 < rows) {
        int32_t sc[2] = {v, v + cols};
        fl_push(&fl, 2, sc);
      }
    }
  int32_t *dom = (int32_t *)malloc(sizeof(int32_t) * n);
  for (int i = 0; i < n; i++) dom[i] = d;
  gen_instance *g = assemble(n, dom, &fl, 0);
  fill_int_tables(g, 100, p2, &rs);
  free(dom);
  fl_free(&fl);
  return g;
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

gen_instance *gen_belief_net(int32_t n, int32_t dmin, int32_t dmax, int32_t maxpar,
                             int32_t window, uint64_t seed) {
  if (n < 1 || dmin < 1 || dmax < dmin) return NULL;
  uint64_t rs = mix_seed(seed, 0);
  int32_t *dom = (int32_t *)malloc(sizeof(int32_t) * n);
  for (int i = 0; i < n; i++) dom[i] = dmin + (int32_t)rand_below(&rs, (uint64_t)(dmax - dmin + 1));
  fn_list fl = {0};
  int32_t *sc = (int32_t *)malloc(sizeof(int32_t) * (maxpar + 1));
  int32_t *pool = (int32_t *)malloc(sizeof(int32_t) * (window > 0 ? window : 1));
  for (int v = 0; v < n; v++) {
    int lo = v - window < 0 ? 0 : v - window;
    int avail = v - lo;
    int np = maxpar < avail ? maxpar : avail;
    for (int i = 0; i < avail; i++) pool[i] = lo + i;
    for (int i = 0; i < np; i++) {
      int j = i + (int)rand_below(&rs, (uint64_t)(avail - i));
      int32_t t = pool[i];
      pool[i] = pool[j];
      pool[j] = t;
      sc[i] = pool[i];
    }
    qsort(sc, np, sizeof(int32_t), cmp_i32);
    sc[np] = v;
    fl_push(&fl, np + 1, sc);
  }
  gen_instance *g = assemble(n, dom, &fl, 1);
  /* CPT rows ~ Dirichlet(1): normalised iid Exp(1) draws; stored -log p */
  for (int f = 0; f < g->nf; f++) {
    int child = g->scopes[g->scope_off[f] + g->arity[f] - 1];
    int dc = dom[child];
    int64_t cells = g->table_off[f + 1] - g->table_off[f];
    double *t = g->fcost + g->table_off[f];
    double *e = (double *)malloc(sizeof(double) * dc);
    for (int64_t row = 0; row < cells / dc; row++) {
      double s = 0;
      for (int c = 0; c < dc; c++) {
        e[c] = -log(rand_unit_open0(&rs));
        s += e[c];
      }
      for (int c = 0; c < dc; c++) {
        double nl = -log(e[c] / s);
        t[row * dc + c] = nl > 0.0 ? nl : 0.0; /* never -0.0 */
      }
    }
    free(e);
  }
  free(sc);
  free(pool);
  free(dom);
  fl_free(&fl);
  return g;
}

static gen_instance *random_network_common(int32_t n, int32_t dmin, int32_t dmax,
                                           int32_t nf, int32_t amin, int32_t amax,
                                           int is_f64, uint64_t *rs) {
  if (n < 1 || dmin < 1 || dmax < dmin || amin < 0 || amax < amin || amax > n) return NULL;
  int32_t *dom = (int32_t *)malloc(sizeof(int32_t) * n);
  for (int i = 0; i < n; i++) dom[i] = dmin + (int32_t)rand_below(rs, (uint64_t)(dmax - dmin + 1));
  fn_list fl = {0};
  int32_t *pool = (int32_t *)malloc(sizeof(int32_t) * n);
  for (int f = 0; f < nf; f++) {
    int a = amin + (int)rand_below(rs, (uint64_t)(amax - amin + 1));
    for (int i = 0; i < n; i++) pool[i] = i;
    for (int i = 0; i < a; i++) {
      int j = i + (int)rand_below(rs, (uint64_t)(n - i));
      int32_t t = pool[i];
      pool[i] = pool[j];
      pool[j] = t;
    }
    fl_push(&fl, a, pool);
  }
  gen_instance *g = assemble(n, dom, &fl, is_f64);
  free(pool);
  free(dom);
  fl_free(&fl);
  return g;
}

gen_instance *gen_random_network(int32_t n, int32_t dmin, int32_t dmax, int32_t nf,
                                 int32_t amin, int32_t amax, int32_t cmax, double p2,
                                 uint64_t seed) {
  uint64_t rs = mix_seed(seed, 0);
  gen_instance *g = random_network_common(n, dmin, dmax, nf, amin, amax, 0, &rs);
  if (g) fill_int_tables(g, cmax, p2, &rs);
  return g;
}

gen_instance *gen_random_network_f64(int32_t n, int32_t dmin, int32_t dmax, int32_t nf,
                                     int32_t amin, int32_t amax, double fmax, double p2,
                                     uint64_t seed) {
  uint64_t rs = mix_seed(seed, 0);
  gen_instance *g = random_network_common(n, dmin, dmax, nf, amin, amax, 1, &rs);
  if (g) fill_f64_tables(g, fmax, p2, &rs);
  return g;
}

void gen_free(gen_instance *g) {
  if (!g) return;
  free(g->dom);
  free(g->arity);
  free(g->scope_off);
  free(g->scopes);
  free(g->table_off);
  free(g->icost);
  free(g->fcost);
  free(g);
}
