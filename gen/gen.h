/* gen.h — seeded synthetic instance generators shared by the oracle and the
 * CUDA path.
 *
 * This module holds NO arithmetic of the method (no ordering, no bucket,
 * no aggregation/elimination).  It only draws graphs and cost tables with a
 * counter-based generator (splitmix64), so the oracle (oracle/) and the
 * product library (paper_1608_05288_b200/csrc) can consume byte-identical
 * inputs without sharing any method code.
 *
 * Topologies follow the paper's instance description, §8.1
 * (P:919-929): random, scale-free Barabasi-Albert, grid
 * (P:926); integer costs uniform in [0,100], a fraction p2 of the cells set to
 * "infinity".  Belief networks (§3) carry CPTs
 * stored as -log p in float64 (reading A10).
 *
 * Table layout: every function's table is stored in DECLARED scope order,
 * lexicographic, first scope variable most significant (§6.1
 * P:553-554).  Integer infinity is GEN_INF_I32 = 2^30 (reading A9).
 */
#ifndef GBE_GEN_H
#define GBE_GEN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GEN_INF_I32 (1 << 30)

typedef struct gen_instance {
  int32_t n;          /* number of variables                              */
  int32_t nf;         /* number of functions                              */
  int32_t is_f64;     /* 0: int32 costs in icost; 1: f64 costs in fcost   */
  int32_t *dom;       /* [n] domain sizes                                 */
  int32_t *arity;     /* [nf]                                             */
  int64_t *scope_off; /* [nf+1] offsets into scopes                       */
  int32_t *scopes;    /* [scope_off[nf]] variable ids, declared order     */
  int64_t *table_off; /* [nf+1] offsets into icost/fcost                  */
  int32_t *icost;     /* [table_off[nf]] or NULL                          */
  double *fcost;      /* [table_off[nf]] or NULL                          */
} gen_instance;

/* Random graph with exactly `nedges` distinct edges drawn uniformly among all
 * pairs, resampled (sub-seed +1) until connected.
 * mode 0: uniform pairs; mode 1: uniform random spanning tree (Pruefer code)
 * plus (nedges - (n-1)) uniform extra edges.  Returns NULL on failure. */
gen_instance *gen_random_graph(int32_t n, int32_t d, int64_t nedges, int32_t mode,
                               double p2, uint64_t seed);

/* Barabasi-Albert scale-free graph: start from a connected 2-node
 * network, add each new node with m=2 edges to distinct existing nodes chosen
 * with probability proportional to degree; 2(n-2)+1 edges in total. */
gen_instance *gen_scalefree(int32_t n, int32_t d, double p2, uint64_t seed);

/* rows x cols 4-neighbour lattice. Variable id = r*cols + c. */
gen_instance *gen_grid(int32_t rows, int32_t cols, int32_t d, double p2,
                       uint64_t seed);

/* Belief network in topological order 0..n-1: domains iid
 * U{dmin..dmax}; variable v gets min(maxpar, v, window) distinct parents drawn
 * uniformly from the `window` preceding variables; one CPT per variable with
 * declared scope (parents ascending..., v); each CPT row ~ Dirichlet(1),
 * stored as -log p in float64. */
gen_instance *gen_belief_net(int32_t n, int32_t dmin, int32_t dmax, int32_t maxpar,
                             int32_t window, uint64_t seed);

/* General random cost network for unit tests: n variables with domains iid
 * U{dmin..dmax}, nf functions with arity iid U{amin..amax} (distinct random
 * variables, random declared order), integer costs U[0,cmax], floor(p2*cells)
 * infinite cells.  No connectivity guarantee. */
gen_instance *gen_random_network(int32_t n, int32_t dmin, int32_t dmax, int32_t nf,
                                 int32_t amin, int32_t amax, int32_t cmax,
                                 double p2, uint64_t seed);

/* Same as gen_random_network but float64 costs uniform in [0, fmax) with
 * floor(p2*cells) +inf cells. */
gen_instance *gen_random_network_f64(int32_t n, int32_t dmin, int32_t dmax,
                                     int32_t nf, int32_t amin, int32_t amax,
                                     double fmax, double p2, uint64_t seed);

void gen_free(gen_instance *g);

/* splitmix64 counter-based generator, exported so tests can draw the same
 * streams (e.g. random assignments) on either side. */
uint64_t gen_splitmix64(uint64_t *state);

#ifdef __cplusplus
}
#endif
#endif
