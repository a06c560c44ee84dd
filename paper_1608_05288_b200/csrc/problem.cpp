// problem.cpp — problem creation, WCSP / UAI loaders, synthetic generation,
// evaluation.  WCSP model <X,D,C>, belief networks / MPE
// (P:347-392), file layouts from SPEC.md S:507-525.
#include <cerrno>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>

#include "common.h"
#include "gen.h"

namespace gbe {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
const char *last_error() { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// JSON (flat)

Json Json::parse(const char *text) {
  Json j;
  if (!text) return j;
  const char *s = text;
  auto ws = [&]() { while (*s == ' ' || *s == '\n' || *s == '\t' || *s == '\r') s++; };
  auto str = [&]() -> std::string {
    if (*s != '"') GBE_FAIL(GBE_E_INVALID, "json: expected string at offset %d", int(s - text));
    s++;
    std::string out;
    while (*s && *s != '"') {
      if (*s == '\\' && s[1]) s++;
      out.push_back(*s++);
    }
    if (*s != '"') GBE_FAIL(GBE_E_INVALID, "json: unterminated string");
    s++;
    return out;
  };
  ws();
  if (*s == 0) return j;
  if (*s != '{') GBE_FAIL(GBE_E_INVALID, "json: expected '{'");
  s++;
  ws();
  if (*s == '}') return j;
  while (true) {
    ws();
    std::string k = str();
    ws();
    if (*s != ':') GBE_FAIL(GBE_E_INVALID, "json: expected ':' after \"%s\"", k.c_str());
    s++;
    ws();
    std::string v;
    if (*s == '"') {
      v = str();
    } else {
      while (*s && *s != ',' && *s != '}' && *s != ' ' && *s != '\n') v.push_back(*s++);
      if (v.empty()) GBE_FAIL(GBE_E_INVALID, "json: empty value for \"%s\"", k.c_str());
    }
    j.kv[k] = v;
    ws();
    if (*s == ',') {
      s++;
      continue;
    }
    if (*s == '}') break;
    GBE_FAIL(GBE_E_INVALID, "json: expected ',' or '}' at offset %d", int(s - text));
  }
  return j;
}

int64_t Json::i(const std::string &k, int64_t def) const {
  auto it = kv.find(k);
  if (it == kv.end()) return def;
  char *end = nullptr;
  double v = std::strtod(it->second.c_str(), &end);
  if (end == it->second.c_str()) GBE_FAIL(GBE_E_INVALID, "json: \"%s\" is not a number", k.c_str());
  return (int64_t)v;
}
double Json::f(const std::string &k, double def) const {
  auto it = kv.find(k);
  if (it == kv.end()) return def;
  char *end = nullptr;
  double v = std::strtod(it->second.c_str(), &end);
  if (end == it->second.c_str()) GBE_FAIL(GBE_E_INVALID, "json: \"%s\" is not a number", k.c_str());
  return v;
}
std::string Json::s(const std::string &k, const std::string &def) const {
  auto it = kv.find(k);
  return it == kv.end() ? def : it->second;
}
bool Json::b(const std::string &k, bool def) const {
  auto it = kv.find(k);
  if (it == kv.end()) return def;
  return it->second == "true" || it->second == "1";
}

// ---------------------------------------------------------------------------
// creation + validation

std::shared_ptr<Problem> problem_create(int32_t n, const int32_t *dom, int32_t nf,
                                        const int32_t *arity, const int32_t *scopes,
                                        gbe_semiring sr, const void *costs) {
  if (n < 0 || nf < 0) GBE_FAIL(GBE_E_INVALID, "negative n or nf");
  if (sr != GBE_MINSUM_I32 && sr != GBE_MINSUM_F64) GBE_FAIL(GBE_E_INVALID, "unknown semiring");
  if ((n && !dom) || (nf && (!arity || !costs))) GBE_FAIL(GBE_E_INVALID, "null array");
  auto p = std::make_shared<Problem>();
  p->n = n;
  p->nf = nf;
  p->sr = sr;
  p->dom.assign(dom, dom + n);
  for (int v = 0; v < n; v++)
    if (dom[v] < 1 || dom[v] > GBE_MAX_DOMAIN)
      GBE_FAIL(GBE_E_INVALID, "variable %d: domain size %d outside [1,%d]", v, dom[v], GBE_MAX_DOMAIN);
  p->arity.assign(arity, arity + nf);
  p->scope_off.assign(nf + 1, 0);
  p->table_off.assign(nf + 1, 0);
  for (int f = 0; f < nf; f++) {
    if (arity[f] < 0) GBE_FAIL(GBE_E_INVALID, "function %d: negative arity", f);
    p->scope_off[f + 1] = p->scope_off[f] + arity[f];
  }
  p->scopes.assign(scopes, scopes + p->scope_off[nf]);
  std::vector<char> seen(n, 0);
  for (int f = 0; f < nf; f++) {
    int64_t cells = 1;
    const int32_t *sc = p->scope(f);
    for (int a = 0; a < arity[f]; a++) {
      if (sc[a] < 0 || sc[a] >= n) GBE_FAIL(GBE_E_INVALID, "function %d: variable id %d out of range", f, sc[a]);
      if (seen[sc[a]]) GBE_FAIL(GBE_E_INVALID, "function %d: duplicate scope variable %d", f, sc[a]);
      seen[sc[a]] = 1;
      cells *= dom[sc[a]];
      if (cells > (int64_t)1 << 40) GBE_FAIL(GBE_E_INVALID, "function %d: table too large", f);
    }
    for (int a = 0; a < arity[f]; a++) seen[sc[a]] = 0;
    p->table_off[f + 1] = p->table_off[f] + cells;
  }
  int64_t tot = p->table_off[nf];
  if (sr == GBE_MINSUM_I32) {
    const int32_t *c = (const int32_t *)costs;
    p->icost.assign(c, c + tot);
    int64_t maxsum = 0;
    for (int f = 0; f < nf; f++) {
      int64_t mx = 0;
      for (int64_t i = p->table_off[f]; i < p->table_off[f + 1]; i++) {
        int32_t &x = p->icost[i];
        if (x < 0) GBE_FAIL(GBE_E_INVALID, "function %d: negative cost %d", f, x);
        if (x >= kInfI32) {
          x = kInfI32;
          p->has_inf = true;
        } else if (x > mx) {
          mx = x;
        }
      }
      maxsum += mx;
    }
    // A9: exactness of saturating arithmetic needs finite sums < 2^30
    if (maxsum >= kInfI32)
      GBE_FAIL(GBE_E_INVALID, "sum of the largest finite costs (%lld) >= 2^30", (long long)maxsum);
    p->maxsum = maxsum;
  } else {
    const double *c = (const double *)costs;
    p->fcost.assign(c, c + tot);
    for (int64_t i = 0; i < tot; i++)
      if (std::isnan(p->fcost[i])) GBE_FAIL(GBE_E_INVALID, "NaN cost at flat index %lld", (long long)i);
  }
  return p;
}

// ---------------------------------------------------------------------------
// WCSP text

namespace {
struct LineReader {
  std::ifstream in;
  int line = 0;
  std::vector<std::string> next(const char *what) {
    std::string s;
    while (std::getline(in, s)) {
      line++;
      std::istringstream is(s);
      std::vector<std::string> tok;
      std::string t;
      while (is >> t) tok.push_back(t);
      if (!tok.empty()) return tok;
    }
    GBE_FAIL(GBE_E_PARSE, "line %d: unexpected end of file (expected %s)", line + 1, what);
  }
};

int64_t to_i64(const std::string &t, int line) {
  char *end = nullptr;
  errno = 0;
  long long v = std::strtoll(t.c_str(), &end, 10);
  if (*end || errno) GBE_FAIL(GBE_E_PARSE, "line %d: bad integer '%s'", line, t.c_str());
  return v;
}
}  // namespace

std::shared_ptr<Problem> problem_load_wcsp(const char *path) {
  LineReader r;
  r.in.open(path);
  if (!r.in) GBE_FAIL(GBE_E_PARSE, "cannot open '%s'", path ? path : "(null)");
  auto h = r.next("header");
  if (h.size() < 5) GBE_FAIL(GBE_E_PARSE, "line %d: header needs 'name n maxdom nf ub'", r.line);
  int64_t n = to_i64(h[1], r.line), nf = to_i64(h[3], r.line), ub = to_i64(h[4], r.line);
  if (n < 0 || nf < 0 || n > (1 << 24)) GBE_FAIL(GBE_E_PARSE, "line %d: bad sizes", r.line);
  std::vector<int32_t> dom;
  while ((int64_t)dom.size() < n) {
    auto t = r.next("domain sizes");
    for (auto &x : t) dom.push_back((int32_t)to_i64(x, r.line));
  }
  if ((int64_t)dom.size() != n) GBE_FAIL(GBE_E_PARSE, "line %d: %zu domain sizes for n=%lld", r.line, dom.size(), (long long)n);
  std::vector<int32_t> arity, scopes, costs;
  for (int64_t f = 0; f < nf; f++) {
    auto t = r.next("function header");
    int64_t a = to_i64(t[0], r.line);
    if (a < 0 || (int64_t)t.size() != a + 3)
      GBE_FAIL(GBE_E_PARSE, "line %d: function header needs 'arity vars... default ntuples'", r.line);
    std::vector<int32_t> sc;
    int64_t cells = 1;
    for (int64_t q = 0; q < a; q++) {
      int64_t v = to_i64(t[1 + q], r.line);
      if (v < 0 || v >= n) GBE_FAIL(GBE_E_PARSE, "line %d: variable %lld out of range", r.line, (long long)v);
      sc.push_back((int32_t)v);
      cells *= dom[v];
    }
    int64_t def = to_i64(t[a + 1], r.line), nt = to_i64(t[a + 2], r.line);
    auto clampc = [&](int64_t c) -> int32_t { return c >= ub ? kInfI32 : (int32_t)std::min<int64_t>(c, kInfI32); };
    std::vector<int32_t> tab(cells, clampc(def));
    for (int64_t k = 0; k < nt; k++) {
      auto u = r.next("tuple");
      if ((int64_t)u.size() != a + 1) GBE_FAIL(GBE_E_PARSE, "line %d: tuple needs %lld values and a cost", r.line, (long long)a);
      int64_t idx = 0;
      for (int64_t q = 0; q < a; q++) {
        int64_t val = to_i64(u[q], r.line);
        if (val < 0 || val >= dom[sc[q]]) GBE_FAIL(GBE_E_PARSE, "line %d: value %lld outside domain", r.line, (long long)val);
        idx = idx * dom[sc[q]] + val;
      }
      tab[idx] = clampc(to_i64(u[a], r.line));
    }
    arity.push_back((int32_t)a);
    scopes.insert(scopes.end(), sc.begin(), sc.end());
    costs.insert(costs.end(), tab.begin(), tab.end());
  }
  return problem_create((int32_t)n, dom.data(), (int32_t)nf, arity.data(), scopes.data(),
                        GBE_MINSUM_I32, costs.data());
}

// ---------------------------------------------------------------------------
// UAI: probabilities stored as -log p

std::shared_ptr<Problem> problem_load_uai(const char *model, const char *evid) {
  std::ifstream in(model ? model : "");
  if (!in) GBE_FAIL(GBE_E_PARSE, "cannot open '%s'", model ? model : "(null)");
  // token stream with line numbers
  std::vector<std::pair<std::string, int>> tok;
  {
    std::string s;
    int line = 0;
    while (std::getline(in, s)) {
      line++;
      std::istringstream is(s);
      std::string t;
      while (is >> t) tok.push_back({t, line});
    }
  }
  size_t k = 0;
  auto next = [&](const char *what) -> std::pair<std::string, int> {
    if (k >= tok.size()) GBE_FAIL(GBE_E_PARSE, "unexpected end of file (expected %s)", what);
    return tok[k++];
  };
  auto h = next("BAYES|MARKOV");
  if (h.first != "BAYES" && h.first != "MARKOV") GBE_FAIL(GBE_E_PARSE, "line %d: expected BAYES or MARKOV", h.second);
  auto nt = next("n");
  int64_t n = to_i64(nt.first, nt.second);
  std::vector<int32_t> dom(n);
  for (int64_t v = 0; v < n; v++) {
    auto t = next("domain");
    dom[v] = (int32_t)to_i64(t.first, t.second);
  }
  auto ft = next("nf");
  int64_t nf = to_i64(ft.first, ft.second);
  std::vector<int32_t> arity(nf), scopes;
  for (int64_t f = 0; f < nf; f++) {
    auto t = next("arity");
    arity[f] = (int32_t)to_i64(t.first, t.second);
    for (int q = 0; q < arity[f]; q++) {
      auto u = next("scope variable");
      int64_t v = to_i64(u.first, u.second);
      if (v < 0 || v >= n) GBE_FAIL(GBE_E_PARSE, "line %d: variable %lld out of range", u.second, (long long)v);
      scopes.push_back((int32_t)v);
    }
  }
  std::vector<double> costs;
  size_t so = 0;
  for (int64_t f = 0; f < nf; f++) {
    int64_t cells = 1;
    for (int q = 0; q < arity[f]; q++) cells *= dom[scopes[so + q]];
    so += arity[f];
    auto t = next("table size");
    if (to_i64(t.first, t.second) != cells) GBE_FAIL(GBE_E_PARSE, "line %d: table size mismatch", t.second);
    for (int64_t c = 0; c < cells; c++) {
      auto u = next("probability");
      char *end = nullptr;
      double pr = std::strtod(u.first.c_str(), &end);
      if (*end || pr < 0 || std::isnan(pr)) GBE_FAIL(GBE_E_PARSE, "line %d: bad probability '%s'", u.second, u.first.c_str());
      double nl = pr > 0 ? -std::log(pr) : std::numeric_limits<double>::infinity();
      costs.push_back(nl > 0 ? nl : 0.0);
    }
  }
  // evidence: condition by a hard unary constraint (0 at the observed value,
  // +inf elsewhere) -- MPE given E (Eq. 2)
  if (evid) {
    std::ifstream ev(evid);
    if (!ev) GBE_FAIL(GBE_E_PARSE, "cannot open evidence '%s'", evid);
    std::vector<int64_t> e;
    int64_t x;
    while (ev >> x) e.push_back(x);
    if (e.empty()) GBE_FAIL(GBE_E_PARSE, "empty evidence file");
    int64_t cnt = e[0];
    if ((int64_t)e.size() < 1 + 2 * cnt) GBE_FAIL(GBE_E_PARSE, "evidence: expected %lld pairs", (long long)cnt);
    for (int64_t i = 0; i < cnt; i++) {
      int64_t v = e[1 + 2 * i], val = e[2 + 2 * i];
      if (v < 0 || v >= n) GBE_FAIL(GBE_E_INVALID, "evidence variable %lld out of range", (long long)v);
      if (val < 0 || val >= dom[v]) GBE_FAIL(GBE_E_INVALID, "evidence value %lld outside the domain of %lld", (long long)val, (long long)v);
      arity.push_back(1);
      scopes.push_back((int32_t)v);
      for (int c = 0; c < dom[v]; c++) costs.push_back(c == val ? 0.0 : std::numeric_limits<double>::infinity());
    }
  }
  return problem_create((int32_t)n, dom.data(), (int32_t)arity.size(), arity.data(), scopes.data(),
                        GBE_MINSUM_F64, costs.data());
}

// ---------------------------------------------------------------------------
// synthetic instances through the shared generator module gen/

std::shared_ptr<Problem> problem_generate(const char *json) {
  Json j = Json::parse(json);
  std::string topo = j.s("topology", "");
  uint64_t seed = (uint64_t)j.i("seed", 0);
  double p2 = j.f("p2", 0.0);
  gen_instance *g = nullptr;
  if (topo == "random")
    g = gen_random_graph((int32_t)j.i("n", 10), (int32_t)j.i("d", 3), j.i("edges", 10),
                         (int32_t)j.i("mode", 0), p2, seed);
  else if (topo == "scalefree")
    g = gen_scalefree((int32_t)j.i("n", 10), (int32_t)j.i("d", 3), p2, seed);
  else if (topo == "grid")
    g = gen_grid((int32_t)j.i("rows", 10), (int32_t)j.i("cols", 10), (int32_t)j.i("d", 3), p2, seed);
  else if (topo == "bn")
    g = gen_belief_net((int32_t)j.i("n", 10), (int32_t)j.i("dmin", 2), (int32_t)j.i("dmax", 4),
                       (int32_t)j.i("maxpar", 3), (int32_t)j.i("window", 20), seed);
  else if (topo == "network")
    g = gen_random_network((int32_t)j.i("n", 10), (int32_t)j.i("dmin", 2), (int32_t)j.i("dmax", 4),
                           (int32_t)j.i("nf", 10), (int32_t)j.i("amin", 1), (int32_t)j.i("amax", 3),
                           (int32_t)j.i("cmax", 100), p2, seed);
  else
    GBE_FAIL(GBE_E_INVALID, "generate: unknown topology '%s'", topo.c_str());
  if (!g) GBE_FAIL(GBE_E_INVALID, "generate: infeasible parameters for '%s'", topo.c_str());
  std::shared_ptr<Problem> p;
  try {
    p = problem_create(g->n, g->dom, g->nf, g->arity, g->scopes,
                       g->is_f64 ? GBE_MINSUM_F64 : GBE_MINSUM_I32,
                       g->is_f64 ? (const void *)g->fcost : (const void *)g->icost);
  } catch (...) {
    gen_free(g);
    throw;
  }
  gen_free(g);
  return p;
}

// ---------------------------------------------------------------------------
// evaluate (Eq. 1)

gbe_value problem_evaluate(const Problem &p, const int32_t *assign) {
  for (int v = 0; v < p.n; v++)
    if (assign[v] < 0 || assign[v] >= p.dom[v])
      GBE_FAIL(GBE_E_INVALID, "assignment of variable %d (%d) outside its domain", v, assign[v]);
  gbe_value out{0, 0, 0.0};
  if (p.is_f64()) {
    double s = 0.0;
    for (int f = 0; f < p.nf; f++) {
      int64_t idx = 0;
      const int32_t *sc = p.scope(f);
      for (int a = 0; a < p.arity[f]; a++) idx = idx * p.dom[sc[a]] + assign[sc[a]];
      s = s + p.fcost[p.table_off[f] + idx];
    }
    out.f = s;
    out.is_inf = std::isinf(s) ? 1 : 0;
  } else {
    int64_t s = 0;
    for (int f = 0; f < p.nf; f++) {
      int64_t idx = 0;
      const int32_t *sc = p.scope(f);
      for (int a = 0; a < p.arity[f]; a++) idx = idx * p.dom[sc[a]] + assign[sc[a]];
      s = std::min<int64_t>(s + p.icost[p.table_off[f] + idx], kInfI32);
    }
    out.i = s;
    out.is_inf = s >= kInfI32 ? 1 : 0;
  }
  return out;
}

}  // namespace gbe
