// kernels.h — host-side launchers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <tuple>
#include <utility>
#include <vector>

#include "gbe.h"

namespace gbe {

struct InPtrs {
  const void *p[GBE_MAX_INPUTS];
};

// Value-phase program (Alg. 1 lines 6-7; MBE reading A7)
struct VStep {
  int32_t var;      // variable assigned by this step
  int32_t kind;     // 0: argmin lookup in `ptr` (uint8); 1: member sum
  int32_t d;        // domain size of var
  int32_t nterm;    // kind 0: row terms
  int64_t term_off; // kind 0: first VTerm
  int64_t lo, hi;   // kind 0: rows held locally [lo, hi) (row sharding)
  const void *ptr;  // kind 0: argmin table (first local row)
  int32_t nmem;     // kind 1: members
  int32_t pad;
  int64_t mem_off;  // kind 1: first VMember
};
struct VMember {
  const void *ptr;  // member table (scope ascending by position, var last)
  int64_t term_off; // first VTerm
  int32_t nterm;
  int32_t pad;
};
struct VTerm {
  int32_t var;
  int32_t pad;
  int64_t stride;
};

// Kernel variants for the fused aggregate+project bucket kernel (BK)
enum BkVariant { BK_AUTO = -1, BK_GENERIC = 0 };

// Tile enumeration order of a full-range launch (host): the high output
// digits p[0..n) are reordered so that the digits an input lacks vary
// fastest, the largest input first: tiles that re-read one slice of an input
// run back to back, so its re-reads hit L2 instead of HBM.  Lexicographic
// over the inputs by decreasing size (a digit the largest input lacks goes
// after one it has; ties by the next input; stable), so a bucket with
// several large inputs that lack different digits gets L2 reuse for all of
// them (with only the largest input's digits moved, C4-d4's x0 re-read its
// two other 1e9-cell inputs from HBM 16-64 times).
inline void order_high_digits(const gbe_bucket_desc &h, int *p, int n) {
  const int k = h.ninputs, m = h.nsep;
  // rank: mode 0 (default) by size; mode 1: the inputs of >= 16 MB by the
  // re-use factor of their slices over the high digits (product of the
  // radices of the high digits they lack) -- their re-reads then happen
  // within the fewest tiles -- then the rest by size (GBE_TILE_ORDER: knob)
  static const int mode = [] {
    const char *e = std::getenv("GBE_TILE_ORDER");
    return e ? std::atoi(e) : 0;
  }();
  const double es = h.semiring == GBE_MINSUM_I32 ? 4.0 : 8.0;
  std::vector<std::tuple<int, double, double, int>> by;  // (group, -reuse, -cells, j)
  for (int j = 0; j < k; j++) {
    double c = h.d, reuse = 1;
    for (int q = 0; q < m; q++) {
      if (h.stride[j][q]) c *= h.radix[q];
    }
    for (int i = 0; i < n; i++)
      if (!h.stride[j][p[i]]) reuse *= h.radix[p[i]];
    const bool large = c * es >= 16.0 * (1 << 20);
    if (mode == 1)
      by.emplace_back(large ? 0 : 1, large ? -reuse : 0.0, -c, j);
    else
      by.emplace_back(0, 0.0, -c, j);
  }
  std::stable_sort(by.begin(), by.end());
  std::stable_sort(p, p + n, [&](int a, int b) {
    for (auto &e : by) {
      const int j = std::get<3>(e);
      const bool la = h.stride[j][a] == 0, lb = h.stride[j][b] == 0;
      if (la != lb) return lb;  // a before b when only b is lacked (b varies faster)
    }
    return false;
  });
}

// Describes how the launcher tiles one bucket (computed on the host from the
// descriptor; see kernels.cu).
struct BkLaunchInfo {
  int variant;
  int nlow, plow;  // low digits per tile, rows per tile
  int grid, block;
  size_t smem;
};

BkLaunchInfo bk_plan_launch(const gbe_bucket_desc &h, int64_t row_begin, int64_t row_end,
                            int variant, int num_sms);

// dev_desc: device copy of `h` (the launcher reads scalars from `h`).
cudaError_t bk_launch(const gbe_bucket_desc &h, const gbe_bucket_desc *dev_desc,
                      const InPtrs &in, void *out, uint8_t *arg, int64_t row_begin,
                      int64_t row_end, const BkLaunchInfo &li, cudaStream_t stream);

// Counting bucket, (min, count) semiring:
// bk_generic's tiling; cin.p[j] = count table of input j (nullptr: every
// entry 1).  cnt[r] = number of completions attaining out[r] (0 if infinite);
// consistent: every finite entry reads as cost 0.
cudaError_t bk_count_launch(const gbe_bucket_desc &h, const gbe_bucket_desc *dev_desc, const InPtrs &in,
                            const InPtrs &cin, void *out, double *cnt, uint8_t *arg, int64_t row_begin,
                            int64_t row_end, bool consistent, cudaStream_t stream);
// count = prod of the n constant counts cc[k][0] (nullptr: 1), 0 if some
// constant cptrs[k][0] is infinite; consistent: *optimum = 0 or INF.
cudaError_t count_total_launch(bool f64, const void *const *cptrs, const double *const *cc, int n,
                               bool consistent, void *optimum, double *count, cudaStream_t stream);

// Relayout of the original tables from declared to sorted scope order
// (P:624): for each function f, out[off[f] + i] = in[off[f] + sum_q
// digit_q(i) * pstride[poff[f] + q]] with digits over radices prad.
cudaError_t relayout_launch(const void *in, void *out, int elem, int nf, const int64_t *off,
                            const int32_t *poff, const int32_t *prad, const int32_t *pstride,
                            cudaStream_t stream);

// Value phase over steps [s0, s1); single warp.  If gvar >= 0 the kernel
// first sets assign[gvar] = max(gathered[0..W)).  If nconst >= 0 it first
// sums the nconst constants (canonical order) into *optimum.
cudaError_t value_launch(bool f64, const VStep *steps, int s0, int s1, const VMember *mems,
                         const VTerm *terms, int32_t *assign, const int32_t *gathered, int gvar,
                         int W, const void *const *cptrs, int nconst, void *optimum,
                         cudaStream_t stream);

}  // namespace gbe
