// kernels.cu — sm_100a kernels of the bucket (UTIL-message) computation.
//
// BK fuses Gpu::Aggregate (Proc. 4) and Gpu::Eliminate (Proc. 5,
// P:781-792): for each output row r of a (mini-)bucket and each value v of
// the eliminated variable, s_v = (+)_j T_j[off_j(r) + v]; out[r] = min_v s_v,
// arg[r] = first minimiser (A8).  The d^{|sep|+1} aggregated table of the
// paper is never materialised.  off_j(r) restates the index map Eq.
// as precomputed per-input strides ("mul/div/mod").
//
// Semirings: int32 min-sum with INF = 2^30 and clamp after every add (A9);
// float64 min-sum (MPE on -log p, A10), inputs added in canonical order;
// float64 sum-product: the same sums, eliminated by
// -log sum_v exp(-s_v) (online log-sum-exp over v), arg = 0.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "kernels.h"

namespace gbe {
namespace {

constexpr uint32_t kInf = GBE_INF_I32;

// ---------------------------------------------------------------------------
// semiring traits

template <typename T>
struct Sr;

template <>
struct Sr<int32_t> {
  using Acc = uint32_t;  // a, b <= 2^30 -> a + b <= 2^31: no wrap
  __device__ __forceinline__ static Acc zero() { return 0u; }
  __device__ __forceinline__ static Acc load(const int32_t *p, int64_t i) {
    return (uint32_t)__ldg(p + i);
  }
  __device__ __forceinline__ static Acc add(Acc a, Acc b) {
    uint32_t s = a + b;
    return s < kInf ? s : kInf;
  }
  __device__ __forceinline__ static int32_t out(Acc a) { return (int32_t)a; }
};

template <>
struct Sr<double> {
  using Acc = double;
  __device__ __forceinline__ static Acc zero() { return 0.0; }
  __device__ __forceinline__ static Acc load(const double *p, int64_t i) { return __ldg(p + i); }
  __device__ __forceinline__ static Acc add(Acc a, Acc b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double out(Acc a) { return a; }
  __device__ __forceinline__ static double inf() { return __longlong_as_double(0x7ff0000000000000LL); }
};

// Element offset in input j of the first row of tile t: the mixed-radix
// digits of t over the high output digits [0, nhigh) times the input's
// strides.  32-bit division when the tile index fits (every practical
// launch: the serial 64-bit div/mod chain dominated large d = 1 merges).
__device__ __forceinline__ int64_t tile_base(const gbe_bucket_desc *__restrict__ D, int j, int64_t t, int nhigh) {
  int64_t o = 0;
  if (t < ((int64_t)1 << 32)) {
    uint32_t rem = (uint32_t)t;
    for (int q = nhigh - 1; q >= 0 && rem; q--) {
      const uint32_t r = (uint32_t)D->radix[q], qt = rem / r;
      o += (int64_t)(rem - qt * r) * D->stride[j][q];
      rem = qt;
    }
  } else {
    int64_t rem = t;
    for (int q = nhigh - 1; q >= 0; q--) {
      const int r = D->radix[q];
      o += (rem % r) * D->stride[j][q];
      rem /= r;
    }
  }
  return o - D->shift[j];
}

// ---------------------------------------------------------------------------
// BK generic: tiles of `plow` consecutive rows (= all values of the `nlow`
// least-significant output digits).  Per CTA: the low-digit offsets of every
// input are built once in shared memory; per tile: one base offset per input
// from the high digits.  Per row: k shared-memory offsets + k*d loads.

template <typename T, bool SP>
__global__ void __launch_bounds__(256) bk_generic(const gbe_bucket_desc *__restrict__ D,
                                                  InPtrs in, T *__restrict__ out,
                                                  uint8_t *__restrict__ arg, int64_t row_begin,
                                                  int64_t row_end, int nlow, int plow) {
  using S = Sr<T>;
  using Acc = typename S::Acc;
  extern __shared__ int32_t loff[];  // [k][plow]
  __shared__ int64_t base[GBE_MAX_INPUTS];
  const int m = D->nsep, k = D->ninputs, d = D->d;
  for (int idx = threadIdx.x; idx < k * plow; idx += blockDim.x) {
    int j = idx / plow, l = idx - j * plow;
    int64_t o = 0;
    for (int q = m - 1; q >= m - nlow; q--) {
      int r = D->radix[q];
      o += (int64_t)(l % r) * D->stride[j][q];
      l /= r;
    }
    loff[idx] = (int32_t)o;
  }
  const int64_t t0 = row_begin / plow, t1 = (row_end - 1) / plow;
  for (int64_t t = t0 + blockIdx.x; t <= t1; t += gridDim.x) {
    __syncthreads();
    if (threadIdx.x < k) base[threadIdx.x] = tile_base(D, threadIdx.x, t, m - nlow);
    __syncthreads();
    for (int l = threadIdx.x; l < plow; l += blockDim.x) {
      int64_t r = t * plow + l;
      if (r < row_begin || r >= row_end) continue;
      Acc best = S::zero();
      int bv = 0;
      double z = 0.0;  // SP: sum_v exp(best - s_v), rescaled whenever best drops
      for (int v = 0; v < d; v++) {
        Acc s = S::zero();
        for (int j = 0; j < k; j++)
          s = S::add(s, S::load((const T *)in.p[j], base[j] + loff[j * plow + l] + v));
        if constexpr (SP) {
          if (v == 0 || s < best) {
            z = (v == 0 || best == Sr<double>::inf()) ? 1.0 : z * exp((double)s - (double)best) + 1.0;
            best = s;
          } else if (s < Sr<double>::inf()) {
            z += exp((double)best - (double)s);
          }
        } else if (v == 0 || s < best) {
          best = s;
          bv = v;
        }
      }
      if constexpr (SP) {
        if ((double)best < Sr<double>::inf()) best = (Acc)((double)best - log(z));
      }
      out[r - row_begin] = S::out(best);
      if (arg) arg[r - row_begin] = (uint8_t)bv;
    }
  }
}

// ---------------------------------------------------------------------------
// Counting bucket ("as a byproduct ... BE can
// compute the number of consistent solutions"): the (min, count) semiring.
// Same tiling and index maps as bk_generic; every message input j also has a
// count table cin.p[j] (nullptr for an original function: count 1).  For
// theta.v: s_v = the saturating / IEEE sum of the inputs (CONS: every finite
// entry read as 0), c_v = prod_j count_j (input order); the row keeps
// out = min_v s_v, arg = first minimiser (A8) and cnt = sum of c_v over the v
// attaining the minimum in ascending v (0 when the minimum is infinite).

template <typename T, bool CONS>
__global__ void __launch_bounds__(256) bk_count(const gbe_bucket_desc *__restrict__ D, InPtrs in,
                                                InPtrs cin, T *__restrict__ out,
                                                double *__restrict__ cnt, uint8_t *__restrict__ arg,
                                                int64_t row_begin, int64_t row_end, int nlow, int plow) {
  using S = Sr<T>;
  using Acc = typename S::Acc;
  extern __shared__ int32_t loff[];  // [k][plow]
  __shared__ int64_t base[GBE_MAX_INPUTS];
  const int m = D->nsep, k = D->ninputs, d = D->d;
  for (int idx = threadIdx.x; idx < k * plow; idx += blockDim.x) {
    int j = idx / plow, l = idx - j * plow;
    int64_t o = 0;
    for (int q = m - 1; q >= m - nlow; q--) {
      int r = D->radix[q];
      o += (int64_t)(l % r) * D->stride[j][q];
      l /= r;
    }
    loff[idx] = (int32_t)o;
  }
  const int64_t t0 = row_begin / plow, t1 = (row_end - 1) / plow;
  for (int64_t t = t0 + blockIdx.x; t <= t1; t += gridDim.x) {
    __syncthreads();
    if (threadIdx.x < k) base[threadIdx.x] = tile_base(D, threadIdx.x, t, m - nlow);
    __syncthreads();
    for (int l = threadIdx.x; l < plow; l += blockDim.x) {
      int64_t r = t * plow + l;
      if (r < row_begin || r >= row_end) continue;
      Acc best = S::zero();
      double bc = 0.0;
      int bv = 0;
      for (int v = 0; v < d; v++) {
        Acc s = S::zero();
        double c = 1.0;
        for (int j = 0; j < k; j++) {
          const int64_t i = base[j] + loff[j * plow + l] + v;
          Acc x = S::load((const T *)in.p[j], i);
          if constexpr (CONS) {
            if constexpr (sizeof(T) == 4)
              x = x < kInf ? 0u : kInf;
            else
              x = x < Sr<double>::inf() ? 0.0 : Sr<double>::inf();
          }
          s = S::add(s, x);
          if (cin.p[j]) c = c * __ldg((const double *)cin.p[j] + i);
        }
        if (v == 0 || s < best) {
          best = s;
          bv = v;
          bc = c;
        } else if (s == best) {
          bc = bc + c;
        }
      }
      bool inf;
      if constexpr (sizeof(T) == 4)
        inf = (uint32_t)best >= kInf;
      else
        inf = !((double)best < Sr<double>::inf());
      out[r - row_begin] = S::out(best);
      cnt[r - row_begin] = inf ? 0.0 : bc;
      if (arg) arg[r - row_begin] = (uint8_t)bv;
    }
  }
}

// number of solutions = product of the constant messages' counts (the
// components multiply; an original constant counts 1), 0 if the optimum is
// infinite.  CONS: the reported value is 0 (or INF) -- every finite cost
// reads as 0.
template <typename T>
__global__ void count_total_kernel(const void *const *cptrs, const double *const *cc, int n, int cons,
                                   T *optimum, double *count) {
  double c = 1.0;
  bool inf = false;
  for (int k = 0; k < n; k++) {
    if (cc[k]) c = c * cc[k][0];
    const T x = ((const T *)cptrs[k])[0];
    if constexpr (sizeof(T) == 4)
      inf = inf || (uint32_t)x >= kInf;
    else
      inf = inf || !(x < Sr<double>::inf());
  }
  if (cons) {
    if constexpr (sizeof(T) == 4)
      *optimum = inf ? (T)kInf : (T)0;
    else
      *optimum = inf ? Sr<double>::inf() : 0.0;
  }
  *count = inf ? 0.0 : c;
}

// ---------------------------------------------------------------------------
// relayout of the original tables (declared -> ascending position order)

template <typename T>
__global__ void relayout_kernel(const T *__restrict__ in, T *__restrict__ out, int nf,
                                const int64_t *__restrict__ off, const int32_t *__restrict__ poff,
                                const int32_t *__restrict__ prad,
                                const int32_t *__restrict__ pstride) {
  for (int f = blockIdx.x; f < nf; f += gridDim.x) {
    const int64_t a = off[f], cells = off[f + 1] - a;
    const int q0 = poff[f], ar = poff[f + 1] - q0;
    for (int64_t i = threadIdx.x; i < cells; i += blockDim.x) {
      int64_t rem = i, src = 0;
      for (int q = ar - 1; q >= 0; q--) {
        int r = prad[q0 + q];
        src += (rem % r) * pstride[q0 + q];
        rem /= r;
      }
      out[a + i] = in[a + src];
    }
  }
}

// ---------------------------------------------------------------------------
// value phase: one warp walks the forward order

template <typename T>
__global__ void value_kernel(const VStep *__restrict__ steps, int s0, int s1,
                             const VMember *__restrict__ mems, const VTerm *__restrict__ terms,
                             int32_t *assign, const int32_t *__restrict__ gathered, int gvar, int W,
                             const void *const *__restrict__ cptrs, int nconst, T *optimum) {
  using S = Sr<T>;
  using Acc = typename S::Acc;
  const int lane = threadIdx.x;
  if (lane == 0) {
    if (nconst >= 0) {  // optimum = sum of the constants
      Acc s = S::zero();
      for (int c = 0; c < nconst; c++) s = S::add(s, S::load((const T *)cptrs[c], 0));
      *optimum = S::out(s);
    }
    if (gvar >= 0) {
      int v = -1;
      for (int w = 0; w < W; w++) v = max(v, gathered[w]);
      assign[gvar] = v;
    }
  }
  __syncwarp();
  for (int si = s0; si < s1; si++) {
    const VStep st = steps[si];
    if (st.kind == 0) {
      if (lane == 0) {
        int64_t row = 0;
        for (int q = 0; q < st.nterm; q++) row += (int64_t)assign[terms[st.term_off + q].var] * terms[st.term_off + q].stride;
        assign[st.var] = (row >= st.lo && row < st.hi) ? (int)((const uint8_t *)st.ptr)[row - st.lo] : -1;
      }
    } else {
      Acc best = S::zero();
      int bv = 1 << 30;
      for (int v = lane; v < st.d; v += 32) {
        Acc s = S::zero();
        for (int mi = 0; mi < st.nmem; mi++) {
          const VMember mm = mems[st.mem_off + mi];
          int64_t b = 0;
          for (int q = 0; q < mm.nterm; q++) b += (int64_t)assign[terms[mm.term_off + q].var] * terms[mm.term_off + q].stride;
          s = S::add(s, S::load((const T *)mm.ptr, b + v));
        }
        if (bv == (1 << 30) || s < best) {
          best = s;
          bv = v;
        }
      }
      // lexicographic (value, index) min over the warp
      for (int o = 16; o > 0; o >>= 1) {
        Acc ob = __shfl_down_sync(0xffffffffu, best, o);
        int ov = __shfl_down_sync(0xffffffffu, bv, o);
        if (ov != (1 << 30) && (bv == (1 << 30) || ob < best || (!(best < ob) && ov < bv))) {
          best = ob;
          bv = ov;
        }
      }
      if (lane == 0) assign[st.var] = bv;
    }
    __syncwarp();
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers

BkLaunchInfo bk_plan_launch(const gbe_bucket_desc &h, int64_t row_begin, int64_t row_end,
                            int variant, int num_sms) {
  BkLaunchInfo li{};
  li.variant = BK_GENERIC;
  const int k = h.ninputs > 0 ? h.ninputs : 1;
  const int plow_max = std::max(1, std::min(1024, 12288 / k));  // <= 48 KB smem
  int nlow = 0, plow = 1;
  // the per-CTA low-digit offsets are int32: stop before any input's largest
  // in-tile offset reaches 2^31 (only arbitrary strides of the bare primitive)
  std::vector<int64_t> maxoff(k, 0);
  while (nlow < h.nsep && (int64_t)plow * h.radix[h.nsep - 1 - nlow] <= plow_max) {
    const int q = h.nsep - 1 - nlow;
    bool fits = true;
    for (int j = 0; j < h.ninputs; j++)
      if (maxoff[j] + (int64_t)(h.radix[q] - 1) * h.stride[j][q] >= (int64_t(1) << 31)) fits = false;
    if (!fits) break;
    for (int j = 0; j < h.ninputs; j++) maxoff[j] += (int64_t)(h.radix[q] - 1) * h.stride[j][q];
    plow *= h.radix[q];
    nlow++;
  }
  li.nlow = nlow;
  li.plow = plow;
  li.block = plow >= 256 ? 256 : (plow >= 128 ? 128 : (plow >= 64 ? 64 : 32));
  li.smem = (size_t)h.ninputs * plow * sizeof(int32_t);
  int64_t tiles = row_end > row_begin ? (row_end - 1) / plow - row_begin / plow + 1 : 0;
  int64_t g = std::min<int64_t>(tiles, (int64_t)num_sms * 8);
  li.grid = (int)std::max<int64_t>(g, 1);
  (void)variant;
  return li;
}

cudaError_t bk_launch(const gbe_bucket_desc &h, const gbe_bucket_desc *dev_desc,
                      const InPtrs &in, void *out, uint8_t *arg, int64_t row_begin,
                      int64_t row_end, const BkLaunchInfo &li, cudaStream_t stream) {
  if (row_end <= row_begin) return cudaSuccess;
  if (h.semiring == GBE_SUMPROD_F64)
    bk_generic<double, true><<<li.grid, li.block, li.smem, stream>>>(
        dev_desc, in, (double *)out, arg, row_begin, row_end, li.nlow, li.plow);
  else if (h.semiring == GBE_MINSUM_F64)
    bk_generic<double, false><<<li.grid, li.block, li.smem, stream>>>(
        dev_desc, in, (double *)out, arg, row_begin, row_end, li.nlow, li.plow);
  else
    bk_generic<int32_t, false><<<li.grid, li.block, li.smem, stream>>>(
        dev_desc, in, (int32_t *)out, arg, row_begin, row_end, li.nlow, li.plow);
  return cudaGetLastError();
}

cudaError_t relayout_launch(const void *in, void *out, int elem, int nf, const int64_t *off,
                            const int32_t *poff, const int32_t *prad, const int32_t *pstride,
                            cudaStream_t stream) {
  if (nf <= 0) return cudaSuccess;
  int grid = nf < 4096 ? nf : 4096;
  if (elem == 8)
    relayout_kernel<double><<<grid, 128, 0, stream>>>((const double *)in, (double *)out, nf, off,
                                                      poff, prad, pstride);
  else
    relayout_kernel<int32_t><<<grid, 128, 0, stream>>>((const int32_t *)in, (int32_t *)out, nf,
                                                       off, poff, prad, pstride);
  return cudaGetLastError();
}

cudaError_t value_launch(bool f64, const VStep *steps, int s0, int s1, const VMember *mems,
                         const VTerm *terms, int32_t *assign, const int32_t *gathered, int gvar,
                         int W, const void *const *cptrs, int nconst, void *optimum,
                         cudaStream_t stream) {
  if (f64)
    value_kernel<double><<<1, 32, 0, stream>>>(steps, s0, s1, mems, terms, assign, gathered, gvar,
                                                W, cptrs, nconst, (double *)optimum);
  else
    value_kernel<int32_t><<<1, 32, 0, stream>>>(steps, s0, s1, mems, terms, assign, gathered,
                                                 gvar, W, cptrs, nconst, (int32_t *)optimum);
  return cudaGetLastError();
}

cudaError_t bk_count_launch(const gbe_bucket_desc &h, const gbe_bucket_desc *dev_desc, const InPtrs &in,
                            const InPtrs &cin, void *out, double *cnt, uint8_t *arg, int64_t row_begin,
                            int64_t row_end, bool consistent, cudaStream_t stream) {
  if (row_end <= row_begin) return cudaSuccess;
  const BkLaunchInfo li = bk_plan_launch(h, row_begin, row_end, BK_GENERIC, 148);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((int64_t)li.grid, (int64_t)nsm * 8);
#define GBE_CNT(T, C) \
  bk_count<T, C><<<grid, li.block, li.smem, stream>>>(dev_desc, in, cin, (T *)out, cnt, arg, row_begin, row_end, li.nlow, li.plow)
  if (h.semiring == GBE_MINSUM_I32) {
    if (consistent) GBE_CNT(int32_t, true); else GBE_CNT(int32_t, false);
  } else {
    if (consistent) GBE_CNT(double, true); else GBE_CNT(double, false);
  }
#undef GBE_CNT
  return cudaGetLastError();
}

cudaError_t count_total_launch(bool f64, const void *const *cptrs, const double *const *cc, int n,
                               bool consistent, void *optimum, double *count, cudaStream_t stream) {
  if (f64)
    count_total_kernel<double><<<1, 1, 0, stream>>>(cptrs, cc, n, consistent, (double *)optimum, count);
  else
    count_total_kernel<int32_t><<<1, 1, 0, stream>>>(cptrs, cc, n, consistent, (int32_t *)optimum, count);
  return cudaGetLastError();
}

}  // namespace gbe
