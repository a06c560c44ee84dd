// bk_stream.cu — the streaming bucket kernel (BK, warp-per-row-group).
//
// The same operation as every BK variant (Proc. 4 + Proc. 5 fused,
// P:705-792): out[r] = min_v (+)_j T_j[off_j(r) + v], arg[r] = first
// minimiser (A8), off_j(r) the index map of Eq. with precomputed
// strides.  Where the tiled kernel (bk_fast.cu) stages tile slices in shared
// memory through a TMA ring, this one loads straight from global memory with
// many warps in flight: it is the variant for buckets whose inputs are few
// and large (a register-blocked tile saves nothing when every input spans
// the tile -- e.g. a single input eliminated, C5's k = 1 buckets), for f64
// tables (whose tile slices leave the ring too few bytes in flight), and for
// any domain size d up to 256.
//
//  * Rows are grouped by LPR lanes ("lanes per row", 1..32): the LPR lanes of
//    a row split the eliminated variable's domain (lane s takes v = s, s+LPR,
//    ...) and combine (value, index) pairs with a lexicographic warp-shuffle
//    min (A8) -- the north star's lanes-over-v mapping; LPR = 1 for d <= 5,
//    where each lane owns whole rows.  The LPR lanes of a row read
//    consecutive elements and a warp's row groups are consecutive rows, so a
//    table spanning the trailing digits is read fully coalesced.
//  * A warp-tile = all values of the trailing output digits (PL rows); the
//    in-tile offset of every input is one shared-memory table built once per
//    CTA (no per-row div/mod).  Warps take warp-tiles round robin; a tile's
//    base offsets come from one parallel mixed-radix decode (lane q: digit
//    q; lane j: input j's base).  For a full-range launch the tiles are
//    enumerated with the digits absent from the largest input varying
//    fastest, so the tiles that re-read one slice of it are in flight
//    together and hit L2.
//  * Loads: each lane issues the loads of UN rows of up to KU inputs before
//    the first add (memory-level parallelism without the shared-memory ring
//    of the tiled kernel); vector loads (16 B) where the layout allows.
//  * int32: saturating adds (A9); f64: IEEE adds in input order (A10);
//    sum-product: m - log sum_v exp(m - s_v) (A18).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "bk_stream.h"

namespace gbe {
namespace {

constexpr uint32_t kInf = GBE_INF_I32;
constexpr int kBlock = 256;

template <typename T>
struct SrS;
template <>
struct SrS<int32_t> {
  using Acc = uint32_t;
  __device__ __forceinline__ static Acc zero() { return 0u; }
  __device__ __forceinline__ static Acc inf() { return kInf; }
  __device__ __forceinline__ static Acc ld(const int32_t *p) { return (uint32_t)__ldg(p); }
  __device__ __forceinline__ static Acc add(Acc a, Acc b) { return min(a + b, kInf); }
  __device__ __forceinline__ static int32_t out(Acc a) { return (int32_t)a; }
};
template <>
struct SrS<double> {
  using Acc = double;
  __device__ __forceinline__ static Acc zero() { return 0.0; }
  __device__ __forceinline__ static Acc inf() { return __longlong_as_double(0x7ff0000000000000LL); }
  __device__ __forceinline__ static Acc ld(const double *p) { return __ldg(p); }
  __device__ __forceinline__ static Acc add(Acc a, Acc b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double out(Acc a) { return a; }
};

// staged mode: mbarrier / TMA bulk-copy wrappers (PTX)
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *smem_dst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// An opaque copy of a pointer: the compiler then adds each row's 32-bit
// offset to it with one IMAD.WIDE instead of re-associating (base + offset)
// into a 64-bit sign-extended add and a scaled add per row (4 instructions)
template <typename P>
__device__ __forceinline__ const P *opaque(const P *p) {
  uint64_t x = (uint64_t)p;
  asm("" : "+l"(x));
  return (const P *)x;
}

__device__ __forceinline__ int64_t shfl64(int64_t x, int src) {
  return (int64_t)__shfl_sync(0xffffffffu, (long long)x, src);
}

// LPR lanes per row, VPL values per lane, UN row groups per lane per pass.
// VEC = 1: lane s of a row takes v = s + i * LPR (scalar loads); VEC > 1:
// lane s takes the VPL = VEC contiguous values v = s * VEC + i with ONE
// vector load per input (16 or 8 bytes), so the warp's loads of a table that
// spans the trailing digits are contiguous (needs every offset a multiple of
// VEC and aligned tables: checked on the host and at launch).  DV > 0: the
// domain size is that compile-time constant; DV = 0: runtime d, masked.
// (SM: the pointer is into shared memory -- the staged mode -- and takes a
// plain load instead of the read-only global path)
template <typename T, int VEC>
struct VecLd;
template <>
struct VecLd<double, 2> {
  template <bool SM>
  __device__ __forceinline__ static void ld(const double *p, double *v) {
    const double2 x = SM ? *(const double2 *)p : __ldg((const double2 *)p);
    v[0] = x.x;
    v[1] = x.y;
  }
};
template <>
struct VecLd<int32_t, 4> {
  template <bool SM>
  __device__ __forceinline__ static void ld(const int32_t *p, uint32_t *v) {
    const int4 x = SM ? *(const int4 *)p : __ldg((const int4 *)p);
    v[0] = (uint32_t)x.x;
    v[1] = (uint32_t)x.y;
    v[2] = (uint32_t)x.z;
    v[3] = (uint32_t)x.w;
  }
};
template <>
struct VecLd<int32_t, 2> {
  template <bool SM>
  __device__ __forceinline__ static void ld(const int32_t *p, uint32_t *v) {
    const int2 x = SM ? *(const int2 *)p : __ldg((const int2 *)p);
    v[0] = (uint32_t)x.x;
    v[1] = (uint32_t)x.y;
  }
};

template <typename T, bool SP, int LPR, int VPL, int DV, int UN, int VEC = 1, bool BD = false, bool HX = false,
          int B2 = 1, bool STG = false>
__global__ void __launch_bounds__(kBlock, 2) bk_stream(const StreamDesc *__restrict__ D, InPtrs in,
                                                    T *__restrict__ out, uint8_t *__restrict__ arg,
                                                    int64_t row_begin, int64_t row_end, int64_t t0,
                                                    int64_t ntiles, bool pf) {
  using S = SrS<T>;
  using Acc = typename S::Acc;
  extern __shared__ int32_t loff[];  // [k][PL] in-tile element offsets
  const int k = D->k, PL = D->PL, nlow = D->nlow, nhigh = D->nhigh;
  const int d = DV > 0 ? DV : D->d;
  for (int idx = threadIdx.x; idx < k * PL; idx += blockDim.x) {
    const int j = idx / PL;
    int l = idx - j * PL, o = 0;
    for (int q = nlow - 1; q >= 0; q--) {
      const int r = D->lrad[q];
      o += (l % r) * D->lstr[q][j];
      l /= r;
    }
    loff[idx] = o;
  }
  // blocked high digits: output-row offset of every in-tile row
  constexpr bool hxt = HX;
  int64_t *rowoff = (int64_t *)(loff + ((k * PL + 1) & ~1));
  if constexpr (HX)
    for (int l0 = threadIdx.x; l0 < PL; l0 += blockDim.x) {
      int l = l0;
      int64_t o = 0;
      for (int q = nlow - 1; q >= 0; q--) {
        const int r = D->lrad[q];
        o += (int64_t)(l % r) * D->lrowst[q];
        l /= r;
      }
      rowoff[l0] = o;
    }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= ntiles) return;
  // staged mode (STG): each warp owns two shared-memory buffers; buffer b
  // holds the input slices of one of its tiles, filled by TMA bulk copies
  // (one per input, issued by lane j) one tile ahead of the compute, with
  // completion on the buffer's mbarrier -- the bytes in flight no longer
  // cost registers and the copies of tile i+1 overlap the compute of tile i
  [[maybe_unused]] unsigned char *wbuf = nullptr;
  [[maybe_unused]] uint64_t *wbar = nullptr;
  if constexpr (STG) {
    unsigned char *sm = (unsigned char *)loff;
    const int w = threadIdx.x >> 5;
    wbar = (uint64_t *)(sm + D->stg_off) + 2 * w;
    wbuf = sm + D->stg_off + 16 * (kBlock / 32) + (size_t)w * 2 * D->stg_buf;
    if (lane == 0) {
      mbar_init(&wbar[0], 1);
      mbar_init(&wbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
  }
  // tile decode: lane q < nhigh computes high digit q of the tile index
  // (32-bit division when the index fits), lane j < k sums its input's base
  // offset and every lane the tile's first output row.  Warps take tiles
  // round robin, so the tiles in flight at any moment form one window of
  // the enumeration and the tiles re-reading a slice of the largest input
  // (its absent digits vary fastest) hit L2.
  int64_t base = 0, row0 = 0;
  auto decode = [&](int64_t t, int64_t &base, int64_t &row0) {
    int dig = 0;
    if (lane < nhigh) {
      const uint32_t hr = (uint32_t)D->hrad[lane];
      if (t < (int64_t(1) << 32) && D->hdiv[lane] < (int64_t(1) << 32))
        dig = (int)(((uint32_t)t / (uint32_t)D->hdiv[lane]) % hr);
      else
        dig = (int)((t / D->hdiv[lane]) % hr);
    }
    base = 0;
    row0 = 0;
    for (int q = 0; q < nhigh; q++) {
      const int dq = __shfl_sync(0xffffffffu, dig, q);
      if (lane < k) base += (int64_t)dq * D->hstr[q][lane];
      row0 += (int64_t)dq * D->hrow[q];
    }
    if (lane < k) base -= D->shift[lane];
  };
  constexpr int G = 32 / LPR;  // row groups per pass
  const int grp = lane / LPR, sub = lane % LPR;
  static_assert(VEC == 1 || (VPL % VEC == 0 && DV == LPR * VPL), "vector path: whole vectors per lane, exact d");
  static_assert(!BD || LPR == 1, "broadcast digits: one lane per row");
  static_assert(B2 == 1 || (BD && UN % B2 == 0), "second broadcast digit: UN = B1 * B2 rows per lane");
  // broadcast digits: pass rows are i = l0 + grp (i < PL / UN enumerates the
  // rows whose broadcast digits are 0) and the lane's UN rows lb(i) + u * bs,
  // u = u1 * B2 + u2 (u1: digit b1, u2: digit b2 when B2 > 1)
  const int bs = BD ? D->bd_stride : 0;
  const uint32_t bhas = BD ? D->bd_has : 0u;
  const uint32_t bhas2 = B2 > 1 ? D->bd_has2 : ~0u;
  const int64_t brs = BD ? (D->bd_rowstride ? D->bd_rowstride : (int64_t)bs) : 0;  // output-row stride of b1
  const int64_t brs2 = B2 > 1 ? D->bd_rowstride2 : 0;                               // ... of b2
  const int PLi = BD ? PL / UN : PL;
  // value index of this lane's i-th value
  auto vix = [&](int i) { return VEC > 1 ? sub * VPL + i : sub + i * LPR; };
  // inputs in chunks of KU: every load of a chunk is issued before the
  // first add (the adds keep the input order), so a lane has KU * UN * VPL
  // loads in flight instead of one input's worth per round trip
  constexpr int kLaneBytes = UN * VPL * (int)sizeof(T);
  constexpr int KU = kLaneBytes <= 32 ? 2 : 1;
  const int lane_off = VEC > 1 ? sub * VPL : sub;
  const T *pb[KU];  // this tile's first KU input pointers (hoisted per tile)
  int64_t trow = 0;
  [[maybe_unused]] const unsigned char *wb = nullptr;  // STG: this tile's buffer
  [[maybe_unused]] int32_t skew = 0;                  // STG: lane j: 16-byte phase of input j's slice
  // STG: element pointer of input j in this tile's buffer
  auto sptr = [&](int j) -> const T * {
    return (const T *)(wb + D->stg_soff[j] + __shfl_sync(0xffffffffu, skew, j)) + lane_off;
  };
  // one pass = UN row groups of this warp (rows l0 + u * G + grp of the
  // tile); MASK: rows past the tile or outside [row_begin, row_end) skipped
  auto pass = [&](auto maskc, int l0) {
    constexpr bool MASK = decltype(maskc)::value;
    Acc acc[UN][VPL];
    bool valid[UN];
    int lrow[UN];  // in-tile row (offset-table index) of each of this lane's UN rows
    [[maybe_unused]] int lb = 0;
    if constexpr (BD) {
      const int i = l0 + grp;
      lb = (i / bs) * bs * UN + i % bs;
#pragma unroll
      for (int u = 0; u < UN; u++) lrow[u] = lb + u * bs;
    } else {
#pragma unroll
      for (int u = 0; u < UN; u++) lrow[u] = l0 + u * G + grp;
    }
    // output row of row u relative to the tile's first row (formed where used)
    auto grow = [&](int u) -> int64_t {
      if constexpr (BD) return lb + (u / B2) * brs + (u % B2) * brs2;
      return (hxt && lrow[u] < PL) ? rowoff[lrow[u]] : (int64_t)lrow[u];
    };
#pragma unroll
    for (int u = 0; u < UN; u++) {
      if constexpr (MASK) {
        const int l = lrow[u];
        const int64_t r = trow + grow(u);
        valid[u] = (BD ? l0 + grp < PLi : l < PL) && r >= row_begin && r < row_end;
      } else {
        valid[u] = true;
      }
#pragma unroll
      for (int i = 0; i < VPL; i++) acc[u][i] = S::zero();
    }
    // input 0 lands straight in the accumulators (0 + x = x: the clamp of A9
    // and IEEE addition leave it unchanged), later inputs in KU chunks (the
    // first chunk peeled, so every register array is indexed statically)
    auto chunk = [&](auto firstc, int j0) {
      constexpr bool FIRST = decltype(firstc)::value;
      Acc x[KU][UN][VPL];
#pragma unroll
      for (int jj = 0; jj < KU; jj++) {
        const int j = j0 + jj;
        if (j >= k) break;
        const T *pj = FIRST ? pb[jj] : (STG ? sptr(j) : opaque((const T *)in.p[j] + shfl64(base, j) + lane_off));
        const int32_t *lo = loff + j * PL;
        // an input without a broadcast digit: the rows that differ only in
        // the digits it lacks share one load (row u copies row src(u))
        const bool h1 = !BD || ((bhas >> j) & 1u), h2 = (bhas2 >> j) & 1u;
#pragma unroll
        for (int u = 0; u < UN; u++) {
          if (MASK && !valid[u]) continue;
          Acc *dst = (FIRST && jj == 0) ? acc[u] : x[jj][u];
          if constexpr (BD) {
            // src(u) = u with the digits the input lacks set to 0; every
            // branch indexes the register arrays with compile-time constants
            const int u1 = u / B2, u2 = u % B2;
            auto from = [&](int sidx) {  // (sidx constant after unrolling)
              const Acc *sp = (FIRST && jj == 0) ? acc[sidx] : x[jj][sidx];
#pragma unroll
              for (int i = 0; i < VPL; i++) dst[i] = sp[i];
            };
            if (!h1 && !h2) {
              if (u != 0 && (!MASK || valid[0])) {
                from(0);
                continue;
              }
            } else if (!h1) {
              if (u1 != 0 && (!MASK || valid[u2])) {
                from(u2);
                continue;
              }
            } else if (!h2) {
              if (u2 != 0 && (!MASK || valid[u1 * B2])) {
                from(u1 * B2);
                continue;
              }
            }
          }
          const T *q = pj + lo[lrow[u]];
          if constexpr (VEC > 1) {
#pragma unroll
            for (int i = 0; i < VPL; i += VEC) VecLd<T, VEC>::template ld<STG>(q + i, dst + i);
          } else {
#pragma unroll
            for (int i = 0; i < VPL; i++)
              if (DV > 0 || sub + i * LPR < d) dst[i] = STG ? (Acc)q[i * LPR] : S::ld(q + i * LPR);
          }
        }
      }
#pragma unroll
      for (int jj = FIRST ? 1 : 0; jj < KU; jj++) {
        if (j0 + jj >= k) break;
#pragma unroll
        for (int u = 0; u < UN; u++)
#pragma unroll
          for (int i = 0; i < VPL; i++)
            if (DV > 0 || vix(i) < d) acc[u][i] = S::add(acc[u][i], x[jj][u][i]);
      }
    };
    chunk(std::true_type{}, 0);
    for (int j0 = KU; j0 < k; j0 += KU) chunk(std::false_type{}, j0);
#pragma unroll
    for (int u = 0; u < UN; u++) {
      // this lane's minimum over its values (ascending v: first wins)
      Acc best = acc[u][0];
      int bv = vix(0);
#pragma unroll
      for (int i = 1; i < VPL; i++)
        if ((DV > 0 || vix(i) < d) && acc[u][i] < best) {
          best = acc[u][i];
          bv = vix(i);
        }
      // lexicographic (value, index) min over the row's LPR lanes
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) {
        const Acc ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bv, o);
        if (ob < best || (ob == best && oi < bv)) {
          best = ob;
          bv = oi;
        }
      }
      if constexpr (SP) {  // -log sum_v exp(-s_v) = m - log sum_v exp(m - s_v)
        double z = 0.0;
        if (best < S::inf()) {
#pragma unroll
          for (int i = 0; i < VPL; i++)
            if (DV > 0 || vix(i) < d) z += exp((double)best - (double)acc[u][i]);
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
        if (best < S::inf()) best = best - log(z);
        bv = 0;
      }
      if (sub == 0 && (!MASK || valid[u])) {
        const int64_t r = trow + grow(u) - row_begin;
        out[r] = S::out(best);
        if (arg) arg[r] = (uint8_t)bv;
      }
    }
  };
  // the NEXT tile of this warp is decoded one tile ahead and its input
  // slices prefetched into L2 with one bulk (TMA) prefetch per input: the
  // loads of a tile then find their data in L2, so a warp keeps a whole
  // tile of bytes in flight without holding registers for them
  // STG: the bulk copies of the tile whose input bases are tb (lane j) into
  // buffer bb (one per input, its 16-byte-aligned covering range); returns
  // lane j's skew (the slice's 16-byte phase)
  [[maybe_unused]] auto issue = [&](int bb, int64_t tb) -> int32_t {
    uintptr_t a16 = 0;
    uint32_t bytes = 0, sk = 0;
    if (lane < k) {
      const uintptr_t a = (uintptr_t)((const T *)in.p[lane] + tb);
      a16 = a & ~(uintptr_t)15;
      bytes = (uint32_t)((a + (uintptr_t)D->stg_slice[lane] - a16 + 15) & ~(uintptr_t)15);
      sk = (uint32_t)(a - a16);
    }
    const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
    // the buffer's previous reads (generic proxy) before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(&wbar[bb], total);
    __syncwarp();
    if (bytes) tma_load_1d(wbuf + (size_t)bb * D->stg_buf + D->stg_soff[lane], (const void *)a16, bytes, &wbar[bb]);
    return (int32_t)sk;
  };
  decode(t0 + gw, base, row0);
  [[maybe_unused]] int bcur = 0;
  [[maybe_unused]] uint32_t bph = 0;
  [[maybe_unused]] int32_t nskew = 0;
  if constexpr (STG) skew = issue(0, base);
  for (int64_t tt = gw; tt < ntiles; tt += nwarps) {
    int64_t nbase = 0, nrow0 = 0;
    if (tt + nwarps < ntiles) {
      decode(t0 + tt + nwarps, nbase, nrow0);
      if constexpr (STG) {
        nskew = issue(bcur ^ 1, nbase);
      } else if (pf && lane < k && D->pf_bytes[lane] > 0) {
        const uintptr_t a = (uintptr_t)((const T *)in.p[lane] + nbase);
        const uintptr_t a16 = a & ~(uintptr_t)15;
        const uint32_t bytes = (uint32_t)((a + D->pf_bytes[lane] - a16 + 15) & ~(uintptr_t)15);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a16), "r"(bytes) : "memory");
      }
    }
    trow = row0;
    if constexpr (STG) {
      mbar_wait(&wbar[bcur], bph);
      wb = wbuf + (size_t)bcur * D->stg_buf;
#pragma unroll
      for (int jj = 0; jj < KU; jj++)
        if (jj < k) pb[jj] = sptr(jj);
    } else {
#pragma unroll
      for (int jj = 0; jj < KU; jj++)
        if (jj < k) pb[jj] = opaque((const T *)in.p[jj] + shfl64(base, jj) + lane_off);
    }
    int l0 = 0;
    constexpr int kStep = BD ? G : G * UN;  // pass rows (BD: rows with digit b = 0)
    // whole tile: unmasked passes (a tile with a high broadcast digit spans
    // rows up to trow + (UN - 1) * brs + PL / UN)
    const int64_t tspan = (BD && brs != bs) ? (int64_t)(UN / B2 - 1) * brs + (int64_t)(B2 - 1) * brs2 + PLi
                                            : (hxt ? int64_t(0) : (int64_t)PL);
    if (trow >= row_begin && trow + tspan <= row_end)
      for (; l0 + kStep <= PLi; l0 += kStep) pass(std::false_type{}, l0);
    for (; l0 < PLi; l0 += kStep) pass(std::true_type{}, l0);
    if constexpr (STG) {
      __syncwarp();  // every lane done with buffer bcur before it is refilled
      skew = nskew;
      bcur ^= 1;
      if (bcur == 0) bph ^= 1;
    }
    base = nbase;
    row0 = nrow0;
  }
}

template <typename T, bool SP, int LPR, int VPL, int DV, int UN, int VEC = 1, bool BD = false, bool HX = false,
          int B2 = 1, bool STG = false>
cudaError_t launch(const StreamDesc *dd, const BksLaunch &L, const InPtrs &in, void *out, uint8_t *arg,
                   int64_t rb, int64_t re, cudaStream_t s) {
  auto kern = bk_stream<T, SP, LPR, VPL, DV, UN, VEC, BD, HX, B2, STG>;
  if (L.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem);
    if (e != cudaSuccess) return e;
  }
  // one wave: the CTAs that are resident at once (registers / shared memory
  // of this instantiation) and no more, so every warp walks its tiles round
  // robin in one window of the L2-friendly tile order (C5: 15.3 -> 14.8 ms
  // against 8 CTAs per SM in waves; GBE_STREAM_WAVES=1 restores waves)
  static const bool waves = [] {
    const char *e = std::getenv("GBE_STREAM_WAVES");
    return e && std::atoi(e) == 1;
  }();
  int grid = L.grid;
  if (!waves) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kBlock, L.smem) == cudaSuccess && nb > 0)
      grid = (int)std::min<int64_t>(grid, (int64_t)nb * L.sms);
  }
  kern<<<grid, kBlock, L.smem, s>>>(dd, in, (T *)out, arg, rb, re, L.t0, L.ntiles, L.pf);
  return cudaGetLastError();
}

template <typename T, bool SP>
cudaError_t dispatch(const StreamDesc *dd, const BksLaunch &L, const InPtrs &in, void *out, uint8_t *arg,
                     int64_t rb, int64_t re, cudaStream_t s) {
  if constexpr (!SP) {  // staged mode (d = 2..5, one lane per row, the unstaged shapes' rows per lane)
    if (L.stg) {
      bool al = L.vec > 1;
      for (int j = 0; j < L.k && al; j++)
        if ((uintptr_t)in.p[j] % 16) al = false;
      constexpr bool F = sizeof(T) == 8;
      constexpr int V4 = F ? 2 : 4;
      switch (L.d) {
        case 2:
          if (al) return launch<T, SP, 1, 2, 2, 4, 2, false, false, 1, true>(dd, L, in, out, arg, rb, re, s);
          return launch<T, SP, 1, 2, 2, F ? 4 : 8, 1, false, false, 1, true>(dd, L, in, out, arg, rb, re, s);
        case 3: return launch<T, SP, 1, 3, 3, F ? 4 : 8, 1, false, false, 1, true>(dd, L, in, out, arg, rb, re, s);
        case 4:
          // (f64: 2 rows per lane -- 4 spill at the 128-register cap; shared-
          // memory loads need fewer rows in flight than global ones)
          if (al) return launch<T, SP, 1, 4, 4, F ? 2 : 4, V4, false, false, 1, true>(dd, L, in, out, arg, rb, re, s);
          return launch<T, SP, 1, 4, 4, F ? 2 : 4, 1, false, false, 1, true>(dd, L, in, out, arg, rb, re, s);
        case 5: return launch<T, SP, 1, 5, 5, F ? 2 : 4, 1, false, false, 1, true>(dd, L, in, out, arg, rb, re, s);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  if constexpr (!SP) {  // blocked high digits (full-range launches, d <= 5, min-sum)
    if (L.hx) {
      bool al = true;
      for (int j = 0; j < L.k; j++)
        if ((uintptr_t)in.p[j] % 16) al = false;
      if constexpr (sizeof(T) == 4) {
        static const int hxun = [] {  // GBE_STREAM_HXUN: rows per lane (tuning knob)
          const char *e = std::getenv("GBE_STREAM_HXUN");
          return e ? std::atoi(e) : 8;
        }();
        if (L.d == 4 && L.vec == 4 && al) {
          if (hxun == 4) return launch<T, SP, 1, 4, 4, 4, 4, false, true>(dd, L, in, out, arg, rb, re, s);
          return launch<T, SP, 1, 4, 4, 8, 4, false, true>(dd, L, in, out, arg, rb, re, s);
        }
      } else {
        if (L.d == 4 && L.vec == 2 && al) return launch<T, SP, 1, 4, 4, 4, 2, false, true>(dd, L, in, out, arg, rb, re, s);
      }
      switch (L.d) {
        case 2: return launch<T, SP, 1, 2, 2, sizeof(T) == 8 ? 4 : 8, 1, false, true>(dd, L, in, out, arg, rb, re, s);
        case 3: return launch<T, SP, 1, 3, 3, sizeof(T) == 8 ? 4 : 8, 1, false, true>(dd, L, in, out, arg, rb, re, s);
        case 4: return launch<T, SP, 1, 4, 4, 4, 1, false, true>(dd, L, in, out, arg, rb, re, s);
        case 5: return launch<T, SP, 1, 5, 5, sizeof(T) == 8 ? 2 : 4, 1, false, true>(dd, L, in, out, arg, rb, re, s);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  if constexpr (!SP) {  // broadcast digits: L.bd rows per lane (one digit, or two of radix 2)
    if (L.bd) {
      bool al = L.vec > 1;
      for (int j = 0; j < L.k && al; j++)
        if ((uintptr_t)in.p[j] % 16) al = false;
      constexpr int V2 = 2, V4 = sizeof(T) == 8 ? 2 : 4;  // vector widths for d = 2, 4
#define GBE_BD(DVc, UNc, B2c)                                                                           \
  if (L.d == DVc) {                                                                                     \
    if constexpr (DVc == 2) {                                                                           \
      if (al) return launch<T, SP, 1, 2, 2, UNc, V2, true, false, B2c>(dd, L, in, out, arg, rb, re, s); \
    }                                                                                                   \
    if constexpr (DVc == 4) {                                                                           \
      if (al) return launch<T, SP, 1, 4, 4, UNc, V4, true, false, B2c>(dd, L, in, out, arg, rb, re, s); \
    }                                                                                                   \
    return launch<T, SP, 1, DVc, DVc, UNc, 1, true, false, B2c>(dd, L, in, out, arg, rb, re, s);        \
  }
      if (L.bd2 == 2 && L.bd == 4) {
        GBE_BD(2, 4, 2) GBE_BD(3, 4, 2) GBE_BD(4, 4, 2) GBE_BD(5, 4, 2)
      } else if (L.bd2 <= 1) {
        if (L.bd == 2) { GBE_BD(2, 2, 1) GBE_BD(3, 2, 1) GBE_BD(4, 2, 1) GBE_BD(5, 2, 1) }
        if (L.bd == 3) { GBE_BD(2, 3, 1) GBE_BD(3, 3, 1) GBE_BD(4, 3, 1) GBE_BD(5, 3, 1) }
        if (L.bd == 4) { GBE_BD(2, 4, 1) GBE_BD(3, 4, 1) GBE_BD(4, 4, 1) GBE_BD(5, 4, 1) }
      }
#undef GBE_BD
      return cudaErrorInvalidValue;
    }
  }
  // vector path: every input 16-byte aligned (offsets are multiples of VEC,
  // checked by bks_build)
  bool aligned = L.vec > 1;
  for (int j = 0; j < L.k && aligned; j++)
    if ((uintptr_t)in.p[j] % 16) aligned = false;
  if (aligned) {
    if constexpr (sizeof(T) == 8) {
      // (d = 4 with two lanes per row and one 16-byte load each measured
      // slower on C5 than one lane per row: x57 3.38 vs 2.30 ms)
      // d = 4: one lane per row, two 16-byte loads (GBE_STREAM_V4=0: scalar, A/B knob)
      static const bool v4 = [] {
        const char *e = std::getenv("GBE_STREAM_V4");
        return !(e && std::atoi(e) == 0);
      }();
      if (L.d == 2) return launch<T, SP, 1, 2, 2, 4, 2>(dd, L, in, out, arg, rb, re, s);
      if (L.d == 4 && v4) return launch<T, SP, 1, 4, 4, 4, 2>(dd, L, in, out, arg, rb, re, s);
      if (L.d == 8) return launch<T, SP, 4, 2, 8, 4, 2>(dd, L, in, out, arg, rb, re, s);
    } else {
      if (L.d == 2) return launch<T, SP, 1, 2, 2, 4, 2>(dd, L, in, out, arg, rb, re, s);
      if (L.d == 4) return launch<T, SP, 1, 4, 4, 4, 4>(dd, L, in, out, arg, rb, re, s);
      if (L.d == 8) return launch<T, SP, 2, 4, 8, 4, 4>(dd, L, in, out, arg, rb, re, s);
      if (L.d == 16) return launch<T, SP, 4, 4, 16, 4, 4>(dd, L, in, out, arg, rb, re, s);
    }
  }
  constexpr bool F = sizeof(T) == 8;
  static const int un = [] {  // GBE_STREAM_UN: rows per lane per pass for d <= 5 (tuning knob)
    const char *e = std::getenv("GBE_STREAM_UN");
    return e ? std::atoi(e) : 0;
  }();
#define GBE_UN(DVc, UNdef)                                                                       \
  {                                                                                              \
    const int u = un ? un : (UNdef);                                                             \
    if (u <= 2) return launch<T, SP, 1, DVc, DVc, 2>(dd, L, in, out, arg, rb, re, s);            \
    if (u <= 4 || F) return launch<T, SP, 1, DVc, DVc, 4>(dd, L, in, out, arg, rb, re, s);       \
    if constexpr (!F) return launch<T, SP, 1, DVc, DVc, 8>(dd, L, in, out, arg, rb, re, s);      \
  }
  switch (L.d) {
    case 1: GBE_UN(1, 8)
    case 2: GBE_UN(2, 8)
    case 3: GBE_UN(3, F ? 4 : 8)
    case 4: GBE_UN(4, 4)
    case 5: GBE_UN(5, F ? 2 : 4)
    default: break;
  }
#undef GBE_UN
  // large domains: rows per lane per pass (GBE_STREAM_UNL: tuning knob; the
  // lanes of a row reduce with shuffles, so several rows per pass overlap
  // their loads and reduction chains)
  static const int unl = [] {
    const char *e = std::getenv("GBE_STREAM_UNL");
    return e ? std::atoi(e) : 0;
  }();
  if (L.d <= 8) return launch<T, SP, 2, 4, 0, 2>(dd, L, in, out, arg, rb, re, s);
  if (L.d <= 16) return launch<T, SP, 4, 4, 0, 2>(dd, L, in, out, arg, rb, re, s);
  constexpr int UL = F ? 2 : 4;  // (f64 with 4 rows per lane spills at the 128-register cap)
  if (L.d <= 32) return launch<T, SP, 8, 4, 0, 2>(dd, L, in, out, arg, rb, re, s);  // (4 rows: d = 25 slower)
  if (L.d <= 64) {
    if (unl == 1) return launch<T, SP, 16, 4, 0, 1>(dd, L, in, out, arg, rb, re, s);
    return launch<T, SP, 16, 4, 0, UL>(dd, L, in, out, arg, rb, re, s);
  }
  if (L.d <= 128) {
    if (unl == 1) return launch<T, SP, 32, 4, 0, 1>(dd, L, in, out, arg, rb, re, s);
    return launch<T, SP, 32, 4, 0, UL>(dd, L, in, out, arg, rb, re, s);
  }
  if constexpr (F) {
    return launch<T, SP, 32, 8, 0, 1>(dd, L, in, out, arg, rb, re, s);
  } else {
    if (unl == 1) return launch<T, SP, 32, 8, 0, 1>(dd, L, in, out, arg, rb, re, s);
    return launch<T, SP, 32, 8, 0, 2>(dd, L, in, out, arg, rb, re, s);
  }
}

}  // namespace

int bks_lanes_per_row(int d) {
  if (d <= 5) return 1;
  if (d <= 8) return 2;
  if (d <= 16) return 4;
  if (d <= 32) return 8;
  if (d <= 64) return 16;
  return 32;
}

bool bks_build(const gbe_bucket_desc &h, int64_t row_begin, int64_t row_end, int num_sms, StreamDesc &S,
               BksLaunch &L, bool stage, int pl_cap_rows) {
  const int m = h.nsep, k = h.ninputs, d = h.d;
  if (k < 1 || k > 32 || d < 1 || d > GBE_MAX_DOMAIN || row_end <= row_begin) return false;
  // warp-tile: trailing output digits while the CTA's offset table stays
  // <= 32 KB (k * PL int32) and every in-tile offset fits int32
  static const int pl_cap = [] {  // GBE_STREAM_PLMAX: warp-tile rows cap (tuning knob)
    const char *e = std::getenv("GBE_STREAM_PLMAX");
    return e ? std::max(32, std::atoi(e)) : 4096;
  }();
  const int pl_max = std::max(1, std::min(pl_cap_rows > 0 ? std::min(pl_cap, pl_cap_rows) : pl_cap, 8192 / k));
  int nlow = 0;
  int64_t PL = 1;
  int64_t maxoff[32] = {0};
  while (nlow < m && PL * h.radix[m - 1 - nlow] <= pl_max) {
    const int q = m - 1 - nlow;
    bool fits = true;
    for (int j = 0; j < k; j++)
      if (maxoff[j] + (int64_t)(h.radix[q] - 1) * h.stride[j][q] >= (int64_t(1) << 31)) fits = false;
    if (!fits) break;
    for (int j = 0; j < k; j++) maxoff[j] += (int64_t)(h.radix[q] - 1) * h.stride[j][q];
    PL *= h.radix[q];
    nlow++;
  }
  // small buckets: shorter warp-tiles, so that every warp of a full grid
  // gets one (down to 128 rows)
  const int64_t want_tiles = (int64_t)num_sms * 2 * (kBlock / 32);
  while (nlow > 0 && PL > 128 && (row_end - row_begin + PL - 1) / PL < want_tiles) {
    nlow--;
    const int q = m - 1 - nlow;
    PL /= h.radix[q];
  }
  // staged mode: every input's slice over the in-tile digits must be one
  // dense range (bulk-copyable), and two per-warp buffers of them plus the
  // offset table must fit the CTA's shared-memory budget
  // (GBE_STREAM_STAGE_KB, default 100 KB: two CTAs per SM): drop low digits
  // until they do
  const int esz = h.semiring == GBE_MINSUM_I32 ? 4 : 8;
  std::vector<int64_t> sbytes(k, 0);
  int64_t sbuf = 0;
  if (stage) {
    if (d < 2 || d > 5 || h.semiring == GBE_SUMPROD_F64) return false;
    static const int stg_kb = [] {
      const char *e = std::getenv("GBE_STREAM_STAGE_KB");
      return e ? std::max(16, std::min(220, std::atoi(e))) : 100;
    }();
    for (;;) {
      bool dense = true;
      sbuf = 0;
      for (int j = 0; j < k; j++) {
        int64_t want = d, span = 1;
        for (int q = nlow - 1; q >= 0; q--) {
          const int p = m - nlow + q;
          if (!h.stride[j][p]) continue;
          if (h.stride[j][p] != want) dense = false;
          want *= h.radix[p];
          span *= h.radix[p];
        }
        sbytes[j] = span * d * esz;
        sbuf += ((sbytes[j] + 15) & ~int64_t(15)) + 32;
      }
      if (!dense) return false;
      const int64_t need = ((4 * (int64_t)k * PL + 15) & ~int64_t(15)) + 16 * (kBlock / 32) + 2 * (kBlock / 32) * sbuf;
      if (need <= (int64_t)stg_kb * 1024) break;
      if (nlow <= 1 || PL / h.radix[m - nlow] < 32) return false;
      PL /= h.radix[m - nlow];  // drop the most significant low digit
      nlow--;
    }
  }
  std::memset(&S, 0, sizeof(S));
  L.pf_ok = false;
  L.pf = false;
  L.stg = stage;
  const bool full = row_begin == 0 && row_end == h.rows;
  std::vector<int64_t> cells(k, d);
  int big = 0;
  for (int j = 0; j < k; j++) {
    for (int p = 0; p < m; p++)
      if (h.stride[j][p]) cells[j] *= h.radix[p];
    if (cells[j] > cells[big]) big = j;
  }
  std::vector<int64_t> rowstride(m + 1, 1);
  for (int p = m - 1; p >= 0; p--) rowstride[p] = rowstride[p + 1] * h.radix[p];
  for (int p = 0; p < m; p++) rowstride[p] = rowstride[p + 1];
  // broadcast digit (d <= 5, min-sum): a digit b of radix 2..4
  // the largest input lacks; a lane's rows are the rows that differ only in
  // b and every input without b is loaded once for all of them.  b is an
  // in-tile digit when one qualifies, else (full-range launches) a high
  // digit placed on top of the warp-tile, whose rows then form radix(b) runs
  // of PL rows.  Chosen to minimise the loads per row sum_j (has b ? 1 : 1/r).
  // blocked high digits (full-range launches): inputs of >= 16 MB that are
  // not the two largest have their re-use served inside a tile -- the high
  // digits they lack go on top of the warp-tile (the tile order serves the
  // two largest inputs through L2).  A bucket with three large inputs that
  // lack different digits (C4-d4's 4^16-row bucket) otherwise re-reads the
  // third from HBM once per combination of its absent digits.
  std::vector<int> hxd;
  int64_t hxprod = 1;
  {
    const char *e = std::getenv("GBE_STREAM_HX");  // A/B knob (0: off)
    const bool hx_off = (e && std::atoi(e) == 0) || d > 5 || d < 2 || h.semiring == GBE_SUMPROD_F64 || stage;
    const double es = h.semiring == GBE_MINSUM_I32 ? 4.0 : 8.0;
    std::vector<std::pair<double, int>> large;
    for (int j = 0; j < k; j++)
      if (cells[j] * es >= 16.0 * (1 << 20)) large.push_back({-(double)cells[j], j});
    std::stable_sort(large.begin(), large.end());
    for (size_t r = 2; full && !hx_off && r < large.size(); r++) {
      const int j = large[r].second;
      std::vector<int> cand;
      int64_t prod = 1;
      for (int p = 0; p < m - nlow; p++)
        if (h.radix[p] > 1 && !h.stride[j][p] && std::find(hxd.begin(), hxd.end(), p) == hxd.end()) {
          cand.push_back(p);
          prod *= h.radix[p];
        }
      if (cand.empty()) continue;
      // room: drop low digits (keeping >= 16 contiguous rows) until it fits
      int nl = nlow;
      int64_t pl = PL;
      while (pl * hxprod * prod > pl_max && nl > 1 && pl / h.radix[m - nl] >= 16) {
        pl /= h.radix[m - nl];
        nl--;
      }
      if (pl * hxprod * prod > pl_max) continue;
      bool fits = true;  // in-tile offsets stay int32
      for (int jj = 0; jj < k; jj++) {
        int64_t mo = 0;
        for (int q = m - nl; q < m; q++) mo += (int64_t)(h.radix[q] - 1) * h.stride[jj][q];
        for (int p : hxd) mo += (int64_t)(h.radix[p] - 1) * h.stride[jj][p];
        for (int p : cand) mo += (int64_t)(h.radix[p] - 1) * h.stride[jj][p];
        if (mo >= (int64_t(1) << 31)) fits = false;
      }
      if (!fits) continue;
      nlow = nl;
      PL = pl;
      hxd.insert(hxd.end(), cand.begin(), cand.end());
      hxprod *= prod;
    }
    std::sort(hxd.begin(), hxd.end());  // most significant first
  }
  int bd_low = -1, bd_high = -1, bd_r = 0;
  int64_t bd_stride = 0;
  if (hxd.empty()) {
    // measured slower on C5 (x57 2.55 -> 2.69 ms, x77 1.39 -> 1.56, x91
    // 1.30 -> 1.63 with the tiled kernel then winning): the rows per lane
    // drop to radix(b) and with them the loads in flight, while the re-reads
    // it saves were L1 hits.  Off unless GBE_STREAM_BD=1 (read per build, so
    // tests can enable it)
    const char *bd_env = std::getenv("GBE_STREAM_BD");
    const bool bd_off = !(bd_env && std::atoi(bd_env) == 1);
    if (!bd_off && !stage && d <= 5 && d >= 2 && h.semiring != GBE_SUMPROD_F64 && k >= 1) {
      auto cost = [&](int p) {
        double c = 0;
        for (int j = 0; j < k; j++) c += h.stride[j][p] ? 1.0 : 1.0 / h.radix[p];
        return c;
      };
      double best = (double)k - 1e-9;
      int64_t stride = 1;
      for (int q = nlow - 1; q >= 0; q--) {  // in-tile digits, least significant first
        const int p = m - nlow + q;
        const int r = h.radix[p];
        if (r >= 2 && r <= 4 && !h.stride[big][p] && cost(p) < best) {
          best = cost(p);
          bd_low = p;
          bd_r = r;
          bd_stride = stride;
        }
        stride *= r;
      }
      if (bd_low < 0 && full && nlow > 0) {
        for (int p = 0; p < m - nlow; p++) {
          const int r = h.radix[p];
          if (r >= 2 && r <= 4 && !h.stride[big][p] && cost(p) < best - 1e-9) {
            best = cost(p);
            bd_high = p;
            bd_r = r;
          }
        }
        if (bd_high >= 0) {  // keep the offset table within its budget
          bool ok = true;
          for (int j = 0; j < k; j++)
            if (maxoff[j] + (int64_t)(bd_r - 1) * h.stride[j][bd_high] >= (int64_t(1) << 31)) ok = false;
          while (ok && nlow > 1 && PL * bd_r > pl_max) {
            const int q = m - nlow;  // drop the most significant low digit
            PL /= h.radix[q];
            nlow--;
          }
          if (!ok || PL * bd_r > pl_max) bd_high = -1;
        }
      }
    }
  }
  // high broadcast digits (opt-in: GBE_STREAM_BD2=1, read per build): when
  // the largest input lacks high output digits, a lane's rows are the
  // combinations of two radix-2 such digits (or all values of one of radix
  // 3-4) placed on top of the warp-tile, and every input lacking one of them
  // is loaded once per combination of the others -- its re-reads come from
  // registers instead of L1/L2/HBM.  Measured SLOWER although it halves the
  // loads (C5 x57 1.89 -> 2.37 ms, x77 1.37 -> 1.50, x91 1.22 -> 1.48;
  // C4-d4 x80 2.62 -> 4.42): the kernel is bound by the latency of its
  // loads, not their number, and the lane's rows are no longer contiguous
  // (GBE_STREAM_BD2=2: on for inputs >= 16 MB, the rule it was measured with)
  int bd_high2 = -1;
  if (!stage && hxd.empty() && bd_low < 0 && bd_high < 0 && full && nlow > 0 && d >= 2 && d <= 5 &&
      h.semiring != GBE_SUMPROD_F64) {
    const char *e2 = std::getenv("GBE_STREAM_BD2");
    const double es = h.semiring == GBE_MINSUM_I32 ? 4.0 : 8.0;
    const int bd2_env = e2 ? std::atoi(e2) : 0;
    if (bd2_env == 1 || (bd2_env == 2 && cells[big] * es >= 16.0 * (1 << 20))) {
      std::vector<int> lack;  // high digits of radix 2..4 the largest input lacks
      for (int p = 0; p < m - nlow; p++)
        if (h.radix[p] >= 2 && h.radix[p] <= 4 && !h.stride[big][p]) lack.push_back(p);
      auto cost = [&](int p1, int p2) {  // loads per row
        double c = 0;
        for (int j = 0; j < k; j++)
          c += 1.0 / ((h.stride[j][p1] ? 1 : h.radix[p1]) * (p2 >= 0 && !h.stride[j][p2] ? h.radix[p2] : 1));
        return c;
      };
      double best = (double)k - 0.25;
      int b1 = -1, b2 = -1;
      for (size_t a = 0; a < lack.size(); a++) {
        const int p1 = lack[a];
        if (h.radix[p1] >= 3 && cost(p1, -1) < best) {
          best = cost(p1, -1);
          b1 = p1;
          b2 = -1;
        }
        for (size_t b = a + 1; b < lack.size(); b++) {
          const int p2 = lack[b];
          if (h.radix[p1] == 2 && h.radix[p2] == 2 && cost(p1, p2) < best - 1e-9) {
            best = cost(p1, p2);
            b1 = p1;
            b2 = p2;
          }
        }
      }
      if (b1 >= 0) {
        const int un = h.radix[b1] * (b2 >= 0 ? 2 : 1);
        bool ok = true;  // in-tile offsets stay int32
        for (int j = 0; j < k; j++) {
          int64_t mo = maxoff[j] + (int64_t)(h.radix[b1] - 1) * h.stride[j][b1];
          if (b2 >= 0) mo += h.stride[j][b2];
          if (mo >= (int64_t(1) << 31)) ok = false;
        }
        while (ok && nlow > 1 && PL * un > pl_max) {
          const int q = m - nlow;  // drop the most significant low digit
          PL /= h.radix[q];
          nlow--;
        }
        if (ok && PL * un <= pl_max) {
          bd_high = b1;
          bd_high2 = b2;
          bd_r = h.radix[b1];
        }
      }
    }
  }
  S.k = k;
  S.d = d;
  const int nbd = bd_high < 0 ? 0 : (bd_high2 >= 0 ? 2 : 1);
  const int top = nbd ? nbd : (int)hxd.size();  // in-tile digits above the low ones
  S.nlow = nlow + top;
  S.PL = (int32_t)(PL * (bd_high >= 0 ? bd_r * (bd_high2 >= 0 ? 2 : 1) : hxprod));
  S.hx = (int32_t)hxd.size();
  if (bd_high >= 0) {
    S.lrad[0] = bd_r;
    for (int j = 0; j < k; j++) S.lstr[0][j] = (int32_t)h.stride[j][bd_high];
  }
  if (bd_high2 >= 0) {
    S.lrad[1] = 2;
    for (int j = 0; j < k; j++) S.lstr[1][j] = (int32_t)h.stride[j][bd_high2];
    S.bd_rowstride2 = rowstride[bd_high2];
    for (int j = 0; j < k; j++)
      if (h.stride[j][bd_high2]) S.bd_has2 |= 1u << j;
  }
  for (size_t q = 0; q < hxd.size(); q++) {
    S.lrad[q] = h.radix[hxd[q]];
    S.lrowst[q] = rowstride[hxd[q]];
    for (int j = 0; j < k; j++) S.lstr[q][j] = (int32_t)h.stride[j][hxd[q]];
  }
  for (int q = 0; q < nlow; q++) {  // low digits, most significant first
    const int p = m - nlow + q;
    S.lrad[top + q] = h.radix[p];
    S.lrowst[top + q] = rowstride[p];
    for (int j = 0; j < k; j++) S.lstr[top + q][j] = (int32_t)h.stride[j][p];
  }
  if (bd_low >= 0 || bd_high >= 0) {
    const int p = bd_low >= 0 ? bd_low : bd_high;
    S.bd_rad = bd_r;
    S.bd_stride = (int32_t)(bd_low >= 0 ? bd_stride : PL);
    S.bd_rowstride = bd_low >= 0 ? 0 : rowstride[p];
    for (int j = 0; j < k; j++)
      if (h.stride[j][p]) S.bd_has |= 1u << j;
  }
  // high digits (radix-1 digits are always 0 and are dropped).  A launch
  // over all rows enumerates tiles with the digits absent from the largest
  // input varying fastest: the tiles re-reading one slice of it then run
  // back to back in a warp and hit L1/L2 instead of HBM
  int hd[GBE_MAX_SEP], nh = 0;
  for (int p = 0; p < m - nlow; p++)
    if (h.radix[p] > 1 && p != bd_high && p != bd_high2 && std::find(hxd.begin(), hxd.end(), p) == hxd.end())
      hd[nh++] = p;
  if (nh > 32) return false;
  if (full)
    order_high_digits(h, hd, nh);
  L.natural = !full;
  S.nhigh = nh;
  int64_t div = 1;
  for (int e = nh - 1; e >= 0; e--) {
    const int p = hd[e];
    S.hrad[e] = h.radix[p];
    S.hdiv[e] = div;
    div *= h.radix[p];
    for (int j = 0; j < k; j++) S.hstr[e][j] = h.stride[j][p];
    S.hrow[e] = rowstride[p];
  }
  for (int j = 0; j < k; j++) S.shift[j] = h.shift[j];
  // L2 prefetch extent of each input's tile slice: [base, base + maxoff + d)
  // is the whole slice when the input's in-tile offsets are one dense block
  // (canonical layouts); otherwise no prefetch.  Measured on C5: buckets
  // with k >= 2 inputs gain (x91 1.43 -> 1.29 ms, x77 1.42 -> 1.39 ms),
  // single-input buckets lose (x26 0.51 -> 0.79 ms), so it is on for k >= 2;
  // GBE_STREAM_PF=0 / 1 forces it off / on (A/B knob)
  static const int pf_env = [] {
    const char *e = std::getenv("GBE_STREAM_PF");
    return e ? std::atoi(e) : -1;
  }();
  // pf_ok: some input can be prefetched; L.pf: on by default (the executor's
  // autotuning also times the other setting)
  const bool no_pf = pf_env == 0 || bd_high >= 0 || !hxd.empty() || stage;
  L.pf = !no_pf && (pf_env == 1 || k >= 2);
  for (int j = 0; j < k; j++) {
    int64_t want = d, span = 1;
    bool dense = true;
    for (int q = nlow - 1; q >= 0; q--) {
      const int p = m - nlow + q;
      if (!h.stride[j][p]) continue;
      if (h.stride[j][p] != want) dense = false;
      want *= h.radix[p];
      span *= h.radix[p];
    }
    const int64_t bytes = span * d * (h.semiring == GBE_MINSUM_I32 ? 4 : 8);
    S.pf_bytes[j] = (dense && !no_pf && bytes >= 256 && bytes < (int64_t(1) << 30)) ? bytes : 0;
    if (S.pf_bytes[j]) L.pf_ok = true;
  }
  if (!L.pf_ok) L.pf = false;
  // vector loads: one 16-byte (f64 d = 2, 4, 8; int32 d = 4, 8, 16) or
  // 8-byte (int32 d = 2) load per lane when every offset is a multiple of VEC
  {
    const int es = h.semiring == GBE_MINSUM_I32 ? 4 : 8;
    int vec = 0;
    if (es == 8 && (d == 2 || d == 4 || d == 8)) vec = 2;
    if (es == 4 && (d == 4 || d == 8 || d == 16)) vec = 4;
    if (es == 4 && d == 2) vec = 2;
    for (int j = 0; j < k && vec; j++) {
      if (h.shift[j] % vec) vec = 0;
      for (int p = 0; p < m && vec; p++)
        if (h.stride[j][p] % vec) vec = 0;
    }
    L.vec = vec;
  }
  L.bd = S.bd_rad * (bd_high2 >= 0 ? 2 : 1);
  L.bd2 = bd_high2 >= 0 ? 2 : 1;
  L.hx = S.hx;
  L.k = k;
  L.d = d;
  L.f64 = h.semiring != GBE_MINSUM_I32;
  L.sp = h.semiring == GBE_SUMPROD_F64;
  L.t0 = row_begin / S.PL;
  L.ntiles = (row_end - 1) / S.PL - L.t0 + 1;
  L.smem = (int)(sizeof(int32_t) * (size_t)(((k * S.PL + 1) & ~1)) + (hxd.empty() ? 0 : 8 * (size_t)S.PL));
  if (stage) {  // [offset table][per-warp mbarriers][per-warp buffers x 2]
    if (L.pf) L.pf = false;
    S.stg_off = (int32_t)((4 * (int64_t)k * S.PL + 15) & ~int64_t(15));
    S.stg_buf = (int32_t)sbuf;
    int64_t o = 0;
    for (int j = 0; j < k; j++) {
      S.stg_soff[j] = (int32_t)o;
      S.stg_slice[j] = (int32_t)sbytes[j];
      o += ((sbytes[j] + 15) & ~int64_t(15)) + 32;
    }
    L.smem = (int)(S.stg_off + 16 * (kBlock / 32) + 2 * (kBlock / 32) * sbuf);
  }
  // CTAs: as many as fit, at least one warp-tile per warp
  static const int grid_cap = [] {  // GBE_STREAM_PER_SM: CTAs per SM cap (tuning knob: the window of
    const char *e = std::getenv("GBE_STREAM_PER_SM");  // tiles in flight against L2 re-use)
    return e ? std::max(1, std::atoi(e)) : 8;
  }();
  const int per_sm = std::max(1, std::min(grid_cap, (200 * 1024) / std::max(L.smem + 1024, 1)));
  const int64_t want = (L.ntiles + (kBlock / 32) - 1) / (kBlock / 32);
  L.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * per_sm, want));
  L.sms = num_sms;
  return true;
}

cudaError_t bks_launch(const StreamDesc *dev_s, const BksLaunch &L, const InPtrs &in, void *out, uint8_t *arg,
                       int64_t row_begin, int64_t row_end, cudaStream_t s) {
  if (L.sp) return dispatch<double, true>(dev_s, L, in, out, arg, row_begin, row_end, s);
  if (L.f64) return dispatch<double, false>(dev_s, L, in, out, arg, row_begin, row_end, s);
  return dispatch<int32_t, false>(dev_s, L, in, out, arg, row_begin, row_end, s);
}

}  // namespace gbe
