// bk_fast.cu — the tiled, TMA-staged, register-blocked bucket kernel (BK).
//
// Same operation as bk_generic (Proc. 4 + Proc. 5 fused), mapped
// to sm_100a:
//  * A tile = all values of the trailing output digits L (P_L rows).  For every
//    input j the tile's slice is ONE contiguous range of d*prod(L ∩ S_j)
//    elements (the eliminated variable and the trailing output variables are
//    the least-significant digits of every input; bkf_build checks
//    that the tile digits of every input form a dense stride suffix), so each
//    tile needs one 1-D TMA bulk copy (cp.async.bulk, UBLKCP) per input.
//  * One CTA per SM, warp-specialised: NG = 2 consumer groups of GW = 4 warps,
//    one producer warp per group and one storer warp.  The producers keep ONE
//    ring of up to 8 input stages full (full/empty mbarriers); CTA tile i goes
//    to stage i mod nstages and to group i mod 2.  Consumers never block on a
//    CTA barrier.
//  * Inside a tile each thread owns R x R2 x d cells: all values of one or two
//    chosen "group" digits g1, g2 in L and of the eliminated variable.  Inputs
//    are split by which group digits they contain; an input missing a group
//    digit is loaded once and reused across that digit's R values, so the
//    shared-memory loads and adds per cell drop from k to
//    sum_j R^-|{g1,g2} \ S_j| (the host picks g1, g2 to minimise this).
//  * Index math is per tile (a batched mixed-radix decode by the producer
//    warps) and per thread group (a shared-memory offset table built once per
//    CTA): no per-row div/mod.
//  * Output rows and argmins are staged in shared memory (2-3 buffers per
//    group) and written by TMA bulk stores issued by the storer warp; or,
//    in the direct-store mode (DS, a per-bucket autotuning candidate), the
//    consumers write them straight to global memory and the staging
//    buffers' shared memory becomes ring stages.
//  * Tile order: the output digits missing from the largest input vary
//    fastest, so tiles that re-read the same input slice run back to back and
//    hit L2 instead of HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bk_fast.h"

namespace gbe {
namespace {

constexpr uint32_t kInf = GBE_INF_I32;
constexpr int kMaxStages = 8;
constexpr int kOutBufsMax = 3;  // output staging buffers per consumer group (2 or 3)
constexpr int64_t kMinCells = 1 << 10;  // measured: the tiled kernel beats bk_generic from ~1e3 cells
constexpr int kSmemCap = 220 * 1024;  // dynamic shared memory cap per CTA (static use ~5 KB of the 227 KB)

template <typename T>
struct SrF;
template <>
struct SrF<int32_t> {
  using Acc = uint32_t;
  static constexpr bool kInt = true;
  // sums of <= 3 clamped partials (each <= 2^30) fit uint32 without clamping
  __device__ __forceinline__ static Acc add_nc(Acc a, Acc b) { return a + b; }
  __device__ __forceinline__ static Acc add3_nc(Acc a, Acc b, Acc c) { return a + b + c; }
  __device__ __forceinline__ static Acc inf() { return kInf; }
  __device__ __forceinline__ static Acc zero() { return 0u; }
  __device__ __forceinline__ static Acc add(Acc a, Acc b) {
    uint32_t s = a + b;
    return s < kInf ? s : kInf;
  }
  __device__ __forceinline__ static Acc add3(Acc a, Acc b, Acc c) {  // a,b,c <= 2^30
    uint32_t s = a + b + c;
    return s < kInf ? s : kInf;
  }
  __device__ __forceinline__ static int32_t out(Acc a) { return (int32_t)a; }
};
template <>
struct SrF<double> {
  using Acc = double;
  static constexpr bool kInt = false;
  __device__ __forceinline__ static Acc add_nc(Acc a, Acc b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static Acc add3_nc(Acc a, Acc b, Acc c) { return __dadd_rn(__dadd_rn(a, b), c); }
  __device__ __forceinline__ static Acc inf() { return __longlong_as_double(0x7ff0000000000000LL); }
  __device__ __forceinline__ static Acc zero() { return 0.0; }
  __device__ __forceinline__ static Acc add(Acc a, Acc b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static Acc add3(Acc a, Acc b, Acc c) { return __dadd_rn(__dadd_rn(a, b), c); }
  __device__ __forceinline__ static double out(Acc a) { return a; }
};

// exp(x) for x <= 0 (x = m - c_v of the sum-product elimination, m the row
// minimum), branch-free so the R*R2*DV independent evaluations of a thread
// interleave (the library exp's special-case branch serialises them).
// x is clamped at -708 (e^-708 ~ 3e-308 vanishes next to the row's own
// term 1); x = n ln2 + r, |r| <= ln2/2 (magic-number rounding, two-part
// ln2); e^r by its degree-12 Taylor polynomial (truncation r^13/13! < 2e-16
// relative); 2^n from the exponent bits (n >= -1021, a normal double).
// Constants live in a constant bank: DFMA takes c[][] operands directly,
// whereas 64-bit literals are rematerialised (UMOV/IMAD pairs) per use under
// the kernel's register pressure.
__constant__ double kExpC[16] = {
    1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0,
    1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0, 1.0,
    1.4426950408889634,        // [13] log2(e)
    -0.6931471805599453,       // [14] -ln2 (high part)
    -2.3190468138462996e-17};  // [15] -ln2 (low part)

__device__ __forceinline__ double exp_nonpos(double x) {
  x = fmax(x, -708.0);
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double kn = fma(x, kExpC[13], kMagic);
  const double n = kn - kMagic;
  double r = fma(n, kExpC[14], x);
  r = fma(n, kExpC[15], r);
  double p = kExpC[0];
#pragma unroll
  for (int i = 1; i <= 12; i++) p = fma(p, r, kExpC[i]);
  const int ni = __double2loint(kn);  // n in the low word (two's complement)
  return p * __hiloint2double((ni + 1023) << 20, 0);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
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

__device__ __forceinline__ void tma_store_1d(void *gdst, const void *smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}


// Producer-side tile decode, batched: lane L decodes the CTA's tile
// t + L*G (G = gridDim.x) — its mixed-radix high digits (one division chain
// per lane, all lanes in parallel) — into the element offset of every input
// slice, tb[L][j], and its first output row, trow[L].  One batch serves the
// next 32 tiles, so the per-tile issue path is a few shared-memory reads.
constexpr int kMaxH = 32;
// Decode tables live in dynamic shared memory sized by the input count k
// (f.off_prod): hstr[nH][k], then per producer warp trow[32] and tb[32][k]
// (a static [32][32] layout cost 25 KB, a ring stage's worth, on every bucket)
struct ProdTiles {      // one producer's decoded batch (views into dynamic smem)
  int64_t *tb;          // [tile in batch][class-ordered input] element offset (shift applied)
  int64_t *trow;        // [tile in batch] first output row of the tile
};
struct ProdSmem {
  int64_t hrow[kMaxH];
  int64_t shift[32];
  uint32_t hrad[kMaxH];
  int64_t *hstr;        // [high digit][class-ordered input]
};

__device__ __forceinline__ void decode_batch(ProdSmem &ps, ProdTiles &pt, const FastHot &f, int64_t t, int64_t step,
                                             int64_t t_end) {
  const int lane = threadIdx.x & 31;
  const int k = f.k;
  const int64_t tl = t + (int64_t)lane * step;
  if (tl < t_end) {
    uint32_t x = (uint32_t)tl;
    int dg[kMaxH];
#pragma unroll
    for (int e = kMaxH - 1; e >= 0; e--) {
      dg[e] = 0;
      if (e < f.nH) {
        const uint32_t r = ps.hrad[e];
        const uint32_t qt = x / r;
        dg[e] = (int)(x - qt * r);
        x = qt;
      }
    }
    int64_t rs = 0;
#pragma unroll
    for (int e = 0; e < kMaxH; e++)
      if (e < f.nH) rs += (int64_t)dg[e] * ps.hrow[e];
    pt.trow[lane] = rs;
    for (int j = 0; j < k; j++) {
      int64_t acc = -ps.shift[j];
#pragma unroll
      for (int e = 0; e < kMaxH; e++)
        if (e < f.nH) acc += (int64_t)dg[e] * ps.hstr[e * k + j];
      pt.tb[lane * k + j] = acc;
    }
  }
  __syncwarp();
}

// The producer warp issues the TMA copies of batch slot L into stage s (one
// 1-D bulk copy per input: the 16-byte aligned range covering the slice) and
// publishes the slice bases for the consumers.
__device__ __forceinline__ void issue_tile(const ProdTiles &ps, const FastHot &f, const char *my_in, int L,
                                           int s, unsigned char *sm, uint64_t *full, int32_t *sbase,
                                           int64_t *rowstart) {
  const int lane = threadIdx.x & 31;
  uintptr_t a16 = 0;
  uint32_t bytes = 0, skew = 0;
  if (lane < f.k) {
    const char *p = my_in + ps.tb[L * f.k + lane] * f.es;
    a16 = (uintptr_t)p & ~(uintptr_t)15;
    const uintptr_t e16 = ((uintptr_t)p + (uintptr_t)f.slen[lane] * f.es + 15) & ~(uintptr_t)15;
    bytes = (uint32_t)(e16 - a16);
    skew = (uint32_t)((uintptr_t)p - a16);
    sbase[s * 32 + lane] = s * f.stage_bytes + f.soff[lane] + (int32_t)skew;
  }
  const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
  __syncwarp();  // every lane's sbase store before lane 0's release (redux.sync does not order memory)
  if (lane == 0) {
    rowstart[s] = ps.trow[L];
    __threadfence_block();
    mbar_arrive_expect_tx(&full[s], total);
  }
  __syncwarp();
  if (bytes) tma_load_1d(sm + s * f.stage_bytes + f.soff[lane], (const void *)a16, bytes, &full[s]);
}

// in-tile row offset a * rs1 + b * rs2 of register-block row (a, b), formed
// where it is used (two live registers instead of R * R2)
struct RowOff {
  int rs1, rs2;
  __device__ __forceinline__ int operator()(int a, int b) const { return a * rs1 + b * rs2; }
};

// cell (a, b, v) = P0[v] (+ P1[a][v]) (+ P2[b][v]) (+ P3[a][b][v]) with the
// saturating adds of A9; min over v, first minimiser (A8); staged in smem.
template <typename T, int R, int R2, int DV, bool H1, bool H2, bool H3, bool SP>
__device__ __forceinline__ void combine(const typename SrF<T>::Acc (&P0)[DV],
                                        const typename SrF<T>::Acc (&P1)[R][DV],
                                        const typename SrF<T>::Acc (&P2)[R2][DV],
                                        const typename SrF<T>::Acc (&P3)[R][R2][DV], T *outs,
                                        uint8_t *args, const RowOff &loff,
                                        typename SrF<T>::Acc &gmax) {
  using S = SrF<T>;
  using Acc = typename S::Acc;
#pragma unroll
  for (int a = 0; a < R; a++) {
    Acc Q[DV];  // clamped: P0 + P1 can reach 2^31
#pragma unroll
    for (int v = 0; v < DV; v++) Q[v] = H1 ? S::add(P0[v], P1[a][v]) : P0[v];
#pragma unroll
    for (int b = 0; b < R2; b++) {
      // unclamped cell sums (int: <= 3 * 2^30 < 2^32); min over v, then one
      // clamp per row.  If the row minimum is infinite every value clamps to
      // INF and the first index wins (A8).
      Acc c[DV];
#pragma unroll
      for (int v = 0; v < DV; v++) {
        if (H2 && H3)
          c[v] = S::add3_nc(Q[v], P2[b][v], P3[a][b][v]);
        else if (H2)
          c[v] = S::add_nc(Q[v], P2[b][v]);
        else if (H3)
          c[v] = S::add_nc(Q[v], P3[a][b][v]);
        else
          c[v] = Q[v];
      }
      const int l = loff(a, b);
      if constexpr (SP) {  // -log sum_v exp(-c_v) = m - log sum_v exp(m - c_v)
        Acc m = c[0];
#pragma unroll
        for (int v = 1; v < DV; v++) m = fmin(m, c[v]);
        if (m < S::inf()) {
          double z = 0.0;
#pragma unroll
          for (int v = 0; v < DV; v++) z += exp_nonpos(m - c[v]);
          m -= log(z);
        }
        outs[l] = S::out(m);
        if (args) args[l] = 0;
      } else {
        Acc best = c[0];
        int bv = 0;
#pragma unroll
        for (int v = 1; v < DV; v++)
          if (c[v] < best) {
            best = c[v];
            bv = v;
          }
        if (S::kInt) gmax = gmax > best ? gmax : best;  // infinite rows fixed per group
        outs[l] = S::out(best);
        if (args) args[l] = (uint8_t)bv;
      }
    }
  }
}

// Infinity-free int32 tables (the plan proved every entry finite and
// (sum of the largest entries) << SH < 2^32): every cell sum is exact in
// uint32 without clamping, and the first minimiser comes out of ONE unsigned
// min over packed keys (sum << SH) | v — ties on the sum resolve to the
// smaller v, i.e. A8.  The shift is folded into the per-cell add (IMAD/LEA)
// and into group-amortised partial sums.
template <int R, int R2, int DV, bool H1, bool H2, bool H3>
__device__ __forceinline__ void combine_nf(const uint32_t (&P0)[DV], const uint32_t (&P1)[R][DV],
                                           const uint32_t (&P2)[R2][DV], const uint32_t (&P3)[R][R2][DV],
                                           int32_t *outs, uint8_t *args, const RowOff &loff) {
  constexpr int SH = DV <= 4 ? 2 : 3;
  constexpr uint32_t MASK = (1u << SH) - 1u;
  auto emit = [&](const uint32_t (&key)[DV], int l) {
    uint32_t m = key[0];
#pragma unroll
    for (int v = 1; v < DV; v++) m = min(m, key[v]);
    outs[l] = (int32_t)(m >> SH);
    if (args) args[l] = (uint8_t)(m & MASK);  // (null only for direct stores without argmins)
  };
  if constexpr (!H1) {
    uint32_t B[R2][DV];  // ((P0 + P2[b]) << SH) + v, shared by every a
#pragma unroll
    for (int b = 0; b < R2; b++)
#pragma unroll
      for (int v = 0; v < DV; v++) B[b][v] = ((H2 ? P0[v] + P2[b][v] : P0[v]) << SH) + (uint32_t)v;
#pragma unroll
    for (int a = 0; a < R; a++)
#pragma unroll
      for (int b = 0; b < R2; b++) {
        uint32_t key[DV];
#pragma unroll
        for (int v = 0; v < DV; v++) key[v] = H3 ? B[b][v] + (P3[a][b][v] << SH) : B[b][v];
        emit(key, loff(a, b));
      }
  } else {
    uint32_t P2s[R2][DV];
    if constexpr (H2) {
#pragma unroll
      for (int b = 0; b < R2; b++)
#pragma unroll
        for (int v = 0; v < DV; v++) P2s[b][v] = P2[b][v] << SH;
    }
#pragma unroll
    for (int a = 0; a < R; a++) {
      uint32_t A[DV];  // ((P0 + P1[a]) << SH) + v, shared by every b
#pragma unroll
      for (int v = 0; v < DV; v++) A[v] = ((P0[v] + P1[a][v]) << SH) + (uint32_t)v;
#pragma unroll
      for (int b = 0; b < R2; b++) {
        uint32_t key[DV];
#pragma unroll
        for (int v = 0; v < DV; v++) {
          uint32_t x = H2 ? A[v] + P2s[b][v] : A[v];
          key[v] = H3 ? x + (P3[a][b][v] << SH) : x;
        }
        emit(key, loff(a, b));
      }
    }
  }
}

// One CTA = NG consumer groups of GW warps + one producer warp.  The
// producer fills ONE ring of f.nstages input stages; tile i of this CTA goes
// to stage i mod nstages and to consumer group i mod NG, so a group computing
// one tile never holds back the loads of the next ones (NG = 2: up to
// nstages - 2 tiles in flight per SM).  Each group stages its rows in its own
// output buffers and stores them with TMA bulk copies.
// CS >= 0 fixes the class structure at compile time (bit 3: class 0 present,
// bits 0-2: classes 1-3 present), so only that combine and those loads are
// emitted; CS = -1 reads it from the descriptor.
// DS: direct stores -- consumers write rows and argmins straight to global
// memory (no staging buffers, no storer work), which frees the staging
// buffers' shared memory for more ring stages
template <typename T, int R, int R2, int DV, bool SP, bool NF, int NG, int GW, int CS = -1, bool DS = false>
// (registers: 2 groups of GW = 4 warps + producer + storer put 3 warps on one
// SM sub-partition: 168 per thread)
__global__ void __launch_bounds__((NG * GW + 1 + NG) * 32, 1)
    bk_fast_kernel(const FastDesc *__restrict__ Fg, InPtrs in, T *__restrict__ out,
                   uint8_t *__restrict__ arg, int64_t row_begin, int64_t t_begin, int64_t t_end) {
  using S = SrF<T>;
  using Acc = typename S::Acc;
  constexpr int kGT = GW * 32;  // threads per consumer group
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ FastHot f;
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ int32_t sbase[kMaxStages * 32];
  __shared__ int64_t rowstart[kMaxStages];
  // output staging handshake: ofull[g][b] completes when the GW warps of group
  // g have staged a tile in buffer b; oempty[g][b] when its bulk store has
  // read it; ostart[g][b] = that tile's first output row (relative)
  __shared__ uint64_t ofull[NG][kOutBufsMax], oempty[NG][kOutBufsMax];
  __shared__ int64_t ostart[NG][kOutBufsMax];
  __shared__ ProdSmem ps;  // producer's decode tables (the large ones in dynamic smem)
  {
    const int kk = Fg->hot.k, nh = Fg->hot.nH;
    ps.hstr = (int64_t *)(sm + Fg->hot.off_prod);
    for (int i = threadIdx.x; i < nh * kk; i += blockDim.x) ps.hstr[i] = Fg->hstr[i / kk][i % kk];
  }
  if (threadIdx.x < kMaxH) {
    ps.hrow[threadIdx.x] = Fg->hrow[threadIdx.x];
    ps.hrad[threadIdx.x] = (uint32_t)Fg->hrad[threadIdx.x];
    ps.shift[threadIdx.x] = Fg->shift[threadIdx.x];
  }
  {
    const int *src = (const int *)&Fg->hot;
    int *dst = (int *)&f;
    for (int i = threadIdx.x; i < (int)(sizeof(FastHot) / 4); i += blockDim.x) dst[i] = src[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GW);
    }
    for (int g = 0; g < NG; g++)
      for (int b = 0; b < kOutBufsMax; b++) {
        mbar_init(&ofull[g][b], GW);
        mbar_init(&oempty[g][b], 1);
      }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int k = f.k, Pmid = f.Pmid, nst = f.nstages;
  int32_t *offtab = (int32_t *)(sm + f.off_tab);
  int32_t *mrowoff = (int32_t *)(sm + f.off_mrow);
  // per-CTA tables: slice offset of every thread group, per input; row offset
  const bool qperm = Fg->qperm_on != 0;
  for (int idx = threadIdx.x; idx < (k + 1) * Pmid; idx += blockDim.x) {
    int jj = idx / Pmid, q = idx - jj * Pmid;
    if (qperm) q = Fg->qperm[q];
    int off = 0;
    for (int e = f.nmid - 1; e >= 0; e--) {
      int r = f.mrad[e], dg = q % r;
      q /= r;
      off += dg * (jj < k ? f.mstr[e][jj] : f.mrow[e]);
    }
    if (jj < k)
      offtab[idx] = off * (int)sizeof(T);
    else
      mrowoff[idx - k * Pmid] = off;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;

  if (warp >= NG * GW + 1) {  // ---- producer warps (one per group): TMA ring ----
    // producer p issues the tiles of group p (CTA tiles i = p mod NG, stages
    // i mod nst -- the ring length is a multiple of NG), so one producer's
    // batch decode overlaps the other's issuing
    const int lane = threadIdx.x & 31;
    const int p = warp - NG * GW - 1;
    ProdTiles pt;
    {
      int64_t *pb = (int64_t *)(sm + f.off_prod) + f.nH * k + p * 32 * (k + 1);
      pt.trow = pb;
      pt.tb = pb + 32;
    }
    const char *my_in = lane < k ? (const char *)in.p[f.in_idx[lane]] : nullptr;
    int s = p % nst, L = 0;
    uint32_t ph = (uint32_t)((p / nst) & 1);
    for (int64_t t = t_begin + blockIdx.x + (int64_t)p * gridDim.x; t < t_end; t += (int64_t)NG * gridDim.x) {
      if (L == 0) decode_batch(ps, pt, f, t, (int64_t)NG * gridDim.x, t_end);
      mbar_wait(&empty[s], ph ^ 1u);
      issue_tile(pt, f, my_in, L, s, sm, full, sbase, rowstart);
      s += NG;
      if (s >= nst) {
        s -= nst;
        ph ^= 1u;
      }
      L = (L + 1) & 31;
    }
    return;
  }
  const int PL = f.PL, es = (int)sizeof(T);
  const int nob = f.nout;

  if (DS && warp == NG * GW) return;  // direct stores: no storer work
  if (warp == NG * GW) {  // ---- storer warp: TMA bulk stores of staged tiles ----
    // tiles in CTA order (tile i: group i mod NG, its buffer (i / NG) mod nob);
    // the buffer of tile i - 1 is released once tile i is committed and at
    // most one store group is still reading shared memory
    const int lane = threadIdx.x & 31;
    int i = 0, pg = -1, pb = 0;
    for (int64_t t = t_begin + blockIdx.x; t < t_end; t += gridDim.x, i++) {
      const int g = i % NG, jg = i / NG, b = jg % nob;
      mbar_wait(&ofull[g][b], (uint32_t)((jg / nob) & 1));
      const int64_t o0 = ostart[g][b];
      T *outs = (T *)(sm + f.off_out + (g * nob + b) * f.out_bytes) + (int)((((uintptr_t)(out + o0)) & 15) / es);
      uint8_t *args = sm + f.off_arg + (g * nob + b) * f.arg_bytes + (int)(((uintptr_t)(arg + o0)) & 15);
      T *gout = out + o0;
      const int h = (int)(((16 - (((uintptr_t)gout) & 15)) & 15) / es);
      const int hh = min(h, PL);
      const int nmid = ((PL - hh) * es / 16) * 16 / es;
      const int tl = PL - hh - nmid;
      if (lane == 0 && nmid > 0) tma_store_1d(gout + hh, outs + hh, (uint32_t)(nmid * es));
      if (lane < hh) gout[lane] = outs[lane];
      if (lane < tl) gout[hh + nmid + lane] = outs[hh + nmid + lane];
      if (arg) {
        uint8_t *ga = arg + o0;
        const int ha = min((int)((16 - (((uintptr_t)ga) & 15)) & 15), PL);
        const int nmida = ((PL - ha) / 16) * 16;
        const int tla = PL - ha - nmida;
        if (lane == 0 && nmida > 0) tma_store_1d(ga + ha, args + ha, (uint32_t)nmida);
        if (lane < ha) ga[lane] = args[lane];
        if (lane < tla) ga[ha + nmida + lane] = args[ha + nmida + lane];
      }
      __syncwarp();  // ragged ends read before the buffer is released
      if (lane == 0) {
        bulk_commit();
        if (pg >= 0) {
          bulk_wait_read<1>();
          mbar_arrive(&oempty[pg][pb]);
        }
      }
      pg = g;
      pb = b;
    }
    if (lane == 0) bulk_wait_all();
    return;
  }

  // ---- consumer groups ----
  const int g = warp / GW;
  const int ctid = threadIdx.x - g * kGT;  // 0 .. kGT-1 inside the group
  const int c0 = f.cls_off[0], c1 = f.cls_off[1], c2 = f.cls_off[2], c3 = f.cls_off[3], c4 = f.cls_off[4];
  const int sel = CS >= 0 ? (CS & 7) : ((c2 > c1 ? 1 : 0) | (c3 > c2 ? 2 : 0) | (c4 > c3 ? 4 : 0));
  const bool has0 = CS >= 0 ? (CS & 8) != 0 : c1 > c0;
  const RowOff loff{f.rs1, f.rs2};  // in-tile row offsets of the group digits
  unsigned char *const obase = sm + f.off_out + g * nob * f.out_bytes;
  unsigned char *const abase = sm + f.off_arg + g * nob * f.arg_bytes;
  uint32_t oph = 0;  // use round of the group's staging buffers (parity)
  int s = g % nst, b = 0;
  uint32_t ph = (uint32_t)((g / nst) & 1);
  for (int64_t t = t_begin + blockIdx.x + (int64_t)g * gridDim.x; t < t_end; t += (int64_t)NG * gridDim.x) {
    mbar_wait(&full[s], ph);
    if (!DS) mbar_wait(&oempty[g][b], oph ^ 1u);  // staging buffer b: previous store has read it
    const int32_t *sb = sbase + s * 32;
    const int64_t o0 = rowstart[s] - row_begin;
    // staging: element l of this tile lives at index l + sh (16-byte phase of
    // its global address), so the aligned interior is one TMA bulk store
    const int sh = (int)((((uintptr_t)(out + o0)) & 15) / es);
    const int sha = (int)(((uintptr_t)(arg + o0)) & 15);
    T *outs = DS ? out + o0 : (T *)(obase + b * f.out_bytes) + sh;
    uint8_t *args = DS ? (arg ? arg + o0 : nullptr) : abase + b * f.arg_bytes + sha;
    for (int q = ctid; q < Pmid; q += kGT) {
      Acc P0[DV], P1[R][DV], P2[R2][DV], P3[R][R2][DV];
      // class 0 (no group digit): P0[v]
      if (has0) {
        const unsigned char *p = sm + sb[c0] + offtab[c0 * Pmid + q];
#pragma unroll
        for (int v = 0; v < DV; v++) P0[v] = (Acc)((const T *)p)[v];
#pragma unroll 1
        for (int jj = c0 + 1; jj < c1; jj++) {
          const unsigned char *pj = sm + sb[jj] + offtab[jj * Pmid + q];
#pragma unroll
          for (int v = 0; v < DV; v++) P0[v] = NF ? S::add_nc(P0[v], (Acc)((const T *)pj)[v]) : S::add(P0[v], (Acc)((const T *)pj)[v]);
        }
      } else {
#pragma unroll
        for (int v = 0; v < DV; v++) P0[v] = S::zero();
      }
      // class 1 (g1 only): P1[a][v]
      if (sel & 1) {
        const unsigned char *p = sm + sb[c1] + offtab[c1 * Pmid + q];
        const int s1 = f.sg1[c1];
#pragma unroll
        for (int a = 0; a < R; a++)
#pragma unroll
          for (int v = 0; v < DV; v++) P1[a][v] = (Acc)((const T *)(p + a * s1))[v];
#pragma unroll 1
        for (int jj = c1 + 1; jj < c2; jj++) {
          const unsigned char *pj = sm + sb[jj] + offtab[jj * Pmid + q];
          const int t1 = f.sg1[jj];
#pragma unroll
          for (int a = 0; a < R; a++)
#pragma unroll
            for (int v = 0; v < DV; v++) {
              const Acc x = (Acc)((const T *)(pj + a * t1))[v];
              P1[a][v] = NF ? S::add_nc(P1[a][v], x) : S::add(P1[a][v], x);
            }
        }
      }
      // class 2 (g2 only): P2[b][v]
      if (sel & 2) {
        const unsigned char *p = sm + sb[c2] + offtab[c2 * Pmid + q];
        const int s2 = f.sg2[c2];
#pragma unroll
        for (int bb = 0; bb < R2; bb++)
#pragma unroll
          for (int v = 0; v < DV; v++) P2[bb][v] = (Acc)((const T *)(p + bb * s2))[v];
#pragma unroll 1
        for (int jj = c2 + 1; jj < c3; jj++) {
          const unsigned char *pj = sm + sb[jj] + offtab[jj * Pmid + q];
          const int t2 = f.sg2[jj];
#pragma unroll
          for (int bb = 0; bb < R2; bb++)
#pragma unroll
            for (int v = 0; v < DV; v++) {
              const Acc x = (Acc)((const T *)(pj + bb * t2))[v];
              P2[bb][v] = NF ? S::add_nc(P2[bb][v], x) : S::add(P2[bb][v], x);
            }
        }
      }
      // class 3 (both): P3[a][b][v]
      if (sel & 4) {
        const unsigned char *p = sm + sb[c3] + offtab[c3 * Pmid + q];
        const int s1 = f.sg1[c3], s2 = f.sg2[c3];
#pragma unroll
        for (int a = 0; a < R; a++)
#pragma unroll
          for (int bb = 0; bb < R2; bb++)
#pragma unroll
            for (int v = 0; v < DV; v++) P3[a][bb][v] = (Acc)((const T *)(p + a * s1 + bb * s2))[v];
#pragma unroll 1
        for (int jj = c3 + 1; jj < c4; jj++) {
          const unsigned char *pj = sm + sb[jj] + offtab[jj * Pmid + q];
          const int t1 = f.sg1[jj], t2 = f.sg2[jj];
#pragma unroll
          for (int a = 0; a < R; a++)
#pragma unroll
            for (int bb = 0; bb < R2; bb++)
#pragma unroll
              for (int v = 0; v < DV; v++) {
                const Acc x = (Acc)((const T *)(pj + a * t1 + bb * t2))[v];
                P3[a][bb][v] = NF ? S::add_nc(P3[a][bb][v], x) : S::add(P3[a][bb][v], x);
              }
        }
      }
      const int row0 = mrowoff[q];
      T *outq = outs + row0;
      uint8_t *argq = args + row0;
      if constexpr (NF) {
        // (T = int32: Acc = uint32)
#define GBE_NF(h1, h2, h3) \
  combine_nf<R, R2, DV, h1, h2, h3>(P0, P1, P2, P3, (int32_t *)outq, argq, loff)
        switch (sel) {
          case 0: GBE_NF(false, false, false); break;
          case 1: GBE_NF(true, false, false); break;
          case 2: GBE_NF(false, true, false); break;
          case 3: GBE_NF(true, true, false); break;
          case 4: GBE_NF(false, false, true); break;
          case 5: GBE_NF(true, false, true); break;
          case 6: GBE_NF(false, true, true); break;
          default: GBE_NF(true, true, true); break;
        }
#undef GBE_NF
      } else {
        Acc gmax = S::zero();
        switch (sel) {
          case 0: combine<T, R, R2, DV, false, false, false, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
          case 1: combine<T, R, R2, DV, true, false, false, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
          case 2: combine<T, R, R2, DV, false, true, false, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
          case 3: combine<T, R, R2, DV, true, true, false, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
          case 4: combine<T, R, R2, DV, false, false, true, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
          case 5: combine<T, R, R2, DV, true, false, true, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
          case 6: combine<T, R, R2, DV, false, true, true, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
          default: combine<T, R, R2, DV, true, true, true, SP>(P0, P1, P2, P3, outq, argq, loff, gmax); break;
        }
        // a row whose minimum is infinite clamps every value to INF, so its
        // first index wins (A8); rare, so handled once per group
        if (S::kInt && gmax >= S::inf()) {
#pragma unroll
          for (int a = 0; a < R; a++)
#pragma unroll
            for (int bb = 0; bb < R2; bb++) {
              const int l = loff(a, bb);
              if ((uint32_t)outq[l] >= kInf) {
                outq[l] = (T)kInf;
                if (argq) argq[l] = 0;
              }
            }
        }
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);  // input stage free
    if (!DS) {
      fence_proxy_async_smem();  // staged rows -> async proxy (the storer's bulk copy)
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        if (ctid == 0) ostart[g][b] = o0;
        mbar_arrive(&ofull[g][b]);
      }
    }
    s += NG;
    if (s >= nst) {
      s -= nst;
      ph ^= 1u;
    }
    if (++b == nob) {
      b = 0;
      oph ^= 1u;
    }
  }
}

// ---------------------------------------------------------------------------
// dispatch table over (semiring, R, DV)

template <typename T, int R, int R2, int DV, bool SP, bool NF, int NG, int GW, int CS = -1, bool DS = false>
cudaError_t launch_one(const FastDesc *d, const InPtrs &in, void *out, uint8_t *arg, int64_t rb,
                       int64_t t0, int64_t t1, int grid, int block, int smem, cudaStream_t s) {
  auto kern = bk_fast_kernel<T, R, R2, DV, SP, NF, NG, GW, CS, DS>;
  // the shared-memory opt-in is per device: one bit per device ordinal
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  kern<<<grid, block, smem, s>>>(d, in, (T *)out, arg, rb, t0, t1);
  return cudaGetLastError();
}

// two consumer groups of 4 warps per CTA (one CTA per SM, shared ring; 10
// warps, 168 registers per thread).  Measured against 8-warp groups at 96
// registers (int32 shapes): each thread now owns ~2 register blocks per
// tile, so the per-tile work is amortised, and no shape is register-capped
// (C4 31.4 -> 29.6 ms, C3 MBE(16) 32.4 -> 31.4 ms; f64 shapes already used 4).
constexpr int ng_of(int, int, int, int) { return 2; }
constexpr int gw_of(int, int, int, int) { return 4; }

// the hottest shape (C4, C3: d = 3, two radix-3 group digits, infinity-free)
// with its class structure as a template parameter
template <int CS>
cudaError_t launch_333_cs(const FastDesc *d, const InPtrs &in, void *out, uint8_t *arg, int64_t rb, int64_t t0,
                          int64_t t1, int grid, int block, int smem, cudaStream_t s) {
  return launch_one<int32_t, 3, 3, 3, false, true, 2, 4, CS>(d, in, out, arg, rb, t0, t1, grid, block, smem, s);
}
template <int CS>
cudaError_t launch_333_cs_ds(const FastDesc *d, const InPtrs &in, void *out, uint8_t *arg, int64_t rb, int64_t t0,
                             int64_t t1, int grid, int block, int smem, cudaStream_t s) {
  return launch_one<int32_t, 3, 3, 3, false, true, 2, 4, CS, true>(d, in, out, arg, rb, t0, t1, grid, block, smem,
                                                                    s);
}
using Launch333 = cudaError_t (*)(const FastDesc *, const InPtrs &, void *, uint8_t *, int64_t, int64_t, int64_t,
                                  int, int, int, cudaStream_t);
constexpr Launch333 kLaunch333[16] = {
    launch_333_cs<0>, launch_333_cs<1>, launch_333_cs<2>,  launch_333_cs<3>,  launch_333_cs<4>,  launch_333_cs<5>,
    launch_333_cs<6>, launch_333_cs<7>, launch_333_cs<8>,  launch_333_cs<9>,  launch_333_cs<10>, launch_333_cs<11>,
    launch_333_cs<12>, launch_333_cs<13>, launch_333_cs<14>, launch_333_cs<15>};
constexpr Launch333 kLaunch333ds[16] = {
    launch_333_cs_ds<0>,  launch_333_cs_ds<1>,  launch_333_cs_ds<2>,  launch_333_cs_ds<3>,
    launch_333_cs_ds<4>,  launch_333_cs_ds<5>,  launch_333_cs_ds<6>,  launch_333_cs_ds<7>,
    launch_333_cs_ds<8>,  launch_333_cs_ds<9>,  launch_333_cs_ds<10>, launch_333_cs_ds<11>,
    launch_333_cs_ds<12>, launch_333_cs_ds<13>, launch_333_cs_ds<14>, launch_333_cs_ds<15>};

template <typename T, bool SP, bool NF>
cudaError_t dispatch(int R, int R2, int DV, int NGr, const FastDesc *d, const InPtrs &in, void *out,
                     uint8_t *arg, int64_t rb, int64_t t0, int64_t t1, int grid, int block,
                     int smem, cudaStream_t s, int cs = -1, bool ds = false) {
  if constexpr (sizeof(T) == 4 && NF && !SP) {
    static const bool cs_off = std::getenv("GBE_FAST_NO_CS") != nullptr;  // A/B knob
    if (ds && R == 3 && R2 == 3 && DV == 3 && cs >= 0)
      return kLaunch333ds[cs](d, in, out, arg, rb, t0, t1, grid, block, smem, s);
    if (!ds && R == 3 && R2 == 3 && DV == 3 && cs >= 0 && !cs_off)
      return kLaunch333[cs](d, in, out, arg, rb, t0, t1, grid, block, smem, s);
  }
#define GBE_CASE(r, r2, dv)                                                                                  \
  if (R == r && R2 == r2 && DV == dv) {                                                                      \
    constexpr int ng = ng_of((int)sizeof(T), r, r2, dv), gw = gw_of((int)sizeof(T), r, r2, dv);             \
    if (NGr != ng) return cudaErrorInvalidValue;                                                             \
    if (ds) return launch_one<T, r, r2, dv, SP, NF, ng, gw, -1, true>(d, in, out, arg, rb, t0, t1, grid, block, \
                                                                      smem, s);                              \
    return launch_one<T, r, r2, dv, SP, NF, ng, gw>(d, in, out, arg, rb, t0, t1, grid, block, smem, s);      \
  }
  GBE_CASE(2, 2, 2) GBE_CASE(2, 2, 3) GBE_CASE(2, 2, 4) GBE_CASE(2, 2, 5) GBE_CASE(3, 3, 2) GBE_CASE(3, 3, 3)
  GBE_CASE(3, 1, 2) GBE_CASE(3, 1, 3) GBE_CASE(3, 1, 4) GBE_CASE(3, 1, 5)
  GBE_CASE(4, 1, 2) GBE_CASE(4, 1, 3) GBE_CASE(4, 1, 4) GBE_CASE(4, 1, 5)
  GBE_CASE(5, 1, 2) GBE_CASE(5, 1, 3) GBE_CASE(5, 1, 4)
  GBE_CASE(4, 4, 2)
  if constexpr (sizeof(T) == 4) {  // f64 register budget (ptxas caps it at 168)
    GBE_CASE(3, 3, 4) GBE_CASE(3, 3, 5) GBE_CASE(4, 4, 3) GBE_CASE(5, 1, 5)
  }
#undef GBE_CASE
  return cudaErrorInvalidValue;
}

bool supported(int R, int R2, int DV, int es) {
  if (DV < 2 || DV > 5) return false;
  if (R2 == R) {
    if (R == 2) return true;
    if (R == 3) return DV <= 3 || es == 4;
    if (R == 4) return DV == 2 || (DV == 3 && es == 4);
    return false;
  }
  if (R2 != 1) return false;
  if (R == 3 || R == 4) return true;
  return R == 5 && (DV <= 4 || es == 4);
}

}  // namespace

// ---------------------------------------------------------------------------
// host: choose L (tile digits), the group digits, the tile order, the smem
// layout; false when the bucket does not fit this kernel (-> bk_generic)

namespace {
// Shared-memory bank conflicts of the consumers' loads and staging stores
// depend on which 32 mid-digit combinations a warp handles together: the
// natural order puts combinations whose offsets agree mod 32 banks in one
// warp (radix-3 strides: 2 wavefronts per LDS / STS on C4's largest
// buckets).  Greedy assignment: combinations in order of how crowded their
// residues are, each to the warp where it adds the fewest same-bank
// collisions, weighted by how many loads (stores) per register block the
// input (the output) issues.
void build_qperm(FastDesc &F, int es, int R, int R2, int Pmid, int64_t rows) {
  F.qperm_on = 0;
  // measured SLOWER on C4 (kernel sum 28.0 -> 29.2 ms: x57 7.09 -> 7.48,
  // x9 6.13 -> 6.47; the scattered argmin byte stores it causes are not in
  // its model), so it is off unless GBE_FAST_QPERM=1 (A/B knob)
  static const bool off = std::getenv("GBE_FAST_QPERM") == nullptr;
  const FastHot &f = F.hot;
  if (off || es != 4 || Pmid < 64 || Pmid > kMaxPmid || rows < (int64_t(1) << 22)) return;
  const int nw = (Pmid + 31) / 32;
  const int ns = f.k + 1;  // streams: inputs, then the output rows
  std::vector<int> res((size_t)Pmid * ns);
  std::vector<int> w(ns);
  for (int q = 0; q < Pmid; q++) {
    int x = q;
    std::vector<int> dg(f.nmid);
    for (int e = f.nmid - 1; e >= 0; e--) {
      dg[e] = x % f.mrad[e];
      x /= f.mrad[e];
    }
    for (int j = 0; j < ns; j++) {
      int64_t o = 0;
      for (int e = 0; e < f.nmid; e++) o += (int64_t)dg[e] * (j < f.k ? f.mstr[e][j] : f.mrow[e]);
      res[(size_t)q * ns + j] = (int)(o & 31);
    }
  }
  for (int j = 0; j < ns; j++) {  // loads (stores) per register block
    if (j == f.k) {
      w[j] = 2 * R * R2;  // outputs + argmins
      continue;
    }
    const bool h1 = f.sg1[j] != 0, h2 = f.sg2[j] != 0;
    w[j] = f.DV * (h1 ? R : 1) * (h2 ? R2 : 1);
  }
  std::vector<int> freq((size_t)ns * 32, 0);
  for (int q = 0; q < Pmid; q++)
    for (int j = 0; j < ns; j++) freq[(size_t)j * 32 + res[(size_t)q * ns + j]] += w[j];
  std::vector<int> order(Pmid);
  for (int q = 0; q < Pmid; q++) order[q] = q;
  std::vector<int> crowd(Pmid, 0);
  for (int q = 0; q < Pmid; q++)
    for (int j = 0; j < ns; j++) crowd[q] += freq[(size_t)j * 32 + res[(size_t)q * ns + j]];
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return crowd[a] > crowd[b]; });
  std::vector<int> cnt((size_t)nw * ns * 32, 0), fill(nw, 0);
  std::vector<std::vector<int>> slots(nw);
  for (int q : order) {
    int best = -1;
    int64_t bc = INT64_MAX;
    for (int wi = 0; wi < nw; wi++) {
      const int cap = wi == nw - 1 ? Pmid - 32 * (nw - 1) : 32;
      if (fill[wi] >= cap) continue;
      int64_t c = 0;
      for (int j = 0; j < ns; j++) c += (int64_t)w[j] * cnt[((size_t)wi * ns + j) * 32 + res[(size_t)q * ns + j]];
      c = c * 64 + fill[wi];  // ties: the emptier warp
      if (c < bc) {
        bc = c;
        best = wi;
      }
    }
    fill[best]++;
    slots[best].push_back(q);
    for (int j = 0; j < ns; j++) cnt[((size_t)best * ns + j) * 32 + res[(size_t)q * ns + j]]++;
  }
  int pos = 0;
  for (int wi = 0; wi < nw; wi++)
    for (int q : slots[wi]) F.qperm[pos++] = (uint16_t)q;
  F.qperm_on = 1;
}
}  // namespace

bool bkf_build(const gbe_bucket_desc &h, int64_t row_begin, int64_t row_end, int num_sms,
               FastDesc &F, BkfLaunch &L, bool noinf, bool ds) {
  const int m = h.nsep, k = h.ninputs, DV = h.d;
  const int es = h.semiring == GBE_MINSUM_I32 ? 4 : 8;
  if (m < 2 || k < 1 || k > 32 || DV < 2 || DV > 5) return false;
  if (row_end <= row_begin) return false;
  // tiny buckets: the tiled kernel's per-CTA setup (descriptor copy, offset
  // tables, mbarrier ring) costs more than the bucket; bk_generic is faster
  if ((row_end - row_begin) * DV < kMinCells) return false;
  static const int64_t kPLMax = [] {  // rows per tile cap (GBE_FAST_PLMAX: tuning knob)
    const char *e = std::getenv("GBE_FAST_PLMAX");
    return e ? std::max<int64_t>(8, std::atoll(e)) : int64_t(16384);
  }();
  // one CTA per SM: dynamic shared-memory budget; GBE_FAST_SMEM_KB overrides
  // it for tuning experiments
  static const char *smem_env = std::getenv("GBE_FAST_SMEM_KB");
  static const int kStagesMax = [] {
    const char *e = std::getenv("GBE_FAST_STAGES");
    return e ? std::max(2, std::min(kMaxStages, std::atoi(e))) : kMaxStages;
  }();
  // stages wanted in the ring: with two consumer groups, two stages can be
  // held by compute while the rest are in flight
  static const int kStagesWant = [] {
    const char *e = std::getenv("GBE_FAST_WANT_STAGES");
    return e ? std::max(2, std::min(kMaxStages, std::atoi(e))) : 4;
  }();
  // inputs' sizes (cells) to find the largest
  auto has = [&](int j, int p) { return h.stride[j][p] != 0; };
  std::vector<int64_t> cells(k, DV);
  for (int j = 0; j < k; j++)
    for (int p = 0; p < m; p++)
      if (has(j, p)) cells[j] *= h.radix[p];
  int big = 0;
  for (int j = 1; j < k; j++)
    if (cells[j] > cells[big]) big = j;

  // pass 0: the largest tile whose ring holds kStagesWant stages; pass 1: the
  // largest tile that fits at all
  for (int pass = 0; pass < 2; pass++) {
  for (int nl = m; nl >= 2; nl--) {
    int64_t PL = 1;
    for (int p = m - nl; p < m; p++) PL *= h.radix[p];
    if (PL > kPLMax) continue;
    // group digits: the pair (equal radix) or single digit with a supported
    // register-blocking shape that minimises the per-cell shared-memory
    // loads sum_j R^-|G \ S_j|; pairs win ties (more reuse per group)
    double bestc = 1e30;
    int g1 = -1, g2 = -1, bestw = 1 << 30;
    static const bool single_only = std::getenv("GBE_FAST_SINGLE") != nullptr;  // tuning knob
    // ties on the load cost: the pair whose first warp's 32 output rows
    // (register-block row 0 of slots q = 0..31) fall in the fewest shared-
    // memory banks per bank -- the staging stores' conflict degree -- then
    // the later pair (GBE_FAST_BANKTIE=0: the later pair only)
    static const bool banktie = [] {
      const char *e = std::getenv("GBE_FAST_BANKTIE");
      return !(e && std::atoi(e) == 0);
    }();
    std::vector<int64_t> rowst_all(m);
    {
      int64_t r = 1;
      for (int p = m - 1; p >= 0; p--) {
        rowst_all[p] = r;
        r *= h.radix[p];
      }
    }
    auto store_ways = [&](int a, int b) {  // max rows of warp 0 per bank
      if (!banktie) return 0;
      std::vector<int> mids;
      for (int p = m - nl; p < m; p++)
        if (p != a && p != b) mids.push_back(p);
      int cnt[32] = {0}, w = 0;
      for (int q = 0; q < 32; q++) {
        int x = q;
        int64_t row = 0;
        for (int e = (int)mids.size() - 1; e >= 0; e--) {
          row += (int64_t)(x % h.radix[mids[e]]) * rowst_all[mids[e]];
          x /= h.radix[mids[e]];
        }
        if (x) break;  // fewer than 32 slots
        w = std::max(w, ++cnt[row & 31]);
      }
      return w;
    };
    // GBE_FAST_BANKTOL (tuning knob): also accept pairs whose load cost is
    // within that fraction of the best when their stores conflict less
    static const double banktol = [] {
      const char *e = std::getenv("GBE_FAST_BANKTOL");
      return e ? std::atof(e) : 0.0;
    }();
    double minc = 1e30;
    for (int a = m - nl; a < m && !single_only; a++)
      for (int b = a + 1; b < m; b++) {
        int R = h.radix[a];
        if (h.radix[b] != R || !supported(R, R, DV, es)) continue;
        double c = 0;
        for (int j = 0; j < k; j++) c += 1.0 / ((has(j, a) ? 1 : R) * (has(j, b) ? 1 : R));
        minc = std::min(minc, c);
      }
    const double cap = minc * (1.0 + banktol) + 1e-12;
    for (int a = m - nl; a < m && !single_only; a++)
      for (int b = a + 1; b < m; b++) {
        int R = h.radix[a];
        if (h.radix[b] != R || !supported(R, R, DV, es)) continue;
        double c = 0;
        for (int j = 0; j < k; j++) c += 1.0 / ((has(j, a) ? 1 : R) * (has(j, b) ? 1 : R));
        if (c > cap) continue;
        const int w = store_ways(a, b);
        if (w < bestw || (w == bestw && (c < bestc - 1e-12 || (c < bestc + 1e-12 && b > g2)))) {
          bestc = c;
          g1 = a;
          g2 = b;
          bestw = w;
        }
      }
    if (g1 < 0)
      for (int a = m - nl; a < m; a++) {
        int R = h.radix[a];
        if (!supported(R, 1, DV, es)) continue;
        double c = 0;
        for (int j = 0; j < k; j++) c += 1.0 / (has(j, a) ? 1 : R);
        if (c < bestc - 1e-12 || (c < bestc + 1e-12 && a > g1)) {
          bestc = c;
          g1 = a;
        }
      }
    if (g1 < 0) continue;
    const int R = h.radix[g1];
    const int R2 = g2 >= 0 ? R : 1;
    const int64_t Pmid = PL / (R * R2);
    if (row_begin % PL || row_end % PL) continue;
    const int NG = ng_of(es, R, R2, DV), GW = gw_of(es, R, R2, DV);
    const size_t kSmemMax = (size_t)(smem_env ? std::atoi(smem_env) : 220) * 1024;
    const int min_st = pass == 0 ? std::max(kStagesWant, 2 * NG) : NG;
    // classes
    std::memset(&F, 0, sizeof(F));
    FastHot &f = F.hot;
    f.k = k;
    f.es = es;
    f.PL = (int32_t)PL;
    f.Pmid = (int32_t)Pmid;
    f.R = R;
    f.DV = DV;
    int jj = 0;
    for (int c = 0; c < 4; c++) {
      f.cls_off[c] = jj;
      for (int j = 0; j < k; j++) {
        int cls = (has(j, g1) ? 1 : 0) + (g2 >= 0 && has(j, g2) ? 2 : 0);
        if (cls != c) continue;
        f.in_idx[jj] = j;
        f.sg1[jj] = (int32_t)(h.stride[j][g1] * es);  // bytes
        f.sg2[jj] = g2 >= 0 ? (int32_t)(h.stride[j][g2] * es) : 0;
        int64_t sl = DV;
        for (int p = m - nl; p < m; p++)
          if (has(j, p)) sl *= h.radix[p];
        f.slen[jj] = (int32_t)sl;
        F.shift[jj] = h.shift[j];
        jj++;
      }
    }
    f.cls_off[4] = jj;
    // every input's tile slice must be ONE contiguous range of slen elements:
    // the tile digits it has, walked from the least significant, carry the
    // dense strides DV, DV*r, ... (canonical layouts always do; the bare
    // primitive accepts arbitrary strides, which go to bk_generic)
    bool dense = true;
    for (int j = 0; j < k && dense; j++) {
      int64_t want = DV;
      for (int p = m - 1; p >= m - nl; p--) {
        if (!has(j, p)) continue;
        if (h.stride[j][p] != want) dense = false;
        want *= h.radix[p];
      }
    }
    if (!dense) continue;
    // mid digits (L minus g1, g2), natural order; FastHot holds at most 12
    // (radix-1 digits would let the count exceed it)
    if (nl - (g2 >= 0 ? 2 : 1) > 12) continue;
    f.nmid = 0;
    int64_t rowst = 1;
    std::vector<int64_t> rowstride(m);
    for (int p = m - 1; p >= 0; p--) {
      rowstride[p] = rowst;
      rowst *= h.radix[p];
    }
    for (int p = m - nl; p < m; p++) {
      if (p == g1 || p == g2) continue;
      int e = f.nmid++;
      f.mrad[e] = h.radix[p];
      f.mrow[e] = (int32_t)rowstride[p];
      for (int q = 0; q < k; q++) f.mstr[e][q] = (int32_t)h.stride[f.in_idx[q]][p];
    }
    f.rs1 = (int32_t)rowstride[g1];
    f.rs2 = g2 >= 0 ? (int32_t)rowstride[g2] : 0;
    build_qperm(F, es, R, R2, (int)Pmid, row_end - row_begin);
    // H digits: natural order; for a full-range launch, digits absent from
    // the largest input go last (fastest) so their re-reads hit L2
    std::vector<int> hd;
    for (int p = 0; p < m - nl; p++) hd.push_back(p);
    const bool full = row_begin == 0 && row_end == h.rows;
    if (full)
      order_high_digits(h, hd.data(), (int)hd.size());
    f.nH = (int32_t)hd.size();
    if (f.nH > 31) continue;
    int64_t div = 1;
    for (int e = f.nH - 1; e >= 0; e--) {
      int p = hd[e];
      F.hrad[e] = h.radix[p];
      F.hdiv[e] = div;
      div *= h.radix[p];
      F.hrow[e] = rowstride[p];
      for (int q = 0; q < k; q++) F.hstr[e][q] = h.stride[f.in_idx[q]][p];
    }
    if (!full) {  // natural order: tile index = row / PL
      // (hd already natural)
    }
    // shared-memory layout
    size_t off = 0;
    for (int q = 0; q < k; q++) {
      f.soff[q] = (int32_t)off;
      off += ((size_t)f.slen[q] * es + 32 + 15) & ~size_t(15);
    }
    f.stage_bytes = (int32_t)off;
    f.out_bytes = (int32_t)(((size_t)PL * es + 16 + 127) & ~size_t(127));
    f.arg_bytes = (int32_t)(((size_t)PL + 16 + 127) & ~size_t(127));
    // 3 staging buffers when they fit beside the wanted ring (the store of
    // a tile then has a whole tile of compute to drain), else 2
    const size_t tabs = (size_t)(k + 1) * Pmid * 4 + 256 + 8 * ((size_t)f.nH * k + 64 * (size_t)(k + 1)) + 256;
    const size_t obuf = (size_t)NG * ((size_t)f.out_bytes + f.arg_bytes);
    static const int kNob = [] {  // GBE_FAST_NOUT: tuning knob (2 or 3)
      const char *e = std::getenv("GBE_FAST_NOUT");
      return e ? std::max(1, std::min(kOutBufsMax, std::atoi(e))) : kOutBufsMax;
    }();
    int nob = ds ? 0 : kNob;  // direct stores: no staging buffers
    while (nob > std::min(2, kNob) && obuf * nob + tabs + (size_t)min_st * off > kSmemMax) nob--;
    f.nout = nob;
    size_t fixed = obuf * nob + tabs;
    // the ring length is a multiple of NG: stage s then always serves group
    // s mod NG, so a group waiting on a stage has consumed that stage's
    // previous round itself and the mbarrier parity wait cannot alias a
    // phase two rounds back (with an odd ring a group could wait on a stage
    // whose previous round, the other group's, was not even issued yet)
    int nst = kStagesMax - kStagesMax % NG;
    while (nst > min_st && fixed + nst * off > kSmemMax) nst -= NG;
    if (nst < NG || fixed + nst * off > kSmemMax) continue;
    f.nstages = nst;
    off = nst * off;
    f.off_out = (int32_t)off;
    off += (size_t)NG * nob * f.out_bytes;
    f.off_arg = (int32_t)off;
    off += (size_t)NG * nob * f.arg_bytes;
    f.off_tab = (int32_t)off;
    off += (size_t)k * Pmid * 4;
    f.off_mrow = (int32_t)off;
    off += (size_t)Pmid * 4;
    off = (off + 127) & ~size_t(127);
    f.off_prod = (int32_t)off;  // producer decode tables: hstr[nH][k], 2 x (trow[32], tb[32][k])
    off += 8 * ((size_t)f.nH * k + 2 * 32 * (size_t)(k + 1));
    off = (off + 127) & ~size_t(127);
    if (off > kSmemMax) continue;
    L.smem = (int)off;
    L.cs = (f.cls_off[1] > f.cls_off[0] ? 8 : 0) | (f.cls_off[2] > f.cls_off[1] ? 1 : 0) |
           (f.cls_off[3] > f.cls_off[2] ? 2 : 0) | (f.cls_off[4] > f.cls_off[3] ? 4 : 0);
    L.NG = NG;
    L.g1 = g1;
    L.g2 = g2;
    L.nf = noinf && es == 4 && h.semiring == GBE_MINSUM_I32;
    L.ds = ds;
    L.block = (NG * GW + 1 + NG) * 32;
    L.t_begin = row_begin / PL;
    L.t_end = row_end / PL;
    if (L.t_end >= (int64_t(1) << 32)) return false;  // the producer decodes 32-bit tile indices
    int per_sm = (int)std::min<size_t>(std::max<size_t>(1, (220 * 1024) / (off + 4096)), 2048 / L.block);
    per_sm = std::max(1, std::min(per_sm, NG == 2 ? 1 : 8));
    int64_t tiles = L.t_end - L.t_begin;
    L.grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms * per_sm));
    L.R = R;
    L.R2 = R2;
    L.DV = DV;
    L.es = es;
    L.sp = h.semiring == GBE_SUMPROD_F64;
    return true;
  }
  }
  return false;
}

cudaError_t bkf_launch(const FastDesc *dev_f, const BkfLaunch &L, const InPtrs &in, void *out,
                       uint8_t *arg, int64_t row_begin, cudaStream_t s) {
  if (L.sp)
    return dispatch<double, true, false>(L.R, L.R2, L.DV, L.NG, dev_f, in, out, arg, row_begin, L.t_begin,
                                         L.t_end, L.grid, L.block, L.smem, s, -1, L.ds);
  if (L.es == 8)
    return dispatch<double, false, false>(L.R, L.R2, L.DV, L.NG, dev_f, in, out, arg, row_begin, L.t_begin,
                                          L.t_end, L.grid, L.block, L.smem, s, -1, L.ds);
  if (L.nf)
    return dispatch<int32_t, false, true>(L.R, L.R2, L.DV, L.NG, dev_f, in, out, arg, row_begin, L.t_begin,
                                          L.t_end, L.grid, L.block, L.smem, s, L.cs, L.ds);
  return dispatch<int32_t, false, false>(L.R, L.R2, L.DV, L.NG, dev_f, in, out, arg, row_begin, L.t_begin,
                                         L.t_end, L.grid, L.block, L.smem, s, -1, L.ds);
}

}  // namespace gbe
