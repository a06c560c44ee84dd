// bk_stream.h — descriptor and launcher of the streaming bucket kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace gbe {

// Device descriptor (read through the read-only cache).
struct StreamDesc {
  int32_t k, d, nlow, PL, nhigh, pad;
  // broadcast digit (register reuse): an in-tile output digit b the largest
  // input lacks; a lane's rows are the bd_rad rows that differ only in b (in-
  // tile stride bd_stride), and every input without b is loaded once for all
  // of them (bit j of bd_has: input j has b)
  int32_t bd_rad, bd_stride;
  uint32_t bd_has, pad2;
  int64_t bd_rowstride;  // 0: b is an in-tile digit of the row order; else b is a high
                         // digit placed on top of the tile: output row stride of b
  // a second broadcast digit b2 (high, radix 2, on top of the tile below b):
  // the lane's rows are then (b, b2) pairs; bit j of bd_has2: input j has b2
  uint32_t bd_has2, pad4;
  int64_t bd_rowstride2;  // output row stride of b2
  // blocked high digits: hx > 0 puts hx high output digits on top of the
  // warp-tile (in-tile digits 0..hx-1) so an input lacking them re-reads its
  // slice inside one tile (L1) instead of across tiles; the tile's rows are
  // then not contiguous: output row of in-tile digit q has stride lrowst[q]
  int32_t hx, pad3;
  int64_t lrowst[GBE_MAX_SEP];
  int32_t lrad[GBE_MAX_SEP];       // low (in-tile) digits, most significant first
  int32_t lstr[GBE_MAX_SEP][32];   // their element strides per input
  int32_t hrad[32];                // high digits (radix > 1), most significant first
  int64_t hdiv[32];                // tile-index divisor of each high digit
  int64_t hstr[32][32];            // [digit][input] element stride
  int64_t hrow[32];                // output-row stride of each high digit
  int64_t pf_bytes[32];            // bytes of input j's tile slice to prefetch into L2 (0: none)
  int64_t shift[32];
  // staged mode: dynamic shared memory = [k*PL offset table][per-warp
  // mbarrier pairs at stg_off][per-warp buffer pairs of stg_buf bytes];
  // input j's slice (stg_slice bytes) at stg_soff within a buffer
  int32_t stg_off, stg_buf;
  int32_t stg_soff[32], stg_slice[32];
};

struct BksLaunch {
  int d = 1, k = 1, grid = 1, smem = 0;
  int vec = 0;  // elements per vector load when the layout allows it (0: scalar)
  int bd = 0;   // broadcast digits: rows per lane (0: off)
  int bd2 = 1;  // radix of the second broadcast digit (1: one digit)
  int hx = 0;   // blocked high digits on top of the warp-tile (0: none)
  bool f64 = false, sp = false;
  bool natural = true;  // tiles in row order (partial row ranges); else reordered for L2 reuse
  bool pf_ok = false;   // some input's tile slice can be prefetched into L2 (dense, canonical layout)
  bool pf = false;      // prefetch on (default: k >= 2 inputs; the executor's autotuning may flip it)
  int sms = 1;          // SMs of the device (the grid is one wave of resident CTAs)
  bool stg = false;     // staged mode: per-warp TMA double buffers of the input slices
  int64_t t0 = 0, ntiles = 0;
};

// false when the descriptor does not fit (more than 32 high digits of radix > 1)
// stage: build the staged-mode descriptor (false when the slices are not
// dense ranges or d is outside 2..5 or sum-product)
// pl_cap_rows > 0: warp-tiles of at most that many rows
bool bks_build(const gbe_bucket_desc &h, int64_t row_begin, int64_t row_end, int num_sms, StreamDesc &S,
               BksLaunch &L, bool stage = false, int pl_cap_rows = 0);
cudaError_t bks_launch(const StreamDesc *dev_s, const BksLaunch &L, const InPtrs &in, void *out, uint8_t *arg,
                       int64_t row_begin, int64_t row_end, cudaStream_t s);
// lanes that split one row's domain (1 for d <= 5, up to 32)
int bks_lanes_per_row(int d);

}  // namespace gbe
