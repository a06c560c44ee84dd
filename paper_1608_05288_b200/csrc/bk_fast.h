// bk_fast.h — descriptor and launcher of the tiled TMA bucket kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace gbe {

constexpr int kMaxPmid = 8192;  // PL <= 16384 rows, R * R2 >= 2

// Fields every CTA copies into shared memory (all int32).
struct FastHot {
  int32_t k, es, PL, Pmid, R, DV, nmid, nH;  // R: radix of g1 (g2 has R or is absent)
  int32_t cls_off[5];    // input class ranges: none / g1 / g2 / both
  int32_t in_idx[32];    // class-ordered input -> original input
  int32_t sg1[32], sg2[32];  // byte strides of the group digits (0 if absent)
  int32_t slen[32];      // slice length (elements) per tile
  int32_t soff[32];      // byte offset of the slice inside a stage
  int32_t stage_bytes;
  int32_t rs1, rs2;      // in-tile row strides of g1, g2
  int32_t mrad[12], mrow[12];  // middle digits (L minus group), most significant first
  int32_t mstr[12][32];  // their element strides per input
  int32_t off_out, off_arg, off_tab, off_mrow, off_prod;
  int32_t nstages, out_bytes, arg_bytes, nout;
};

struct FastDesc {
  FastHot hot;
  int32_t hrad[32];      // high digits in tile-enumeration order
  int32_t pad2;
  int64_t hdiv[32];      // tile-index divisor of each high digit
  int64_t hrow[32];      // output row stride of each high digit
  int64_t hstr[32][32];  // element stride per high digit, per (class-ordered) input
  int64_t shift[32];
  // thread-block slot q -> mid-digit combination (the in-tile offsets of slot
  // q are those of combination qperm[q]); chosen on the host so that the 32
  // combinations a warp handles together hit distinct shared-memory banks
  // (qperm_on = 0: identity)
  int32_t qperm_on, pad3;
  uint16_t qperm[kMaxPmid];
};

struct BkfLaunch {
  int R = 0, R2 = 0, DV = 0, es = 4;
  bool sp = false;  // sum-product elimination (GBE_SUMPROD_F64)
  bool nf = false;  // infinity-free int32 tables: packed-key argmin (no clamps)
  int NG = 1;       // consumer groups per CTA
  int g1 = -1, g2 = -1;  // group (register-blocking) digits
  int cs = -1;           // class structure (bit 3: class 0 present, bits 0-2: classes 1-3)
  bool ds = false;       // direct stores: consumers write rows + argmins to global memory (no staging buffers)
  int grid = 1, block = 256, smem = 0;
  int64_t t_begin = 0, t_end = 0;
};

bool bkf_build(const gbe_bucket_desc &h, int64_t row_begin, int64_t row_end, int num_sms,
               FastDesc &F, BkfLaunch &L, bool noinf = false, bool ds = false);
cudaError_t bkf_launch(const FastDesc *dev_f, const BkfLaunch &L, const InPtrs &in, void *out,
                       uint8_t *arg, int64_t row_begin, cudaStream_t s);

}  // namespace gbe
