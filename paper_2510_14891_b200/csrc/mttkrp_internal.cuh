// Internal interface between the MTTKRP front end (mttkrp.cu) and the
// warp-specialized TMA kernel (mttkrp_ws.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cpk_b200.h"

namespace cpk {

// FP64 math of the warp-specialized kernel's consumers.
enum { WS_MATH_DFMA = 0, WS_MATH_DMMA = 1 };

struct WsRequest {
  const double* y;
  int d, k, n_o;
  int64_t dims[CPK_MAX_MODES];
  const double* factors[CPK_MAX_MODES];
  int64_t ld[CPK_MAX_MODES];
  int64_t rank;
  int rank_tile, block_k, splits;
  int math;  // WS_MATH_*
  int32_t y0, y1, z0, z1;  // row blocks / splits of this launch (y1, z1 exclusive)
  double* out;
  int64_t ldo, out_split_stride;
  const double* lam;
  int* sem;  // split-K chain counters (common.cuh), or nullptr
  int fold;  // Khatri-Rao fold: factors[f] is W = KR(A_f, A_o0), rows i_f + I_f i_o0 (WsParams::fold)
};

// TMA tile for a rank tile (DMMA 16 | 32 | 64 | 128 | 256, DFMA 64 | 128 | 256) and math: rows per CTA and chunk depth.
bool ws_shape(int rank_tile, int math, int* block_rows, int* block_k);
bool ws_eligible(const WsRequest& r);
int launch_ws(const WsRequest& r, cudaStream_t st);

}  // namespace cpk
