// Internal interface between the MTTKRP front end (mttkrp.cu) and the
// warp-specialized TMA kernel (mttkrp_ws.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cpk_b200.h"

namespace cpk {

struct WsRequest {
  const double* y;
  int d, k, n_o;
  int64_t dims[CPK_MAX_MODES];
  const double* factors[CPK_MAX_MODES];
  int64_t ld[CPK_MAX_MODES];
  int64_t rank;
  int rank_tile, block_k, splits;
  double* out;
  int64_t ldo, out_split_stride;
  const double* lam;
};

// TMA tile for a rank tile (64 | 128 | 256): rows per CTA and chunk depth.
bool ws_shape(int rank_tile, int* block_rows, int* block_k);
bool ws_eligible(const WsRequest& r);
int launch_ws(const WsRequest& r, cudaStream_t st);

}  // namespace cpk
