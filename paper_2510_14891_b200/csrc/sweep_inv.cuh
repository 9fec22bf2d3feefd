// Gamma^-1 by the multi-CTA blocked sweep (sweep_inv.cu), for the CP-ALS solve.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace cpk {

// R rounded up to whole 32 x 32 tiles (the leading dimension of Gamma^-1)
int64_t sweep_padded(int64_t R);
// Workspace of sweep_inverse: the Rp x Rp matrix (Gamma^-1 on exit, at the
// start of `work`), two tile panels, D, and the info word.
size_t sweep_factor_bytes(int64_t R);
// CTAs of a full-machine launch for this R (one (C)-phase item each, capped
// by co-residency)
int sweep_default_ctas(int64_t R);
// Gamma + eps tr(Gamma)/R I  ->  its inverse (Rp x Rp, row-major, both
// triangles) at `work`; *info = 0, or potrf's 1-based failing column.  One
// cooperative launch of `ctas` CTAs (0 = sweep_default_ctas) on `st`.
int sweep_inverse(const double* gamma, int64_t R, double eps, void* work, size_t work_bytes, int* info, int ctas,
                  cudaStream_t st);
const double* sweep_inverse_matrix(const void* work);

}  // namespace cpk
