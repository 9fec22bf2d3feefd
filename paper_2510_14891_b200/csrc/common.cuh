// Shared helpers for the cpk_b200 C ABI: status plumbing and small PTX wrappers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "cpk_b200.h"

namespace cpk {

// Per-thread last error message (cpk_last_error).
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CPK_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return CPK_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- cp.async (LDGSTS) with zero fill: src_bytes < cp bytes pads with 0 ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- split-K as an ordered chain into G (the private-copy merge of
// mttkrp._run_private_copy, mttkrp.py:279-286, without the partial copies).
// Split z of an output tile waits until splits 0..z-1 have added their
// partials into G, adds its own (G = P_0 on z = 0), folds lam when it is the
// last split, and hands over: G = (((P_0 + P_1) + P_2) + ...) * lam, the
// same additions in the same order as splitk_reduce_f64, so the result is
// bit-identical to the workspace merge and run-to-run reproducible.  The
// predecessor is `tiles` CTAs earlier in the launch order, dispatched
// before this one, so the chain always progresses; the planner uses it only
// when that distance is at least half the resident CTAs (waits are then at
// most one epilogue long).  sem: one counter per output tile, zeroed before
// the first launch of an MTTKRP.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void chain_wait(const int* sem, int z) {
  while (ld_acquire_gpu(sem) < z) __nanosleep(128);
}

// L2 eviction policies for the chain's running sum: it is re-read by the
// next split of the tile about a tile-row of CTAs later, while the tensor
// streams through L2, so its lines are kept (evict_last) until the last
// split, whose store releases them (evict_first).
__device__ __forceinline__ uint64_t l2_policy_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_release() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_l2_hint2(const double* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_l2_hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_l2_hint2(double* a, double x, double y, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(a), "d"(x), "d"(y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_l2_hint(double* a, double x, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(a), "d"(x), "l"(pol) : "memory");
}

// Where an epilogue writes: a partial copy or the final G (plain stores), or
// G as the split chain's running sum (L2 hints; add = z > 0).
struct OutMode {
  bool chain, add, fold;
  bool hint;  // use the L2 policy `pol` on every access
  uint64_t pol;
};

// The epilogue store of two adjacent outputs (j, j + 1) of a row: optional
// running-sum add (chain, z > 0; L2 reads, the tile was written by another
// SM), optional lam fold, one 16-byte store when both columns are live.
__device__ __forceinline__ void store_pair(double* dst, int64_t j, int64_t R, bool vec, double v0, double v1,
                                           const double* lam, const OutMode& m) {
  const bool both = j + 1 < R && vec;
  if (m.add && !m.hint) {
    if (both) {
      const double2 o = __ldcg(reinterpret_cast<const double2*>(dst));
      v0 = o.x + v0;
      v1 = o.y + v1;
    } else {
      if (j < R) v0 = __ldcg(dst) + v0;
      if (j + 1 < R) v1 = __ldcg(dst + 1) + v1;
    }
  } else if (m.add) {
    if (both) {
      const double2 o = ld_l2_hint2(dst, m.pol);
      v0 = o.x + v0;
      v1 = o.y + v1;
    } else {
      if (j < R) v0 = ld_l2_hint(dst, m.pol) + v0;
      if (j + 1 < R) v1 = ld_l2_hint(dst + 1, m.pol) + v1;
    }
  }
  if (m.fold) {
    if (j < R) v0 *= lam[j];
    if (j + 1 < R) v1 *= lam[j + 1];
  }
  if (m.hint) {
    if (both) {
      st_l2_hint2(dst, v0, v1, m.pol);
    } else {
      if (j < R) st_l2_hint(dst, v0, m.pol);
      if (j + 1 < R) st_l2_hint(dst + 1, v1, m.pol);
    }
  } else if (both) {
    *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
  } else {
    if (j < R) dst[0] = v0;
    if (j + 1 < R) dst[1] = v1;
  }
}

// Chain state of split z: add for z > 0, lam on the last split, the L2 policy.
// Without the hints the running sum went to DRAM between splits (c4: 2.05
// GB written, +0.6 GB read per launch); evict_first on the partial copies
// changed nothing (profiles/r02_chain_exp2.log).
__device__ __forceinline__ OutMode chain_mode(bool chain, int z, int n_splits, bool have_lam) {
  OutMode m;
  m.chain = chain;
  m.add = chain && z > 0;
  m.fold = have_lam && (!chain || z == n_splits - 1);
  m.hint = chain;
  m.pol = chain ? (z == n_splits - 1 ? l2_policy_release() : l2_policy_keep()) : 0;
  return m;
}

}  // namespace cpk
