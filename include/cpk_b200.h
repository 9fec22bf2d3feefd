/*
 * cpk_b200.h -- C ABI of the B200-native matrix-free dense MTTKRP and the
 * CP-ALS step kernels that sit behind it.
 *
 * The reference package (`cpkern`, Python + numba, /root/reference/pkg) has no
 * C interface; its "FFI" into compiled code is the numba kernel signature
 *
 *     tile_kernel(data f64[N], dims i64[d], strides i64[d], k,
 *                 fm f64[], foff i64[d], lam f64[R], r, f_cols, n_t, gp)
 *                                      (pkg/src/cpkern/_kernels.py:162-174)
 *
 * i.e. flat buffers, int64 metadata and a caller-owned output.  The entry
 * points below keep that shape with DEVICE pointers: the tensor is one flat
 * float64 buffer in first-mode-fastest order (dtensor.py:3-7), factors are
 * row-major float64 (kruskal.py:18-22, one device pointer per mode instead of
 * the packed `fm`/`foff` pair, _kernels.py:25-36), weights are folded exactly
 * once (README.md:155-156), and the result is the I_k x R row-major matrix
 * (mttkrp.py:114-117).  Every call is stream-ordered and asynchronous on the
 * caller's cudaStream_t (passed as void*), never allocates on the hot path
 * (the split-K workspace is caller-provided), and returns a status code that
 * maps 1:1 onto the reference's exception classes (errors.py:4-25).
 *
 * No torch types cross this boundary.  Python binds it with ctypes
 * (paper_2510_14891_b200/_lib.py); INTEGRATION.md shows the binding.
 */
#ifndef CPK_B200_H
#define CPK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  errors.py:4-25: CpkernError > {ShapeError, IndexRangeError,
 * ParameterError, ResourceError, FormatError}; CUDA and NCCL failures are new
 * (the reference has no device) and surface as CpkernError subclasses. */
enum {
  CPK_OK = 0,
  CPK_ERR_SHAPE = 1,     /* ShapeError      (mttkrp.py:120-122)          */
  CPK_ERR_INDEX = 2,     /* IndexRangeError (mttkrp.py:123-124, 248-249) */
  CPK_ERR_PARAM = 3,     /* ParameterError  (mttkrp.py:76-89)          */
  CPK_ERR_RESOURCE = 4,  /* ResourceError   (workspace too small)        */
  CPK_ERR_CUDA = 5,      /* launch / runtime failure                     */
  CPK_ERR_NOT_PD = 6,    /* Cholesky failed: Gamma not positive definite */
  CPK_ERR_LIB = 7,       /* cuSOLVER failure                             */
  CPK_ERR_FORMAT = 8     /* FormatError     (dtensor.py:359-382)         */
};

#define CPK_MAX_MODES 16

/* Kernel knobs.  Mirrors MttkrpPlan (mttkrp.py:53-89): `unroll` (F) and
 * `tile_volume` (N_T) keep their meaning; `rank_tile` is the GPU rank tile
 * (the paper's F*b_y column block); `splits` is the number of CTAs sharing
 * one output tile along the contraction (the reference's tiles-per-slice,
 * mttkrp.py:354-355).  Zero in any field means "choose" (cpk_plan_resolve). */
typedef struct cpk_plan {
  int32_t rank_tile;    /* 0 | 16 | 32 | 64 | 128 | 256 (engine-dependent) */
  int32_t block_rows;   /* 0, else the tile's mode-k rows per CTA     */
  int64_t tile_volume;  /* in-slice elements per CTA work item, 0=auto */
  int32_t splits;       /* split-K factor, 0 = derive from tile_volume */
  int32_t sm_count;     /* 0 = query the device                        */
  int32_t block_k;      /* 0 | 16 | 32: chunk depth (contraction tile) */
  int32_t engine;       /* CPK_ENGINE_*: data-movement engine          */
  int32_t merge;        /* CPK_MERGE_*: small-mode merging              */
} cpk_plan;

/* merge: a mode far smaller than the row tile can run as the (d-1)-way
 * problem with its neighbour (mode-1 or mode+1) merged into the output rows,
 * plus a small contraction with that neighbour's factor.  AUTO decides (only
 * when rank_tile, block_rows, tile_volume, splits and block_k are all 0);
 * cpk_plan_resolve then reports PREV/NEXT and the other fields describe the
 * merged problem, so passing the resolved plan back runs the same thing. */
#define CPK_MERGE_AUTO 0
#define CPK_MERGE_NONE (-1)
#define CPK_MERGE_PREV 1
#define CPK_MERGE_NEXT 2
/* KR: the two fastest non-k modes run as one virtual mode whose factor is
 * their Khatri-Rao product, materialized in the workspace (longer o-groups
 * for the kernel's per-group scaling).  AUTO picks it for automatic plans
 * when those modes are short and the factor small (d >= 4: o-groups under
 * 64 chunks; d = 3, where it is the whole product: under 16 chunks);
 * resolve reports KR, and passing it back runs the same merged problem. */
#define CPK_MERGE_KR 3
/* KR_FOLD: for d >= 4 when k sits between the fastest non-k mode f and the
 * first other mode o0 (so KR cannot reshape them), the DMMA kernel reads
 * W = KR(A_f, A_o0) (rows i_f + I_f i_o0, materialized in the workspace) as
 * its factor rows and an all-ones factor for o0: o-groups run I_o0 times
 * longer.  AUTO picks it for automatic plans under the same conditions as
 * KR; resolve reports it and passing it back runs the same thing. */
#define CPK_MERGE_KR_FOLD 4

/* engine: AUTO picks the warp-specialized TMA kernel with DMMA consumers
 * when the problem is aligned (even I_0 and leading dimensions, 16-byte
 * aligned bases, d <= 5), else the cp.async kernel; the rank tile minimizes
 * padded work / measured rate (cpk_plan_resolve). */
#define CPK_ENGINE_AUTO 0
#define CPK_ENGINE_CPASYNC 1
#define CPK_ENGINE_TMA 2
/* TMA data movement (as CPK_ENGINE_TMA) with the FP64 math on mma.sync
 * m8n8k4 f64 (DMMA) instead of DFMA outer products; rank tiles 64/128/256. */
#define CPK_ENGINE_DMMA 3
/* cp.async data movement (any shape / alignment, as CPK_ENGINE_CPASYNC) with
 * the DMMA consumers; rank tiles 64 (256 rows) and 128 (128 rows).  Picked
 * where TMA cannot describe the tensor (odd I_0, misaligned factors). */
#define CPK_ENGINE_CPDMMA 4

/* Last error message of the calling thread (never NULL). */
const char* cpk_last_error(void);
/* Library version string. */
const char* cpk_version(void);

/* Fill every zero field of *plan for this problem; validates the problem.
 * Replaces the CPU worker-pool / tile-volume resolution of
 * mttkrp.py:127-144 and plan_for_mode's clamp (mttkrp.py:394-401). */
int cpk_plan_resolve(int d, const int64_t* dims, int mode, int64_t rank,
                     cpk_plan* plan);

/* Bytes of workspace cpk_mttkrp_f64 needs for the same (request) plan:
 * split-K partials plus, for merged plans, the merged output or the
 * Khatri-Rao factor (0 when nothing is needed).  plan may be NULL: the
 * all-zero automatic request, as cpk_mttkrp_f64 treats a NULL plan. */
int cpk_mttkrp_workspace_bytes(int d, const int64_t* dims, int mode,
                               int64_t rank, const cpk_plan* plan,
                               size_t* bytes);

/*
 * G = Y_(mode) (A_{d-1} (.) ... (.) A_{mode+1} (.) A_{mode-1} (.) ... (.) A_0) diag(lam)
 *
 * Replaces mttkrp_tile / tile_kernel (mttkrp.py:345-375, _kernels.py:96-174)
 * and, with splits == 1, mttkrp_slice (mttkrp.py:317-342).
 *   y        device, N = prod(dims) float64, first mode fastest
 *   factors  host array of d device pointers; factors[m] is dims[m] x ld[m]
 *            row-major (ld[m] >= rank); factors[mode] is not read
 *   ld       host array of d leading dimensions (NULL = rank for all)
 *   lam      device, rank float64, or NULL for unit weights
 *   G        device, dims[mode] x ldg row-major (ldg >= rank)
 *   workspace device scratch of cpk_mttkrp_workspace_bytes (may be NULL if 0)
 *   stream   cudaStream_t (NULL = legacy default stream)
 */
int cpk_mttkrp_f64(const double* y, int d, const int64_t* dims, int mode,
                   const double* const* factors, const int64_t* ld,
                   const double* lam, int64_t rank, double* G, int64_t ldg,
                   const cpk_plan* plan, void* workspace, size_t ws_bytes,
                   void* stream);

/* The same MTTKRP, launched piecewise while the tensor streams in: only
 * the work whose tensor slices along the slowest mode (d-1) all lie in
 * [0, landed_hi) and not all in [0, landed_lo).  Calling it with
 * (0, h_1), (h_1, h_2), ..., (h_{n-1}, dims[d-1]) in stream order launches
 * every work item exactly once; the first call (landed_lo = 0) starts the
 * MTTKRP and the last completes the split-K merge, so G is bit-identical to
 * cpk_mttkrp_f64's.  Same plan, workspace and pointers on every call (the
 * workspace carries the partial sums or the split-chain counters). */
int cpk_mttkrp_f64_landed(const double* y, int d, const int64_t* dims,
                          int mode, const double* const* factors,
                          const int64_t* ld, const double* lam, int64_t rank,
                          double* G, int64_t ldg, const cpk_plan* plan,
                          void* workspace, size_t ws_bytes, void* stream,
                          int64_t landed_lo, int64_t landed_hi);

/* Float32 MTTKRP (the north star's optional float32 path, <= 1e-4 relative
 * Frobenius): tcgen05.mma kind::tf32 with a 3xTF32 split (hi*hi + hi*lo +
 * lo*hi) so results keep fp32 accuracy; fp32 accumulation in TMEM, split-K
 * partials merged in FP64.  Needs 2 <= d <= 5, a 16-byte aligned tensor
 * with I_0 % 4 == 0, and 16-byte aligned factors with ld % 4 == 0 (TMA
 * strides).  splits = 0 chooses; the workspace holds splits x I_k x
 * round4(R) floats (0 bytes when splits == 1). */
int cpk_mttkrp_f32_workspace_bytes(int d, const int64_t* dims, int mode,
                                   int64_t rank, int splits, size_t* bytes);
int cpk_mttkrp_f32(const float* y, int d, const int64_t* dims, int mode,
                   const float* const* factors, const int64_t* ld,
                   const float* lam, int64_t rank, float* G, int64_t ldg,
                   int splits, void* workspace, size_t ws_bytes, void* stream);

/* The paper's baseline matrix-free GPU kernel MTTKRP-ELEM (PAPER.md:203-243,
 * _kernels.py:60-93): one FP64 atomic per element and column (N R logical
 * atomics).  For Fig. 4-style comparisons only: zero-fills G, then adds in
 * atomic order (not bit-reproducible).  Same argument meaning as
 * cpk_mttkrp_f64, no plan or workspace. */
int cpk_mttkrp_elem_f64(const double* y, int d, const int64_t* dims, int mode,
                        const double* const* factors, const int64_t* ld,
                        const double* lam, int64_t rank, double* G,
                        int64_t ldg, void* stream);

/* Gram matrix A^T A (R x R), symmetrized exactly: upper triangle computed,
 * lower mirrored -- kruskal.gram (kruskal.py:110-114). */
int cpk_gram_f64(const double* A, int64_t rows, int64_t rank, int64_t lda,
                 double* gram, void* stream);

/* out = (*) of grams[m] over m != skip (skip < 0: all), elementwise, in
 * ascending m order starting from ones -- cpals.py:129-132 and the fit's H
 * (cpals.py:143-145); kruskal.hadamard_gram (kruskal.py:74-83). */
int cpk_hadamard_f64(const double* const* grams, int n, int skip,
                     int64_t rank, double* out, void* stream);

/* Solve X Gamma = G in place (G is rows x rank row-major, Gamma rank x rank
 * SPD) with the regularization ladder of cpals._solve_normal
 * (cpals.py:75-89): Cholesky; on failure Gamma + eps tr(Gamma)/R I with
 * eps = 1e-12, x1e3, up to 5 tries.  `work` is caller scratch of
 * cpk_solve_workspace_bytes.  Returns CPK_ERR_NOT_PD if every rung fails
 * (the caller then takes the least-squares path). Synchronizes the stream
 * only to read the Cholesky info flag. */
int cpk_solve_workspace_bytes(int64_t rows, int64_t rank, size_t* bytes);
int cpk_solve_normal_f64(const double* gamma, double* G, int64_t rows,
                         int64_t rank, void* work, size_t work_bytes,
                         void* stream);

/* Speculative, sync-free form of the same solve for graph-captured sweeps:
 * rung 0 only (plain Cholesky + solve), the potrf info flag written to the
 * DEVICE int *info_out and never read back here.  A nonzero flag means G
 * holds garbage; the caller (cp_als) then restores the sweep's inputs and
 * reruns it through cpk_solve_normal_f64's full ladder. */
int cpk_solve_normal_spec_f64(const double* gamma, double* G, int64_t rows,
                              int64_t rank, void* work, size_t work_bytes,
                              int* info_out, void* stream);

/* Dimension-tree CP-ALS, in-group step (no reference counterpart as one
 * call: it is the second half of the reference sweep's mode-k MTTKRP,
 * cpals.py:121-124, when the sweep splits the modes into two groups).
 * W (prod(ext) x rank, row stride ldw, group multi-index first-mode-fastest)
 * is the MTTKRP of the tensor over the modes OUTSIDE a group of g modes with
 * extents ext[0..g-1]; out (ext[j] x rank, row stride ldo) =
 *   sum over i_l, l != j, of W[i, r] * prod_{l != j} factors[l][i_l, r],
 * i.e. group mode j's MTTKRP.  factors[j] is not read (may be NULL);
 * factors[l] has row stride lda[l].  Deterministic (fixed summation order). */
int cpk_dimtree_contract_f64(const double* W, int64_t ldw, int g,
                             const int64_t* ext, int j,
                             const double* const* factors, const int64_t* lda,
                             int64_t rank, double* out, int64_t ldo,
                             void* stream);

/* The same speculative solve in its two halves, so the factorization (which
 * needs only Gamma) can run on a side stream while the mode's MTTKRP
 * produces G: _factor writes the Cholesky factor into `work` and the flag
 * into *info_out; _apply (same work / rank, stream-ordered after _factor)
 * solves G in place, and skips when *info_out != 0. */
int cpk_solve_factor_spec_f64(const double* gamma, int64_t rank, void* work,
                              size_t work_bytes, int* info_out, void* stream);
int cpk_solve_apply_spec_f64(double* G, int64_t rows, int64_t rank, void* work,
                             size_t work_bytes, const int* info_out, void* stream);

/* Column 2-norms of A (rows x rank), A[:, nz] /= nrm, lam = where(nz, nrm, 0)
 * -- cpals.py:134-137.  Split in two so the sharded driver can allreduce the
 * squared norms of a row-partitioned factor in between:
 *   cpk_colnorms_sq_f64:  normsq[j] = sum_i A[i, j]^2 (deterministic order)
 *   cpk_scale_columns_f64: nrm = sqrt(normsq); A[:, nrm > 0] /= nrm; lam = nrm */
int cpk_colnorms_sq_f64(const double* A, int64_t rows, int64_t rank,
                        int64_t lda, double* normsq, void* stream);
int cpk_scale_columns_f64(double* A, int64_t rows, int64_t rank, int64_t lda,
                          const double* normsq, double* lam, void* stream);
int cpk_normalize_columns_f64(double* A, int64_t rows, int64_t rank,
                              int64_t lda, double* lam, double* normsq_work,
                              void* stream);

/* Fit terms (cpals.py:143-150): out[0] = lam^T H lam, out[1] =
 * sum((G * lam) * A), both as device scalars. */
int cpk_fit_terms_f64(const double* H, const double* lam, const double* G,
                      const double* A, int64_t rows, int64_t rank,
                      double* out2, void* stream);

/* Sum of squares of a flat device vector (for ||Y||^2), deterministic:
 * `work` holds CPK_SUMSQ_PARTIALS doubles of block partials. */
#define CPK_SUMSQ_PARTIALS 1024
int cpk_sumsq_f64(const double* x, int64_t n, double* work, double* out,
                  void* stream);

/* Fill x[i] = U[0,1) from the counter-based generator
 * u = (splitmix64(seed * 2^32 + offset + i) >> 11) * 2^-53, used to create
 * BASELINE tensors too large to stage through the host.  The CPU twin is
 * oracle/gen.py:splitmix_uniform. */
int cpk_fill_uniform_f64(double* x, int64_t n, uint64_t seed, int64_t offset,
                         void* stream);

/* The slab [lo, hi) along `mode` of the d-way splitmix tensor of global
 * shape global_dims, stored as its own first-mode-fastest tensor: the
 * per-rank shard of the sharded driver, generated on the device. */
int cpk_fill_uniform_slab_f64(double* x, int d, const int64_t* global_dims,
                              int mode, int64_t lo, int64_t hi, uint64_t seed,
                              void* stream);

/* DTEN v1 files (dtensor.py:334-382): shape of the file's tensor (header
 * validated as the reference does, 1..64 modes; FormatError ->
 * CPK_ERR_FORMAT).  dims must hold CPK_DTEN_MAX_MODES entries.  Files with
 * more modes than the kernels take (CPK_MAX_MODES) still load: the limit
 * applies to the MTTKRP, not to ingest. */
#define CPK_DTEN_MAX_MODES 64
int cpk_dten_read_header(const char* path, int* d, int64_t* dims);

/* Load the slab [lo, hi) along `mode` of a DTEN file straight into device
 * memory `dst` (dst_elems = the slab's volume), as its own first-mode-fastest
 * tensor: pread through `threads` reader threads (0 = host cores, 8..32) into two pinned
 * staging buffers, each streamed with cudaMemcpyAsync on `stream` while the
 * other fills.  (lo, hi) = (0, dims[mode]) loads the whole tensor; the
 * sharded driver loads only its rows.  Returns after the last copy has
 * been enqueued and the staging buffers have drained. */
int cpk_dten_load_slab_f64(const char* path, int mode, int64_t lo, int64_t hi,
                           double* dst, int64_t dst_elems, int threads,
                           void* stream);

/* Device-side FP64 pipe probe: the larger achieved FLOP/s of a
 * register-resident DFMA loop and a register-resident DMMA (mma.sync
 * m8n8k4 f64) loop over the whole chip -- the FP64 roofline peak
 * (MEASURED_PEAKS.json has no FP64 figure).  Synchronous. */
int cpk_fp64_peak_probe(double* flops_per_s, double* seconds);

#ifdef __cplusplus
}
#endif

#endif /* CPK_B200_H */
