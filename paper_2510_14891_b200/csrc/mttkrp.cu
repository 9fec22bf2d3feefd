// Matrix-free dense MTTKRP for B200 (sm_100a), FP64 on the CUDA-core DFMA pipe.
//
// What it computes (reference: mttkrp_tile / tile_kernel / accum_tile,
// pkg/src/cpkern/mttkrp.py:345-375 and _kernels.py:96-174):
//
//     G[n, j] = lam[j] * sum_{i : i_k = n} y[i] * prod_{m != k} A_m[i_m, j]
//
// B200 design.  The contraction over the N_S in-slice elements of every
// mode-k slice is run as an on-the-fly GEMM
//
//     G (I_k x R) = Y_(k) (I_k x N_S) . Z (N_S x R),   Z = Khatri-Rao rows
//
// without ever materializing Z.  The in-slice elements are walked in the
// reference's own first-mode-fastest order and cut into *chunks*: BK
// consecutive values of the fastest non-k mode f, with every other non-k
// index ("o" modes) fixed.  For one chunk the Khatri-Rao rows are
//
//     Z[c, j] = A_f[i_f0 + c, j] * P_o[j],   P_o[j] = prod_{m in o} A_m[o_m, j]
//
// so one chunk needs BK factor rows of A_f plus one row per o-mode.  They are
// staged with cp.async into shared memory next to the BM x BK tensor tile and
// each thread scales its own B-tile chunks by P_o in place (the Khatri-Rao row
// is formed once per CTA per chunk, amortized over BM output rows).  The math
// is a register-tiled DFMA outer product: 8x8 accumulators per thread, operand
// fragments read with 128-bit LDS in broadcast-friendly layouts.
//
//   * mode 0     : tensor tile is "M-major" (the mode-0 index n is contiguous),
//                  staged as As[k][m]
//   * mode k > 0 : tensor tile is "K-major" (the contraction index i_0 is
//                  contiguous), staged as As[m][k] with a 2-double row pad
//                  so the 8 row reads of a warp hit distinct banks
//
// Parallelism: grid = (rank tiles, row tiles, splits).  Rank tiles are the
// fastest grid index so the CTAs that share one tensor tile run together and
// the tile is read from HBM once and from L2 R/BN times.  `splits` cuts the
// chunk sequence (the reference's tiles-per-slice, mttkrp.py:354-355) into
// contiguous ranges; partials land in a [splits, I_k, R] workspace that one
// deterministic kernel sums in split order -- no floating-point atomics, so
// results are bit-reproducible run to run.
#include "common.cuh"
#include "mttkrp_cp.cuh"
#include "mttkrp_internal.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace cpk {
// Deterministic split-K reduction (the private-copy merge of
// mttkrp._run_private_copy, mttkrp.py:279-286: partials summed in a fixed
// order, then lam folded once).
__global__ void splitk_reduce_f64(const double* __restrict__ w, int splits, int64_t Ik, int64_t R,
                                  int64_t ldw, int64_t split_stride, const double* __restrict__ lam,
                                  double* __restrict__ G, int64_t ldg) {
  const int64_t total = Ik * R;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = idx / R, j = idx - n * R;
    const double* src = w + n * ldw + j;
    double s = 0.0;
    int sp = 0;
    for (; sp + 4 <= splits; sp += 4) {
      const double v0 = src[(sp + 0) * split_stride];
      const double v1 = src[(sp + 1) * split_stride];
      const double v2 = src[(sp + 2) * split_stride];
      const double v3 = src[(sp + 3) * split_stride];
      s += v0;
      s += v1;
      s += v2;
      s += v3;
    }
    for (; sp < splits; ++sp) s += src[sp * split_stride];
    if (lam) s *= lam[j];
    G[n * ldg + j] = s;
  }
}

// ---------------------------------------------------------------------------
// host side

struct Problem {
  int d, k, f;
  int64_t dims[CPK_MAX_MODES];
  int64_t strides[CPK_MAX_MODES];
  int64_t N, Ik, NS, R;
  int n_o;
  int o_modes[CPK_MAX_MODES];
};

static int make_problem(int d, const int64_t* dims, int mode, int64_t rank, Problem* pr) {
  if (d < 1 || d > CPK_MAX_MODES) return fail(CPK_ERR_PARAM, "order d=%d unsupported (1..%d)", d, CPK_MAX_MODES);
  if (!dims) return fail(CPK_ERR_SHAPE, "dims is NULL");
  if (mode < 0 || mode >= d) return fail(CPK_ERR_INDEX, "mode %d out of range [0, %d]", mode, d - 1);
  if (rank < 1) return fail(CPK_ERR_PARAM, "rank must be >= 1, got %lld", (long long)rank);
  pr->d = d;
  pr->k = mode;
  pr->R = rank;
  int64_t s = 1;
  for (int m = 0; m < d; ++m) {
    if (dims[m] < 1) return fail(CPK_ERR_SHAPE, "every extent must be >= 1 (mode %d is %lld)", m, (long long)dims[m]);
    pr->dims[m] = dims[m];
    pr->strides[m] = s;
    if (s > INT64_MAX / dims[m]) return fail(CPK_ERR_SHAPE, "volume does not fit in int64");
    s *= dims[m];
  }
  pr->N = s;
  pr->Ik = dims[mode];
  pr->NS = s / dims[mode];
  pr->f = d == 1 ? -1 : (mode == 0 ? 1 : 0);
  pr->n_o = 0;
  for (int m = 0; m < d; ++m)
    if (m != mode && m != pr->f) pr->o_modes[pr->n_o++] = m;
  return CPK_OK;
}

// engine CPK_ENGINE_CPASYNC: DFMA tiles; CPK_ENGINE_CPDMMA: 8-warp DMMA tiles
// (rank tile 64 -> 256 rows, 128 -> 128 rows, as the TMA DMMA kernel's)
static KernelInfo pick_kernel(int rank_tile, int bk, bool kmaj, int vec, int no, bool dmma = false) {
  return dmma ? pick_kernel_dmma(rank_tile, bk, kmaj, vec, no) : pick_kernel_dfma(rank_tile, bk, kmaj, vec, no);
}
static int block_rows_for(int rank_tile, bool dmma = false) {
  if (dmma) return rank_tile == 64 ? 256 : 128;
  return rank_tile == 32 ? 64 : 128;
}

static int device_sms(int* out) {
  static int cached = 0;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    int dev = 0;
    err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
  });
  if (err != cudaSuccess) return fail(CPK_ERR_CUDA, "device query: %s", cudaGetErrorString(err));
  *out = cached;
  return CPK_OK;
}

// CTAs of the chosen kernel that fit on one SM (1 for the 256-thread tile).
static int ctas_per_sm(const KernelInfo& ki) {
  int n = 0;
  if (cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ki.smem)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ki.fn, ki.threads, ki.smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    return 1;
  }
  return n;
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int64_t n_chunks_of(const Problem& pr, int bk) {
  if (pr.f < 0) return 1;
  int64_t n = ceil_div(pr.dims[pr.f], bk);
  for (int i = 0; i < pr.n_o; ++i) n *= pr.dims[pr.o_modes[i]];
  return n;
}

// Choose the split count.  Two pressures:
//  * CTAs that share a tensor tile (the rank tiles of one row tile) read it
//    through L2 only while they stay close in time; long-running CTAs drift
//    apart and re-read it from HBM.  At c4 DRAM reads fall from 3.0x to
//    1.2x the tensor going from 15 to 148 splits (profiles/
//    r01_exp_splits.log), so each CTA walks at most kChunksPerCta chunks.
//  * the split-K workspace (splits x I_k x R doubles, read back once by the
//    reduction) stays under kWorkspaceBudget.
// Within those bounds, the split count minimizing a time model in units of
// one CTA's chunk: waves x (chunks per CTA + a fixed per-CTA cost) + the
// merge's read of the partial copies.  Filling the last wave is not free
// when it takes many short CTAs: the dimension tree's c3 view (16384 x 128 x
// 128, R = 256; 256 tiles, 1024 chunks) ran 15 splits (99.8 % wave fill)
// 3 % slower than 4 (98.8 %); the model ranks the measured plans in order
// (profiles/r02_c3_view_plan_sweep.log).
constexpr int64_t kChunksPerCta = 512;
constexpr int64_t kMaxSplits = 4096;
constexpr double kWorkspaceBudget = 2.0 * (1 << 30);
constexpr double kCtaFixedSeconds = 5e-6;   // prologue (TMEM, barriers, pipeline fill) + epilogue store
constexpr double kSmFp64Flops = 2.0 * 64 * 1.9e9;  // one SM's FP64 (DFMA = DMMA) rate
constexpr double kHbmBytesPerSecond = 6.5e12;

static int auto_splits(int64_t tiles, int64_t chunks, int slots, double bytes_per_split, double chunk_seconds) {
  const int64_t cap = std::max<int64_t>(1, int64_t(kWorkspaceBudget / std::max(bytes_per_split, 1.0)));
  const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>({chunks / 4, kMaxSplits, cap}));
  const int64_t lo = std::min<int64_t>(max_s, std::max<int64_t>(1, ceil_div(chunks, kChunksPerCta)));
  const double fixed = kCtaFixedSeconds / chunk_seconds;
  const double merge = 2.0 * bytes_per_split / kHbmBytesPerSecond / chunk_seconds;  // write + read back, per split
  double best = 1e300;
  int64_t best_s = lo;
  for (int64_t s = lo; s <= max_s; ++s) {
    const int64_t waves = ceil_div(tiles * s, slots);
    const double cost = double(waves) * (double(ceil_div(chunks, s)) + fixed) + (s > 1 ? double(s) * merge : 0.0);
    if (cost < best * (1 - 1e-9)) {
      best = cost;
      best_s = s;
    }
  }
  return int(best_s);
}

// Can the TMA kernel take this problem (dims-only view: the launch re-checks
// pointer alignment and leading dimensions)?
static bool tma_possible(const Problem& pr) {
  if (pr.d < 2 || pr.d > 5 || pr.n_o > 3 || pr.dims[0] % 2 != 0 || pr.R % 2 != 0) return false;
  for (int m = 0; m < pr.d; ++m)
    if (pr.dims[m] >= (int64_t(1) << 31)) return false;
  return true;
}

// Relative FP64 efficiency of each (engine, rank tile) against the DFMA TMA
// kernel at tile 128, from the c2-c5 sweeps (profiles/r01_sweep_*.agg.csv,
// profiles/r01_sweep_*_dmma.agg.csv); the auto plan minimizes padded work /
// rate.  A rate of 0 would make an engine explicit-only.
struct TileChoice {
  int engine, rank_tile;
  double rate;
};
static const TileChoice kChoices[] = {
    {CPK_ENGINE_TMA, 256, 0.95}, {CPK_ENGINE_TMA, 128, 1.00}, {CPK_ENGINE_TMA, 64, 0.93},
    {CPK_ENGINE_DMMA, 256, 1.02}, {CPK_ENGINE_DMMA, 128, 1.23}, {CPK_ENGINE_DMMA, 64, 1.26},
    {CPK_ENGINE_DMMA, 32, 1.15}, {CPK_ENGINE_DMMA, 16, 0.90},
    {CPK_ENGINE_CPDMMA, 128, 0.97}, {CPK_ENGINE_CPDMMA, 64, 0.88},
    {CPK_ENGINE_CPASYNC, 128, 0.92}, {CPK_ENGINE_CPASYNC, 64, 0.78}, {CPK_ENGINE_CPASYNC, 32, 0.55},
};

static bool is_tma(int engine) { return engine == CPK_ENGINE_TMA || engine == CPK_ENGINE_DMMA; }

static int rows_for(int engine, int rank_tile, int* bm, int* bk_fixed) {
  if (is_tma(engine)) {
    int bk;
    if (!ws_shape(rank_tile, engine == CPK_ENGINE_DMMA ? WS_MATH_DMMA : WS_MATH_DFMA, bm, &bk)) return fail(CPK_ERR_PARAM, "TMA engine has no rank_tile %d tile", rank_tile);
    *bk_fixed = bk;
    return CPK_OK;
  }
  if (engine == CPK_ENGINE_CPDMMA) {
    if (rank_tile != 64 && rank_tile != 128)
      return fail(CPK_ERR_PARAM, "cp.async DMMA engine rank_tile must be 64 or 128 (got %d)", rank_tile);
    *bm = block_rows_for(rank_tile, true);
    *bk_fixed = 0;
    return CPK_OK;
  }
  if (rank_tile != 32 && rank_tile != 64 && rank_tile != 128)
    return fail(CPK_ERR_PARAM, "cp.async engine rank_tile must be 32, 64 or 128 (got %d)", rank_tile);
  *bm = block_rows_for(rank_tile);
  *bk_fixed = 0;
  return CPK_OK;
}

static int resolve(const Problem& pr, cpk_plan* plan) {
  if (plan->engine < CPK_ENGINE_AUTO || plan->engine > CPK_ENGINE_CPDMMA)
    return fail(CPK_ERR_PARAM, "engine must be 0 (auto), 1 (cp.async), 2 (TMA), 3 (TMA + DMMA) or 4 (cp.async + DMMA)");
  const bool tma_ok = tma_possible(pr);
  if (plan->engine == CPK_ENGINE_AUTO || plan->rank_tile == 0) {
    // (engine, rank tile) minimizing padded rows x padded columns / rate
    double best = 1e300;
    int best_e = 0, best_rt = 0;
    for (const TileChoice& c : kChoices) {
      if (plan->engine != CPK_ENGINE_AUTO && c.engine != plan->engine) continue;
      if (plan->engine == CPK_ENGINE_AUTO && c.rate <= 0) continue;  // explicit-only engines
      if (plan->rank_tile != 0 && c.rank_tile != plan->rank_tile) continue;
      if (is_tma(c.engine) && !tma_ok) continue;
      int bm, bk;
      if (rows_for(c.engine, c.rank_tile, &bm, &bk)) continue;
      const double cost =
          double(ceil_div(pr.Ik, bm) * bm) * double(ceil_div(pr.R, c.rank_tile) * c.rank_tile) / c.rate;
      if (cost < best * (1 - 1e-9)) {
        best = cost;
        best_e = c.engine;
        best_rt = c.rank_tile;
      }
    }
    if (best_e == 0) {
      if (is_tma(plan->engine) && !tma_ok)
        return fail(CPK_ERR_PARAM, "TMA engine needs 2 <= d <= 5, even I_0 and even rank");
      return fail(CPK_ERR_PARAM, "no kernel for rank_tile %d", plan->rank_tile);
    }
    plan->engine = best_e;
    plan->rank_tile = best_rt;
  }
  if (is_tma(plan->engine) && !tma_ok)
    return fail(CPK_ERR_PARAM, "TMA engine needs 2 <= d <= 5, even I_0 and even rank");
  int bm, bk_fixed;
  int rc = rows_for(plan->engine, plan->rank_tile, &bm, &bk_fixed);
  if (rc) return rc;
  if (plan->block_rows == 0) plan->block_rows = bm;
  if (plan->block_rows != bm)
    return fail(CPK_ERR_PARAM, "block_rows %d does not match rank_tile %d (expects %d)", plan->block_rows,
                plan->rank_tile, bm);
  if (plan->sm_count == 0) {
    rc = device_sms(&plan->sm_count);
    if (rc) return rc;
  }
  if (plan->block_k == 0) {
    if (bk_fixed) {
      plan->block_k = bk_fixed;
    } else {
      // 32-deep chunks halve the per-stage overhead, but only the 256-thread
      // 128x128 cp.async tile keeps 2 warps per SMSP at that stage size (the
      // 128x64 tile drops to 1 CTA/SM: 30 vs 45 TFLOP/s on config 2,
      // profiles/r01_sweep_c2.agg.csv); needs the 16-byte path (even I_0)
      plan->block_k =
          (plan->rank_tile == 128 && pr.f >= 0 && pr.dims[0] % 2 == 0 && pr.dims[pr.f] >= 32) ? 32 : 16;
    }
  }
  if (plan->block_k != 16 && plan->block_k != 32)
    return fail(CPK_ERR_PARAM, "block_k must be 16 or 32 (got %d)", plan->block_k);
  if (bk_fixed && plan->block_k != bk_fixed)
    return fail(CPK_ERR_PARAM, "TMA rank_tile %d uses block_k %d (got %d)", plan->rank_tile, bk_fixed,
                plan->block_k);
  const int64_t chunks = n_chunks_of(pr, plan->block_k);
  const int64_t cols_per_chunk = pr.f < 0 ? 1 : std::min<int64_t>(plan->block_k, pr.dims[pr.f]);
  if (plan->tile_volume < 0 || plan->tile_volume > pr.NS)
    return fail(CPK_ERR_PARAM, "tile_volume %lld out of range [1, %lld]", (long long)plan->tile_volume,
                (long long)pr.NS);
  if (plan->splits < 0) return fail(CPK_ERR_PARAM, "splits must be >= 0");
  if (plan->splits == 0) {
    if (plan->tile_volume > 0) {
      // N_T -> chunks per split; the reference's tiles land in W private
      // copies (mttkrp.py:279-286), so the split count (= partial copies)
      // is capped like the auto plan's: <= kMaxSplits and the workspace budget
      const int64_t cps = std::max<int64_t>(1, plan->tile_volume / cols_per_chunk);
      const double per_split = double(pr.Ik) * double((pr.R + 1) & ~int64_t(1)) * sizeof(double);
      const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(kMaxSplits, int64_t(kWorkspaceBudget / per_split)));
      plan->splits = int(std::min<int64_t>(ceil_div(chunks, cps), cap));
    } else {
      const int64_t tiles = ceil_div(pr.Ik, bm) * ceil_div(pr.R, plan->rank_tile);
      int per_sm = 1;  // the TMA kernels take one CTA per SM
      if (plan->engine == CPK_ENGINE_CPASYNC || plan->engine == CPK_ENGINE_CPDMMA) {
        KernelInfo ki = pick_kernel(plan->rank_tile, plan->block_k, pr.k != 0, 2, std::min(pr.n_o, 3),
                                    plan->engine == CPK_ENGINE_CPDMMA);
        per_sm = ki.fn ? ctas_per_sm(ki) : 1;
      }
      const double ldw = double((pr.R + 1) & ~int64_t(1));
      // one chunk of one CTA: its FP64 work at the SM's rate, or its share of
      // the tensor tile's HBM bytes (the rank tiles split them) if larger;
      // CTAs sharing an SM share its rate
      const double n_rt = double(ceil_div(pr.R, plan->rank_tile));
      const double t_flop = 2.0 * plan->block_k * bm * plan->rank_tile / kSmFp64Flops;
      const double t_hbm = double(plan->block_k) * bm * sizeof(double) / n_rt / (kHbmBytesPerSecond / plan->sm_count);
      const double chunk_s = std::max(t_flop, t_hbm) * per_sm;
      plan->splits =
          auto_splits(tiles, chunks, plan->sm_count * per_sm, double(pr.Ik) * ldw * sizeof(double), chunk_s);
    }
  }
  if (plan->splits > chunks) plan->splits = int(chunks);
  // no empty splits: recompute from the per-split chunk count
  const int64_t cps = ceil_div(chunks, plan->splits);
  plan->splits = int(ceil_div(chunks, cps));
  plan->tile_volume = std::min<int64_t>(pr.NS, cps * cols_per_chunk);
  return CPK_OK;
}

// Split-K merge.  Default: partial copies in the workspace, summed in split
// order by splitk_reduce_f64 (the private-copy merge, mttkrp.py:279-286).
// CPK_SPLIT_CHAIN=1 selects the ordered chain into G (common.cuh) for plans
// whose output tiles number at least half the SMs (an output tile's
// consecutive splits are then at least half a wave apart in launch order,
// so the chain never waits long): the same sums in the same order (identical
// bits), no partial copies through HBM (c4: -2.1 GB written and read per
// launch), but each CTA's epilogue becomes a wait + read-modify-write of its
// tile, which with one CTA per SM the next CTA cannot hide: measured +1.0 to
// +1.3 ms per c4 mode (+0.9 %), so it is opt-in.
static int64_t out_tiles(const Problem& pr, const cpk_plan& plan) {
  return ceil_div(pr.Ik, plan.block_rows) * ceil_div(pr.R, plan.rank_tile);
}
static bool chain_merge(const Problem& pr, const cpk_plan& plan) {
  const char* want = getenv("CPK_SPLIT_CHAIN");
  if (plan.splits <= 1 || !want || want[0] != '1') return false;
  return 2 * out_tiles(pr, plan) >= int64_t(plan.sm_count);
}

static size_t ws_bytes_for(const Problem& pr, const cpk_plan& plan) {
  if (plan.splits <= 1) return 0;
  if (chain_merge(pr, plan)) return ((size_t(out_tiles(pr, plan)) * sizeof(int) + 255) / 256) * 256;
  const int64_t ldw = (pr.R + 1) & ~int64_t(1);
  return size_t(plan.splits) * size_t(pr.Ik) * size_t(ldw) * sizeof(double);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace cpk

using namespace cpk;

// ---- small-extent modes: merge the output mode with an adjacent one
// A mode of extent I_k far below the row tile (paper tensor A: I_2 = 12 in
// 64-row tiles) wastes most of every CTA.  Merging it with a neighbour a
// (adjacent in memory, so the tensor is simply reinterpreted as (d-1)-way)
// gives I_k * I_a output rows: the kernel computes the partial MTTKRP
// G'[(i_a, i_k), :] without A_a, and a small contraction finishes
// G[i_k, :] = sum_{i_a} G'[(i_a, i_k), :] * A_a[i_a, :] (the same split the
// reference's GEMM baseline makes for interior modes, mttkrp.py:257-265).
// Only for auto plans (no rank tile / split / N_T / chunk depth forced).
struct Merge {
  int a = -1;                         // merged neighbour, -1 = none
  int d2 = 0, mode2 = 0;
  int64_t dims2[CPK_MAX_MODES] = {};
  int64_t scale_last = 1;             // merged-mode slices per original last-mode slice
};

static double rate_of(int engine, int rank_tile) {
  for (const TileChoice& c : kChoices)
    if (c.engine == engine && c.rank_tile == rank_tile) return c.rate;
  return 1.0;
}

// issued work per output row for the resolved plan (padded rows x padded
// rank / rate / rows)
static bool padded_cost(const Problem& pr, const cpk_plan& in, double* cost) {
  cpk_plan p = in;
  if (resolve(pr, &p) != CPK_OK) return false;
  *cost = double(ceil_div(pr.Ik, p.block_rows) * p.block_rows) * double(ceil_div(pr.R, p.rank_tile) * p.rank_tile) /
          rate_of(p.engine, p.rank_tile) / double(pr.Ik);
  return true;
}

static bool plan_is_auto(const cpk_plan* p) {
  return !p || (p->rank_tile == 0 && p->splits == 0 && p->tile_volume == 0 && p->block_rows == 0 && p->block_k == 0);
}

static bool merged_problem(const Problem& pr, int a, Merge* m) {
  if (pr.d < 3 || a < 0 || a >= pr.d || (a != pr.k - 1 && a != pr.k + 1)) return false;
  m->a = a;
  m->d2 = pr.d - 1;
  const int lo = std::min(a, pr.k);
  for (int i = 0, j = 0; i < pr.d; ++i) {
    if (i == lo + 1) continue;
    m->dims2[j++] = i == lo ? pr.dims[lo] * pr.dims[lo + 1] : pr.dims[i];
  }
  m->mode2 = lo;
  m->scale_last = (lo + 1 == pr.d - 1) ? pr.dims[pr.d - 2] : 1;
  return true;
}

// The merge a plan asks for: forced PREV/NEXT, NONE, or (AUTO with an
// otherwise automatic plan) the neighbour that cuts the padding overhead by
// more than 15 %.
static Merge choose_merge(const Problem& pr, const cpk_plan* plan_in) {
  Merge best;
  const int want = plan_in ? plan_in->merge : CPK_MERGE_AUTO;
  if (want == CPK_MERGE_PREV || want == CPK_MERGE_NEXT) {
    Merge m;
    if (merged_problem(pr, want == CPK_MERGE_PREV ? pr.k - 1 : pr.k + 1, &m)) best = m;
    return best;
  }
  if (want != CPK_MERGE_AUTO || pr.d < 3 || !plan_is_auto(plan_in)) return best;
  cpk_plan base = plan_in ? *plan_in : cpk_plan{0, 0, 0, 0, 0, 0, 0, 0};
  base.merge = CPK_MERGE_NONE;
  double c_direct;
  if (!padded_cost(pr, base, &c_direct)) return best;
  double c_best = 0.85 * c_direct;  // merge only for a clear win
  for (int a : {pr.k - 1, pr.k + 1}) {
    Merge m;
    if (!merged_problem(pr, a, &m)) continue;
    Problem p2;
    if (make_problem(m.d2, m.dims2, m.mode2, pr.R, &p2) != CPK_OK || p2.n_o > 3) continue;
    double c;
    if (!padded_cost(p2, base, &c)) continue;
    // both costs are padding overheads (issued / useful work): the merged
    // problem does the same useful work, N x R per mode
    if (c < c_best) {
      c_best = c;
      best = m;
    }
  }
  return best;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// bytes of G' (merged rows x rank) placed after the inner workspace
static size_t merged_out_bytes(const Problem& pr, const Merge& m) {
  return size_t(pr.Ik) * size_t(pr.dims[m.a]) * size_t(pr.R) * sizeof(double);
}

__global__ static void merged_contract_f64(const double* __restrict__ gp, int64_t Ik, int64_t Ia, int64_t R,
                                           int a_faster, const double* __restrict__ A, int64_t lda,
                                           double* __restrict__ G, int64_t ldg) {
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < Ik * R;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = idx / R, j = idx - n * R;
    double s = 0.0;
    for (int64_t ia = 0; ia < Ia; ++ia) {
      const int64_t row = a_faster ? ia + Ia * n : n + Ik * ia;
      s = fma(gp[row * R + j], A[ia * lda + j], s);
    }
    G[n * ldg + j] = s;
  }
}

// Khatri-Rao merge of the two fastest non-k modes.  The DMMA kernel folds
// the o-row product into a TMEM total once per o-group (the chunks_per_f =
// I_f / BK chunks that share the o-digits, mttkrp_ws.cu og_flush), so short
// o-groups cost flushes: c3 (128^4) has 4 chunks per group.  For d >= 4 the
// two fastest non-k modes f and f + 1 (adjacent, both before the last mode)
// are merged into one virtual mode whose factor W[i_f + I_f i_g, :] =
// A_f[i_f, :] o A_g[i_g, :] is materialized in the workspace (c3: 128 x 128
// rows x R = 32 MB); the (d-1)-way problem then has I_f I_g / BK chunks per
// o-group.  For d = 3 the pair is both non-k modes (W is the full
// Khatri-Rao product) and only very short o-groups merge; when g is the
// slowest mode, streamed (landed) slabs [lo, hi) of g map to the merged
// range [lo I_f, hi I_f).  Automatic plans only; off when a small-mode merge
// applies or W would exceed kKrMergeBytes.
constexpr size_t kKrMergeBytes = size_t(256) << 20;
constexpr int64_t kKrMergeMinGroup = 64;  // merge while an o-group is shorter than this many chunks
constexpr int64_t kKrMergeMinGroup3 = 16;  // the same for the full-product merge of a 3-way tensor

struct KrMerge {
  bool on = false;
  int f = -1, d2 = 0, mode2 = 0;
  int64_t dims2[CPK_MAX_MODES] = {};
  int64_t ldw = 0;
  size_t w_bytes = 0;
};

static KrMerge choose_kr_merge(const Problem& pr, const cpk_plan* plan_in) {
  KrMerge m;
  const bool forced = plan_in && plan_in->merge == CPK_MERGE_KR;
  if (!forced && (!plan_is_auto(plan_in) || (plan_in && plan_in->merge != CPK_MERGE_AUTO))) return m;
  const int f = pr.f, g = f + 1;
  if (pr.d < 3 || f < 0 || g == pr.k || g >= pr.d) return m;
  // g the slowest mode (every 3-way case): the merged mode becomes the
  // slowest one, and a streamed (landed) slab [lo, hi) of g is the merged
  // range [lo I_f, hi I_f); CPK_KR_MERGE_LAST=0 restricts merges to d >= 4
  // with g below the slowest mode (the round-2 rule)
  if (g == pr.d - 1 || pr.d < 4) {
    static const bool last_ok = [] {
      const char* e = getenv("CPK_KR_MERGE_LAST");
      return !(e && e[0] == '0');
    }();
    if (!last_ok && !forced) return m;
    // a 3-way merge is the whole Khatri-Rao product: only for very short
    // o-groups (the dimension tree's c3 views, I_f = 128: +5 %); at I_f = 512
    // (c2) W's extra pass loses 11-14 % (profiles/r02_kr_merge_last_ab.md)
    if (!forced && pr.dims[f] / 16 >= kKrMergeMinGroup3) return m;
  }
  if (!forced && pr.dims[f] / 16 >= kKrMergeMinGroup) return m;  // o-groups already long (BK >= 16)
  m.ldw = (pr.R + 1) & ~int64_t(1);
  m.w_bytes = size_t(pr.dims[f]) * size_t(pr.dims[g]) * size_t(m.ldw) * sizeof(double);
  if (!forced && m.w_bytes > kKrMergeBytes) return m;
  m.on = true;
  m.f = f;
  m.d2 = pr.d - 1;
  for (int i = 0, j = 0; i < pr.d; ++i) {
    if (i == g) continue;
    m.dims2[j++] = i == f ? pr.dims[f] * pr.dims[g] : pr.dims[i];
  }
  m.mode2 = pr.k < f ? pr.k : pr.k - 1;
  return m;
}

// Orders beyond the kernels' three o-modes (d >= 6, or d >= 7 after the
// Khatri-Rao merge of f): merge the fastest adjacent pair of o-modes
// (neither k nor f, not the slowest mode, so the streamed/landed contract
// holds) into one virtual o-mode with a materialized Khatri-Rao factor
// W[i_a + I_a i_b] = A_a[i_a] o A_b[i_b]; each level of mttkrp_impl removes
// one mode until three o-modes remain.  Any plan (a necessity, not a tuning
// choice); the plan is unchanged by it (I_k, R, f and the chunk count are).
static KrMerge choose_order_merge(const Problem& pr) {
  KrMerge m;
  if (pr.n_o <= 3) return m;
  for (int a = 0; a + 1 < pr.d - 1; ++a) {
    const int b = a + 1;
    if (a == pr.k || b == pr.k || a == pr.f || b == pr.f) continue;
    m.ldw = (pr.R + 1) & ~int64_t(1);
    m.w_bytes = size_t(pr.dims[a]) * size_t(pr.dims[b]) * size_t(m.ldw) * sizeof(double);
    m.on = true;
    m.f = a;
    m.d2 = pr.d - 1;
    for (int i = 0, j = 0; i < pr.d; ++i) {
      if (i == b) continue;
      m.dims2[j++] = i == a ? pr.dims[a] * pr.dims[b] : pr.dims[i];
    }
    m.mode2 = pr.k < a ? pr.k : pr.k - 1;
    return m;
  }
  return m;
}

// Workspace of a problem including any order merges: [inner][W] per level.
static int order_ws(const Problem& pr, const cpk_plan& q, size_t* bytes) {
  if (pr.n_o <= 3) {
    *bytes = ws_bytes_for(pr, q);
    return CPK_OK;
  }
  const KrMerge km = choose_order_merge(pr);
  if (!km.on) return fail(CPK_ERR_PARAM, "order d=%d: no pair of o-modes to merge", pr.d);
  Problem p2;
  int rc = make_problem(km.d2, km.dims2, km.mode2, pr.R, &p2);
  if (rc) return rc;
  size_t inner = 0;
  rc = order_ws(p2, q, &inner);
  if (rc) return rc;
  *bytes = align256(inner) + km.w_bytes;
  return CPK_OK;
}

// Khatri-Rao fold (CPK_MERGE_KR_FOLD): when the fastest non-k mode f is
// short and k sits between it and the first o-mode o0 (c3's mode 1), the
// reshape of choose_kr_merge is impossible, but the DMMA kernel can read
// W = KR(A_f, A_o0) (rows i_f + I_f i_o0) as its factor rows and an all-ones
// factor for o0: the chunk walk and the tensor tiles are unchanged, P_o no
// longer changes with i_o0, so an o-group is I_o0 times longer
// (WsParams::fold).  Needs the resolved plan: DMMA engine, I_f a multiple of
// the chunk depth.  W is a two-mode partial Khatri-Rao product (d >= 4: the
// other o-modes stay on the fly), capped like the KR merge.
struct KrFold {
  bool on = false;
  int o0 = -1;
  int64_t ldw = 0;
  size_t w_bytes = 0, ones_bytes = 0;
};

static KrFold choose_kr_fold(const Problem& pr, const cpk_plan& resolved, const cpk_plan* plan_in) {
  KrFold m;
  const bool forced = plan_in && plan_in->merge == CPK_MERGE_KR_FOLD;
  if (!forced && (!plan_is_auto(plan_in) || (plan_in && plan_in->merge != CPK_MERGE_AUTO))) return m;
  if (pr.d < 4 || pr.f < 0 || pr.n_o < 2 || pr.n_o > 3 || resolved.engine != CPK_ENGINE_DMMA) return m;
  if (resolved.block_k <= 0 || pr.dims[pr.f] % resolved.block_k != 0) return m;
  if (!forced && pr.dims[pr.f] / resolved.block_k >= kKrMergeMinGroup) return m;  // o-groups already long
  const int o0 = pr.o_modes[0];
  m.ldw = (pr.R + 1) & ~int64_t(1);
  m.w_bytes = size_t(pr.dims[pr.f]) * size_t(pr.dims[o0]) * size_t(m.ldw) * sizeof(double);
  m.ones_bytes = size_t(pr.dims[o0]) * size_t(m.ldw) * sizeof(double);
  if (!forced && m.w_bytes > kKrMergeBytes) return m;
  m.on = true;
  m.o0 = o0;
  return m;
}

static size_t fold_bytes(const KrFold& kf) { return kf.on ? align256(kf.w_bytes) + align256(kf.ones_bytes) : 0; }

__global__ static void fill_f64(double* x, int64_t n, double v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] = v;
}

__global__ static void kr_pair_f64(const double* __restrict__ Af, int64_t ldf, const double* __restrict__ Ag,
                                   int64_t ldg, int64_t If, int64_t rows, int64_t R, double* __restrict__ W,
                                   int64_t ldw) {
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < rows * R;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = idx / R, j = idx - row * R;
    const int64_t i_g = row / If, i_f = row - i_g * If;
    W[row * ldw + j] = Af[i_f * ldf + j] * Ag[i_g * ldg + j];
  }
}

extern "C" int cpk_plan_resolve(int d, const int64_t* dims, int mode, int64_t rank, cpk_plan* plan) {
  if (!plan) return fail(CPK_ERR_PARAM, "plan is NULL");
  Problem pr;
  int rc = make_problem(d, dims, mode, rank, &pr);
  if (rc) return rc;
  const Merge mg = choose_merge(pr, plan);
  if (mg.a >= 0) {  // the plan of the merged (d-1)-way problem the kernel runs
    Problem p2;
    rc = make_problem(mg.d2, mg.dims2, mg.mode2, rank, &p2);
    if (rc) return rc;
    plan->merge = mg.a < mode ? CPK_MERGE_PREV : CPK_MERGE_NEXT;
    return resolve(p2, plan);
  }
  if (plan->merge != CPK_MERGE_AUTO && plan->merge != CPK_MERGE_NONE && plan->merge != CPK_MERGE_KR &&
      plan->merge != CPK_MERGE_KR_FOLD)
    return fail(CPK_ERR_PARAM, "merge %d impossible for mode %d of a %d-way tensor", plan->merge, mode, d);
  const KrMerge km = choose_kr_merge(pr, plan);
  if (plan->merge == CPK_MERGE_KR && !km.on)
    return fail(CPK_ERR_PARAM, "Khatri-Rao merge impossible for mode %d of a %d-way tensor", mode, d);
  const cpk_plan request = *plan;
  plan->merge = km.on ? CPK_MERGE_KR : CPK_MERGE_NONE;
  if (km.on) {  // the plan of the (d-1)-way problem with f and f + 1 merged
    Problem p2;
    rc = make_problem(km.d2, km.dims2, km.mode2, rank, &p2);
    if (rc) return rc;
    return resolve(p2, plan);
  }
  rc = resolve(pr, plan);
  if (rc) return rc;
  const KrFold kf = choose_kr_fold(pr, *plan, &request);
  if (request.merge == CPK_MERGE_KR_FOLD && !kf.on)
    return fail(CPK_ERR_PARAM, "Khatri-Rao fold impossible for mode %d of a %d-way tensor", mode, d);
  if (kf.on) plan->merge = CPK_MERGE_KR_FOLD;
  return CPK_OK;
}

extern "C" int cpk_mttkrp_workspace_bytes(int d, const int64_t* dims, int mode, int64_t rank,
                                          const cpk_plan* plan_or_null, size_t* bytes) {
  if (!bytes) return fail(CPK_ERR_PARAM, "NULL argument");
  // a NULL plan is the all-zero request, exactly as cpk_mttkrp_f64 reads it
  const cpk_plan auto_plan{0, 0, 0, 0, 0, 0, 0, 0};
  const cpk_plan* plan = plan_or_null ? plan_or_null : &auto_plan;
  Problem pr;
  int rc = make_problem(d, dims, mode, rank, &pr);
  if (rc) return rc;
  const Merge mg = choose_merge(pr, plan);
  if (mg.a >= 0) {
    Problem p2;
    rc = make_problem(mg.d2, mg.dims2, mg.mode2, rank, &p2);
    if (rc) return rc;
    cpk_plan q = *plan;
    rc = resolve(p2, &q);
    if (rc) return rc;
    size_t inner = 0;
    rc = order_ws(p2, q, &inner);
    if (rc) return rc;
    *bytes = align256(inner) + merged_out_bytes(pr, mg);
    return CPK_OK;
  }
  const KrMerge km = choose_kr_merge(pr, plan);
  if (km.on) {
    Problem p2;
    rc = make_problem(km.d2, km.dims2, km.mode2, rank, &p2);
    if (rc) return rc;
    cpk_plan q = *plan;
    rc = resolve(p2, &q);
    if (rc) return rc;
    size_t inner = 0;
    rc = order_ws(p2, q, &inner);
    if (rc) return rc;
    *bytes = align256(inner) + km.w_bytes;
    return CPK_OK;
  }
  cpk_plan p = *plan;
  rc = resolve(pr, &p);
  if (rc) return rc;
  rc = order_ws(pr, p, bytes);
  if (rc) return rc;
  const KrFold kf = choose_kr_fold(pr, p, plan);
  if (kf.on) *bytes = align256(*bytes) + fold_bytes(kf);
  return CPK_OK;
}

// d == 1: G[n, j] = lam[j] * y[n] (ref_kernel with no factor products).
__global__ static void mttkrp_order1(const double* y, int64_t I, int64_t R, const double* lam, double* G,
                                     int64_t ldg) {
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < I * R;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = idx / R, j = idx % R;
    G[n * ldg + j] = lam ? lam[j] * y[n] : y[n];
  }
}

// Work items of a launch that are complete once the slices [0, h) of the
// slowest mode (d-1) are in memory.  mode == d-1: row blocks (each needs its
// own BM slices); else splits (split z needs the slices its last chunk
// touches; chunks run f fastest, then the o modes ascending).
struct Landed {
  int64_t bm, bk, n_chunks, cps;
  int64_t rows_ready(const Problem& pr, int64_t h) const {
    return h >= pr.Ik ? ceil_div(pr.Ik, bm) : h / bm;
  }
  int64_t need(const Problem& pr, int64_t z) const {
    const int64_t qe = std::min((z + 1) * cps, n_chunks) - 1;
    const int last = pr.d - 1;
    if (pr.f == last) return std::min((qe + 1) * bk, pr.dims[last]);  // d == 2, mode 0
    return qe / (n_chunks / pr.dims[last]) + 1;
  }
  int64_t splits_ready(const Problem& pr, int64_t splits, int64_t h) const {
    int64_t z = 0;
    while (z < splits && need(pr, z) <= h) ++z;
    return z;
  }
};

static int mttkrp_impl(const double* y, int d, const int64_t* dims, int mode, const double* const* factors,
                       const int64_t* ld, const double* lam, int64_t rank, double* G, int64_t ldg,
                       const cpk_plan* plan_in, void* workspace, size_t ws_bytes, void* stream, int64_t landed_lo,
                       int64_t landed_hi, bool allow_merge = true) {
  const bool ranged = landed_hi >= 0;
  Problem pr;
  int rc = make_problem(d, dims, mode, rank, &pr);
  if (rc) return rc;
  if (!y || !G) return fail(CPK_ERR_PARAM, "tensor or output pointer is NULL");
  if (ldg < rank) return fail(CPK_ERR_PARAM, "ldg %lld < rank %lld", (long long)ldg, (long long)rank);
  cudaStream_t st = as_stream(stream);
  if (ranged && (landed_lo < 0 || landed_hi < landed_lo || landed_hi > dims[d - 1]))
    return fail(CPK_ERR_PARAM, "landed range [%lld, %lld) not within [0, %lld]", (long long)landed_lo,
                (long long)landed_hi, (long long)dims[d - 1]);
  if (d == 1) {
    if (ranged && landed_hi < dims[0]) return CPK_OK;  // rows all land together: run once at the end
    mttkrp_order1<<<256, 256, 0, st>>>(y, pr.Ik, rank, lam, G, ldg);
    return check_launch("mttkrp_order1");
  }
  if (!factors) return fail(CPK_ERR_PARAM, "factors is NULL");
  for (int m = 0; m < d; ++m) {
    if (m == mode) continue;
    if (!factors[m]) return fail(CPK_ERR_PARAM, "factor %d is NULL", m);
    if (ld && ld[m] < rank) return fail(CPK_ERR_PARAM, "ld[%d] < rank", m);
  }
  const Merge mg = allow_merge ? choose_merge(pr, plan_in) : Merge{};
  if (allow_merge && mg.a < 0 && plan_in && (plan_in->merge == CPK_MERGE_PREV || plan_in->merge == CPK_MERGE_NEXT))
    return fail(CPK_ERR_PARAM, "merge %d impossible for mode %d of a %d-way tensor", plan_in->merge, mode, d);
  if (mg.a >= 0) {
    Problem p2;
    rc = make_problem(mg.d2, mg.dims2, mg.mode2, rank, &p2);
    if (rc) return rc;
    cpk_plan q = plan_in ? *plan_in : cpk_plan{0, 0, 0, 0, 0, 0, 0, 0};
    rc = resolve(p2, &q);
    if (rc) return rc;
    size_t inner_raw = 0;
    rc = order_ws(p2, q, &inner_raw);
    if (rc) return rc;
    const size_t inner = align256(inner_raw);
    if (!workspace || ws_bytes < inner + merged_out_bytes(pr, mg))
      return fail(CPK_ERR_RESOURCE, "merged-mode workspace needs %zu bytes, got %zu", inner + merged_out_bytes(pr, mg),
                  ws_bytes);
    double* gp = reinterpret_cast<double*>(static_cast<char*>(workspace) + inner);
    const double* f2[CPK_MAX_MODES];
    int64_t ld2[CPK_MAX_MODES];
    const int lo = std::min(mg.a, mode);
    for (int i = 0, j = 0; i < d; ++i) {
      if (i == lo + 1) continue;
      f2[j] = (i == lo) ? nullptr : factors[i];
      ld2[j] = (i == lo) ? rank : (ld ? ld[i] : rank);
      ++j;
    }
    const int64_t l_lo = ranged ? landed_lo * mg.scale_last : -1, l_hi = ranged ? landed_hi * mg.scale_last : -1;
    rc = mttkrp_impl(y, mg.d2, mg.dims2, mg.mode2, f2, ld2, lam, rank, gp, rank, &q, workspace, inner, stream, l_lo,
                     l_hi, false);
    if (rc) return rc;
    if (ranged && landed_hi < dims[d - 1]) return CPK_OK;  // contraction once everything landed
    const int64_t total = pr.Ik * rank;
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 148 * 8)));
    merged_contract_f64<<<blocks, 256, 0, st>>>(gp, pr.Ik, pr.dims[mg.a], rank, mg.a < mode ? 1 : 0, factors[mg.a],
                                                ld ? ld[mg.a] : rank, G, ldg);
    return check_launch("merged_contract");
  }
  if (allow_merge) {
    const KrMerge km = choose_kr_merge(pr, plan_in);
    if (!km.on && plan_in && plan_in->merge == CPK_MERGE_KR)
      return fail(CPK_ERR_PARAM, "Khatri-Rao merge impossible for mode %d of a %d-way tensor", mode, d);
    if (km.on) {
      Problem p2;
      rc = make_problem(km.d2, km.dims2, km.mode2, rank, &p2);
      if (rc) return rc;
      cpk_plan q = plan_in ? *plan_in : cpk_plan{0, 0, 0, 0, 0, 0, 0, 0};
      rc = resolve(p2, &q);
      if (rc) return rc;
      size_t inner_raw = 0;
      rc = order_ws(p2, q, &inner_raw);
      if (rc) return rc;
      const size_t inner = align256(inner_raw);
      if (!workspace || ws_bytes < inner + km.w_bytes)
        return fail(CPK_ERR_RESOURCE, "Khatri-Rao merge workspace needs %zu bytes, got %zu", inner + km.w_bytes,
                    ws_bytes);
      double* W = reinterpret_cast<double*>(static_cast<char*>(workspace) + inner);
      const int f = km.f, g = f + 1;
      const int64_t wrows = dims[f] * dims[g];
      const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(wrows * rank, 256), 148 * 8)));
      kr_pair_f64<<<blocks, 256, 0, st>>>(factors[f], ld ? ld[f] : rank, factors[g], ld ? ld[g] : rank, dims[f],
                                          wrows, rank, W, km.ldw);
      rc = check_launch("kr_pair");
      if (rc) return rc;
      const double* f2[CPK_MAX_MODES];
      int64_t ld2[CPK_MAX_MODES];
      for (int i = 0, j = 0; i < d; ++i) {
        if (i == g) continue;
        f2[j] = i == f ? W : factors[i];
        ld2[j] = i == f ? km.ldw : (ld ? ld[i] : rank);
        ++j;
      }
      const int64_t sc = (g == d - 1) ? dims[f] : 1;  // merged slowest mode: i_f + I_f i_g
      return mttkrp_impl(y, km.d2, km.dims2, km.mode2, f2, ld2, lam, rank, G, ldg, &q, workspace, inner, stream,
                         ranged ? landed_lo * sc : landed_lo, ranged ? landed_hi * sc : landed_hi, false);
    }
  }
  if (pr.n_o > 3) {  // more o-modes than the kernels take: merge a pair of them (choose_order_merge)
    const KrMerge km = choose_order_merge(pr);
    if (!km.on) return fail(CPK_ERR_PARAM, "order d=%d: no pair of o-modes to merge", d);
    Problem p2;
    rc = make_problem(km.d2, km.dims2, km.mode2, rank, &p2);
    if (rc) return rc;
    cpk_plan q = plan_in ? *plan_in : cpk_plan{0, 0, 0, 0, 0, 0, 0, 0};
    q.merge = CPK_MERGE_NONE;
    rc = resolve(p2, &q);
    if (rc) return rc;
    size_t inner_raw = 0;
    rc = order_ws(p2, q, &inner_raw);
    if (rc) return rc;
    const size_t inner = align256(inner_raw);
    if (!workspace || ws_bytes < inner + km.w_bytes)
      return fail(CPK_ERR_RESOURCE, "order-merge workspace needs %zu bytes, got %zu", inner + km.w_bytes, ws_bytes);
    double* W = reinterpret_cast<double*>(static_cast<char*>(workspace) + inner);
    const int a = km.f, b = a + 1;
    const int64_t wrows = dims[a] * dims[b];
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(wrows * rank, 256), 148 * 8)));
    kr_pair_f64<<<blocks, 256, 0, st>>>(factors[a], ld ? ld[a] : rank, factors[b], ld ? ld[b] : rank, dims[a], wrows,
                                        rank, W, km.ldw);
    rc = check_launch("kr_pair (order merge)");
    if (rc) return rc;
    const double* f2[CPK_MAX_MODES];
    int64_t ld2[CPK_MAX_MODES];
    for (int i = 0, j = 0; i < d; ++i) {
      if (i == b) continue;
      f2[j] = i == a ? W : factors[i];
      ld2[j] = i == a ? km.ldw : (ld ? ld[i] : rank);
      ++j;
    }
    return mttkrp_impl(y, km.d2, km.dims2, km.mode2, f2, ld2, lam, rank, G, ldg, &q, workspace, inner, stream,
                       landed_lo, landed_hi, false);
  }

  cpk_plan plan = plan_in ? *plan_in : cpk_plan{0, 0, 0, 0, 0, 0, 0, 0};
  rc = resolve(pr, &plan);
  if (rc) return rc;
  const KrFold kf = choose_kr_fold(pr, plan, plan_in);
  if (plan_in && plan_in->merge == CPK_MERGE_KR_FOLD && !kf.on)
    return fail(CPK_ERR_PARAM, "Khatri-Rao fold impossible for mode %d of a %d-way tensor", mode, d);
  const size_t split_need = ws_bytes_for(pr, plan);
  const size_t need = kf.on ? align256(split_need) + fold_bytes(kf) : split_need;
  if (need > 0 && (!workspace || ws_bytes < need))
    return fail(CPK_ERR_RESOURCE, "split-K workspace needs %zu bytes, got %zu", need, ws_bytes);

  auto ldof = [&](int m) { return ld ? ld[m] : rank; };
  MttkrpParams p{};
  p.y = y;
  p.fac_f = factors[pr.f];
  p.ld_f = ldof(pr.f);
  for (int i = 0; i < pr.n_o; ++i) {
    const int m = pr.o_modes[i];
    p.fac_o[i] = factors[m];
    p.ld_o[i] = ldof(m);
    p.dim_o[i] = pr.dims[m];
    p.stride_o[i] = pr.strides[m];
  }
  p.Ik = pr.Ik;
  p.stride_k = pr.strides[pr.k];
  p.If = pr.dims[pr.f];
  p.stride_f = pr.strides[pr.f];
  const bool direct = plan.splits == 1;
  const bool chain = chain_merge(pr, plan);  // splits accumulate into G in order (no partial copies)
  double* out = (direct || chain) ? G : static_cast<double*>(workspace);
  const int64_t ldo = (direct || chain) ? ldg : ((rank + 1) & ~int64_t(1));
  const int64_t out_split_stride = (direct || chain) ? 0 : pr.Ik * ldo;
  const double* lam_fold = (direct || chain) ? lam : nullptr;
  int* sem = chain ? static_cast<int*>(workspace) : nullptr;
  if (chain && (!ranged || landed_lo == 0)) {  // a (streamed) MTTKRP starts: zero the tile counters
    if (cudaMemsetAsync(sem, 0, size_t(out_tiles(pr, plan)) * sizeof(int), st) != cudaSuccess)
      return fail(CPK_ERR_CUDA, "split-K counters memset failed");
  }

  if (is_tma(plan.engine)) {
    WsRequest wr{};
    wr.math = plan.engine == CPK_ENGINE_DMMA ? WS_MATH_DMMA : WS_MATH_DFMA;
    wr.y = y;
    wr.d = d;
    wr.k = mode;
    wr.n_o = pr.n_o;
    for (int m = 0; m < d; ++m) {
      wr.dims[m] = pr.dims[m];
      wr.factors[m] = factors[m];
      wr.ld[m] = ldof(m);
    }
    wr.rank = rank;
    wr.rank_tile = plan.rank_tile;
    wr.block_k = plan.block_k;
    wr.splits = plan.splits;
    wr.out = out;
    wr.ldo = ldo;
    wr.out_split_stride = out_split_stride;
    wr.lam = lam_fold;
    wr.sem = sem;
    if (ws_eligible(wr) && kf.on) {
      // the fold's factors: W = KR(A_f, A_o0) and all-ones rows for o0, once
      // per MTTKRP (the first landed piece) in the workspace after the split state
      char* base = static_cast<char*>(workspace) + align256(split_need);
      double* W = reinterpret_cast<double*>(base);
      double* ones = reinterpret_cast<double*>(base + align256(kf.w_bytes));
      const int f = pr.f, o0 = kf.o0;
      if (!ranged || landed_lo == 0) {
        const int64_t wrows = pr.dims[f] * pr.dims[o0];
        const unsigned blocks =
            unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(wrows * rank, 256), 148 * 8)));
        kr_pair_f64<<<blocks, 256, 0, st>>>(factors[f], ldof(f), factors[o0], ldof(o0), pr.dims[f], wrows, rank, W,
                                            kf.ldw);
        fill_f64<<<unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(pr.dims[o0] * kf.ldw, 256), 1024))),
                   256, 0, st>>>(ones, pr.dims[o0] * kf.ldw, 1.0);
        rc = check_launch("kr fold factors");
        if (rc) return rc;
      }
      wr.factors[f] = W;
      wr.ld[f] = kf.ldw;
      wr.factors[o0] = ones;
      wr.ld[o0] = kf.ldw;
      wr.fold = 1;
    }
    if (ws_eligible(wr)) {
      Landed ld_{plan.block_rows, plan.block_k, 0, 0};
      ld_.n_chunks = n_chunks_of(pr, plan.block_k);
      ld_.cps = ceil_div(ld_.n_chunks, plan.splits);
      wr.y1 = int32_t(ceil_div(pr.Ik, plan.block_rows));
      wr.z1 = plan.splits;
      if (ranged) {
        if (mode == d - 1) {
          wr.y0 = int32_t(ld_.rows_ready(pr, landed_lo));
          wr.y1 = int32_t(ld_.rows_ready(pr, landed_hi));
        } else {
          wr.z0 = int32_t(ld_.splits_ready(pr, plan.splits, landed_lo));
          wr.z1 = int32_t(ld_.splits_ready(pr, plan.splits, landed_hi));
        }
      }
      if (wr.y1 > wr.y0 && wr.z1 > wr.z0) {
        rc = launch_ws(wr, st);
        if (rc) return rc;
      }
      goto reduce;
    }
    if (plan_in && is_tma(plan_in->engine))
      return fail(CPK_ERR_PARAM, "TMA engine needs even leading dimensions and 16-byte aligned bases");
    // auto plan, misaligned buffers: same splits (same workspace) on cp.async
    // (the DMMA tiles where the rank tile has one)
    const bool cpd = plan.engine == CPK_ENGINE_DMMA && (plan.rank_tile == 64 || plan.rank_tile == 128);
    plan.engine = cpd ? CPK_ENGINE_CPDMMA : CPK_ENGINE_CPASYNC;
    plan.rank_tile = std::min(plan.rank_tile, 128);
    plan.block_rows = block_rows_for(plan.rank_tile, cpd);
    plan.block_k = 16;
  }
  {
    // 16-byte cp.async needs even element offsets everywhere: I_0 even, even
    // leading dimensions, 16-byte aligned bases.
    bool vec2 = (pr.dims[0] % 2 == 0) && aligned16(y) && aligned16(p.fac_f) && (p.ld_f % 2 == 0);
    for (int i = 0; i < pr.n_o; ++i) vec2 = vec2 && aligned16(p.fac_o[i]) && (p.ld_o[i] % 2 == 0);
    const int bk = (plan.block_k == 32 && vec2) ? 32 : 16;
    p.chunks_per_f = ceil_div(p.If, bk);
    p.n_chunks = n_chunks_of(pr, bk);
    p.chunks_per_split = ceil_div(p.n_chunks, plan.splits);
    p.R = rank;
    p.out = out;
    p.ldo = ldo;
    p.out_split_stride = out_split_stride;
    p.lam = lam_fold;
    p.sem = sem;
    p.n_splits = plan.splits;
    KernelInfo ki = pick_kernel(plan.rank_tile, bk, pr.k != 0, vec2 ? 2 : 1, pr.n_o, plan.engine == CPK_ENGINE_CPDMMA);
    if (!ki.fn) return fail(CPK_ERR_PARAM, "no kernel for rank_tile %d", plan.rank_tile);
    if (cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ki.smem)) != cudaSuccess)
      return check_launch("cudaFuncSetAttribute");
    int64_t y0 = 0, y1 = ceil_div(pr.Ik, plan.block_rows), z0 = 0, z1 = plan.splits;
    if (ranged) {
      const Landed ld_{plan.block_rows, bk, p.n_chunks, p.chunks_per_split};
      if (mode == d - 1) {
        y0 = ld_.rows_ready(pr, landed_lo);
        y1 = ld_.rows_ready(pr, landed_hi);
      } else {
        z0 = ld_.splits_ready(pr, plan.splits, landed_lo);
        z1 = ld_.splits_ready(pr, plan.splits, landed_hi);
      }
    }
    p.z0 = int32_t(z0);
    if (z1 - z0 > 65535) return fail(CPK_ERR_PARAM, "grid too large (splits)");
    // row blocks beyond the 65535 grid-y limit go in several launches
    for (int64_t yb = y0; yb < y1 && z1 > z0; yb += 65535) {
      p.y0 = int32_t(yb);
      dim3 grid(unsigned(ceil_div(rank, plan.rank_tile)), unsigned(std::min<int64_t>(y1 - yb, 65535)),
                unsigned(z1 - z0));
      void* args[] = {&p};
      cudaError_t e = cudaLaunchKernel(ki.fn, grid, dim3(ki.threads), args, ki.smem, st);
      if (e != cudaSuccess) return fail(CPK_ERR_CUDA, "mttkrp launch: %s", cudaGetErrorString(e));
    }
  }
reduce:
  if (!direct && !chain && (!ranged || landed_hi == dims[d - 1])) {
    const int64_t total = pr.Ik * rank;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(total, threads), int64_t(plan.sm_count) * 16);
    splitk_reduce_f64<<<unsigned(std::max<int64_t>(blocks, 1)), threads, 0, st>>>(
        out, plan.splits, pr.Ik, rank, ldo, out_split_stride, lam, G, ldg);
    return check_launch("splitk_reduce");
  }
  return CPK_OK;
}

extern "C" int cpk_mttkrp_f64(const double* y, int d, const int64_t* dims, int mode, const double* const* factors,
                              const int64_t* ld, const double* lam, int64_t rank, double* G, int64_t ldg,
                              const cpk_plan* plan_in, void* workspace, size_t ws_bytes, void* stream) {
  return mttkrp_impl(y, d, dims, mode, factors, ld, lam, rank, G, ldg, plan_in, workspace, ws_bytes, stream, -1, -1);
}

extern "C" int cpk_mttkrp_f64_landed(const double* y, int d, const int64_t* dims, int mode,
                                     const double* const* factors, const int64_t* ld, const double* lam,
                                     int64_t rank, double* G, int64_t ldg, const cpk_plan* plan_in, void* workspace,
                                     size_t ws_bytes, void* stream, int64_t landed_lo, int64_t landed_hi) {
  if (landed_hi < 0) return fail(CPK_ERR_PARAM, "landed_hi must be >= 0");
  return mttkrp_impl(y, d, dims, mode, factors, ld, lam, rank, G, ldg, plan_in, workspace, ws_bytes, stream,
                     landed_lo, landed_hi);
}
