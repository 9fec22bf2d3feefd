// cp.async MTTKRP kernel with DFMA consumers (mttkrp_cp.cuh): dispatch over
// the rank tiles; each tile's instantiations live in their own unit
// (mttkrp_cp_dfma_rt*.cu) so the build compiles them in parallel.
#include "mttkrp_cp.cuh"

namespace cpk {

KernelInfo pick_dfma_rt128(int bk, bool kmaj, int vec, int no);
KernelInfo pick_dfma_rt64(int bk, bool kmaj, int vec, int no);
KernelInfo pick_dfma_rt32(int bk, bool kmaj, int vec, int no);

KernelInfo pick_kernel_dfma(int rank_tile, int bk, bool kmaj, int vec, int no) {
  switch (rank_tile) {
    case 128: return pick_dfma_rt128(bk, kmaj, vec, no);
    case 64: return pick_dfma_rt64(bk, kmaj, vec, no);
    case 32: return pick_dfma_rt32(bk, kmaj, vec, no);
    default: return {nullptr, 0, 0, 0};
  }
}

}  // namespace cpk
