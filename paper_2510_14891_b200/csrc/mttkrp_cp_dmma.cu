// Instantiations of the cp.async MTTKRP kernel with DMMA consumers
// (mttkrp_cp.cuh, engine CPK_ENGINE_CPDMMA): rank tile 128 -> 128 rows,
// 64 -> 256 rows.
#include "mttkrp_cp.cuh"

namespace cpk {

KernelInfo pick_kernel_dmma(int rank_tile, int bk, bool kmaj, int vec, int no) {
  switch (rank_tile) {
    case 128: return pick_layout<128, 128, true>(bk, kmaj, vec, no);
    case 64: return pick_layout<256, 64, true>(bk, kmaj, vec, no);
    default: return {nullptr, 0, 0, 0};
  }
}

}  // namespace cpk
