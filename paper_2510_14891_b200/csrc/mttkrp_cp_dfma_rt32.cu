// cp.async DFMA MTTKRP instantiations, rank tile 32 (64 rows per CTA).
#include "mttkrp_cp.cuh"

namespace cpk {

KernelInfo pick_dfma_rt32(int bk, bool kmaj, int vec, int no) { return pick_layout<64, 32>(bk, kmaj, vec, no); }

}  // namespace cpk
