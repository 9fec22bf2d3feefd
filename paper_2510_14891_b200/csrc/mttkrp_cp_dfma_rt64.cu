// cp.async DFMA MTTKRP instantiations, rank tile 64 (128 rows per CTA).
#include "mttkrp_cp.cuh"

namespace cpk {

KernelInfo pick_dfma_rt64(int bk, bool kmaj, int vec, int no) { return pick_layout<128, 64>(bk, kmaj, vec, no); }

}  // namespace cpk
