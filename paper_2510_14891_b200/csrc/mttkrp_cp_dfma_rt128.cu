// cp.async DFMA MTTKRP instantiations, rank tile 128 (128 rows per CTA).
#include "mttkrp_cp.cuh"

namespace cpk {

KernelInfo pick_dfma_rt128(int bk, bool kmaj, int vec, int no) { return pick_layout<128, 128>(bk, kmaj, vec, no); }

}  // namespace cpk
