// Instantiations of the batched local band solve for rf 2..3 (split across
// translation units so they compile in parallel; see hg_local_impl.cuh).
#include "hg_local_impl.cuh"

namespace hg {

LocalKernel pick_local_multi_lo(int rf, int rb) {
  switch (rf) {
    case 2: return pick_rb<2, HG_MAX_RHS>(rb);
    case 3: return pick_rb<3, HG_MAX_RHS>(rb);
    default: return nullptr;
  }
}

}  // namespace hg
