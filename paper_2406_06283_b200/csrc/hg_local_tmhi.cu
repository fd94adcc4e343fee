// Instantiations of the batched local band solve for rf 5..6 (split across
// translation units so they compile in parallel; see hg_local_impl.cuh).
#include "hg_local_impl.cuh"

namespace hg {

LocalKernel pick_local_multi_hi(int rf, int rb) {
  switch (rf) {
    case 5: return pick_rb<5, HG_MAX_RHS>(rb);
    case 6: return pick_rb<6, HG_MAX_RHS>(rb);
    default: return nullptr;
  }
}

}  // namespace hg
