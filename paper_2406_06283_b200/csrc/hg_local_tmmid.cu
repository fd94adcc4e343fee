// Instantiations of the batched local band solve for rf 4 (split across
// translation units so they compile in parallel; see hg_local_impl.cuh).
#include "hg_local_impl.cuh"

namespace hg {

LocalKernel pick_local_multi_mid(int rf, int rb) {
  switch (rf) {
    case 4: return pick_rb<4, HG_MAX_RHS>(rb);
    default: return nullptr;
  }
}

}  // namespace hg
