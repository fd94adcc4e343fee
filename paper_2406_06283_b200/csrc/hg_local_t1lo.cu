// Instantiations of the single-RHS local band solve for rf 2..3 (split across
// translation units so they compile in parallel; see hg_local_impl.cuh).
#include "hg_local_impl.cuh"

namespace hg {

LocalKernel pick_local_single_lo(int rf, int rb) {
  switch (rf) {
    case 2: return pick_rb<2, 1>(rb);
    case 3: return pick_rb<3, 1>(rb);
    default: return nullptr;
  }
}

}  // namespace hg
