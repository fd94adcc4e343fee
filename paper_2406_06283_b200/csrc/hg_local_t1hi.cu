// Instantiations of the single-RHS local band solve for rf 4..6 (split across
// translation units so they compile in parallel; see hg_local_impl.cuh).
#include "hg_local_impl.cuh"

namespace hg {

LocalKernel pick_local_single_hi(int rf, int rb) {
  switch (rf) {
    case 4: return pick_rb<4, 1>(rb);
    case 5: return pick_rb<5, 1>(rb);
    case 6: return pick_rb<6, 1>(rb);
    default: return nullptr;
  }
}

}  // namespace hg
