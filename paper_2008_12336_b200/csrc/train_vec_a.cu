// Instantiations of the training kernels for the small vector layouts.
#include "train_kernels.cuh"

namespace gb {
namespace tk {
Variant vec_variant_a(int G, int NV) {
  if (G == 2 && NV == 1) return make_variant<VecRow<2, 1>, false, true>();
  if (G == 4 && NV == 1) return make_variant<VecRow<4, 1>, false, true>();
  if (G == 8 && NV == 1) return make_variant<VecRow<8, 1>, false, true>();
  if (G == 16 && NV == 1) return make_variant<VecRow<16, 1>, false, true>();
  return Variant{};
}
}  // namespace tk
}  // namespace gb
