// Instantiations of the training kernels for the d=64/128 vector layouts.
#include "train_kernels.cuh"

namespace gb {
namespace tk {
Variant vec_variant_b(int G, int NV) {
  if (G == 8 && NV == 2) return make_variant<VecRow<8, 2>, false, true>();
  if (G == 32 && NV == 1) return make_variant<VecRow<32, 1>, false, true>();
  if (G == 16 && NV == 2) return make_variant<VecRow<16, 2>, false, true>();
  return Variant{};
}
}  // namespace tk
}  // namespace gb
