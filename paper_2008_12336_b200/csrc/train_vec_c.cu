// Instantiations of the training kernels for the 4-float4-per-lane layouts.
#include "train_kernels.cuh"

namespace gb {
namespace tk {
Variant vec_variant_c(int G, int NV) {
  if (G == 8 && NV == 4) return make_variant<VecRow<8, 4>, false, true>();
  if (G == 16 && NV == 4) return make_variant<VecRow<16, 4>, false, true>();
  if (G == 32 && NV == 2) return make_variant<VecRow<32, 2>, false, true>();
  if (G == 32 && NV == 4) return make_variant<VecRow<32, 4>, false, true>();
  return Variant{};
}
}  // namespace tk
}  // namespace gb
