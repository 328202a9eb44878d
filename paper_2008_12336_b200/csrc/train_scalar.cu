// Instantiations of the any-dim (scalar) layouts, fast and exact.
#include "train_kernels.cuh"

namespace gb {
namespace tk {
Variant scalar_variant(int NS, bool exact) {
#define GB_S(ns)                                                                  \
  if (NS == ns)                                                                   \
    return exact ? make_variant<ScalarRow<ns>, true>() : make_variant<ScalarRow<ns>, false>();
  GB_S(1) GB_S(2) GB_S(4) GB_S(8) GB_S(16)
#undef GB_S
  return Variant{};
}
}  // namespace tk
}  // namespace gb
