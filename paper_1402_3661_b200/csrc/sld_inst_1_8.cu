// Kernel instantiations for moduli of 1..8 32-bit limbs.
#include "sld_ops.cuh"

namespace sld {
void fill_ops_1_8(LOps* t) { fill_ops_range<8, 1>(t); }
}  // namespace sld
