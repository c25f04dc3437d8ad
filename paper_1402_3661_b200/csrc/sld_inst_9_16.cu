// Kernel instantiations for moduli of 9..16 32-bit limbs.
#include "sld_ops.cuh"

namespace sld {
void fill_ops_9_16(LOps* t) { fill_ops_range<16, 9>(t); }
}  // namespace sld
