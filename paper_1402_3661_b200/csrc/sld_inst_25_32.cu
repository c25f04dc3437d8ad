// Kernel instantiations for moduli of 25..32 32-bit limbs.
#include "sld_ops.cuh"

namespace sld {
void fill_ops_25_32(LOps* t) { fill_ops_range<32, 25>(t); }
}  // namespace sld
