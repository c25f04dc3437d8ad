// Kernel instantiations for moduli of 17..24 32-bit limbs.
#include "sld_ops.cuh"

namespace sld {
void fill_ops_17_24(LOps* t) { fill_ops_range<24, 17>(t); }
}  // namespace sld
