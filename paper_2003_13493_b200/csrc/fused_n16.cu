// Fused detector kernels for arc length N = 16 (see kernels_fused.cuh).
#include "fused_dispatch.hpp"

FLKB_FUSED_INSTANTIATE(16)
