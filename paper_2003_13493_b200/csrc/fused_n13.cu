// Fused detector kernels for arc length N = 13 (see kernels_fused.cuh).
#include "fused_dispatch.hpp"

FLKB_FUSED_INSTANTIATE(13)
