// Kernel-pointer dispatch for the fused detector: one translation unit per
// arc length N instantiates the 3 score kinds x {radius 1, generic radius} x
// {plain, counting (stats)}.
#pragma once

#include "kernels_fused.cuh"

namespace flkb {
namespace fused {

using KernelFn = void (*)(const Params);

KernelFn kernel_n9(int kind, int radius, bool stats);
KernelFn kernel_n10(int kind, int radius, bool stats);
KernelFn kernel_n11(int kind, int radius, bool stats);
KernelFn kernel_n12(int kind, int radius, bool stats);
KernelFn kernel_n13(int kind, int radius, bool stats);
KernelFn kernel_n14(int kind, int radius, bool stats);
KernelFn kernel_n15(int kind, int radius, bool stats);
KernelFn kernel_n16(int kind, int radius, bool stats);

inline KernelFn kernel_for(int n, int kind, int radius, bool stats) {
  switch (n) {
    case 9: return kernel_n9(kind, radius, stats);
    case 10: return kernel_n10(kind, radius, stats);
    case 11: return kernel_n11(kind, radius, stats);
    case 12: return kernel_n12(kind, radius, stats);
    case 13: return kernel_n13(kind, radius, stats);
    case 14: return kernel_n14(kind, radius, stats);
    case 15: return kernel_n15(kind, radius, stats);
    default: return kernel_n16(kind, radius, stats);
  }
}

}  // namespace fused
}  // namespace flkb

// Body of kernel_nN: expanded once per arc length in fused_nN.cu.
#define FLKB_FUSED_PICK(NN, S)                                            \
  if (radius == 1) {                                                      \
    if (kind == kSadB) return k_detect<NN, kSadB, 1, S>;                  \
    if (kind == kSadA) return k_detect<NN, kSadA, 1, S>;                  \
    return k_detect<NN, kMt, 1, S>;                                       \
  }                                                                       \
  if (kind == kSadB) return k_detect<NN, kSadB, 0, S>;                    \
  if (kind == kSadA) return k_detect<NN, kSadA, 0, S>;                    \
  return k_detect<NN, kMt, 0, S>;

#define FLKB_FUSED_INSTANTIATE(NN)                                        \
  namespace flkb {                                                        \
  namespace fused {                                                       \
  KernelFn kernel_n##NN(int kind, int radius, bool stats) {               \
    if (stats) {                                                          \
      FLKB_FUSED_PICK(NN, true)                                           \
    }                                                                     \
    FLKB_FUSED_PICK(NN, false)                                            \
  }                                                                       \
  }                                                                       \
  }
