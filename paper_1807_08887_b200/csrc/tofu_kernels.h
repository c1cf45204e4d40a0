// Kernel-level entry points of libtofu (device work).  Declared publicly in include/tofu.h;
// this internal header only repeats the argument structs for the .cu translation units.
#pragma once
#include <cstdlib>

#include "../../include/tofu.h"

namespace tofu {
// Stream-K share of a persistent tcgen05 launch (common.cuh WorkList): 0 = all tiles data-parallel.  Used when
// the data-parallel waves would leave SMs idle (tile count not a multiple of the SM count, efficiency < 92%),
// the caller supplied a stream-K workspace, and every CTA gets at least 4 k-blocks.  The stream-K region is
// the last partial wave plus one full wave (all tiles when there is less than two waves).
// splitk_alt: the kernel has split-K with a parallel plane reduction, which is used instead when the tiles
// fill at most half the SMs (stream-K would leave the whole reduction to one finisher CTA per tile).
// intensity: algorithmic flops / HBM bytes of the launch.  Stream-K pays an fp32 partial round trip per cut
// tile and only helps compute-bound launches (a memory-bound launch's last partial wave runs at full HBM
// bandwidth anyway): it is used from 2.5x the B200 ridge point (1343 TFLOP/s / 6.5 TB/s ~ 200 flop/B) up.
// Measured on the WResNet 1x1 shapes (tools/sk_bench.py): wins at >= 615 flop/B, loses at <= 424.
inline double sk_min_intensity() {  // TOFU_SK_AI overrides the threshold (A/B measurements)
  static const double v = [] {
    const char* e = std::getenv("TOFU_SK_AI");
    return e ? std::atof(e) : 500.0;
  }();
  return v;
}
inline int sk_tiles_for(int tiles, int nk, int sms, const void* sk_ws, bool splitk_alt, double intensity) {
  if (!sk_ws || tiles <= 0 || nk < 4 || (splitk_alt && tiles * 2 <= sms) || intensity < sk_min_intensity()) return 0;
  const int waves = (tiles + sms - 1) / sms;
  if ((double)tiles / ((double)waves * sms) >= 0.92) return 0;
  const int sk = tiles < 2 * sms ? tiles : tiles % sms + sms;
  if ((int64_t)sk * nk < 4LL * sms) return 0;
  return sk;
}
}  // namespace tofu
