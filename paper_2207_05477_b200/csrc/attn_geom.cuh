// Geometry of one gated-attention call: problems are (batch b, position l);
// the token row of (b, l) in the token-major buffers is b*sb + l*sl and the
// key-mask element is mask[b*msb + l*msl].
#pragma once
#include <stdint.h>

namespace evo {
struct AttnGeom {
  int64_t B, L, H, D, sb, sl, ld, msb, msl;
  __host__ __device__ int64_t tok(int64_t b, int64_t l) const { return b * sb + l * sl; }
};
}  // namespace evo
