// rounding.cuh -- step a2 (round-up of a request), shared by K1 and K2.
//
// PAPER.md:153-154, 256 (i) "rounded up to the nearest hardware-required
// multiple" (512 B); with the NEXT-4 variant torch's
// roundup_power2_divisions:N (reading Q20): a request above
// min_block * N goes to the next multiple of 2^k / N, 2^k <= request < 2^(k+1)
// (a power of two stays). Requests are < 2^40 (XM_MAX_REQUEST), so the result
// is <= 2^40 and fits 32 bits in units of min_block (>= 512 B).
#pragma once
#include <cstdint>

#include "xm_internal.h"

namespace xm_internal {

__device__ __forceinline__ uint32_t round_units(uint64_t mag, const UnitConfig& u) {
  const uint64_t m1 = (1ull << u.unit_shift) - 1;
  if (u.div_shift && mag > (1ull << (u.unit_shift + u.div_shift))) {
    const int k = 63 - __clzll(static_cast<long long>(mag));
    const uint64_t s1 = (1ull << (k - int(u.div_shift))) - 1;   // step - 1, step >= min_block
    return uint32_t(((mag + s1) & ~s1) >> u.unit_shift);
  }
  return uint32_t((mag + m1) >> u.unit_shift);
}

}  // namespace xm_internal
