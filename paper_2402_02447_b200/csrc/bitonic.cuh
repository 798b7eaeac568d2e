// Warp-wide bitonic sort of 32*K keys held K per lane (blocked: element
// i = lane*K + j), ascending; shared by K3 (64-bit composite keys) and the
// Monte-Carlo balance kernel (32-bit lengths).  Padding keys sort last when
// they are the type's maximum.
#pragma once

namespace b2 {

template <int K, typename T>
__device__ __forceinline__ void warp_bitonic_sort(T (&key)[K], int lane) {
  constexpr int n = 32 * K;
#pragma unroll
  for (int size = 2; size <= n; size <<= 1) {
#pragma unroll
    for (int d = size >> 1; d > 0; d >>= 1) {
      if (d >= K) {  // partner in another lane, same slot
        const int lm = d / K;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const T other = __shfl_xor_sync(0xffffffffu, key[j], lm);
          const int i = lane * K + j;
          const bool up = (i & size) == 0;
          const bool take_min = (lower == up);
          const T mn = key[j] < other ? key[j] : other;
          const T mx = key[j] < other ? other : key[j];
          key[j] = take_min ? mn : mx;
        }
      } else {  // both elements in this lane
#pragma unroll
        for (int j = 0; j < K; ++j) {
          if ((j & d) == 0) {
            const int i = lane * K + j;
            const bool up = (i & size) == 0;
            const T a = key[j], b = key[j | d];
            if ((a > b) == up) {
              key[j] = b;
              key[j | d] = a;
            }
          }
        }
      }
    }
  }
}

}  // namespace b2
