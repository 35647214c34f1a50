// Division by a runtime-invariant 32-bit divisor as one multiply-high and a
// shift (round-up reciprocal, exact for dividends < 2^31), so the fused
// kernels' strip -> (frame, block row, strip column) decomposition costs a
// handful of integer instructions instead of a 64-bit division call and the
// branches around it (which also split the strip body's basic block).
#pragma once
#include <cstdint>

namespace dctf {
struct FastDiv {
  uint32_t d, m, s;
};
__host__ __device__ __forceinline__ FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0u, 0u};
  if (d > 1) {
#ifdef __CUDA_ARCH__
    const uint32_t l = 32u - static_cast<uint32_t>(__clz(d - 1));  // ceil(log2 d)
#else
    const uint32_t l = 32u - static_cast<uint32_t>(__builtin_clz(d - 1));
#endif
    const uint32_t p = 31u + l;
    f.m = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
    f.s = p - 32u;
  }
  return f;
}
__device__ __forceinline__ uint32_t fdiv(const FastDiv& f, uint32_t n) {
  return f.d == 1 ? n : (__umulhi(n, f.m) >> f.s);
}
}  // namespace dctf
