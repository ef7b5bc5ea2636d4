// vecreg.cuh — one feature vector per thread, in registers (select.cu,
// forest.cu): 256-bit / 128-bit loads of the row and x[f] by a compile-time
// select tree.  Internal to libadapt.so.
#pragma once
#include <cstdint>

namespace adapt {

// x[f] of a vector held in registers (N = 4, 8 or 16, a power of two): a
// select tree on the bits of f, all indices compile-time, no local memory
template <int N>
__device__ __forceinline__ float pick(const float (&x)[N], int f) {
  float t[N];
#pragma unroll
  for (int i = 0; i < N; i++) t[i] = x[i];
#pragma unroll
  for (int b = 0; (1 << b) < N; b++) {
    const bool hi = (f >> b) & 1;
#pragma unroll
    for (int i = 0; i < (N >> (b + 1)); i++) t[i] = hi ? t[2 * i + 1] : t[2 * i];
  }
  return t[0];
}

// a vector's F floats (F a multiple of 4; rows 16-byte aligned, 32-byte when
// `wide`) straight from global memory into registers
template <int F>
__device__ __forceinline__ void load_vec(const float *__restrict__ p, bool wide, float (&x)[F]) {
  if constexpr (F % 8 == 0) {
    if (wide) {
#pragma unroll
      for (int i = 0; i < F; i += 8)
        asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(x[i]), "=f"(x[i + 1]), "=f"(x[i + 2]), "=f"(x[i + 3]), "=f"(x[i + 4]), "=f"(x[i + 5]),
              "=f"(x[i + 6]), "=f"(x[i + 7])
            : "l"(p + i));
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < F; i += 4) {
    const float4 v = __ldcs(reinterpret_cast<const float4 *>(p + i));
    x[i] = v.x;
    x[i + 1] = v.y;
    x[i + 2] = v.z;
    x[i + 3] = v.w;
  }
}

}  // namespace adapt
