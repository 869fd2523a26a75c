// Exact separable translation shifts (M2M up, L2L down), shared by the
// cascade kernels (expand.cu) and the separable M2L epilogue (m2l_sep.cu).
#pragma once
#include "common.cuh"

namespace fc2t2 {

template <int RHO, int AXIS, bool UP>
__device__ __forceinline__ void shift_axis(const float (&in)[MI<RHO>::P], float (&out)[MI<RHO>::P],
                                           const float (&t)[RHO + 1]) {
  constexpr MI<RHO> mi{};
  constexpr int P = MI<RHO>::P;
#pragma unroll
  for (int n = 0; n < P; ++n) {
    const int e0 = mi.e0[n], e1 = mi.e1[n], e2 = mi.e2[n];
    float s = 0.f;
#pragma unroll
    for (int m = 0; m <= RHO; ++m) {
      const int d0 = AXIS == 0 ? (UP ? -m : m) : 0;
      const int d1 = AXIS == 1 ? (UP ? -m : m) : 0;
      const int d2 = AXIS == 2 ? (UP ? -m : m) : 0;
      const int j = MI<RHO>::index(e0 + d0, e1 + d1, e2 + d2);
      if (j >= 0) s = fmaf(in[j], t[m], s);
    }
    out[n] = s;
  }
}

template <int RHO, bool UP>
__device__ __forceinline__ void shift3(float (&v)[MI<RHO>::P], float dx, float dy, float dz) {
  constexpr int P = MI<RHO>::P;
  float tx[RHO + 1], ty[RHO + 1], tz[RHO + 1];
  tx[0] = ty[0] = tz[0] = 1.f;
#pragma unroll
  for (int m = 1; m <= RHO; ++m) {
    tx[m] = tx[m - 1] * dx / (float)m;
    ty[m] = ty[m - 1] * dy / (float)m;
    tz[m] = tz[m - 1] * dz / (float)m;
  }
  float u[P];
  shift_axis<RHO, 0, UP>(v, u, tx);
  shift_axis<RHO, 1, UP>(u, v, ty);
  shift_axis<RHO, 2, UP>(v, u, tz);
#pragma unroll
  for (int n = 0; n < P; ++n) v[n] = u[n];
}

}  // namespace fc2t2
