// Register-window correlation helpers shared by the certificate (eta.cu)
// and the 1-D pass kernels (psf.cu).
#pragma once

#include <utility>

#include "internal.cuh"

namespace sfw3d {

template <typename T>
__device__ __forceinline__ void ld4(const T* p, T& a, T& b, T& c, T& d) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    a = v.x; b = v.y; c = v.z; d = v.w;
  } else {
    const double2 v0 = *reinterpret_cast<const double2*>(p);
    const double2 v1 = *reinterpret_cast<const double2*>(p + 2);
    a = v0.x; b = v0.y; c = v1.x; d = v1.y;
  }
}

// shared-memory 4-vector load as a volatile asm statement: ptxas keeps the
// program order of these loads, so the folded kernel's loads stay exactly one
// step ahead of their use instead of being hoisted (register pressure)
template <typename T>
__device__ __forceinline__ void lds4v(const T* p, T& a, T& b, T& c, T& d) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(p));
  if constexpr (sizeof(T) == 4) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "r"(sa));
  } else {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(sa));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(c), "=d"(d) : "r"(sa + 16));
  }
}

template <typename T>
__device__ __forceinline__ void ldg4(const T* p, T& a, T& b, T& c, T& d) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    a = v.x; b = v.y; c = v.z; d = v.w;
  } else {
    const double2 v0 = __ldg(reinterpret_cast<const double2*>(p));
    const double2 v1 = __ldg(reinterpret_cast<const double2*>(p + 2));
    a = v0.x; b = v0.y; c = v1.x; d = v1.y;
  }
}

// acc[j] += sum_{c < 4 ns} trow[c] * (sum_{r < NR} q_r[j + c]),  j < KJ
// (q_r, trow in shared memory, 16-byte aligned). Each thread slides a
// (KJ + 4)-register window along its row(s), 4 taps per step:
//   sum the NR rows' next 4 columns (loaded one step earlier) into the slots
//   freed by the previous step, issue the loads for the following step and
//   the next 4 taps, then 4 KJ FFMA (tap-major, KJ independent chains).
// The window rotation is resolved at compile time (no register moves); the
// loads are volatile asm so they stay one step ahead (register pressure).
// Reads q_r[0 .. KJ + 4 ns + 4) and trow[0 .. 4 ns + 4).
template <typename T, int KJ, int NR>
struct Fold {
  static constexpr int W = KJ + 4;  // window registers
  static constexpr int NS = W / 4;  // steps per full rotation

  template <int R>
  static __device__ __forceinline__ void step(T (&acc)[KJ], T (&buf)[W], T (&tc)[4], T (&u)[NR][4],
                                              const T* __restrict__ tnext,
                                              const T* const (&q)[NR], int col) {
    // columns KJ..KJ+3 of this window (loaded last step) into freed slots
#pragma unroll
    for (int i = 0; i < 4; ++i) buf[(4 * R + KJ + i) % W] = NR == 2 ? u[0][i] + u[NR - 1][i] : u[0][i];
    // next step's new columns and taps
#pragma unroll
    for (int r = 0; r < NR; ++r) lds4v(q[r] + col + KJ + 4, u[r][0], u[r][1], u[r][2], u[r][3]);
    T n0, n1, n2, n3;
    lds4v(tnext, n0, n1, n2, n3);  // shared-memory tap row (broadcast)
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < KJ; ++j) acc[j] = fma(tc[k], buf[(4 * R + j + k) % W], acc[j]);
    tc[0] = n0;
    tc[1] = n1;
    tc[2] = n2;
    tc[3] = n3;
  }

  static __device__ __forceinline__ void row(T (&acc)[KJ], const T* __restrict__ trow,
                                             const T* const (&q)[NR], int ns) {
    T buf[W], tc[4], u[NR][4];
    lds4v(trow, tc[0], tc[1], tc[2], tc[3]);
#pragma unroll
    for (int g = 0; g < KJ / 4; ++g) {
      T s0, s1, s2, s3;
      lds4v(q[0] + 4 * g, s0, s1, s2, s3);
      if constexpr (NR == 2) {
        T v0, v1, v2, v3;
        lds4v(q[1] + 4 * g, v0, v1, v2, v3);
        s0 += v0; s1 += v1; s2 += v2; s3 += v3;
      }
      buf[4 * g] = s0;
      buf[4 * g + 1] = s1;
      buf[4 * g + 2] = s2;
      buf[4 * g + 3] = s3;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) lds4v(q[r] + KJ, u[r][0], u[r][1], u[r][2], u[r][3]);
    int s = 0;
    for (; s + NS <= ns; s += NS) unrolled(acc, buf, tc, u, trow, q, s, std::make_integer_sequence<int, NS>{});
    const int rem = ns - s;
    tail(acc, buf, tc, u, trow, q, s, rem, std::make_integer_sequence<int, NS - 1>{});
  }

  template <int... R>
  static __device__ __forceinline__ void unrolled(T (&acc)[KJ], T (&buf)[W], T (&tc)[4],
                                                  T (&u)[NR][4], const T* trow,
                                                  const T* const (&q)[NR], int s,
                                                  std::integer_sequence<int, R...>) {
    (step<R>(acc, buf, tc, u, trow + 4 * (s + R) + 4, q, 4 * (s + R)), ...);
  }
  template <int... R>
  static __device__ __forceinline__ void tail(T (&acc)[KJ], T (&buf)[W], T (&tc)[4], T (&u)[NR][4],
                                              const T* trow, const T* const (&q)[NR], int s,
                                              int rem, std::integer_sequence<int, R...>) {
    ((rem > R ? step<R>(acc, buf, tc, u, trow + 4 * (s + R) + 4, q, 4 * (s + R)) : void()), ...);
  }
};

}  // namespace sfw3d
