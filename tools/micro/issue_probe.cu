// Does FFMA2 (fma.rn.f32x2) free issue slots? FMA-pipe work fixed (2 x 8 x NACC
// lane-FMAs per iteration), plus N independent ALU-pipe ops (LOP3) per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_probe issue_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NACC = 16;
__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r;
}
__device__ __forceinline__ void fma2(unsigned long long& c, unsigned long long a, unsigned long long b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}
template <int NALU>
__global__ void __launch_bounds__(256) k_ffma(float* out, const float* taps, int iters) {
  float a[NACC], w[NACC], t = taps[threadIdx.x & 63];
  unsigned x[8];
  for (int i = 0; i < NACC; ++i) { a[i] = 0; w[i] = taps[(threadIdx.x + i) & 63]; }
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * (i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) a[i] = fmaf(t, w[i], a[i]);
#pragma unroll
      for (int q = 0; q < NALU; ++q) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[q & 7]) : "r"(it), "r"(r));
    }
  }
  float s = 0; for (int i = 0; i < NACC; ++i) s += a[i];
  unsigned y = 0; for (int i = 0; i < 8; ++i) y ^= x[i];
  if (s == 1.2345f || y == 12345u) out[0] = s + y;
}
template <int NALU>
__global__ void __launch_bounds__(256) k_ffma2(float* out, const float* taps, int iters) {
  unsigned long long a[NACC / 2], w[NACC / 2], t;
  unsigned x[8];
  float tt = taps[threadIdx.x & 63];
  t = pk(tt, tt);
  for (int i = 0; i < NACC / 2; ++i) { a[i] = 0; w[i] = pk(taps[(threadIdx.x + 2 * i) & 63], taps[(threadIdx.x + 2 * i + 1) & 63]); }
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * (i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int i = 0; i < NACC / 2; ++i) fma2(a[i], t, w[i]);
#pragma unroll
      for (int q = 0; q < NALU; ++q) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[q & 7]) : "r"(it), "r"(r));
    }
  }
  float s = 0; for (int i = 0; i < NACC / 2; ++i) s += __uint_as_float(unsigned(a[i])) + __uint_as_float(unsigned(a[i] >> 32));
  unsigned y = 0; for (int i = 0; i < 8; ++i) y ^= x[i];
  if (s == 1.2345f || y == 12345u) out[0] = s + y;
}
// broadcast operand: (x, x) built from one scalar register per step
__global__ void __launch_bounds__(256) k_bcast(float* out, const float* taps, int iters) {
  unsigned long long a[NACC / 2], w[NACC / 2];
  float t[4];
  for (int i = 0; i < 4; ++i) t[i] = taps[(threadIdx.x + i) & 63];
  for (int i = 0; i < NACC / 2; ++i) { a[i] = 0; w[i] = pk(taps[(threadIdx.x + 2 * i) & 63], taps[(threadIdx.x + 2 * i + 1) & 63]); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const unsigned long long tb = pk(t[(it + r) & 3], t[(it + r) & 3]);
#pragma unroll
      for (int i = 0; i < NACC / 2; ++i) fma2(a[i], tb, w[i]);
    }
    t[it & 3] += 1e-7f;
  }
  float s = 0; for (int i = 0; i < NACC / 2; ++i) s += __uint_as_float(unsigned(a[i])) + __uint_as_float(unsigned(a[i] >> 32));
  if (s == 1.2345f) out[0] = s;
}
int main() {
  float *out, *taps;
  cudaMalloc(&out, 4); cudaMalloc(&taps, 256 * 4);
  float h[256]; for (int i = 0; i < 256; ++i) h[i] = 1e-3f * (i % 17);
  cudaMemcpy(taps, h, sizeof h, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 8192, blocks = sms * 8, threads = 256;
  const double fl = 2.0 * blocks * threads * double(iters) * 2 * NACC;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 3; ++r) launch(); cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-12s %8.2f TFLOP/s (fma part)  %s\n", name, 3 * fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run("ffma+0alu", [&] { k_ffma<0><<<blocks, threads>>>(out, taps, iters); });
  run("ffma+8alu", [&] { k_ffma<8><<<blocks, threads>>>(out, taps, iters); });
  run("ffma+16alu", [&] { k_ffma<16><<<blocks, threads>>>(out, taps, iters); });
  run("ffma2+0alu", [&] { k_ffma2<0><<<blocks, threads>>>(out, taps, iters); });
  run("ffma2+8alu", [&] { k_ffma2<8><<<blocks, threads>>>(out, taps, iters); });
  run("ffma2+16alu", [&] { k_ffma2<16><<<blocks, threads>>>(out, taps, iters); });
  run("ffma2 bcast", [&] { k_bcast<<<blocks, threads>>>(out, taps, iters); });
}
