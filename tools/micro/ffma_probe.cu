// FP32 pipe microbenchmark: FFMA immediate / 3-register / uniform-register
// operand forms and packed FFMA2 (fma.rn.f32x2), to size the FP32 roofline of
// the certificate's 1-D tap loops (taps are register or uniform operands).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_probe ffma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NACC = 16;

__global__ void __launch_bounds__(256) k_imm(float* out, int iters) {
  float a[NACC];
  for (int i = 0; i < NACC; ++i) a[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < NACC; ++i) a[i] = fmaf(a[i], 0.999999f, 1e-7f);
  float s = 0; for (int i = 0; i < NACC; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}

// taps from memory (per-thread registers): FFMA R, R, R
__global__ void __launch_bounds__(256) k_reg(float* out, const float* taps, int iters) {
  float a[NACC], t[8];
  for (int i = 0; i < NACC; ++i) a[i] = threadIdx.x * 1e-7f + i;
  for (int r = 0; r < 8; ++r) t[r] = taps[(threadIdx.x + r) & 63];
  float w = taps[threadIdx.x & 63];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < NACC; ++i) a[i] = fmaf(t[r], w, a[i]) ;
  float s = 0; for (int i = 0; i < NACC; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}

// window x tap like the pass loops: a[i] += tap[r] * win[i + r]
__global__ void __launch_bounds__(256) k_win(float* out, const float* taps, int iters) {
  float a[NACC], win[NACC + 8], t[8];
  for (int i = 0; i < NACC; ++i) a[i] = 0;
  for (int i = 0; i < NACC + 8; ++i) win[i] = taps[(threadIdx.x + i) & 63];
  for (int r = 0; r < 8; ++r) t[r] = taps[r];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < NACC; ++i) a[i] = fmaf(t[r], win[i + r], a[i]);
  float s = 0; for (int i = 0; i < NACC; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}

__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void fma2(unsigned long long& c, unsigned long long a, unsigned long long b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}

// packed: c[i] += (t, t) * (win[2i], win[2i+1]) — NACC/2 FFMA2 = NACC lanes-ops per tap
__global__ void __launch_bounds__(256) k_win2(float* out, const float* taps, int iters) {
  unsigned long long a[NACC / 2], win[NACC / 2 + 4], t[8];
  for (int i = 0; i < NACC / 2; ++i) a[i] = 0;
  for (int i = 0; i < NACC / 2 + 4; ++i) win[i] = pk(taps[(threadIdx.x + 2 * i) & 63], taps[(threadIdx.x + 2 * i + 1) & 63]);
  for (int r = 0; r < 8; ++r) t[r] = pk(taps[r], taps[r]);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < NACC / 2; ++i) fma2(a[i], t[r], win[i + (r >> 1)]);
  float s = 0;
  for (int i = 0; i < NACC / 2; ++i) s += __uint_as_float(unsigned(a[i])) + __uint_as_float(unsigned(a[i] >> 32));
  if (s == 1.2345f) out[0] = s;
}

// taps in shared memory (uniform broadcast LDS per tap, as a kernel streams taps)
__global__ void __launch_bounds__(256) k_smemtap(float* out, const float* taps, int iters) {
  __shared__ float st[64];
  if (threadIdx.x < 64) st[threadIdx.x] = taps[threadIdx.x];
  __syncthreads();
  float a[NACC], win[NACC + 8];
  for (int i = 0; i < NACC; ++i) a[i] = 0;
  for (int i = 0; i < NACC + 8; ++i) win[i] = taps[(threadIdx.x + i) & 63];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float t = st[(it * 8 + r) & 63];
#pragma unroll
      for (int i = 0; i < NACC; ++i) a[i] = fmaf(t, win[i + r], a[i]);
    }
  float s = 0; for (int i = 0; i < NACC; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  float *out, *taps;
  cudaMalloc(&out, 4);
  cudaMalloc(&taps, 256 * 4);
  float h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1e-3f * (i % 17);
  cudaMemcpy(taps, h, sizeof h, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  const double fl = 2.0 * blocks * threads * double(iters) * 8 * NACC;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-10s %8.2f TFLOP/s  (%s)\n", name, 5 * fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run("imm", [&] { k_imm<<<blocks, threads>>>(out, iters); });
  run("reg", [&] { k_reg<<<blocks, threads>>>(out, taps, iters); });
  run("win", [&] { k_win<<<blocks, threads>>>(out, taps, iters); });
  run("win2", [&] { k_win2<<<blocks, threads>>>(out, taps, iters); });
  run("smemtap", [&] { k_smemtap<<<blocks, threads>>>(out, taps, iters); });
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms %d clock %d MHz nominal FFMA peak %.2f TFLOP/s\n", sms, clk / 1000, sms * 128 * 2.0 * clk * 1e3 / 1e12);
}
