// Does a 64 MiB volume stay L2-resident across ping-pong passes on B200?
// copy-like pass A -> B -> A ... with per-access L2 eviction hints.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_pingpong l2_pingpong.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long policy(int kind) {
  unsigned long long p;
  if (kind == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_hint(const float4* p, unsigned long long pol) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(float4* p, float4 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// mode: 0 plain ld / __stcs store; 1 plain ld / plain st; 2 hints (ldk, stk)
__global__ void __launch_bounds__(256) pass(const float4* __restrict__ in, float4* __restrict__ out,
                                            long long n4, int mode, int ldk, int stk, int reverse) {
  const unsigned long long pl = policy(ldk), ps = policy(stk);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride) {
    const long long i = reverse ? n4 - 1 - i0 : i0;
    float4 v = mode == 2 ? ld_hint(in + i, pl) : in[i];
    v.x = v.x * 1.0001f + 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
    if (mode == 0) __stcs(out + i, v);
    else if (mode == 1) out[i] = v;
    else st_hint(out + i, v, ps);
  }
}

int main(int argc, char** argv) {
  const double mib = argc > 1 ? atof(argv[1]) : 64.0;
  const long long n4 = (long long)(mib * 1024 * 1024 / 16);
  float4 *a, *b;
  cudaMalloc(&a, n4 * 16); cudaMalloc(&b, n4 * 16);
  cudaMemset(a, 0, n4 * 16); cudaMemset(b, 0, n4 * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148 * 8;
  struct Cfg { const char* name; int mode, ldk, stk, rev; } cfgs[] = {
    {"ld plain / st.cs", 0, 0, 0, 0}, {"ld plain / st plain", 1, 0, 0, 0},
    {"ld first / st last", 2, 0, 2, 0}, {"ld first / st normal", 2, 0, 1, 0},
    {"ld normal / st last", 2, 1, 2, 0}, {"ld first / st first", 2, 0, 0, 0},
    {"ld first / st last, alternate direction", 2, 0, 2, 1},
    {"ld plain / st plain, alternate direction", 1, 0, 0, 1},
    {"ld normal / st last, alternate direction", 2, 1, 2, 1},
  };
  for (auto& c : cfgs) {
    const int passes = 24;
    for (int w = 0; w < 4; ++w) pass<<<grid, 256>>>(w % 2 ? b : a, w % 2 ? a : b, n4, c.mode, c.ldk, c.stk, c.rev ? w % 2 : 0);
    cudaEventRecord(e0);
    for (int p = 0; p < passes; ++p)
      pass<<<grid, 256>>>(p % 2 ? b : a, p % 2 ? a : b, n4, c.mode, c.ldk, c.stk, c.rev ? p % 2 : 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%6.0f MiB  %-44s %8.2f us/pass  %8.1f GB/s (read+write)\n", mib, c.name, 1e3 * ms / passes,
           2.0 * n4 * 16 / (ms / passes * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
