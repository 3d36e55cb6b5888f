// Kernel-family timing (sfw3d_ctx_profile) and the FP32 peak probe.
#include "internal.cuh"

namespace sfw3d {

ProfScope::ProfScope(sfw3d_ctx* c, const char* f) : ctx(c), family(f) {
  if (!ctx->profile) return;
  cudaEvent_t start;
  if (cudaEventCreate(&start) != cudaSuccess || cudaEventCreate(&stop) != cudaSuccess) {
    stop = nullptr;
    return;
  }
  cudaEventRecord(start, ctx->stream);
  ctx->marks.push_back({family, start, nullptr});
}

ProfScope::~ProfScope() {
  if (!ctx->profile || !stop) return;
  cudaEventRecord(stop, ctx->stream);
  ctx->marks.back().stop = stop;
}

static void drain_marks(sfw3d_ctx* ctx) {
  for (auto& m : ctx->marks) {
    float ms = 0.f;
    if (m.stop) {
      cudaEventSynchronize(m.stop);
      cudaEventElapsedTime(&ms, m.start, m.stop);
      cudaEventDestroy(m.stop);
    }
    cudaEventDestroy(m.start);
    bool found = false;
    for (auto& t : ctx->totals)
      if (t.first == m.family) {
        t.second.first += ms;
        t.second.second += 1;
        found = true;
      }
    if (!found) ctx->totals.push_back({m.family, {double(ms), 1LL}});
  }
  ctx->marks.clear();
}

namespace probe_detail {
__global__ void __launch_bounds__(256) fma_probe_kernel(float* out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-7f + i;
  const float m = 0.999999f, c = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], m, c);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678f) out[0] = s;  // keep the loop alive
}
}  // namespace

}  // namespace sfw3d

using namespace sfw3d;

extern "C" int sfw3d_ctx_profile(sfw3d_ctx* ctx, int enable) {
  SFW3D_CHECK_ARG(ctx, "ctx is NULL");
  SFW3D_TRY(activate(ctx));
  drain_marks(ctx);
  ctx->totals.clear();
  ctx->profile = enable ? 1 : 0;
  return SFW3D_OK;
}

extern "C" int sfw3d_ctx_profile_read(sfw3d_ctx* ctx, const char* family, double* total_ms,
                                      int64_t* launches) {
  SFW3D_CHECK_ARG(ctx && family, "NULL argument");
  SFW3D_TRY(activate(ctx));
  drain_marks(ctx);
  double ms = 0.0;
  long long n = 0;
  for (auto& t : ctx->totals)
    if (t.first == family) {
      ms = t.second.first;
      n = t.second.second;
    }
  if (total_ms) *total_ms = ms;
  if (launches) *launches = n;
  return SFW3D_OK;
}

extern "C" int sfw3d_probe_fp32(sfw3d_ctx* ctx, double* tflops) {
  SFW3D_CHECK_ARG(ctx && tflops, "NULL argument");
  SFW3D_TRY(begin_call(ctx));
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small, 4096));
  float* out = static_cast<float*>(ctx->ws_small.ptr);
  const int blocks = ctx->num_sms * 8;  // 64 warps per SM
  const int iters = 4096;
  cudaEvent_t a, b;
  SFW3D_CUDA_TRY(cudaEventCreate(&a));
  SFW3D_CUDA_TRY(cudaEventCreate(&b));
  probe_detail::fma_probe_kernel<<<blocks, 256, 0, ctx->stream>>>(out, 64, 1.0f);  // warm-up
  SFW3D_LAUNCH_CHECK(ctx);
  SFW3D_CUDA_TRY(cudaEventRecord(a, ctx->stream));
  probe_detail::fma_probe_kernel<<<blocks, 256, 0, ctx->stream>>>(out, iters, 1.0f);
  SFW3D_LAUNCH_CHECK(ctx);
  SFW3D_CUDA_TRY(cudaEventRecord(b, ctx->stream));
  SFW3D_CUDA_TRY(cudaEventSynchronize(b));
  float ms = 0.f;
  SFW3D_CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const double flops = 2.0 * double(blocks) * 256.0 * iters * 16.0 * 8.0;
  *tflops = flops / (double(ms) * 1e-3) / 1e12;
  return SFW3D_OK;
}
