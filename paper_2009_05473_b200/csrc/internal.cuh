// Internal declarations shared by the sfw3d CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/sfw3d_cuda.h"

namespace sfw3d {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);

struct Status {
  int code;
  Status(int c = SFW3D_OK) : code(c) {}
};

#define SFW3D_CHECK_ARG(cond, msg)                   \
  do {                                               \
    if (!(cond)) {                                   \
      ::sfw3d::set_error(std::string("invalid argument: ") + (msg)); \
      return SFW3D_EINVAL;                           \
    }                                                \
  } while (0)

#define SFW3D_CUDA_TRY(expr)                                                  \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::sfw3d::set_error(std::string("CUDA error ") + cudaGetErrorString(_e) + \
                         " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
      return _e == cudaErrorMemoryAllocation ? SFW3D_ENOMEM : SFW3D_ECUDA;    \
    }                                                                         \
  } while (0)

#define SFW3D_LAUNCH_CHECK(ctx)                 \
  do {                                          \
    (ctx)->launches++;                          \
    SFW3D_CUDA_TRY(cudaGetLastError());         \
  } while (0)

// Records a CUDA event pair around a kernel launch when profiling is on.
#define SFW3D_PROF(ctx, family) ::sfw3d::ProfScope _prof_scope((ctx), (family))

#define SFW3D_TRY(expr)            \
  do {                             \
    int _s = (expr);               \
    if (_s != SFW3D_OK) return _s; \
  } while (0)

// ---------------------------------------------------------------- context
struct Arena {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace sfw3d

struct sfw3d_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t launches = 0;
  // L2 residency of the 1-D pass chains (psf.cu: pass_typed sets it per pass):
  // 1 when a pass's input and output volumes fit the 126 MB L2 together well
  // enough to ping-pong there (input lines evict-first once consumed, output
  // lines kept for the next pass), 0 for streaming volumes
  int l2mode = 0;
  sfw3d::Arena ws;         // device scratch (grown on demand, reused)
  sfw3d::Arena pinned;     // pinned host staging for uploads (bump-allocated)
  size_t pin_off = 0;      // bytes of `pinned` referenced by in-flight copies
  sfw3d::Arena pinned_out; // pinned host buffer for small downloads
  sfw3d::Arena ws_small;   // small device scratch (params, partials)
  sfw3d::Arena ws_aux;     // auxiliary small device scratch (render culling boxes)
  sfw3d::Arena ws_plan;    // atom-sum chunk plan + chunk partials
  sfw3d::Arena pinned_io;  // pinned staging of the .vol reader / writer
  // single-atom ascent evaluations (atoms.cu: refine_sums_impl): ticket + CTA
  // partials on the device, result + sequence flag in mapped pinned memory
  sfw3d::Arena ws_one;
  void* one_host = nullptr;
  void* one_host_dev = nullptr;
  unsigned long long one_seq = 0;
  // kernel-family timing (sfw3d_ctx_profile)
  int profile = 0;
  struct Mark {
    const char* family;
    cudaEvent_t start, stop;
  };
  std::vector<Mark> marks;
  std::vector<std::pair<std::string, std::pair<double, long long>>> totals;
};

namespace sfw3d {

int ensure_device(sfw3d_ctx* ctx, Arena& a, size_t bytes);
int ensure_pinned_io(sfw3d_ctx* ctx, size_t bytes);
// Host->device upload through the pinned staging area (asynchronous on
// ctx->stream). The staging area is recycled at the next begin_call or
// after a synchronising download.
int stage_upload(sfw3d_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
// Device->host copy through pinned memory; synchronises ctx->stream.
int download_sync(sfw3d_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);
// Called at the top of every ABI entry point.
int begin_call(sfw3d_ctx* ctx);
int activate(sfw3d_ctx* ctx);  // cudaSetDevice

struct ProfScope {
  sfw3d_ctx* ctx;
  cudaEvent_t stop = nullptr;
  const char* family;
  ProfScope(sfw3d_ctx* c, const char* f);
  ~ProfScope();
};

// Carves aligned sub-buffers from a workspace arena.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* p) : base(static_cast<char*>(p)) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
  static size_t need(const std::vector<size_t>& sizes) {
    size_t o = 0;
    for (size_t s : sizes) o = ((o + 255) & ~size_t(255)) + s;
    return o + 256;
  }
};

// ---------------------------------------------------------------- atoms
// The reference's tail exponent 2*ln(1/1e-12) (forward.py:34), as the exact
// double numpy produces.
extern const double kTailExponent;

// Per-atom descriptor with the support box resolved on the host exactly as
// forward.py:97-116 does (libm pow/ceil/rint in float64).
struct AtomGeo {
  double w, m[3], sigma, d;
  double inv2sd;     // 0.5 / sigma**d           (forward.py:135)
  double half_d;     // 0.5 * d                   (forward.py:136)
  double log_sigma;  // log(sigma)                (forward.py:150)
  double d_over_sigma;
  int start[3];      // first span value (unwrapped), 0 for a full axis
  int len[3];        // box length per axis
  int full[3];       // 1 when 2R+1 >= n (minimum-image full axis)
  int d2;            // d == 2.0 exactly          (forward.py:136)
  int radius;
  long long nvox;
};

// Builds AtomGeo rows; returns SFW3D_EINVAL for sigma<=0, d<=0 or
// non-finite parameters (forward.py:130-131, measures.py:80-82).
int build_atoms(const int dims[3], const double* params, int k, std::vector<AtomGeo>& out);
// the six unit-atom inner products of ONE atom against a device field, fp64
// math, result returned on the host (the certificate ascent's evaluation)
int refine_sums_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* field,
                     const AtomGeo& atom, double out[6]);

// ---------------------------------------------------------------- PSF
}  // namespace sfw3d

namespace sfw3d { struct PsfFft; }

struct sfw3d_psf {
  int dims[3];
  int separable;
  int lo[3], hi[3];              // non-zero offset box (offset = index - n//2)
  // separable: taps per axis over [lo, hi]; device f64 and f32 copies
  double* taps64[3] = {nullptr, nullptr, nullptr};
  float* taps32[3] = {nullptr, nullptr, nullptr};
  // general: dense box over [lo, hi]^3 (C order)
  double* box64 = nullptr;
  float* box32 = nullptr;
  int device = 0;
  // general kernels at size: cuFFT plans + kernel spectra (fft.cu), lazily
  mutable sfw3d::PsfFft* fft = nullptr;
};

namespace sfw3d {

// Applies the PSF (or its adjoint) on ctx->stream. tmp_dev: one scratch
// volume of the same dtype (may alias nothing else). in != out.
int psf_apply_impl(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in,
                   void* out, int adjoint, void* tmp);

// One circular 1-D correlation pass along `axis`:
//   out[i] = addend_w * addend[i] + w * sum_q taps[q] * in[i + (lo + q) e_axis]
// (addend may be NULL or alias out; taps are device pointers of the dtype).
// Axis-0 output plane range: outputs a in [begin, end) (end < 0: the whole
// axis) are written to plane a + shift of `out`.
struct XRange {
  int begin = 0, end = -1, shift = 0;
  double* sq = nullptr;     // (axis-0 tiled pass with an addend) per-CTA sum of squares
  mutable int nsq = 0;      // number of partials written
};
int corr_pass_impl(sfw3d_ctx* ctx, int dtype, const void* in, void* out, const int dims[3], int axis,
                   const void* taps, int lo, int ntaps, const void* addend, double addend_w,
                   double w, const char* family, const XRange* xr = nullptr);

// x-slab data plane (multi-GPU certificate): the caller's halo exchange and
// all-reduce (include/sfw3d_cuda.h: sfw3d_halo_fn, sfw3d_allreduce_fn).
struct SlabLink {
  sfw3d_halo_fn halo = nullptr;
  sfw3d_allreduce_fn allreduce = nullptr;
  void* user = nullptr;
};
int slab_corr_impl(sfw3d_ctx* ctx, int dtype, const void* in, void* out, const int odims[3],
                   const void* const taps[3], const int lo[3], const int nt[3], void* win, int H,
                   void* tmp, const SlabLink& link, const char* family);
bool psf_use_fft(const sfw3d_psf* psf);
int psf_apply_resid(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                    void* tmp, const void* y, double* sq_parts, int max_parts, int* nparts);
// fixed-order fp64 sum of n partials into *out (atoms.cu)
int sum_parts_impl(sfw3d_ctx* ctx, const double* parts, int n, double* out);
int psf_fft_apply(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                  int adjoint);
void psf_fft_destroy(sfw3d_psf* psf);
int psf_apply_slab(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                   int adjoint, const int odims[3], void* win, int H, void* tmp,
                   const SlabLink& link);

// Launch helpers implemented in the .cu files.
int render_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const std::vector<AtomGeo>& atoms,
                const AtomGeo* atoms_dev,
                int k, void* out);
int atom_sums_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* field,
                   const std::vector<AtomGeo>& atoms, const AtomGeo* atoms_dev,
                   double* sums_dev);

// fp64 block reductions
int sumsq_diff_impl(sfw3d_ctx* ctx, int dtype, int64_t n, const void* a, const void* b,
                    void* diff_out, double* partials, double* result_dev);

// Packed fp32 pairs (sm_100 FFMA2 / FMUL2: two independent RN operations per
// instruction, bit-identical to the scalar ones). Low half = first element.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
  return (f32x2)__float_as_uint(lo) | ((f32x2)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo32(f32x2 v) { return __uint_as_float(unsigned(v)); }
__device__ __forceinline__ float hi32(f32x2 v) { return __uint_as_float(unsigned(v >> 32)); }

// Raise a kernel's dynamic shared-memory limit MONOTONICALLY (per device):
// contexts on several host threads launch the same kernel with different
// sizes, and a per-launch cudaFuncSetAttribute could lower the limit under a
// concurrent launch ("invalid argument").
inline cudaError_t allow_dynamic_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> lim;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> guard(mu);
  size_t& cur = lim[{dev, func}];
  if (bytes <= cur) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// Asynchronous global->shared copies (LDGSTS): staging loops issue all of
// their copies without a register round trip, then wait once.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// L2 eviction policy of a pass's global accesses (first = 1: evict-first)
__device__ __forceinline__ unsigned long long l2_policy(int first) {
  unsigned long long p;
  if (first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16h(void* smem, const void* gmem, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
// this thread's cp.async groups except the N most recent have landed
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

inline int64_t vol_count(const int dims[3]) {
  return int64_t(dims[0]) * dims[1] * dims[2];
}
inline size_t dtype_size(int dtype) { return dtype == SFW3D_F64 ? 8 : 4; }

}  // namespace sfw3d
