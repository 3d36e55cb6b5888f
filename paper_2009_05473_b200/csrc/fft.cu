// K4 for a NON-separable PSF at size: circular convolution through cuFFT,
// i.e. the reference's own algorithm (forward.py:79-94: irfftn(rfftn(v) *
// H_hat), with conj(H_hat) for the adjoint). The kernel spectrum is built once
// per PSF and storage precision on the device (the box scattered to its
// ifftshifted positions, forward.py:58, then R2C) and cached with the plans.
// Small non-separable boxes keep the direct stencil (psf.cu).
#include <cufft.h>

#include "internal.cuh"

namespace sfw3d {

struct PsfFft {
  cufftHandle fwd[2] = {0, 0}, inv[2] = {0, 0};  // [f32, f64]
  bool planned[2] = {false, false};
  void* hat[2] = {nullptr, nullptr};   // kernel spectrum (complex), storage precision
  void* spec[2] = {nullptr, nullptr};  // work spectrum
};

namespace {

#define SFW3D_CUFFT_TRY(x)                                          \
  do {                                                              \
    cufftResult r_ = (x);                                           \
    if (r_ != CUFFT_SUCCESS) {                                      \
      set_error("cuFFT error " + std::to_string(int(r_)) + " at " #x); \
      return SFW3D_ECUDA;                                           \
    }                                                               \
  } while (0)

// dense ifftshifted kernel from the non-zero box: K[(o + n) mod n] = box[o - lo]
template <typename T>
__global__ void scatter_box_kernel(const T* __restrict__ box, int l0, int l1, int l2, int lo0,
                                   int lo1, int lo2, int nx, int ny, int nz, T* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)l0 * l1 * l2) return;
  const int c = int(i % l2), b = int((i / l2) % l1), a = int(i / ((long long)l1 * l2));
  const int x = ((lo0 + a) % nx + nx) % nx, y = ((lo1 + b) % ny + ny) % ny,
            z = ((lo2 + c) % nz + nz) % nz;
  out[((long long)x * ny + y) * nz + z] = box[i];
}

template <typename C>
__global__ void spectrum_product_kernel(C* __restrict__ s, const C* __restrict__ h, long long n,
                                        double scale, int conj_h) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const C a = s[i], b = h[i];
    const double br = b.x, bi = conj_h ? -double(b.y) : double(b.y);
    C r;
    r.x = decltype(a.x)((double(a.x) * br - double(a.y) * bi) * scale);
    r.y = decltype(a.x)((double(a.x) * bi + double(a.y) * br) * scale);
    s[i] = r;
  }
}

int ensure_fft(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype) {
  PsfFft*& f = psf->fft;
  if (!f) f = new PsfFft();
  const int k = dtype == SFW3D_F64 ? 1 : 0;
  if (f->planned[k]) return SFW3D_OK;
  const int* d = psf->dims;
  const long long nspec = (long long)d[0] * d[1] * (d[2] / 2 + 1);
  const size_t cbytes = size_t(nspec) * (k ? sizeof(cufftDoubleComplex) : sizeof(cufftComplex));
  const size_t rbytes = size_t(vol_count(d)) * (k ? 8 : 4);
  SFW3D_CUFFT_TRY(cufftPlan3d(&f->fwd[k], d[0], d[1], d[2], k ? CUFFT_D2Z : CUFFT_R2C));
  SFW3D_CUFFT_TRY(cufftPlan3d(&f->inv[k], d[0], d[1], d[2], k ? CUFFT_Z2D : CUFFT_C2R));
  SFW3D_CUDA_TRY(cudaMalloc(&f->hat[k], cbytes));
  SFW3D_CUDA_TRY(cudaMalloc(&f->spec[k], cbytes));
  // kernel spectrum: dense ifftshifted kernel (in the work spectrum's room
  // when it fits, else a temporary) -> R2C
  void* dense = nullptr;
  SFW3D_CUDA_TRY(cudaMalloc(&dense, rbytes));
  SFW3D_CUDA_TRY(cudaMemsetAsync(dense, 0, rbytes, ctx->stream));
  const int l0 = psf->hi[0] - psf->lo[0] + 1, l1 = psf->hi[1] - psf->lo[1] + 1,
            l2 = psf->hi[2] - psf->lo[2] + 1;
  const long long nb = (long long)l0 * l1 * l2;
  if (k)
    scatter_box_kernel<double><<<unsigned((nb + 255) / 256), 256, 0, ctx->stream>>>(
        psf->box64, l0, l1, l2, psf->lo[0], psf->lo[1], psf->lo[2], d[0], d[1], d[2],
        static_cast<double*>(dense));
  else
    scatter_box_kernel<float><<<unsigned((nb + 255) / 256), 256, 0, ctx->stream>>>(
        psf->box32, l0, l1, l2, psf->lo[0], psf->lo[1], psf->lo[2], d[0], d[1], d[2],
        static_cast<float*>(dense));
  SFW3D_LAUNCH_CHECK(ctx);
  SFW3D_CUFFT_TRY(cufftSetStream(f->fwd[k], ctx->stream));
  if (k)
    SFW3D_CUFFT_TRY(cufftExecD2Z(f->fwd[k], static_cast<cufftDoubleReal*>(dense),
                                 static_cast<cufftDoubleComplex*>(f->hat[k])));
  else
    SFW3D_CUFFT_TRY(cufftExecR2C(f->fwd[k], static_cast<cufftReal*>(dense),
                                 static_cast<cufftComplex*>(f->hat[k])));
  SFW3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  cudaFree(dense);
  f->planned[k] = true;
  return SFW3D_OK;
}

}  // namespace

// box taps above which a non-separable PSF goes through cuFFT
bool psf_use_fft(const sfw3d_psf* psf) {
  const long long taps = (long long)(psf->hi[0] - psf->lo[0] + 1) * (psf->hi[1] - psf->lo[1] + 1) *
                         (psf->hi[2] - psf->lo[2] + 1);
  return !psf->separable && taps > 125;
}

int psf_fft_apply(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                  int adjoint) {
  SFW3D_TRY(ensure_fft(ctx, psf, dtype));
  PsfFft* f = psf->fft;
  const int k = dtype == SFW3D_F64 ? 1 : 0;
  const int* d = psf->dims;
  const long long nspec = (long long)d[0] * d[1] * (d[2] / 2 + 1);
  const double scale = 1.0 / double(vol_count(d));
  SFW3D_PROF(ctx, "psf_fft");
  SFW3D_CUFFT_TRY(cufftSetStream(f->fwd[k], ctx->stream));
  SFW3D_CUFFT_TRY(cufftSetStream(f->inv[k], ctx->stream));
  const unsigned grid = unsigned(std::min<long long>(8LL * ctx->num_sms, (nspec + 255) / 256));
  if (k) {
    SFW3D_CUFFT_TRY(cufftExecD2Z(f->fwd[k], static_cast<cufftDoubleReal*>(const_cast<void*>(in)),
                                 static_cast<cufftDoubleComplex*>(f->spec[k])));
    spectrum_product_kernel<cufftDoubleComplex><<<grid, 256, 0, ctx->stream>>>(
        static_cast<cufftDoubleComplex*>(f->spec[k]),
        static_cast<const cufftDoubleComplex*>(f->hat[k]), nspec, scale, adjoint);
    SFW3D_LAUNCH_CHECK(ctx);
    SFW3D_CUFFT_TRY(cufftExecZ2D(f->inv[k], static_cast<cufftDoubleComplex*>(f->spec[k]),
                                 static_cast<cufftDoubleReal*>(out)));
  } else {
    SFW3D_CUFFT_TRY(cufftExecR2C(f->fwd[k], static_cast<cufftReal*>(const_cast<void*>(in)),
                                 static_cast<cufftComplex*>(f->spec[k])));
    spectrum_product_kernel<cufftComplex><<<grid, 256, 0, ctx->stream>>>(
        static_cast<cufftComplex*>(f->spec[k]), static_cast<const cufftComplex*>(f->hat[k]),
        nspec, scale, adjoint);
    SFW3D_LAUNCH_CHECK(ctx);
    SFW3D_CUFFT_TRY(cufftExecC2R(f->inv[k], static_cast<cufftComplex*>(f->spec[k]),
                                 static_cast<cufftReal*>(out)));
  }
  return SFW3D_OK;
}

void psf_fft_destroy(sfw3d_psf* psf) {
  PsfFft* f = psf->fft;
  if (!f) return;
  for (int k = 0; k < 2; ++k) {
    if (f->planned[k]) {
      cufftDestroy(f->fwd[k]);
      cufftDestroy(f->inv[k]);
    }
    if (f->hat[k]) cudaFree(f->hat[k]);
    if (f->spec[k]) cudaFree(f->spec[k]);
  }
  delete f;
  psf->fft = nullptr;
}

}  // namespace sfw3d
