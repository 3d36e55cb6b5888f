// K4 — circular PSF convolution / adjoint correlation, spatial domain.
//
// Replaces convolve / correlate_adjoint (forward.py:79-94), which the
// reference evaluates as rfftn -> product with kernel_hat -> irfftn. Every
// BASELINE PSF is a box-truncated sampled Gaussian, i.e. exactly separable,
// so the operator is three 1-D circular passes (one per axis) with
// (hi - lo + 1) taps each instead of a 3-D FFT pair; a non-separable kernel
// falls back to a direct 3-D stencil over its non-zero box. Offsets are
// relative to the kernel origin n//2 (forward.py:43-47, ifftshift at :58).
#include "internal.cuh"

namespace sfw3d {
namespace {

// out[a0 + j] = sum_q taps[q] * in[a0 + j + lo + q]   (circular along `axis`)
// Thread layout: (outer, a-block, inner) with inner the contiguous block of
// the axes after `axis`, so a warp reads consecutive addresses for axes 0/1.
template <typename T, int J>
__global__ void __launch_bounds__(256) pass1d_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                     int n_axis, long long stride, long long n_outer,
                                                     const T* __restrict__ taps, int lo, int ntaps) {
  const int nblk = (n_axis + J - 1) / J;
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long total = n_outer * nblk * stride;
  if (t >= total) return;
  long long inner = t % stride;
  long long rest = t / stride;
  int blk = int(rest % nblk);
  long long outer = rest / nblk;
  const long long base = outer * (long long)n_axis * stride + inner;
  const int a0 = blk * J;

  T acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) acc[j] = T(0);

  int idx = (a0 + lo) % n_axis;
  if (idx < 0) idx += n_axis;
  const int nwin = J - 1 + ntaps;
  for (int u = 0; u < nwin; ++u) {
    const T v = in[base + idx * stride];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int q = u - j;
      if (q >= 0 && q < ntaps) acc[j] = fma(taps[q], v, acc[j]);
    }
    if (++idx == n_axis) idx = 0;
  }
#pragma unroll
  for (int j = 0; j < J; ++j)
    if (a0 + j < n_axis) out[base + (long long)(a0 + j) * stride] = acc[j];
}

// General (non-separable) kernel: out[x] = sum_o K(o) in[x + sgn*o] over the
// non-zero offset box [lo, hi]^3; sgn = -1 convolution, +1 correlation.
template <typename T>
__global__ void __launch_bounds__(256) stencil3d_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                        int nx, int ny, int nz,
                                                        const T* __restrict__ box, int lo0, int lo1,
                                                        int lo2, int l0, int l1, int l2, int sgn) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long n = (long long)nx * ny * nz;
  if (t >= n) return;
  int k = int(t % nz);
  int j = int((t / nz) % ny);
  int i = int(t / ((long long)ny * nz));
  T acc = T(0);
  for (int a = 0; a < l0; ++a) {
    int xi = (i + sgn * (lo0 + a)) % nx;
    if (xi < 0) xi += nx;
    for (int b = 0; b < l1; ++b) {
      int yj = (j + sgn * (lo1 + b)) % ny;
      if (yj < 0) yj += ny;
      const T* row = in + ((long long)xi * ny + yj) * nz;
      const T* krow = box + ((long long)a * l1 + b) * l2;
      for (int c = 0; c < l2; ++c) {
        int zk = (k + sgn * (lo2 + c)) % nz;
        if (zk < 0) zk += nz;
        acc = fma(krow[c], row[zk], acc);
      }
    }
  }
  out[t] = acc;
}

template <typename T>
int launch_pass(sfw3d_ctx* ctx, const T* in, T* out, const int dims[3], int axis, const T* taps,
                int lo, int ntaps) {
  long long stride = 1;
  for (int a = axis + 1; a < 3; ++a) stride *= dims[a];
  long long outer = 1;
  for (int a = 0; a < axis; ++a) outer *= dims[a];
  const int n = dims[axis];
  SFW3D_PROF(ctx, "psf_pass");
  if (axis == 2) {
    constexpr int J = 1;
    long long total = outer * ((n + J - 1) / J) * stride;
    pass1d_kernel<T, J><<<unsigned((total + 255) / 256), 256, 0, ctx->stream>>>(
        in, out, n, stride, outer, taps, lo, ntaps);
  } else {
    constexpr int J = 8;
    long long total = outer * ((n + J - 1) / J) * stride;
    pass1d_kernel<T, J><<<unsigned((total + 255) / 256), 256, 0, ctx->stream>>>(
        in, out, n, stride, outer, taps, lo, ntaps);
  }
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

template <typename T>
int apply_typed(sfw3d_ctx* ctx, const sfw3d_psf* psf, const T* in, T* out, int adjoint, T* tmp,
                const T* const taps[3], const T* box) {
  const int* dims = psf->dims;
  if (psf->separable) {
    // adjoint: correlation with taps over [lo, hi]; forward: convolution =
    // correlation with reversed taps over [-hi, -lo] (reversed copies are
    // stored right after the forward taps, see psf_create).
    int lo[3], nt[3];
    const T* tp[3];
    for (int a = 0; a < 3; ++a) {
      nt[a] = psf->hi[a] - psf->lo[a] + 1;
      lo[a] = adjoint ? psf->lo[a] : -psf->hi[a];
      tp[a] = adjoint ? taps[a] : taps[a] + nt[a];
    }
    SFW3D_TRY(launch_pass<T>(ctx, in, out, dims, 2, tp[2], lo[2], nt[2]));
    SFW3D_TRY(launch_pass<T>(ctx, out, tmp, dims, 1, tp[1], lo[1], nt[1]));
    SFW3D_TRY(launch_pass<T>(ctx, tmp, out, dims, 0, tp[0], lo[0], nt[0]));
    return SFW3D_OK;
  }
  long long n = vol_count(dims);
  const int l0 = psf->hi[0] - psf->lo[0] + 1, l1 = psf->hi[1] - psf->lo[1] + 1,
            l2 = psf->hi[2] - psf->lo[2] + 1;
  SFW3D_PROF(ctx, "psf_pass");
  stencil3d_kernel<T><<<unsigned((n + 255) / 256), 256, 0, ctx->stream>>>(
      in, out, dims[0], dims[1], dims[2], box, psf->lo[0], psf->lo[1], psf->lo[2], l0, l1, l2,
      adjoint ? 1 : -1);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

}  // namespace

int psf_apply_impl(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                   int adjoint, void* tmp) {
  if (dtype == SFW3D_F64) {
    const double* taps[3] = {psf->taps64[0], psf->taps64[1], psf->taps64[2]};
    return apply_typed<double>(ctx, psf, static_cast<const double*>(in), static_cast<double*>(out),
                               adjoint, static_cast<double*>(tmp), taps, psf->box64);
  }
  const float* taps[3] = {psf->taps32[0], psf->taps32[1], psf->taps32[2]};
  return apply_typed<float>(ctx, psf, static_cast<const float*>(in), static_cast<float*>(out),
                            adjoint, static_cast<float*>(tmp), taps, psf->box32);
}

}  // namespace sfw3d
