// C-ABI entry points, context / workspace management, atom geometry and the
// PSF object. See include/sfw3d_cuda.h for the contract of every function.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "internal.cuh"

namespace sfw3d {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// 2 * ln(1 / 1e-12) exactly as numpy computes it (forward.py:34)
const double kTailExponent = 0x1.ba18a998fffa0p+5;

int activate(sfw3d_ctx* ctx) {
  SFW3D_CUDA_TRY(cudaSetDevice(ctx->device));
  return SFW3D_OK;
}

int ensure_device(sfw3d_ctx* ctx, Arena& a, size_t bytes) {
  if (a.bytes >= bytes) return SFW3D_OK;
  if (a.ptr) {
    SFW3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    SFW3D_CUDA_TRY(cudaFree(a.ptr));
    a.ptr = nullptr;
    a.bytes = 0;
  }
  size_t want = bytes + bytes / 8 + 4096;
  SFW3D_CUDA_TRY(cudaMalloc(&a.ptr, want));
  a.bytes = want;
  return SFW3D_OK;
}

static int ensure_pinned_arena(sfw3d_ctx* ctx, Arena& a, size_t bytes) {
  if (a.bytes >= bytes) return SFW3D_OK;
  if (a.ptr) {
    SFW3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    SFW3D_CUDA_TRY(cudaFreeHost(a.ptr));
    a.ptr = nullptr;
    a.bytes = 0;
  }
  size_t want = bytes * 2 + 65536;
  SFW3D_CUDA_TRY(cudaMallocHost(&a.ptr, want));
  a.bytes = want;
  return SFW3D_OK;
}

int ensure_pinned_io(sfw3d_ctx* ctx, size_t bytes) { return ensure_pinned_arena(ctx, ctx->pinned_io, bytes); }

int begin_call(sfw3d_ctx* ctx) {
  SFW3D_TRY(activate(ctx));
  if (ctx->pin_off) {
    // an earlier asynchronous call may still be reading the staging area
    SFW3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->pin_off = 0;
  }
  return SFW3D_OK;
}

int stage_upload(sfw3d_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes) {
  if (bytes == 0) return SFW3D_OK;
  size_t need = ((ctx->pin_off + 255) & ~size_t(255)) + bytes;
  if (need > ctx->pinned.bytes) {
    SFW3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->pin_off = 0;
    SFW3D_TRY(ensure_pinned_arena(ctx, ctx->pinned, bytes + 256));
  }
  size_t off = (ctx->pin_off + 255) & ~size_t(255);
  char* p = static_cast<char*>(ctx->pinned.ptr) + off;
  memcpy(p, src_host, bytes);
  SFW3D_CUDA_TRY(cudaMemcpyAsync(dst_dev, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->pin_off = off + bytes;
  return SFW3D_OK;
}

int download_sync(sfw3d_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes) {
  SFW3D_TRY(ensure_pinned_arena(ctx, ctx->pinned_out, bytes));
  SFW3D_CUDA_TRY(cudaMemcpyAsync(ctx->pinned_out.ptr, src_dev, bytes, cudaMemcpyDeviceToHost,
                                 ctx->stream));
  SFW3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ctx->pin_off = 0;
  memcpy(dst_host, ctx->pinned_out.ptr, bytes);
  return SFW3D_OK;
}

// ------------------------------------------------------------ atom geometry
static int axis_geometry(int n, double centre, int radius, int& start, int& len, int& full) {
  if (2LL * radius + 1 >= n) {  // forward.py:107-109
    start = 0;
    len = n;
    full = 1;
  } else {  // forward.py:111-113: round-half-even centre, unwrapped span
    const double c = std::nearbyint(centre);
    start = int(c) - radius;
    len = 2 * radius + 1;
    full = 0;
  }
  return SFW3D_OK;
}

// One atom's geometry (forward.py:97-116, 130-137); returns a status and
// sets the thread's error message on failure.
static int build_one(const int dims[3], const double* r, int i, AtomGeo& a) {
  for (int c = 0; c < 6; ++c)
    if (!std::isfinite(r[c])) {
      set_error("invalid argument: non-finite atom parameters (row " + std::to_string(i) + ")");
      return SFW3D_EINVAL;
    }
  a.w = r[0];
  a.m[0] = r[1];
  a.m[1] = r[2];
  a.m[2] = r[3];
  a.sigma = r[4];
  a.d = r[5];
  if (!(a.sigma > 0.0 && a.d > 0.0)) {
    set_error("invalid argument: sigma and d must be positive (row " + std::to_string(i) + ")");
    return SFW3D_EINVAL;
  }
  // forward.py:97-99 support_radius
  const double rr = std::ceil(a.sigma * std::pow(kTailExponent, 1.0 / a.d));
  if (!(rr < 1e9)) {
    set_error("invalid argument: support radius overflow");
    return SFW3D_EINVAL;
  }
  a.radius = int(rr);
  a.inv2sd = 0.5 / std::pow(a.sigma, a.d);
  a.half_d = 0.5 * a.d;
  a.log_sigma = std::log(a.sigma);
  a.d_over_sigma = a.d / a.sigma;
  a.d2 = (a.d == 2.0) ? 1 : 0;
  a.nvox = 1;
  for (int ax = 0; ax < 3; ++ax) {
    axis_geometry(dims[ax], a.m[ax], a.radius, a.start[ax], a.len[ax], a.full[ax]);
    a.nvox *= a.len[ax];
  }
  return SFW3D_OK;
}

// The host geometry of k atoms (libm pow / ceil / nearbyint exactly as the
// reference). Large k is split over OpenMP threads (the per-atom work is
// independent; a failure is re-run on the calling thread for its message).
int build_atoms(const int dims[3], const double* params, int k, std::vector<AtomGeo>& out) {
  out.resize(k);
  int bad = k;
  const int nth = k >= 512 ? std::min(8, k / 128) : 1;
#pragma omp parallel for num_threads(nth) schedule(static) reduction(min : bad) if (nth > 1)
  for (int i = 0; i < k; ++i)
    if (build_one(dims, params + 6 * i, i, out[i]) != SFW3D_OK) bad = std::min(bad, i);
  if (bad < k) return build_one(dims, params + 6 * bad, bad, out[bad]);
  return SFW3D_OK;
}

static bool dims_ok(const int dims[3]) {
  return dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0;
}

}  // namespace sfw3d

using namespace sfw3d;

// =========================================================== ABI: library
extern "C" int sfw3d_abi_version(void) { return SFW3D_ABI_VERSION; }

extern "C" const char* sfw3d_last_error(void) { return g_last_error.c_str(); }

extern "C" int sfw3d_ctx_create(int device, void* stream, sfw3d_ctx** out) {
  SFW3D_CHECK_ARG(out != nullptr, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  SFW3D_CUDA_TRY(cudaGetDeviceCount(&ndev));
  SFW3D_CHECK_ARG(device >= 0 && device < ndev, "device index out of range");
  auto* ctx = new sfw3d_ctx();
  ctx->device = device;
  ctx->stream = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    set_error(std::string("CUDA error ") + cudaGetErrorString(e));
    delete ctx;
    return SFW3D_ECUDA;
  }
  *out = ctx;
  return SFW3D_OK;
}

extern "C" int sfw3d_ctx_destroy(sfw3d_ctx* ctx) {
  if (!ctx) return SFW3D_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->ws.ptr) cudaFree(ctx->ws.ptr);
  if (ctx->ws_small.ptr) cudaFree(ctx->ws_small.ptr);
  if (ctx->ws_aux.ptr) cudaFree(ctx->ws_aux.ptr);
  if (ctx->ws_plan.ptr) cudaFree(ctx->ws_plan.ptr);
  if (ctx->pinned.ptr) cudaFreeHost(ctx->pinned.ptr);
  if (ctx->pinned_out.ptr) cudaFreeHost(ctx->pinned_out.ptr);
  if (ctx->pinned_io.ptr) cudaFreeHost(ctx->pinned_io.ptr);
  if (ctx->ws_one.ptr) cudaFree(ctx->ws_one.ptr);
  if (ctx->one_host) cudaFreeHost(ctx->one_host);
  delete ctx;
  return SFW3D_OK;
}

extern "C" int sfw3d_ctx_sync(sfw3d_ctx* ctx) {
  SFW3D_CHECK_ARG(ctx, "ctx is NULL");
  SFW3D_TRY(activate(ctx));
  SFW3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ctx->pin_off = 0;
  return SFW3D_OK;
}

extern "C" int64_t sfw3d_ctx_launches(const sfw3d_ctx* ctx) { return ctx ? ctx->launches : 0; }

extern "C" int sfw3d_atom_geometry(const int dims[3], const double* params_host, int k,
                                   int32_t* radius, int32_t* start, int32_t* len, int32_t* full) {
  SFW3D_CHECK_ARG(dims_ok(dims), "dims must be positive");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || params_host), "params");
  std::vector<AtomGeo> atoms;
  SFW3D_TRY(build_atoms(dims, params_host, k, atoms));
  for (int i = 0; i < k; ++i) {
    if (radius) radius[i] = atoms[i].radius;
    for (int a = 0; a < 3; ++a) {
      if (start) start[3 * i + a] = atoms[i].start[a];
      if (len) len[3 * i + a] = atoms[i].len[a];
      if (full) full[3 * i + a] = atoms[i].full[a];
    }
  }
  return SFW3D_OK;
}

// =============================================================== ABI: PSF
extern "C" int sfw3d_psf_create(sfw3d_ctx* ctx, const int dims[3], const double* kernel_host,
                                sfw3d_psf** out) {
  SFW3D_CHECK_ARG(ctx && out && kernel_host, "NULL argument");
  SFW3D_CHECK_ARG(dims_ok(dims), "dims must be positive");
  SFW3D_TRY(begin_call(ctx));
  *out = nullptr;
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  auto at = [&](int i, int j, int l) { return kernel_host[((long long)i * ny + j) * nz + l]; };
  // non-zero bounding box in index space
  int lo_i[3] = {dims[0], dims[1], dims[2]}, hi_i[3] = {-1, -1, -1};
  double peak = 0.0;
  int piv[3] = {0, 0, 0};
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j)
      for (int l = 0; l < nz; ++l) {
        const double v = at(i, j, l);
        if (!std::isfinite(v)) {
          set_error("invalid argument: kernel contains non-finite values");
          return SFW3D_EINVAL;
        }
        if (v != 0.0) {
          const int q[3] = {i, j, l};
          for (int a = 0; a < 3; ++a) {
            lo_i[a] = std::min(lo_i[a], q[a]);
            hi_i[a] = std::max(hi_i[a], q[a]);
          }
          if (std::fabs(v) > peak) {
            peak = std::fabs(v);
            piv[0] = i;
            piv[1] = j;
            piv[2] = l;
          }
        }
      }
  auto* psf = new sfw3d_psf();
  for (int a = 0; a < 3; ++a) psf->dims[a] = dims[a];
  psf->device = ctx->device;
  if (hi_i[0] < 0) {  // all-zero kernel: a single zero tap
    for (int a = 0; a < 3; ++a) lo_i[a] = hi_i[a] = dims[a] / 2;
  }
  for (int a = 0; a < 3; ++a) {
    psf->lo[a] = lo_i[a] - dims[a] / 2;
    psf->hi[a] = hi_i[a] - dims[a] / 2;
  }
  const int l[3] = {hi_i[0] - lo_i[0] + 1, hi_i[1] - lo_i[1] + 1, hi_i[2] - lo_i[2] + 1};
  // rank-1 test through the pivot (exact for sampled separable kernels)
  std::vector<double> f[3];
  bool sep = peak > 0.0;
  if (sep) {
    const double p = at(piv[0], piv[1], piv[2]);
    f[0].resize(l[0]);
    f[1].resize(l[1]);
    f[2].resize(l[2]);
    for (int i = 0; i < l[0]; ++i) f[0][i] = at(lo_i[0] + i, piv[1], piv[2]);
    for (int j = 0; j < l[1]; ++j) f[1][j] = at(piv[0], lo_i[1] + j, piv[2]) / p;
    for (int q = 0; q < l[2]; ++q) f[2][q] = at(piv[0], piv[1], lo_i[2] + q) / p;
    const double tol = 1e-14 * peak;
    for (int i = 0; i < l[0] && sep; ++i)
      for (int j = 0; j < l[1] && sep; ++j)
        for (int q = 0; q < l[2]; ++q) {
          const double rec = f[0][i] * f[1][j] * f[2][q];
          if (std::fabs(rec - at(lo_i[0] + i, lo_i[1] + j, lo_i[2] + q)) > tol) {
            sep = false;
            break;
          }
        }
  }
  psf->separable = sep ? 1 : 0;
  auto fail = [&](cudaError_t e) {
    set_error(std::string("CUDA error ") + cudaGetErrorString(e));
    sfw3d_psf_destroy(psf);
    return e == cudaErrorMemoryAllocation ? SFW3D_ENOMEM : SFW3D_ECUDA;
  };
  if (sep) {
    for (int a = 0; a < 3; ++a) {
      std::vector<double> t64(2 * l[a]);
      std::vector<float> t32(2 * l[a]);
      for (int q = 0; q < l[a]; ++q) {
        t64[q] = f[a][q];
        t64[l[a] + q] = f[a][l[a] - 1 - q];  // reversed: convolution direction
      }
      for (int q = 0; q < 2 * l[a]; ++q) t32[q] = float(t64[q]);
      cudaError_t e = cudaMalloc(&psf->taps64[a], t64.size() * sizeof(double));
      if (e == cudaSuccess) e = cudaMalloc(&psf->taps32[a], t32.size() * sizeof(float));
      if (e == cudaSuccess)
        e = cudaMemcpy(psf->taps64[a], t64.data(), t64.size() * sizeof(double), cudaMemcpyHostToDevice);
      if (e == cudaSuccess)
        e = cudaMemcpy(psf->taps32[a], t32.data(), t32.size() * sizeof(float), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(e);
    }
  } else {
    const size_t nb = size_t(l[0]) * l[1] * l[2];
    std::vector<double> b64(nb);
    std::vector<float> b32(nb);
    for (int i = 0; i < l[0]; ++i)
      for (int j = 0; j < l[1]; ++j)
        for (int q = 0; q < l[2]; ++q) {
          const size_t o = (size_t(i) * l[1] + j) * l[2] + q;
          b64[o] = at(lo_i[0] + i, lo_i[1] + j, lo_i[2] + q);
          b32[o] = float(b64[o]);
        }
    cudaError_t e = cudaMalloc(&psf->box64, nb * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&psf->box32, nb * sizeof(float));
    if (e == cudaSuccess) e = cudaMemcpy(psf->box64, b64.data(), nb * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(psf->box32, b32.data(), nb * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(e);
  }
  *out = psf;
  return SFW3D_OK;
}

extern "C" int sfw3d_psf_info(const sfw3d_psf* psf, int* separable, int32_t lo[3], int32_t hi[3]) {
  SFW3D_CHECK_ARG(psf, "psf is NULL");
  if (separable) *separable = psf->separable;
  for (int a = 0; a < 3; ++a) {
    if (lo) lo[a] = psf->lo[a];
    if (hi) hi[a] = psf->hi[a];
  }
  return SFW3D_OK;
}

extern "C" int sfw3d_psf_destroy(sfw3d_psf* psf) {
  if (!psf) return SFW3D_OK;
  cudaSetDevice(psf->device);
  for (int a = 0; a < 3; ++a) {
    if (psf->taps64[a]) cudaFree(psf->taps64[a]);
    if (psf->taps32[a]) cudaFree(psf->taps32[a]);
  }
  if (psf->box64) cudaFree(psf->box64);
  if (psf->box32) cudaFree(psf->box32);
  psf_fft_destroy(psf);
  delete psf;
  return SFW3D_OK;
}

extern "C" int sfw3d_psf_apply(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in_dev,
                               void* out_dev, int adjoint) {
  SFW3D_CHECK_ARG(ctx && psf && in_dev && out_dev, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(in_dev != out_dev, "in and out must differ");
  SFW3D_TRY(begin_call(ctx));
  const size_t vb = size_t(vol_count(psf->dims)) * dtype_size(dtype);
  SFW3D_TRY(ensure_device(ctx, ctx->ws, vb));
  return psf_apply_impl(ctx, psf, dtype, in_dev, out_dev, adjoint, ctx->ws.ptr);
}

// ============================================================= ABI: atoms
static int upload_atoms(sfw3d_ctx* ctx, const std::vector<AtomGeo>& atoms, AtomGeo* dst) {
  return stage_upload(ctx, dst, atoms.data(), atoms.size() * sizeof(AtomGeo));
}

extern "C" int sfw3d_render(sfw3d_ctx* ctx, int dtype, const int dims[3], const double* params_host,
                            int k, void* out_dev) {
  SFW3D_CHECK_ARG(ctx && out_dev, "NULL argument");
  SFW3D_CHECK_ARG(dims_ok(dims), "dims must be positive");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || params_host), "params");
  SFW3D_TRY(begin_call(ctx));
  std::vector<AtomGeo> atoms;
  SFW3D_TRY(build_atoms(dims, params_host, k, atoms));
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small, (size_t(k) + 1) * sizeof(AtomGeo) + 4096));
  AtomGeo* ad = static_cast<AtomGeo*>(ctx->ws_small.ptr);
  SFW3D_TRY(upload_atoms(ctx, atoms, ad));
  return render_impl(ctx, dtype, dims, atoms, ad, k, out_dev);
}

static int finite_all(const double* x, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return 0;
  return 1;
}

extern "C" int sfw3d_atom_sums(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* field_dev,
                               const double* params_host, int k, double* sums_host) {
  SFW3D_CHECK_ARG(ctx && field_dev && sums_host, "NULL argument");
  SFW3D_CHECK_ARG(dims_ok(dims), "dims must be positive");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || params_host), "params");
  SFW3D_TRY(begin_call(ctx));
  if (k == 0) return SFW3D_OK;
  std::vector<AtomGeo> atoms;
  SFW3D_TRY(build_atoms(dims, params_host, k, atoms));
  const size_t need = Carver::need({size_t(k) * sizeof(AtomGeo), size_t(k) * 6 * sizeof(double)});
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small, need));
  Carver cv(ctx->ws_small.ptr);
  AtomGeo* ad = cv.take<AtomGeo>(k);
  double* sums = cv.take<double>(size_t(k) * 6);
  SFW3D_TRY(upload_atoms(ctx, atoms, ad));
  SFW3D_TRY(atom_sums_impl(ctx, dtype, dims, field_dev, atoms, ad, sums));
  SFW3D_TRY(download_sync(ctx, sums_host, sums, size_t(k) * 6 * sizeof(double)));
  if (!finite_all(sums_host, size_t(k) * 6)) {
    set_error("non-finite atom inner product; atom parameters left the smooth regime");
    return SFW3D_ENONFINITE;
  }
  return SFW3D_OK;
}

extern "C" int sfw3d_cost_grad(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                               const double* params_host, int k, double lam, double* cost_host,
                               double* grad_host, void* back_dev) {
  SFW3D_CHECK_ARG(ctx && psf && y_dev && cost_host, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || params_host), "params");
  SFW3D_CHECK_ARG(lam > 0.0, "lam must be > 0");
  SFW3D_TRY(begin_call(ctx));
  const int* dims = psf->dims;
  std::vector<AtomGeo> atoms;
  SFW3D_TRY(build_atoms(dims, params_host, k, atoms));
  const int64_t n = vol_count(dims);
  const size_t vb = size_t(n) * dtype_size(dtype);
  SFW3D_TRY(ensure_device(ctx, ctx->ws, Carver::need({vb, vb})));
  Carver cw(ctx->ws.ptr);
  void* A = cw.take<char>(vb);
  void* B = cw.take<char>(vb);
  // partials of ||r||^2: the grid-stride reduction, or one per CTA of the
  // fused residual x pass (<= ceil(nx / 64) * ny nz / 64)
  const int nred = int(std::max<long long>(4LL * ctx->num_sms,
                                           (long long)((dims[0] + 63) / 64) * ((long long)dims[1] * dims[2] / 64)));
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small,
                          Carver::need({(size_t(k) + 1) * sizeof(AtomGeo), (size_t(k) * 6 + 1) * sizeof(double),
                                        size_t(nred) * sizeof(double)})));
  Carver cs(ctx->ws_small.ptr);
  AtomGeo* ad = cs.take<AtomGeo>(k + 1);
  double* res = cs.take<double>(size_t(k) * 6 + 1);  // [sumsq, sums...]
  double* partials = cs.take<double>(nred);
  SFW3D_TRY(upload_atoms(ctx, atoms, ad));
  // model = H * sum w G, resid = model - y -> A with ||resid||^2 fused into
  // the PSF's last pass (B scratch); else the separate residual pass
  SFW3D_TRY(render_impl(ctx, dtype, dims, atoms, ad, k, B));
  int nparts = 0;
  SFW3D_TRY(psf_apply_resid(ctx, psf, dtype, B, A, B, y_dev, partials, nred, &nparts));
  if (nparts > 0) {
    SFW3D_TRY(sum_parts_impl(ctx, partials, nparts, res));
  } else {
    SFW3D_TRY(render_impl(ctx, dtype, dims, atoms, ad, k, A));
    SFW3D_TRY(psf_apply_impl(ctx, psf, dtype, A, B, 0, A));
    SFW3D_TRY(sumsq_diff_impl(ctx, dtype, n, B, y_dev, A, partials, res));
  }
  if (grad_host || back_dev) {
    void* back = back_dev ? back_dev : B;
    SFW3D_TRY(psf_apply_impl(ctx, psf, dtype, A, back, 1, back == B ? A : B));
    if (grad_host) SFW3D_TRY(atom_sums_impl(ctx, dtype, dims, back, atoms, ad, res + 1));
  }
  std::vector<double> host(size_t(k) * 6 + 1);
  SFW3D_TRY(download_sync(ctx, host.data(), res, (grad_host ? host.size() : 1) * sizeof(double)));
  double mass = 0.0;
  for (int i = 0; i < k; ++i) mass += atoms[i].w;  // total_mass: sum in order
  *cost_host = 0.5 * host[0] + lam * mass;
  if (grad_host) {
    for (int i = 0; i < k; ++i) {
      const double* s = &host[1 + 6 * i];
      double* g = grad_host + 6 * i;
      g[0] = s[0] + lam;                                   // forward.py:218
      for (int c = 1; c < 6; ++c) g[c] = atoms[i].w * s[c];  // forward.py:219-220
    }
    if (!finite_all(grad_host, size_t(k) * 6)) {
      set_error("non-finite criterion gradient; atom parameters left the smooth regime");
      return SFW3D_ENONFINITE;
    }
  }
  return SFW3D_OK;
}


// ------------------------------------------------ slab-local cost + gradient
// One rank's share of criterion_and_gradient (forward.py:232-257) on its
// x-slab [x0, x1] of a periodic (gnx, ny, nz) volume. The rank holds the
// window of planes x0 - halo .. x1 + halo (halo >= the PSF's x half-extent),
// `psf` is created on those window dims, y_dev is y on the window. Each atom's
// x-span is clipped to the window (one piece per periodic image that meets
// it; the unwrapped offsets p - m are kept), so render and the atom sums run
// on the window only. The residual is formed on the slab planes and zeroed
// elsewhere, so back = H^T (r 1_slab): summed over ranks, the raw sums and
// 1/2 ||r||^2 are exactly the single-volume ones (up to summation order).
namespace sfw3d {
// x-slabs: every atom's unwrapped x-span clipped to the global planes
// [clip0, clip0 + clip_len), one piece per periodic image that meets them,
// in coordinates whose plane 0 is global plane `origin` (start and centre
// shifted by the same integer: the offsets p - m are unchanged)
int clip_atoms_x(const std::vector<AtomGeo>& atoms, int gnx, int clip0, int clip_len, int origin,
                 std::vector<AtomGeo>& pieces, std::vector<int>& owner) {
  pieces.clear();
  owner.clear();
  for (int i = 0; i < int(atoms.size()); ++i) {
    const AtomGeo& a = atoms[i];
    if (a.full[0]) {
      set_error("invalid argument: an atom box spans the x axis; slabs cannot shard it");
      return SFW3D_EINVAL;
    }
    for (int j = -1; j <= 1; ++j) {
      const int s = a.start[0] + j * gnx;
      const int lo = std::max(s, clip0), hi = std::min(s + a.len[0], clip0 + clip_len);
      if (lo >= hi) continue;
      AtomGeo p = a;
      p.m[0] = a.m[0] + double(j * gnx - origin);
      p.start[0] = lo - origin;
      p.len[0] = hi - lo;
      p.nvox = (long long)p.len[0] * p.len[1] * p.len[2];
      pieces.push_back(p);
      owner.push_back(i);
    }
  }
  return SFW3D_OK;
}

// out[0] = 1/2 res[0]; out[1 + 6i + c] = sum of atom i's pieces' res[1 + 6q + c]
// (pieces of one atom are consecutive, in image order)
__global__ void piece_combine_kernel(const int* __restrict__ first, int k,
                                     const double* __restrict__ res, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > 6 * k) return;
  if (i == 0) {
    out[0] = 0.5 * res[0];
    return;
  }
  const int atom = (i - 1) / 6, c = (i - 1) % 6;
  double x = 0.0;
  for (int q = first[atom]; q < first[atom + 1]; ++q) x += res[1 + 6 * q + c];
  out[i] = x;
}
}  // namespace sfw3d

static int cost_grad_slab_impl(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                               const double* params_host, int k, int gnx, int x0, int x1, int halo,
                               double* half_sumsq_host, double* sums_host, double* partials_dev);

extern "C" int sfw3d_cost_grad_slab(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                                    const double* params_host, int k, int gnx, int x0, int x1,
                                    int halo, double* half_sumsq_host, double* sums_host) {
  SFW3D_CHECK_ARG(half_sumsq_host && sums_host, "NULL argument");
  return cost_grad_slab_impl(ctx, psf, dtype, y_dev, params_host, k, gnx, x0, x1, halo,
                             half_sumsq_host, sums_host, nullptr);
}

extern "C" int sfw3d_cost_grad_slab_dev(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype,
                                        const void* y_dev, const double* params_host, int k,
                                        int gnx, int x0, int x1, int halo, double* partials_dev) {
  SFW3D_CHECK_ARG(partials_dev, "NULL argument");
  return cost_grad_slab_impl(ctx, psf, dtype, y_dev, params_host, k, gnx, x0, x1, halo, nullptr,
                             nullptr, partials_dev);
}

static int cost_grad_slab_impl(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                               const double* params_host, int k, int gnx, int x0, int x1, int halo,
                               double* half_sumsq_host, double* sums_host, double* partials_dev) {
  SFW3D_CHECK_ARG(ctx && psf && y_dev, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || params_host), "params");
  const int* dims = psf->dims;
  const int nxl = x1 - x0 + 1 + 2 * halo;
  SFW3D_CHECK_ARG(gnx > 0 && x0 >= 0 && x1 >= x0 && x1 < gnx && halo >= 0, "slab bounds");
  SFW3D_CHECK_ARG(dims[0] == nxl && nxl <= gnx, "psf dims[0] must be x1 - x0 + 1 + 2 halo <= gnx");
  SFW3D_CHECK_ARG(-psf->lo[0] <= halo && psf->hi[0] <= halo,
                  "halo must cover the PSF's x half-extent (else the window convolution wraps)");
  SFW3D_TRY(begin_call(ctx));
  const int gdims[3] = {gnx, dims[1], dims[2]};
  std::vector<AtomGeo> atoms;
  SFW3D_TRY(build_atoms(gdims, params_host, k, atoms));
  // clip every atom's x-span to the window [gx0, gx0 + nxl) (unwrapped)
  const int gx0 = x0 - halo;
  std::vector<AtomGeo> pieces;
  std::vector<int> owner;
  SFW3D_TRY(clip_atoms_x(atoms, gnx, gx0, nxl, gx0, pieces, owner));
  const int kp = int(pieces.size());
  const int64_t n = vol_count(dims);
  const size_t es = dtype_size(dtype), vb = size_t(n) * es;
  SFW3D_TRY(ensure_device(ctx, ctx->ws, Carver::need({vb, vb})));
  Carver cw(ctx->ws.ptr);
  char* A = cw.take<char>(vb);
  char* B = cw.take<char>(vb);
  const int nred = 4 * ctx->num_sms;
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small,
                          Carver::need({(size_t(kp) + 1) * sizeof(AtomGeo), (size_t(kp) * 6 + 1) * sizeof(double),
                                        size_t(nred) * sizeof(double)})));
  Carver cs(ctx->ws_small.ptr);
  AtomGeo* ad = cs.take<AtomGeo>(kp + 1);
  double* res = cs.take<double>(size_t(kp) * 6 + 1);
  double* partials = cs.take<double>(nred);
  SFW3D_TRY(upload_atoms(ctx, pieces, ad));
  SFW3D_TRY(render_impl(ctx, dtype, dims, pieces, ad, kp, A));
  SFW3D_TRY(psf_apply_impl(ctx, psf, dtype, A, B, 0, A));
  // r = model - y on the slab planes only, 0 on the halo planes
  const size_t plane = size_t(dims[1]) * dims[2];
  const size_t off = size_t(halo) * plane * es;
  SFW3D_CUDA_TRY(cudaMemsetAsync(A, 0, vb, ctx->stream));
  SFW3D_TRY(sumsq_diff_impl(ctx, dtype, int64_t(x1 - x0 + 1) * int64_t(plane), B + off,
                            static_cast<const char*>(y_dev) + off, A + off, partials, res));
  SFW3D_TRY(psf_apply_impl(ctx, psf, dtype, A, B, 1, A));
  SFW3D_TRY(atom_sums_impl(ctx, dtype, dims, B, pieces, ad, res + 1));
  if (partials_dev) {  // device output for an in-stream all-reduce: no sync here
    std::vector<int> first(k + 1, 0);
    for (int q = 0, i = 0; i <= k; ++i) {
      while (q < kp && owner[q] < i) ++q;
      first[i] = q;
    }
    SFW3D_TRY(ensure_device(ctx, ctx->ws_aux, first.size() * sizeof(int)));
    int* first_dev = static_cast<int*>(ctx->ws_aux.ptr);
    SFW3D_TRY(stage_upload(ctx, first_dev, first.data(), first.size() * sizeof(int)));
    piece_combine_kernel<<<(6 * k + 1 + 255) / 256, 256, 0, ctx->stream>>>(first_dev, k, res,
                                                                          partials_dev);
    SFW3D_LAUNCH_CHECK(ctx);
    return SFW3D_OK;
  }
  std::vector<double> host(size_t(kp) * 6 + 1);
  SFW3D_TRY(download_sync(ctx, host.data(), res, host.size() * sizeof(double)));
  *half_sumsq_host = 0.5 * host[0];
  std::fill(sums_host, sums_host + size_t(k) * 6, 0.0);
  for (int q = 0; q < kp; ++q)
    for (int c = 0; c < 6; ++c) sums_host[6 * owner[q] + c] += host[1 + 6 * q + c];
  if (!finite_all(sums_host, size_t(k) * 6)) {
    set_error("non-finite criterion gradient; atom parameters left the smooth regime");
    return SFW3D_ENONFINITE;
  }
  return SFW3D_OK;
}

// ------------------------------------------------ x-slab render / atom sums
extern "C" int sfw3d_render_slab(sfw3d_ctx* ctx, int dtype, const int gdims[3],
                                 const double* params_host, int k, int x0, int x1, int halo,
                                 void* out_dev) {
  SFW3D_CHECK_ARG(ctx && out_dev && gdims, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || params_host), "params");
  SFW3D_CHECK_ARG(gdims[0] > 0 && x0 >= 0 && x1 >= x0 && x1 < gdims[0] && halo >= 0,
                  "slab bounds");
  SFW3D_TRY(begin_call(ctx));
  std::vector<AtomGeo> atoms, pieces;
  std::vector<int> owner;
  SFW3D_TRY(build_atoms(gdims, params_host, k, atoms));
  const int nxl = x1 - x0 + 1 + 2 * halo;
  SFW3D_TRY(clip_atoms_x(atoms, gdims[0], x0 - halo, nxl, x0 - halo, pieces, owner));
  const int kp = int(pieces.size());
  const int wd[3] = {nxl, gdims[1], gdims[2]};
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small, (size_t(kp) + 1) * sizeof(AtomGeo) + 4096));
  AtomGeo* ad = static_cast<AtomGeo*>(ctx->ws_small.ptr);
  SFW3D_TRY(upload_atoms(ctx, pieces, ad));
  return render_impl(ctx, dtype, wd, pieces, ad, kp, out_dev);
}

extern "C" int sfw3d_atom_sums_slab(sfw3d_ctx* ctx, int dtype, const int gdims[3],
                                    const void* field_dev, const double* params_host, int k,
                                    int x0, int x1, int halo, double* sums_host) {
  SFW3D_CHECK_ARG(ctx && field_dev && sums_host && gdims, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || params_host), "params");
  SFW3D_CHECK_ARG(gdims[0] > 0 && x0 >= 0 && x1 >= x0 && x1 < gdims[0] && halo >= 0,
                  "slab bounds");
  SFW3D_TRY(begin_call(ctx));
  std::fill(sums_host, sums_host + size_t(k) * 6, 0.0);
  if (k == 0) return SFW3D_OK;
  std::vector<AtomGeo> atoms, pieces;
  std::vector<int> owner;
  SFW3D_TRY(build_atoms(gdims, params_host, k, atoms));
  // the sums run over the OWNED planes [x0, x1]; the field is the window
  // whose plane 0 is global plane x0 - halo
  SFW3D_TRY(clip_atoms_x(atoms, gdims[0], x0, x1 - x0 + 1, x0 - halo, pieces, owner));
  const int kp = int(pieces.size());
  if (kp == 0) return SFW3D_OK;
  const int wd[3] = {x1 - x0 + 1 + 2 * halo, gdims[1], gdims[2]};
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small,
                          Carver::need({size_t(kp) * sizeof(AtomGeo), size_t(kp) * 6 * sizeof(double)})));
  Carver cv(ctx->ws_small.ptr);
  AtomGeo* ad = cv.take<AtomGeo>(kp);
  double* sums = cv.take<double>(size_t(kp) * 6);
  SFW3D_TRY(upload_atoms(ctx, pieces, ad));
  SFW3D_TRY(atom_sums_impl(ctx, dtype, wd, field_dev, pieces, ad, sums));
  std::vector<double> host(size_t(kp) * 6);
  SFW3D_TRY(download_sync(ctx, host.data(), sums, host.size() * sizeof(double)));
  for (int q = 0; q < kp; ++q)
    for (int c = 0; c < 6; ++c) sums_host[6 * owner[q] + c] += host[6 * q + c];
  return SFW3D_OK;
}

// ------------------------------------------------ .vol IO straight to HBM
// volumes.py:96-113 format: b"SFW3DV01", nx, ny, nz (little-endian uint32),
// then nx*ny*nz little-endian float64 in C order. The payload streams through
// two pinned staging buffers (the disk read of chunk i + 1 overlaps the H2D of
// chunk i); fp32 storage converts on the device; a device pass counts
// non-finite values (the reference's VolumeFormatError, here SFW3D_EINVAL).
namespace sfw3d {
namespace {
constexpr size_t kVolChunk = size_t(32) << 20;  // bytes per staging buffer

// dst == NULL: check only (fp64 storage reads straight into place)
template <typename T>
__global__ void vol_convert_kernel(const double* src, T* dst, long long n,
                                   unsigned long long* __restrict__ bad) {
  unsigned long long b = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = src[i];
    b += !isfinite(v);
    if (dst) dst[i] = T(v);
  }
  if (b) atomicAdd(bad, b);  // (an integer count: order-independent)
}

template <typename T>
__global__ void vol_export_kernel(const T* __restrict__ src, double* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = double(src[i]);
}

int vol_header(FILE* f, const char* path, int dims[3], long long* payload) {
  unsigned char h[20];
  if (fread(h, 1, 20, f) != 20) {
    set_error(std::string(path) + ": truncated header");
    return SFW3D_EINVAL;
  }
  if (memcmp(h, "SFW3DV01", 8) != 0) {
    set_error(std::string(path) + ": bad magic");
    return SFW3D_EINVAL;
  }
  long long n = 1;
  for (int a = 0; a < 3; ++a) {
    const uint32_t v = uint32_t(h[8 + 4 * a]) | (uint32_t(h[9 + 4 * a]) << 8) |
                       (uint32_t(h[10 + 4 * a]) << 16) | (uint32_t(h[11 + 4 * a]) << 24);
    if (v < 1 || v > (1u << 30)) {
      set_error(std::string(path) + ": dims must be three positive integers");
      return SFW3D_EINVAL;
    }
    dims[a] = int(v);
    n *= v;
  }
  fseeko(f, 0, SEEK_END);
  const long long size = ftello(f);
  fseeko(f, 20, SEEK_SET);
  if (size != 20 + 8 * n) {
    set_error(std::string(path) + ": payload size mismatch (header says " +
              std::to_string(20 + 8 * n) + " bytes, file has " + std::to_string(size) + ")");
    return SFW3D_EINVAL;
  }
  *payload = n;
  return SFW3D_OK;
}
}  // namespace
}  // namespace sfw3d

extern "C" int sfw3d_volume_info(const char* path, int32_t dims[3]) {
  SFW3D_CHECK_ARG(path && dims, "NULL argument");
  FILE* f = fopen(path, "rb");
  if (!f) {
    set_error(std::string(path) + ": cannot open");
    return SFW3D_EINVAL;
  }
  int d[3];
  long long n = 0;
  const int st = vol_header(f, path, d, &n);
  fclose(f);
  if (st == SFW3D_OK)
    for (int a = 0; a < 3; ++a) dims[a] = d[a];
  return st;
}

extern "C" int sfw3d_volume_read(sfw3d_ctx* ctx, const char* path, int dtype, void* out_dev) {
  SFW3D_CHECK_ARG(ctx && path && out_dev, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_TRY(begin_call(ctx));
  FILE* f = fopen(path, "rb");
  if (!f) {
    set_error(std::string(path) + ": cannot open");
    return SFW3D_EINVAL;
  }
  int dims[3];
  long long n = 0;
  int st = vol_header(f, path, dims, &n);
  if (st != SFW3D_OK) {
    fclose(f);
    return st;
  }
  // staging: 2 pinned host buffers + (fp32) one device f64 chunk + the counter
  SFW3D_TRY(ensure_pinned_io(ctx, 2 * kVolChunk));
  SFW3D_TRY(ensure_device(ctx, ctx->ws_aux, kVolChunk + 256));
  double* dchunk = static_cast<double*>(ctx->ws_aux.ptr);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(
      static_cast<char*>(ctx->ws_aux.ptr) + kVolChunk);
  SFW3D_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(*bad), ctx->stream));
  cudaEvent_t ev[2];
  SFW3D_CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  SFW3D_CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  const long long per = (long long)(kVolChunk / 8);
  long long done = 0;
  int i = 0;
  for (; done < n && st == SFW3D_OK; ++i) {
    const long long cnt = std::min(per, n - done);
    char* host = static_cast<char*>(ctx->pinned_io.ptr) + (i & 1) * kVolChunk;
    if (i >= 2) cudaEventSynchronize(ev[i & 1]);  // that buffer's copy has landed
    if (fread(host, 8, size_t(cnt), f) != size_t(cnt)) {
      set_error(std::string(path) + ": short read");
      st = SFW3D_EINVAL;
      break;
    }
    void* dst = dtype == SFW3D_F64 ? static_cast<void*>(static_cast<double*>(out_dev) + done)
                                   : static_cast<void*>(dchunk);
    cudaMemcpyAsync(dst, host, size_t(cnt) * 8, cudaMemcpyHostToDevice, ctx->stream);
    const unsigned grid = unsigned(std::min<long long>(4LL * ctx->num_sms, (cnt + 255) / 256));
    if (dtype == SFW3D_F64)
      vol_convert_kernel<double><<<grid, 256, 0, ctx->stream>>>(
          static_cast<double*>(dst), nullptr, cnt, bad);
    else
      vol_convert_kernel<float><<<grid, 256, 0, ctx->stream>>>(
          dchunk, static_cast<float*>(out_dev) + done, cnt, bad);
    SFW3D_LAUNCH_CHECK(ctx);
    cudaEventRecord(ev[i & 1], ctx->stream);
    done += cnt;
  }
  fclose(f);
  unsigned long long hbad = 0;
  if (st == SFW3D_OK) st = download_sync(ctx, &hbad, bad, sizeof(hbad));
  else cudaStreamSynchronize(ctx->stream);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (st == SFW3D_OK && hbad) {
    set_error(std::string(path) + ": payload contains non-finite values");
    return SFW3D_EINVAL;
  }
  return st;
}

extern "C" int sfw3d_volume_write(sfw3d_ctx* ctx, const char* path, int dtype, const int dims[3],
                                  const void* in_dev) {
  SFW3D_CHECK_ARG(ctx && path && in_dev && dims, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
  SFW3D_TRY(begin_call(ctx));
  FILE* f = fopen(path, "wb");
  if (!f) {
    set_error(std::string(path) + ": cannot open for writing");
    return SFW3D_EINVAL;
  }
  unsigned char h[20];
  memcpy(h, "SFW3DV01", 8);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 4; ++b) h[8 + 4 * a + b] = (uint32_t(dims[a]) >> (8 * b)) & 255;
  fwrite(h, 1, 20, f);
  SFW3D_TRY(ensure_pinned_io(ctx, 2 * kVolChunk));
  SFW3D_TRY(ensure_device(ctx, ctx->ws_aux, kVolChunk));
  double* dchunk = static_cast<double*>(ctx->ws_aux.ptr);
  const long long n = (long long)dims[0] * dims[1] * dims[2], per = (long long)(kVolChunk / 8);
  int st = SFW3D_OK;
  for (long long done = 0; done < n; done += per) {
    const long long cnt = std::min(per, n - done);
    const double* src = static_cast<const double*>(in_dev) + done;
    if (dtype == SFW3D_F32) {
      vol_export_kernel<float><<<unsigned(std::min<long long>(4LL * ctx->num_sms, (cnt + 255) / 256)),
                                 256, 0, ctx->stream>>>(static_cast<const float*>(in_dev) + done,
                                                        dchunk, cnt);
      src = dchunk;
    }
    char* host = static_cast<char*>(ctx->pinned_io.ptr);
    cudaMemcpyAsync(host, src, size_t(cnt) * 8, cudaMemcpyDeviceToHost, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess ||
        fwrite(host, 8, size_t(cnt), f) != size_t(cnt)) {
      set_error(std::string(path) + ": write failed");
      st = SFW3D_ECUDA;
      break;
    }
  }
  fclose(f);
  return st;
}
