// K5 / K8 / K9 — non-negative LASSO weight step on the device.
//
// nonneg_lasso (solvers.py:111-180) stacks k full blurred-atom volumes and
// forms Gram = Phi Phi^T and b = Phi y with one DGEMM (solvers.py:141-143),
// then runs cyclic coordinate descent in Python. Here:
//  * sfw3d_dots: k inner products <vec_i, v> in fp64 with a fixed block
//    partition and fixed-order combine (deterministic); the host solver keeps
//    the Gram matrix incrementally (one new row per added atom);
//  * sfw3d_nnlasso_cd: one warp runs the reference's exact update sequence
//    in fp64 (same rounding: no FMA where numpy rounds twice);
//  * sfw3d_residual: y - sum_i w_i phi_i in list order (solvers.py:253-257).
#include <cstring>

#include "internal.cuh"

namespace sfw3d {
namespace {

constexpr int kDotThreads = 256;
constexpr int kDotBlocks = 64;  // per vector; fixed so the sum order is fixed

template <typename T>
__global__ void __launch_bounds__(kDotThreads) dots_kernel(const T* const* __restrict__ vecs,
                                                           const T* __restrict__ v, long long n,
                                                           double* __restrict__ partials) {
  const T* a = vecs[blockIdx.y];
  double s = 0.0;
  // 16-byte loads (fixed partition: the sum order depends only on n)
  constexpr int V = 16 / sizeof(T);
  const long long nv = n / V;
  for (long long q = blockIdx.x * (long long)kDotThreads + threadIdx.x; q < nv;
       q += (long long)kDotBlocks * kDotThreads) {
    if constexpr (sizeof(T) == 8) {
      const double2 x = __ldg(reinterpret_cast<const double2*>(a) + q);
      const double2 z = __ldg(reinterpret_cast<const double2*>(v) + q);
      s += x.x * z.x;
      s += x.y * z.y;
    } else {
      const float4 x = __ldg(reinterpret_cast<const float4*>(a) + q);
      const float4 z = __ldg(reinterpret_cast<const float4*>(v) + q);
      s += double(x.x) * double(z.x);
      s += double(x.y) * double(z.y);
      s += double(x.z) * double(z.z);
      s += double(x.w) * double(z.w);
    }
  }
  for (long long i = nv * V + blockIdx.x * (long long)kDotThreads + threadIdx.x; i < n;
       i += (long long)kDotBlocks * kDotThreads)
    s += double(a[i]) * double(v[i]);
  __shared__ double red[kDotThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < kDotThreads / 32; ++w) x += red[w];
    partials[blockIdx.y * kDotBlocks + blockIdx.x] = x;
  }
}

__global__ void dots_combine_kernel(const double* __restrict__ partials, int k,
                                    double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  double x = 0.0;
  for (int b = 0; b < kDotBlocks; ++b) x += partials[i * kDotBlocks + b];
  out[i] = x;
}

template <typename T>
__global__ void __launch_bounds__(256) residual_kernel(const T* __restrict__ y,
                                                       const T* const* __restrict__ phis,
                                                       const double* __restrict__ w, int k,
                                                       long long n, T* __restrict__ out,
                                                       double* __restrict__ partials,
                                                       const int* __restrict__ plane_ptr,
                                                       const int* __restrict__ plane_atoms,
                                                       long long plane) {
  double s = 0.0;
  // plane_ptr / plane_atoms (optional): per x plane the atoms, in list order,
  // whose phi is not identically zero there (CSR); the others are skipped —
  // loads and arithmetic — which leaves every voxel unchanged bit for bit
  // V consecutive voxels per thread (16-byte loads) and 4 atoms' loads issued
  // before their (in-order) updates: the k streams are read with enough
  // loads in flight; the per-voxel update order is the reference's
  constexpr int V = 16 / sizeof(T);
  const long long nv = n / V;
  for (long long q = blockIdx.x * 256LL + threadIdx.x; q < nv; q += (long long)gridDim.x * 256) {
    const long long i = q * V;
    int jb = 0, je = k;
    if (plane_ptr) {
      const int x = int(i / plane);
      jb = plane_ptr[x];
      je = plane_ptr[x + 1];
    }
    // the running residual is kept in fp64 across the atoms (one conversion
    // per phi value; fp32 storage rounds once, at the end) — the conversion
    // pipe, not HBM, bounded the per-atom fp32 round trip
    double r[V];
#pragma unroll
    for (int u = 0; u < V; ++u) r[u] = double(y[i + u]);
    int jj = jb;
    for (; jj + 4 <= je; jj += 4) {
      T ph[4][V];
      int ja[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ja[a] = plane_atoms ? plane_atoms[jj + a] : jj + a;
        if constexpr (sizeof(T) == 8) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(phis[ja[a]] + i));
          ph[a][0] = v.x; ph[a][1] = v.y;
        } else {
          const float4 v = __ldg(reinterpret_cast<const float4*>(phis[ja[a]] + i));
          ph[a][0] = v.x; ph[a][1] = v.y; ph[a][2] = v.z; ph[a][3] = v.w;
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double wj = w[ja[a]];
#pragma unroll
        for (int u = 0; u < V; ++u)
          r[u] = __dsub_rn(r[u], __dmul_rn(wj, double(ph[a][u])));  // data -= w * phi
      }
    }
    for (; jj < je; ++jj) {
      const int j = plane_atoms ? plane_atoms[jj] : jj;
      const double wj = w[j];
#pragma unroll
      for (int u = 0; u < V; ++u) r[u] = __dsub_rn(r[u], __dmul_rn(wj, double(phis[j][i + u])));
    }
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const T rt = T(r[u]);
      if (out) out[i + u] = rt;
      s += double(rt) * double(rt);
    }
  }
  // (tail voxels when n is not a multiple of V)
  for (long long i = nv * V + blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    double rd = double(y[i]);
    int jb = 0, je = k;
    if (plane_ptr) {
      const int x = int(i / plane);
      jb = plane_ptr[x];
      je = plane_ptr[x + 1];
    }
    for (int jj = jb; jj < je; ++jj) {
      const int j2 = plane_atoms ? plane_atoms[jj] : jj;
      rd = __dsub_rn(rd, __dmul_rn(w[j2], double(phis[j2][i])));
    }
    const T r = T(rd);
    if (out) out[i] = r;
    s += double(r) * double(r);
  }
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int q = 0; q < 8; ++q) x += red[q];
    partials[blockIdx.x] = x;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ p, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double x = 0.0;
    for (int i = 0; i < n; ++i) x += p[i];
    *out = x;
  }
}

// One warp; solvers.py:149-180 step for step. Gram rows are read for the
// column update: the host assembles the Gram matrix exactly symmetric.
// GRAM_SMEM: the Gram matrix and b are staged in shared memory first (k <=
// kCdSmemK): the sweep's per-coordinate reads then cost shared-memory
// latency instead of L2 round trips; the arithmetic is unchanged.
template <bool GRAM_SMEM>
__global__ void __launch_bounds__(32) cd_kernel(int k, const double* __restrict__ gram_g,
                                                const double* __restrict__ b_g, double lam,
                                                double tol, int max_iter, double* __restrict__ w_io,
                                                int* __restrict__ info, double* __restrict__ kkt_out) {
  extern __shared__ double sm[];
  double* w = sm;
  double* gw = sm + k;
  const int lane = threadIdx.x;
  const double* gram = gram_g;
  const double* b = b_g;
  if constexpr (GRAM_SMEM) {
    double* sg = sm + 2 * k;
    double* sb = sg + (size_t)k * k;
    for (long long e = lane; e < (long long)k * k; e += 32) sg[e] = gram_g[e];
    for (int i = lane; i < k; i += 32) sb[i] = b_g[i];
    gram = sg;
    b = sb;
  }
  for (int i = lane; i < k; i += 32) w[i] = w_io[i];
  __syncwarp();
  // gw = gram @ w (row order)
  for (int i = lane; i < k; i += 32) {
    double x = 0.0;
    for (int j = 0; j < k; ++j) x = __dadd_rn(x, __dmul_rn(gram[(long long)i * k + j], w[j]));
    gw[i] = x;
  }
  __syncwarp();
  double wmax = 0.0;
  for (int i = 0; i < k; ++i) wmax = (i == 0 || w[i] > wmax) ? w[i] : wmax;
  double w_scale = wmax > 1.0 ? wmax : 1.0;  // max(1.0, max(w))
  double kkt = INFINITY;
  int sweeps = 0, reason = 2;
  for (int sweep = 1; sweep <= max_iter; ++sweep) {
    sweeps = sweep;
    double step = 0.0;
    for (int i = 0; i < k; ++i) {
      const double old = w[i];
      const double gii = gram[(long long)i * k + i];
      const double x = __dadd_rn(old, __ddiv_rn(__dsub_rn(__dsub_rn(b[i], lam), gw[i]), gii));
      const double nw = (x > 0.0) ? x : 0.0;  // Python max(0.0, x)
      __syncwarp();
      if (nw != old) {
        const double dlt = __dsub_rn(nw, old);
        const double* row = gram + (long long)i * k;
        for (int j = lane; j < k; j += 32) gw[j] = __dadd_rn(gw[j], __dmul_rn(dlt, row[j]));
        if (lane == 0) w[i] = nw;
        const double ad = fabs(dlt);
        step = (ad > step) ? ad : step;
      }
      __syncwarp();
    }
    // KKT residual (solvers.py:161-169)
    double ka = 0.0, ki = 0.0;
    int has_a = 0, has_i = 0;
    for (int j = lane; j < k; j += 32) {
      const double slope = __dadd_rn(__dsub_rn(gw[j], b[j]), lam);
      if (w[j] > 0.0) {
        has_a = 1;
        ka = fmax(ka, fabs(slope));
      } else {
        has_i = 1;
        ki = fmax(ki, fmax(0.0, -slope));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ka = fmax(ka, __shfl_xor_sync(0xffffffffu, ka, o));
      ki = fmax(ki, __shfl_xor_sync(0xffffffffu, ki, o));
      has_a |= __shfl_xor_sync(0xffffffffu, has_a, o);
      has_i |= __shfl_xor_sync(0xffffffffu, has_i, o);
    }
    kkt = 0.0;
    if (has_a) kkt = ka;
    if (has_i) kkt = fmax(kkt, ki);
    if (kkt <= tol) {
      reason = 0;
      break;
    }
    double wm = -INFINITY;
    for (int j = lane; j < k; j += 32) wm = fmax(wm, w[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wm = fmax(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    w_scale = (wm > w_scale) ? wm : w_scale;
    if (step <= 1e-14 * w_scale) {
      reason = 1;
      break;
    }
  }
  __syncwarp();
  for (int i = lane; i < k; i += 32) w_io[i] = w[i];
  if (lane == 0) {
    info[0] = sweeps;
    info[1] = reason;
    *kkt_out = kkt;
  }
}

// Active-set solve of the same non-negative LASSO (fp32-storage solves):
// min 1/2 w'Gw - (b - lam)'w subject to w >= 0 is a strictly convex QP
// (Gram of distinct blurred atoms); Lawson-Hanson's active-set iteration
// reaches its exact optimum in a few dense solves instead of hundreds of CD
// sweeps. One CTA: the free set's Gram block is gathered into shared memory
// and Cholesky-factored in place (column-parallel), two triangular solves,
// the step / set update, and the reference's KKT residual as the stop test.
// info[1]: 0 KKT <= tol, 2 iteration cap, 3 factorisation failed (near-
// singular free block: the caller falls back to cd_kernel).
constexpr int kQpThreads = 256;
constexpr int kQpMaxFree = 150;  // free-set block <= 150^2 doubles in shared memory

__device__ double qp_block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < kQpThreads / 32; ++w) r = fmax(r, red[w]);
  return r;
}

__global__ void __launch_bounds__(kQpThreads) nnqp_kernel(int k, const double* __restrict__ G,
                                                         const double* __restrict__ b, double lam,
                                                         double tol, int max_iter,
                                                         double* __restrict__ w_io,
                                                         int* __restrict__ info,
                                                         double* __restrict__ kkt_out) {
  extern __shared__ double sm[];
  double* A = sm;                                   // [kQpMaxFree * kQpMaxFree]
  double* w = A + kQpMaxFree * kQpMaxFree;          // [k]
  double* z = w + k;                                // [k] (free-set solution, slot order)
  double* g = z + k;                                // [k] b - lam - G w
  int* fidx = reinterpret_cast<int*>(g + k);        // [k] free indices
  __shared__ double red[kQpThreads / 32];
  __shared__ int s_nf, s_flag, s_arg;
  __shared__ double s_alpha;
  const int tid = threadIdx.x;
  for (int i = tid; i < k; i += kQpThreads) w[i] = w_io[i];
  double dmax = 0.0;
  for (int i = tid; i < k; i += kQpThreads) dmax = fmax(dmax, G[(long long)i * k + i]);
  dmax = qp_block_max(dmax, red);
  int reason = 2, it = 0;
  double kkt = INFINITY;
  bool solved = false;  // w is the exact solve on its current free set
  for (it = 1; it <= max_iter; ++it) {
    // gradient residual g = (b - lam) - G w and the reference KKT measure
    for (int i = tid; i < k; i += kQpThreads) {
      double x = 0.0;
      const double* row = G + (long long)i * k;
      for (int j = 0; j < k; ++j) x += row[j] * w[j];
      g[i] = (b[i] - lam) - x;
    }
    __syncthreads();
    double ka = 0.0, best = -INFINITY;
    int arg = -1;
    for (int i = tid; i < k; i += kQpThreads) {
      if (w[i] > 0.0) {
        ka = fmax(ka, fabs(g[i]));
      } else {
        ka = fmax(ka, fmax(0.0, g[i]));
        if (g[i] > best) { best = g[i]; arg = i; }
      }
    }
    kkt = qp_block_max(ka, red);
    if (kkt <= tol) { reason = 0; break; }
    // entering index: the inactive coordinate with the largest g (ties: lowest)
    {
      double v = best;
      int a = arg;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oa = __shfl_xor_sync(0xffffffffu, a, o);
        if (ov > v || (ov == v && oa >= 0 && (a < 0 || oa < a))) { v = ov; a = oa; }
      }
      __shared__ double rv[kQpThreads / 32];
      __shared__ int ra[kQpThreads / 32];
      if ((tid & 31) == 0) { rv[tid >> 5] = v; ra[tid >> 5] = a; }
      __syncthreads();
      if (tid == 0) {
        double bv = rv[0];
        int ba = ra[0];
        for (int q = 1; q < kQpThreads / 32; ++q)
          if (rv[q] > bv || (rv[q] == bv && ra[q] >= 0 && (ba < 0 || ra[q] < ba))) { bv = rv[q]; ba = ra[q]; }
        s_arg = bv > tol ? ba : -1;
      }
      __syncthreads();
    }
    const int enter = s_arg;
    if (enter < 0 && solved) {  // KKT limited by rounding on the solved free set
      reason = 0;
      break;
    }
    // inner loop: solve on the free set, step back while the solution leaves w >= 0
    bool entered = false;
    solved = false;
    for (int inner = 0; inner < 4 * k + 4; ++inner) {
      if (tid == 0) {
        int nf = 0;
        for (int i = 0; i < k; ++i)
          if (w[i] > 0.0 || (!entered && i == enter)) fidx[nf++] = i;
        s_nf = nf;
      }
      __syncthreads();
      entered = true;
      const int nf = s_nf;
      if (nf > kQpMaxFree) { reason = 3; break; }
      if (nf == 0) break;
      for (int e = tid; e < nf * nf; e += kQpThreads) {
        const int r = e / nf, c = e - r * nf;
        A[e] = G[(long long)fidx[r] * k + fidx[c]];
      }
      for (int r = tid; r < nf; r += kQpThreads) z[r] = b[fidx[r]] - lam;
      if (tid == 0) s_flag = 0;
      __syncthreads();
      // Cholesky A = L L^T (lower, in place), right-looking
      for (int j = 0; j < nf; ++j) {
        if (tid == 0) {
          const double d = A[j * nf + j];
          if (!(d > 1e-13 * dmax)) s_flag = 1;
          A[j * nf + j] = sqrt(fmax(d, 1e-300));
        }
        __syncthreads();
        if (s_flag) break;
        const double ljj = A[j * nf + j];
        for (int r = j + 1 + tid; r < nf; r += kQpThreads) A[r * nf + j] /= ljj;
        __syncthreads();
        const int m = nf - j - 1;
        for (int e = tid; e < m * m; e += kQpThreads) {
          const int r = j + 1 + e / m, c = j + 1 + e % m;
          if (c <= r) A[r * nf + c] -= A[r * nf + j] * A[c * nf + j];
        }
        __syncthreads();
      }
      if (s_flag) { reason = 3; break; }
      // L y = rhs, L^T z = y (one thread per step: nf <= 150)
      if (tid == 0) {
        for (int r = 0; r < nf; ++r) {
          double x = z[r];
          for (int c = 0; c < r; ++c) x -= A[r * nf + c] * z[c];
          z[r] = x / A[r * nf + r];
        }
        for (int r = nf - 1; r >= 0; --r) {
          double x = z[r];
          for (int c = r + 1; c < nf; ++c) x -= A[c * nf + r] * z[c];
          z[r] = x / A[r * nf + r];
        }
        // feasible: accept; else step from w toward z until a free weight hits 0
        double alpha = 1.0;
        for (int r = 0; r < nf; ++r)
          if (z[r] <= 0.0) {
            const double wi = w[fidx[r]];
            const double a = wi / (wi - z[r]);
            alpha = fmin(alpha, a);
          }
        s_alpha = alpha;
        for (int r = 0; r < nf; ++r) {
          const int i = fidx[r];
          double nw = alpha >= 1.0 ? z[r] : w[i] + alpha * (z[r] - w[i]);
          if (alpha < 1.0 && (z[r] <= 0.0 && w[i] / (w[i] - z[r]) <= alpha)) nw = 0.0;
          w[i] = nw > 0.0 ? nw : 0.0;
        }
      }
      __syncthreads();
      if (s_alpha >= 1.0) {
        solved = true;
        break;
      }
    }
    if (reason == 3) break;
  }
  __syncthreads();
  for (int i = tid; i < k; i += kQpThreads) w_io[i] = w[i];
  if (tid == 0) {
    info[0] = it;
    info[1] = reason;
    *kkt_out = kkt;
  }
}

}  // namespace
}  // namespace sfw3d

using namespace sfw3d;

extern "C" int sfw3d_dots(sfw3d_ctx* ctx, int dtype, int64_t n, const void* const* vecs_host, int k,
                          const void* v_dev, double* out_host) {
  SFW3D_CHECK_ARG(ctx && v_dev && out_host, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(n >= 0 && k >= 0 && (k == 0 || vecs_host), "sizes");
  SFW3D_TRY(begin_call(ctx));
  if (k == 0) return SFW3D_OK;
  for (int i = 0; i < k; ++i) SFW3D_CHECK_ARG(vecs_host[i] != nullptr, "NULL vector");
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small,
                          Carver::need({size_t(k) * sizeof(void*), size_t(k) * kDotBlocks * sizeof(double),
                                        size_t(k) * sizeof(double)})));
  Carver cv(ctx->ws_small.ptr);
  const void** vp = cv.take<const void*>(k);
  double* part = cv.take<double>(size_t(k) * kDotBlocks);
  double* out = cv.take<double>(k);
  SFW3D_TRY(stage_upload(ctx, vp, vecs_host, size_t(k) * sizeof(void*)));
  dim3 grid(kDotBlocks, k);
  SFW3D_PROF(ctx, "dots");
  if (dtype == SFW3D_F64)
    dots_kernel<double><<<grid, kDotThreads, 0, ctx->stream>>>(
        reinterpret_cast<const double* const*>(vp), static_cast<const double*>(v_dev), n, part);
  else
    dots_kernel<float><<<grid, kDotThreads, 0, ctx->stream>>>(
        reinterpret_cast<const float* const*>(vp), static_cast<const float*>(v_dev), n, part);
  SFW3D_LAUNCH_CHECK(ctx);
  dots_combine_kernel<<<(k + 127) / 128, 128, 0, ctx->stream>>>(part, k, out);
  SFW3D_LAUNCH_CHECK(ctx);
  return download_sync(ctx, out_host, out, size_t(k) * sizeof(double));
}

static int residual_run(sfw3d_ctx* ctx, int dtype, int64_t n, const void* y_dev,
                        const void* const* phis_host, const double* w_host, int k, void* out_dev,
                        double* sumsq_host, const int32_t* xrange_host, long long plane);

extern "C" int sfw3d_residual(sfw3d_ctx* ctx, int dtype, int64_t n, const void* y_dev,
                              const void* const* phis_host, const double* w_host, int k,
                              void* out_dev, double* sumsq_host) {
  return residual_run(ctx, dtype, n, y_dev, phis_host, w_host, k, out_dev, sumsq_host, nullptr, 1);
}

extern "C" int sfw3d_residual_ranged(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* y_dev,
                                     const void* const* phis_host, const double* w_host,
                                     const int32_t* xrange_host, int k, void* out_dev,
                                     double* sumsq_host) {
  SFW3D_CHECK_ARG(dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
  SFW3D_CHECK_ARG(k == 0 || xrange_host, "NULL argument");
  for (int i = 0; i < k; ++i)
    SFW3D_CHECK_ARG(xrange_host[2 * i] >= 0 && xrange_host[2 * i] < dims[0] &&
                        xrange_host[2 * i + 1] >= 0 && xrange_host[2 * i + 1] < dims[0], "x range");
  return residual_run(ctx, dtype, vol_count(dims), y_dev, phis_host, w_host, k, out_dev, sumsq_host,
                      xrange_host, (long long)dims[1] * dims[2]);
}

static int residual_run(sfw3d_ctx* ctx, int dtype, int64_t n, const void* y_dev,
                        const void* const* phis_host, const double* w_host, int k, void* out_dev,
                        double* sumsq_host, const int32_t* xrange_host, long long plane) {
  SFW3D_CHECK_ARG(ctx && y_dev, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(n >= 0 && k >= 0 && (k == 0 || (phis_host && w_host)), "sizes");
  SFW3D_TRY(begin_call(ctx));
  const int nblk = 4 * ctx->num_sms;
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small,
                          Carver::need({size_t(k + 1) * sizeof(void*), size_t(k + 1) * sizeof(double),
                                        size_t(nblk) * sizeof(double), sizeof(double)})));
  Carver cv(ctx->ws_small.ptr);
  const void** pp = cv.take<const void*>(k + 1);
  double* wd = cv.take<double>(k + 1);
  double* part = cv.take<double>(nblk);
  double* res = cv.take<double>(1);
  if (k) {
    SFW3D_TRY(stage_upload(ctx, pp, phis_host, size_t(k) * sizeof(void*)));
    SFW3D_TRY(stage_upload(ctx, wd, w_host, size_t(k) * sizeof(double)));
  }
  // per x plane the atoms that reach it, in list order (CSR)
  int* pptr = nullptr;
  int* patoms = nullptr;
  if (xrange_host && k > 0) {
    const int nx = int(n / plane);
    std::vector<int> ptr(nx + 1, 0), list;
    list.reserve(size_t(nx) * 8);
    for (int x = 0; x < nx; ++x) {
      for (int j = 0; j < k; ++j) {
        const int lo = xrange_host[2 * j], hi = xrange_host[2 * j + 1];
        if (lo <= hi ? (x >= lo && x <= hi) : (x >= lo || x <= hi)) list.push_back(j);
      }
      ptr[x + 1] = int(list.size());
    }
    SFW3D_TRY(ensure_device(ctx, ctx->ws_plan, Carver::need({ptr.size() * sizeof(int),
                                                            (list.size() + 1) * sizeof(int)})));
    Carver cp(ctx->ws_plan.ptr);
    pptr = cp.take<int>(ptr.size());
    patoms = cp.take<int>(list.size() + 1);
    SFW3D_TRY(stage_upload(ctx, pptr, ptr.data(), ptr.size() * sizeof(int)));
    if (!list.empty()) SFW3D_TRY(stage_upload(ctx, patoms, list.data(), list.size() * sizeof(int)));
  }
  SFW3D_PROF(ctx, "residual");
  if (dtype == SFW3D_F64)
    residual_kernel<double><<<nblk, 256, 0, ctx->stream>>>(
        static_cast<const double*>(y_dev), reinterpret_cast<const double* const*>(pp), wd, k, n,
        static_cast<double*>(out_dev), part, pptr, patoms, plane);
  else
    residual_kernel<float><<<nblk, 256, 0, ctx->stream>>>(
        static_cast<const float*>(y_dev), reinterpret_cast<const float* const*>(pp), wd, k, n,
        static_cast<float*>(out_dev), part, pptr, patoms, plane);
  SFW3D_LAUNCH_CHECK(ctx);
  if (sumsq_host) {
    sum_partials_kernel<<<1, 32, 0, ctx->stream>>>(part, nblk, res);
    SFW3D_LAUNCH_CHECK(ctx);
    return download_sync(ctx, sumsq_host, res, sizeof(double));
  }
  return SFW3D_OK;
}

static int nnlasso_run(sfw3d_ctx* ctx, int k, const double* gram_host, const double* b_host,
                       double lam, double tol, int max_iter, double* w_host, int32_t* info_host,
                       double* kkt_host, bool qp);

extern "C" int sfw3d_nnlasso_qp(sfw3d_ctx* ctx, int k, const double* gram_host, const double* b_host,
                                double lam, double tol, int max_iter, double* w_host,
                                int32_t* info_host, double* kkt_host) {
  return nnlasso_run(ctx, k, gram_host, b_host, lam, tol, max_iter, w_host, info_host, kkt_host,
                     true);
}

extern "C" int sfw3d_nnlasso_cd(sfw3d_ctx* ctx, int k, const double* gram_host, const double* b_host,
                                double lam, double tol, int max_iter, double* w_host,
                                int32_t* info_host, double* kkt_host) {
  return nnlasso_run(ctx, k, gram_host, b_host, lam, tol, max_iter, w_host, info_host, kkt_host,
                     false);
}

static int nnlasso_run(sfw3d_ctx* ctx, int k, const double* gram_host, const double* b_host,
                       double lam, double tol, int max_iter, double* w_host, int32_t* info_host,
                       double* kkt_host, bool qp) {
  SFW3D_CHECK_ARG(ctx && w_host, "NULL argument");
  SFW3D_CHECK_ARG(k >= 0 && (k == 0 || (gram_host && b_host)), "sizes");
  SFW3D_CHECK_ARG(lam > 0.0, "lam must be > 0");
  SFW3D_CHECK_ARG(max_iter >= 0, "max_iter must be >= 0");
  SFW3D_CHECK_ARG(k <= 6000, "k too large for the single-warp solver (<= 6000)");
  SFW3D_TRY(begin_call(ctx));
  if (k == 0) {
    if (info_host) info_host[0] = info_host[1] = 0;
    if (kkt_host) *kkt_host = 0.0;
    return SFW3D_OK;
  }
  for (int i = 0; i < k; ++i)
    SFW3D_CHECK_ARG(w_host[i] >= 0.0, "w_init must be non-negative with one entry per atom");
  const size_t kk = size_t(k) * k;
  SFW3D_TRY(ensure_device(ctx, ctx->ws_small,
                          Carver::need({kk * sizeof(double), size_t(k) * sizeof(double),
                                        size_t(k) * sizeof(double), 4 * sizeof(int), sizeof(double)})));
  Carver cv(ctx->ws_small.ptr);
  double* g = cv.take<double>(kk);
  double* bd = cv.take<double>(k);
  double* wd = cv.take<double>(k);
  int* info = cv.take<int>(4);
  double* kkt = cv.take<double>(1);
  SFW3D_TRY(stage_upload(ctx, g, gram_host, kk * sizeof(double)));
  SFW3D_TRY(stage_upload(ctx, bd, b_host, size_t(k) * sizeof(double)));
  SFW3D_TRY(stage_upload(ctx, wd, w_host, size_t(k) * sizeof(double)));
  if (qp) {
    if (k > kQpMaxFree) {
      if (info_host) info_host[0] = 0, info_host[1] = 3;  // too large: caller falls back
      return SFW3D_OK;
    }
    const size_t smem = (size_t(kQpMaxFree) * kQpMaxFree + 3 * size_t(k)) * sizeof(double) +
                        size_t(k) * sizeof(int);
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(nnqp_kernel), size_t(int(smem))));
    SFW3D_PROF(ctx, "cd");
    nnqp_kernel<<<1, kQpThreads, smem, ctx->stream>>>(k, g, bd, lam, tol, max_iter, wd, info, kkt);
    SFW3D_LAUNCH_CHECK(ctx);
  } else {
  const bool gs = (kk + 3 * size_t(k)) * sizeof(double) <= 200 * 1024;  // k <= ~158
  const size_t smem = (gs ? kk + 3 * size_t(k) : 2 * size_t(k)) * sizeof(double);
  {
    SFW3D_PROF(ctx, "cd");
    if (gs) {
      if (smem > 48 * 1024)
        SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(cd_kernel<true>), size_t(int(smem))));
      cd_kernel<true><<<1, 32, smem, ctx->stream>>>(k, g, bd, lam, tol, max_iter, wd, info, kkt);
    } else {
      if (smem > 48 * 1024)
        SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(cd_kernel<false>), size_t(int(smem))));
      cd_kernel<false><<<1, 32, smem, ctx->stream>>>(k, g, bd, lam, tol, max_iter, wd, info, kkt);
    }
    SFW3D_LAUNCH_CHECK(ctx);
  }
  }
  // results: w, info, kkt in one pinned download each
  SFW3D_TRY(download_sync(ctx, w_host, wd, size_t(k) * sizeof(double)));
  int hinfo[4];
  SFW3D_TRY(download_sync(ctx, hinfo, info, 4 * sizeof(int)));
  double hk = 0.0;
  SFW3D_TRY(download_sync(ctx, &hk, kkt, sizeof(double)));
  if (info_host) {
    info_host[0] = hinfo[0];
    info_host[1] = hinfo[1];
  }
  if (kkt_host) *kkt_host = hk;
  return SFW3D_OK;
}
