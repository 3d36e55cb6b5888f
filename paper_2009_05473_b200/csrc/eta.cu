// K1 / K2 — dual certificate eta over every voxel x (sigma, d) candidate,
// fused with the windowed argmax.
//
// Reference: build_template_table (certificate.py:65-97) stores
// rfftn(H * G_ij) per candidate and eta_field (certificate.py:140-184) runs
// one irfftn per candidate, keeps every field, and scans the window for the
// first C-order maximum; the global winner is the first candidate reaching
// the maximum (strict '>', sigma-major).
//
// Here the certificate is a DIRECT spatial correlation in factorised form
//     eta_c(m) = (1/lam) * sum_v G_c(v) * b(m + v),   b = H^T * r,
// exact by associativity (corr(r, H*G) = corr(corr(r, H), G)); the PSF
// adjoint is the separable K4 pass, applied once and shared by all
// candidates. b is copied once into a periodically padded volume so the
// correlation kernel needs no wrap logic.
//
// Direct kernel (per candidate): a CTA owns 32 (y) x 64 (z) outputs of one
// x-plane. Warp w handles z-group w (16 consecutive outputs per thread),
// lane l handles row y0+l, so a warp's shared-memory reads hit 32 different
// rows (pitch = 4 mod 32 words: conflict-free LDS.128). For every template
// x-offset a, the residual plane region (32 + template rows - 1) x pitch is
// staged in shared memory; every template row (a, b) then streams its taps
// four at a time: one LDS.128 of the sliding register window, one broadcast
// LDG.128 of taps and 64 FFMA per thread (register window rotated at compile
// time, no moves). fp32 partial sums are promoted to fp64 once per template
// slice. The argmax over the window is reduced warp -> CTA -> candidate
// with the reference's tie rule.
#include <algorithm>
#include <cstring>

#include "internal.cuh"

struct sfw3d_table;

namespace sfw3d {

struct CandHost {
  double sigma, d;
  int lo[3], hi[3];  // template offset box per axis
  int cl, lc4;       // template cols c = cl + col, col in [0, lc4)
  int la, lb;
  std::vector<int2> rows;  // per (a,b): (first step, nsteps), step = 4 cols
  long long taps;          // executed taps per output voxel
  double* t64 = nullptr;
  float* t32 = nullptr;
  int2* rows_dev = nullptr;
};

}  // namespace sfw3d

struct sfw3d_table {
  int dims[3];
  int n_sigma, n_shape;
  const sfw3d_psf* psf;
  std::vector<sfw3d::CandHost> cands;
  int pad[3];       // periodic padding (left) per axis of the padded b volume
  int pdims[3];     // padded dims
  int device;
  long long taps_per_voxel;
};

namespace sfw3d {
namespace {

constexpr int kTY = 32;              // output rows per CTA (one per lane)
constexpr int kJ = 16;               // outputs per thread along z
constexpr int kWarps = 4;            // z-groups per CTA
constexpr int kTZ = kJ * kWarps;     // 64 outputs along z per CTA
constexpr int kThreads = 32 * kWarps;

struct CandDev {
  const void* taps;   // dense [la][lb][lc4] of T
  const int2* rows;   // [la][lb]
  int lo_a, lo_b, la, lb, cl, lc4;
};

struct Geo {
  int nx, ny, nz;
  int px, py, pz;        // padding
  long long pys, pxs;    // padded strides (y, x) in elements
  int win[6];            // argmax window (inclusive)
  int ox0, oy0;          // output tile origin (x plane, y row)
  int zbase;             // first z tile origin (multiple of 4)
  int nty, ntz;          // tiles per plane
  int pitch;             // smem row pitch (elements)
  int brows;             // template rows per staged chunk
  double lam;            // eta = sum / lam (certificate.py:160)
};

struct Best {
  double v;
  long long idx;
};

__device__ __forceinline__ bool better(double v, long long i, double bv, long long bi) {
  // larger value wins; ties -> smaller C-order index (first maximum)
  return (v > bv) || (v == bv && i < bi);
}

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  using type = float4;
};
template <>
struct Vec4<double> {
  using type = double4;
};

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

// One 4-tap step with compile-time window rotation R (0..4): the window
// value at relative column u lives in buf[(4R + u) % 20].
template <typename T, int R>
__device__ __forceinline__ void tap_step(T (&acc)[kJ], T (&buf)[20], const T* trow, const T* srow) {
  T t0, t1, t2, t3;
  ldg4(trow, t0, t1, t2, t3);
#pragma unroll
  for (int j = 0; j < kJ; ++j) {
    acc[j] = fma(t0, buf[(4 * R + j + 0) % 20], acc[j]);
    acc[j] = fma(t1, buf[(4 * R + j + 1) % 20], acc[j]);
    acc[j] = fma(t2, buf[(4 * R + j + 2) % 20], acc[j]);
    acc[j] = fma(t3, buf[(4 * R + j + 3) % 20], acc[j]);
  }
  // slots of columns 0..3 are free now: load columns 20..23
  ld4(srow + 20, buf[(4 * R) % 20], buf[(4 * R + 1) % 20], buf[(4 * R + 2) % 20],
      buf[(4 * R + 3) % 20]);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) eta_direct_kernel(const T* __restrict__ bpad, Geo g,
                                                              CandDev cd, T* __restrict__ field,
                                                              Best* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* region = reinterpret_cast<T*>(smem_raw);
  __shared__ Best wbest[kWarps];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int ty = tile / g.ntz, tz = tile % g.ntz;
  const int x = g.ox0 + blockIdx.y;
  const int y0 = g.oy0 + ty * kTY;
  const int z0 = g.zbase + tz * kTZ;
  const T* taps = static_cast<const T*>(cd.taps);

  double accd[kJ];
#pragma unroll
  for (int j = 0; j < kJ; ++j) accd[j] = 0.0;

  for (int ai = 0; ai < cd.la; ++ai) {
    const int a = cd.lo_a + ai;
    const T* plane = bpad + (long long)(x + g.px + a) * g.pxs;
    for (int b0 = 0; b0 < cd.lb; b0 += g.brows) {
      const int nb = min(g.brows, cd.lb - b0);
      // skip chunks without taps (warp-uniform: every thread reads the same rows)
      bool any = false;
      for (int bi = 0; bi < nb; ++bi) any |= cd.rows[ai * cd.lb + b0 + bi].y > 0;
      if (!any) continue;
      __syncthreads();
      // stage rows y0 + lo_b + b0 .. + (kTY + nb - 1), cols z0 + cl .. + pitch
      const int nrows = kTY + nb - 1;
      const int nvec = g.pitch / 4;
      const T* src0 = plane + (long long)(y0 + g.py + cd.lo_b + b0) * g.pys + (z0 + g.pz + cd.cl);
      for (int e = threadIdx.x; e < nrows * nvec; e += kThreads) {
        const int r = e / nvec, c4 = e % nvec;
        const T* s = src0 + (long long)r * g.pys + 4 * c4;
        T* d = region + r * g.pitch + 4 * c4;
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(d) = __ldg(reinterpret_cast<const float4*>(s));
        } else {
          *reinterpret_cast<double2*>(d) = __ldg(reinterpret_cast<const double2*>(s));
          *reinterpret_cast<double2*>(d + 2) = __ldg(reinterpret_cast<const double2*>(s + 2));
        }
      }
      __syncthreads();
      T acc[kJ];
#pragma unroll
      for (int j = 0; j < kJ; ++j) acc[j] = T(0);
      for (int bi = 0; bi < nb; ++bi) {
        const int2 rr = cd.rows[ai * cd.lb + b0 + bi];
        if (rr.y <= 0) continue;
        const T* trow = taps + ((long long)ai * cd.lb + b0 + bi) * cd.lc4 + 4 * rr.x;
        const T* srow = region + (lane + bi) * g.pitch + warp * kJ + 4 * rr.x;
        T buf[20];
#pragma unroll
        for (int q = 0; q < 5; ++q) ld4(srow + 4 * q, buf[4 * q], buf[4 * q + 1], buf[4 * q + 2], buf[4 * q + 3]);
        int s = 0;
        const int ns = rr.y;
        for (; s + 5 <= ns; s += 5) {
          tap_step<T, 0>(acc, buf, trow + 4 * s, srow + 4 * s);
          tap_step<T, 1>(acc, buf, trow + 4 * s + 4, srow + 4 * s + 4);
          tap_step<T, 2>(acc, buf, trow + 4 * s + 8, srow + 4 * s + 8);
          tap_step<T, 3>(acc, buf, trow + 4 * s + 12, srow + 4 * s + 12);
          tap_step<T, 4>(acc, buf, trow + 4 * s + 16, srow + 4 * s + 16);
        }
        const int rem = ns - s;
        if (rem > 0) tap_step<T, 0>(acc, buf, trow + 4 * s, srow + 4 * s);
        if (rem > 1) tap_step<T, 1>(acc, buf, trow + 4 * s + 4, srow + 4 * s + 4);
        if (rem > 2) tap_step<T, 2>(acc, buf, trow + 4 * s + 8, srow + 4 * s + 8);
        if (rem > 3) tap_step<T, 3>(acc, buf, trow + 4 * s + 12, srow + 4 * s + 12);
      }
#pragma unroll
      for (int j = 0; j < kJ; ++j) accd[j] += double(acc[j]);
    }
  }

  // epilogue: eta = acc / lam, optional field store, windowed argmax
  const int y = y0 + lane;
  Best best{-INFINITY, 0x7fffffffffffffffLL};
  const bool row_ok = y < g.ny;
  const bool row_win = x >= g.win[0] && x <= g.win[1] && y >= g.win[2] && y <= g.win[3];
#pragma unroll
  for (int j = 0; j < kJ; ++j) {
    const int z = z0 + warp * kJ + j;
    if (!row_ok || z >= g.nz) continue;
    const double eta = accd[j] / g.lam;
    const long long lin = ((long long)x * g.ny + y) * g.nz + z;
    if (field) field[lin] = T(eta);
    if (row_win && z >= g.win[4] && z <= g.win[5] && better(eta, lin, best.v, best.idx))
      best = {eta, lin};
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best.v, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, best.idx, o);
    if (better(ov, oi, best.v, best.idx)) best = {ov, oi};
  }
  if (lane == 0) wbest[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best b = wbest[0];
    for (int w = 1; w < kWarps; ++w)
      if (better(wbest[w].v, wbest[w].idx, b.v, b.idx)) b = wbest[w];
    partial[(long long)blockIdx.y * gridDim.x + blockIdx.x] = b;
  }
}

// periodic padding: dst[X][Y][Z] = src[(X-px) mod nx][(Y-py) mod ny][(Z-pz) mod nz]
template <typename T>
__global__ void pad_kernel(const T* __restrict__ src, T* __restrict__ dst, int nx, int ny, int nz,
                           int px, int py, int pz, int PX, int PY, int PZ) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)PX * PY * PZ;
  if (t >= n) return;
  const int Z = int(t % PZ);
  const int Y = int((t / PZ) % PY);
  const int X = int(t / ((long long)PZ * PY));
  int x = (X - px) % nx; if (x < 0) x += nx;
  int y = (Y - py) % ny; if (y < 0) y += ny;
  int z = (Z - pz) % nz; if (z < 0) z += nz;
  dst[t] = src[((long long)x * ny + y) * nz + z];
}

__global__ void best_reduce_kernel(const Best* __restrict__ partial, long long n, Best* __restrict__ out) {
  __shared__ Best sb[32];
  Best b{-INFINITY, 0x7fffffffffffffffLL};
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const Best p = partial[i];
    if (better(p.v, p.idx, b.v, b.idx)) b = p;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, b.v, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, b.idx, o);
    if (better(ov, oi, b.v, b.idx)) b = {ov, oi};
  }
  if (lane == 0) sb[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best r = sb[0];
    for (int w = 1; w < (int)(blockDim.x / 32); ++w)
      if (better(sb[w].v, sb[w].idx, r.v, r.idx)) r = sb[w];
    *out = r;
  }
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// smem row pitch: >= cols needed, and == 4 (mod 32) elements for fp32
// (conflict-free LDS.128 across 8 consecutive rows); fp64 uses == 2 (mod 16).
int region_pitch(int lc4, int esize) {
  int need = lc4 + kTZ + 8;
  int p = round_up(need, 4);
  if (esize == 4) {
    while (p % 32 != 4) p += 4;
  } else {
    while (p % 16 != 4) p += 4;
  }
  return p;
}

}  // namespace

// ------------------------------------------------------------------ table
static int build_candidate(const int dims[3], double sigma, double d, double tap_tol, CandHost& c) {
  c.sigma = sigma;
  c.d = d;
  const double rr = std::ceil(sigma * std::pow(kTailExponent, 1.0 / d));
  const int R = int(rr);
  for (int a = 0; a < 3; ++a) {
    if (2LL * R + 1 >= dims[a]) {
      c.lo[a] = -(dims[a] / 2);
      c.hi[a] = c.lo[a] + dims[a] - 1;
    } else {
      c.lo[a] = -R;
      c.hi[a] = R;
    }
  }
  c.la = c.hi[0] - c.lo[0] + 1;
  c.lb = c.hi[1] - c.lo[1] + 1;
  c.cl = -round_up(-c.lo[2], 4);  // lo[2] rounded down to a multiple of 4
  c.lc4 = round_up(c.hi[2] - c.cl + 1, 4) + 4;
  const double inv2sd = 0.5 / std::pow(sigma, d);
  const double half_d = 0.5 * d;
  const bool d2 = d == 2.0;
  c.rows.assign(size_t(c.la) * c.lb, make_int2(0, 0));
  std::vector<double> t(size_t(c.la) * c.lb * c.lc4, 0.0);
  c.taps = 0;
  for (int ai = 0; ai < c.la; ++ai) {
    const double a = c.lo[0] + ai;
    for (int bi = 0; bi < c.lb; ++bi) {
      const double b = c.lo[1] + bi;
      int cmin = 1 << 30, cmax = -(1 << 30);
      double* row = &t[(size_t(ai) * c.lb + bi) * c.lc4];
      for (int cc = c.lo[2]; cc <= c.hi[2]; ++cc) {
        const double u2 = (a * a + b * b) + double(cc) * cc;
        const double tt = inv2sd * (d2 ? u2 : std::pow(u2, half_d));
        const double v = std::exp(-tt);
        row[cc - c.cl] = v;
        if (tap_tol <= 0.0 || v >= tap_tol) {
          cmin = std::min(cmin, cc);
          cmax = std::max(cmax, cc);
        }
      }
      if (cmax >= cmin) {
        const int s0 = (cmin - c.cl) / 4, s1 = (cmax - c.cl) / 4;
        c.rows[size_t(ai) * c.lb + bi] = make_int2(s0, s1 - s0 + 1);
        c.taps += 4LL * (s1 - s0 + 1);
      }
    }
  }
  cudaError_t e = cudaMalloc(&c.t64, t.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c.t32, t.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&c.rows_dev, c.rows.size() * sizeof(int2));
  if (e != cudaSuccess) {
    set_error(std::string("CUDA error ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SFW3D_ENOMEM : SFW3D_ECUDA;
  }
  std::vector<float> t32(t.begin(), t.end());
  SFW3D_CUDA_TRY(cudaMemcpy(c.t64, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice));
  SFW3D_CUDA_TRY(cudaMemcpy(c.t32, t32.data(), t32.size() * sizeof(float), cudaMemcpyHostToDevice));
  SFW3D_CUDA_TRY(cudaMemcpy(c.rows_dev, c.rows.data(), c.rows.size() * sizeof(int2), cudaMemcpyHostToDevice));
  return SFW3D_OK;
}

}  // namespace sfw3d

using namespace sfw3d;

extern "C" int sfw3d_table_destroy(sfw3d_table* t) {
  if (!t) return SFW3D_OK;
  cudaSetDevice(t->device);
  for (auto& c : t->cands) {
    if (c.t64) cudaFree(c.t64);
    if (c.t32) cudaFree(c.t32);
    if (c.rows_dev) cudaFree(c.rows_dev);
  }
  delete t;
  return SFW3D_OK;
}

extern "C" int sfw3d_table_create(sfw3d_ctx* ctx, const sfw3d_psf* psf, int n_sigma,
                                  const double* sigma_host, int n_shape, const double* shape_host,
                                  double tap_tol, int mode, double basis_tol, sfw3d_table** out) {
  (void)basis_tol;
  SFW3D_CHECK_ARG(ctx && psf && out, "NULL argument");
  SFW3D_CHECK_ARG(n_sigma > 0 && n_shape > 0 && sigma_host && shape_host,
                  "parameter grids must be non-empty");
  SFW3D_CHECK_ARG(mode == 0 || mode == 1, "mode");
  SFW3D_TRY(begin_call(ctx));
  *out = nullptr;
  std::vector<double> sg(sigma_host, sigma_host + n_sigma), dg(shape_host, shape_host + n_shape);
  for (double v : sg) SFW3D_CHECK_ARG(std::isfinite(v) && v > 0.0, "sigma grid values must be > 0");
  for (double v : dg) SFW3D_CHECK_ARG(std::isfinite(v) && v > 0.0, "shape grid values must be > 0");
  std::sort(sg.begin(), sg.end());
  std::sort(dg.begin(), dg.end());
  auto* t = new sfw3d_table();
  for (int a = 0; a < 3; ++a) t->dims[a] = psf->dims[a];
  t->n_sigma = n_sigma;
  t->n_shape = n_shape;
  t->psf = psf;
  t->device = ctx->device;
  t->cands.resize(size_t(n_sigma) * n_shape);
  t->taps_per_voxel = 0;
  int maxlo[3] = {0, 0, 0}, maxhi[3] = {0, 0, 0}, maxpitch = 0;
  for (int i = 0; i < n_sigma; ++i)
    for (int j = 0; j < n_shape; ++j) {
      CandHost& c = t->cands[size_t(i) * n_shape + j];
      int s = build_candidate(t->dims, sg[i], dg[j], tap_tol, c);
      if (s != SFW3D_OK) {
        sfw3d_table_destroy(t);
        return s;
      }
      t->taps_per_voxel += c.taps;
      maxlo[0] = std::max(maxlo[0], -c.lo[0]);
      maxhi[0] = std::max(maxhi[0], c.hi[0]);
      maxlo[1] = std::max(maxlo[1], -c.lo[1]);
      maxhi[1] = std::max(maxhi[1], c.hi[1]);
      maxlo[2] = std::max(maxlo[2], -c.cl);
      maxpitch = std::max(maxpitch, std::max(region_pitch(c.lc4, 8), region_pitch(c.lc4, 4)));
    }
  // padded b: x/y pads cover the template offsets (+ the last partial tile
  // in y), z covers the aligned template start and the widest staged row.
  t->pad[0] = maxlo[0];
  t->pad[1] = maxlo[1];
  t->pad[2] = round_up(maxlo[2], 4);
  t->pdims[0] = t->pad[0] + t->dims[0] + maxhi[0];
  t->pdims[1] = t->pad[1] + round_up(t->dims[1], kTY) + maxhi[1] + kTY;
  t->pdims[2] = round_up(t->pad[2] + round_up(t->dims[2], kTZ) + 4 + maxpitch, 4);
  *out = t;
  return SFW3D_OK;
}

extern "C" int sfw3d_table_info(const sfw3d_table* t, int* n_cand, int* n_direct, int* n_basis,
                                int64_t* taps_per_voxel) {
  SFW3D_CHECK_ARG(t, "table is NULL");
  if (n_cand) *n_cand = int(t->cands.size());
  if (n_direct) *n_direct = int(t->cands.size());
  if (n_basis) *n_basis = 0;
  if (taps_per_voxel) *taps_per_voxel = t->taps_per_voxel;
  return SFW3D_OK;
}

namespace {

template <typename T>
int eta_typed(sfw3d_ctx* ctx, const sfw3d_table* t, const void* residual, double lam,
              const int32_t win_in[6], sfw3d_argmax* best_host, sfw3d_argmax* per_cand_host,
              void* fields) {
  const int* dims = t->dims;
  const int64_t n = vol_count(dims);
  const size_t vb = size_t(n) * sizeof(T);
  const size_t pb = size_t(t->pdims[0]) * t->pdims[1] * t->pdims[2] * sizeof(T);
  const int nc = int(t->cands.size());
  // output tiles: the window, or the whole grid when fields are requested
  int win[6];
  for (int a = 0; a < 6; ++a) win[a] = win_in[a];
  int ow[6];
  if (fields) {
    ow[0] = 0; ow[1] = dims[0] - 1; ow[2] = 0; ow[3] = dims[1] - 1; ow[4] = 0; ow[5] = dims[2] - 1;
  } else {
    for (int a = 0; a < 6; ++a) ow[a] = win[a];
  }
  const int zbase = (ow[4] / 4) * 4;
  const int nty = (ow[3] - ow[2] + 1 + kTY - 1) / kTY;
  const int ntz = (ow[5] - zbase + 1 + kTZ - 1) / kTZ;
  const int nxp = ow[1] - ow[0] + 1;
  const long long nblocks = (long long)nty * ntz * nxp;
  SFW3D_TRY(ensure_device(ctx, ctx->ws, Carver::need({vb, vb, pb, size_t(nblocks) * sizeof(Best),
                                                      size_t(nc) * sizeof(Best)})));
  Carver cv(ctx->ws.ptr);
  T* b = cv.take<T>(n);
  T* tmp = cv.take<T>(n);
  T* bpad = cv.take<T>(size_t(pb / sizeof(T)));
  Best* partial = cv.take<Best>(nblocks);
  Best* cbest = cv.take<Best>(nc);
  // b = H^T * r, then periodic padding
  SFW3D_TRY(psf_apply_impl(ctx, t->psf, sizeof(T) == 8 ? SFW3D_F64 : SFW3D_F32, residual, b, 1, tmp));
  const long long np = (long long)t->pdims[0] * t->pdims[1] * t->pdims[2];
  {
    SFW3D_PROF(ctx, "pad");
    pad_kernel<T><<<unsigned((np + 255) / 256), 256, 0, ctx->stream>>>(
        b, bpad, dims[0], dims[1], dims[2], t->pad[0], t->pad[1], t->pad[2], t->pdims[0],
        t->pdims[1], t->pdims[2]);
    SFW3D_LAUNCH_CHECK(ctx);
  }

  Geo g;
  g.nx = dims[0]; g.ny = dims[1]; g.nz = dims[2];
  g.px = t->pad[0]; g.py = t->pad[1]; g.pz = t->pad[2];
  g.pys = t->pdims[2];
  g.pxs = (long long)t->pdims[1] * t->pdims[2];
  for (int a = 0; a < 6; ++a) g.win[a] = win[a];
  g.ox0 = ow[0];
  g.oy0 = ow[2];
  g.zbase = zbase;
  g.nty = nty;
  g.ntz = ntz;
  g.lam = lam;
  int smem_max = 0;
  SFW3D_CUDA_TRY(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int budget = std::min(smem_max - 2048, 110 * 1024);
  for (int ci = 0; ci < nc; ++ci) {
    const CandHost& c = t->cands[ci];
    CandDev cd;
    cd.taps = sizeof(T) == 8 ? static_cast<const void*>(c.t64) : static_cast<const void*>(c.t32);
    cd.rows = c.rows_dev;
    cd.lo_a = c.lo[0];
    cd.lo_b = c.lo[1];
    cd.la = c.la;
    cd.lb = c.lb;
    cd.cl = c.cl;
    cd.lc4 = c.lc4;
    Geo gc = g;
    gc.pitch = region_pitch(c.lc4, sizeof(T));
    const int row_bytes = gc.pitch * int(sizeof(T));
    const int brows = budget / row_bytes - (kTY - 1);
    if (brows < 1) {
      set_error("certificate template too wide for the shared-memory tile");
      return SFW3D_EINVAL;
    }
    gc.brows = std::min(brows, c.lb);
    const int smem = (kTY + gc.brows - 1) * row_bytes;
    SFW3D_CUDA_TRY(cudaFuncSetAttribute(eta_direct_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid(unsigned(nty * ntz), unsigned(nxp));
    T* fld = fields ? static_cast<T*>(fields) + size_t(ci) * n : nullptr;
    {
      SFW3D_PROF(ctx, "eta_direct");
      eta_direct_kernel<T><<<grid, kThreads, smem, ctx->stream>>>(bpad, gc, cd, fld, partial);
      SFW3D_LAUNCH_CHECK(ctx);
    }
    {
      SFW3D_PROF(ctx, "argmax");
      best_reduce_kernel<<<1, 1024, 0, ctx->stream>>>(partial, nblocks, cbest + ci);
      SFW3D_LAUNCH_CHECK(ctx);
    }
  }
  std::vector<Best> hb(nc);
  SFW3D_TRY(download_sync(ctx, hb.data(), cbest, size_t(nc) * sizeof(Best)));
  int bi = 0;
  double bv = -INFINITY;
  for (int ci = 0; ci < nc; ++ci) {
    if (hb[ci].v > bv) {  // strict '>' over sigma-major candidates (certificate.py:168-172)
      bv = hb[ci].v;
      bi = ci;
    }
  }
  auto rec = [&](int ci) {
    sfw3d_argmax r;
    const long long lin = hb[ci].idx;
    r.pos[2] = int(lin % dims[2]);
    r.pos[1] = int((lin / dims[2]) % dims[1]);
    r.pos[0] = int(lin / ((long long)dims[1] * dims[2]));
    r.cand = ci;
    r.value = hb[ci].v;
    return r;
  };
  if (best_host) *best_host = rec(bi);
  if (per_cand_host)
    for (int ci = 0; ci < nc; ++ci) per_cand_host[ci] = rec(ci);
  if (!std::isfinite(bv)) {
    set_error("non-finite certificate value");
    return SFW3D_ENONFINITE;
  }
  return SFW3D_OK;
}

}  // namespace

extern "C" int sfw3d_eta_argmax(sfw3d_ctx* ctx, const sfw3d_table* t, int dtype,
                                const void* residual_dev, double lam, const int32_t window[6],
                                sfw3d_argmax* best_host, sfw3d_argmax* per_cand_host, void* fields_dev) {
  SFW3D_CHECK_ARG(ctx && t && residual_dev && window, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(lam > 0.0, "lam must be > 0");
  for (int a = 0; a < 3; ++a)
    SFW3D_CHECK_ARG(0 <= window[2 * a] && window[2 * a] <= window[2 * a + 1] &&
                        window[2 * a + 1] < t->dims[a],
                    "window must be a non-empty box inside the grid");
  SFW3D_TRY(begin_call(ctx));
  if (dtype == SFW3D_F64)
    return eta_typed<double>(ctx, t, residual_dev, lam, window, best_host, per_cand_host, fields_dev);
  return eta_typed<float>(ctx, t, residual_dev, lam, window, best_host, per_cand_host, fields_dev);
}
