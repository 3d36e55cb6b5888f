// K1 / K2 — dual certificate eta over every voxel x (sigma, d) candidate,
// fused with the windowed argmax.
//
// Reference: build_template_table (certificate.py:65-97) stores
// rfftn(H * G_ij) per candidate; eta_field (certificate.py:140-184) runs one
// irfftn per candidate, keeps every field, and scans the window for the
// first C-order maximum; the global winner is the first candidate reaching
// the maximum (strict '>', sigma-major).
//
// Here eta is evaluated in the spatial domain in factorised form
//     eta_c(m) = (1/lam) * sum_v G_c(v) * b(m + v),   b = H^T * r,
// exact by associativity (corr(r, H*G) = corr(corr(r, H), G)); b is one
// separable K4 pass shared by all candidates. Evaluators per candidate:
//
//  FOLDED DIRECT (eta_fold_kernel) — symmetric boxes: the radial atom's rows
//   (x +- a, y +- b) share one tap row; per a the CTA stages the summed plane
//   P(x+a) + P(x-a), per b each thread sums rows y +- b and correlates with
//   the tap row through a compile-time-rotated register window (window.cuh).
//  DIRECT (eta_direct_kernel) — any box (full-axis, asymmetric offsets).
//  SHARED BASIS (basis.cu) — d <= 2 candidates as positive Gaussian
//   mixtures on one dictionary shared by the table: separable passes once
//   per shared term, one fused mix + argmax kernel for all members.
//  EXACT REFINEMENT (refine_kernel) — fp64 storage, inexact members: the
//   voxels within 2 E_c of the member's approximate maximum are re-evaluated
//   with the direct taps, so maxima / argmaxima are the direct ones.
#include <algorithm>
#include <mutex>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <string>
#include <utility>

#include "basis.cuh"
#include "window.cuh"

namespace sfw3d {

struct CandHost {
  double sigma, d;
  int lo[3], hi[3];  // template offset box per axis
  // direct
  int cl, lc4;       // template cols c = cl + col, col in [0, lc4)
  int la, lb;
  std::vector<int2> rows;  // per (a,b): (first step, nsteps), step = 4 cols
  long long taps = 0;      // executed direct taps per output voxel
  double* t64 = nullptr;
  float* t32 = nullptr;
  int2* rows_dev = nullptr;
  double fold_flops[2] = {0.0, 0.0};  // flops per voxel of the folded kernel (f32, f64)
};

}  // namespace sfw3d

struct sfw3d_table {
  int dims[3];
  int n_sigma, n_shape;
  const sfw3d_psf* psf;
  std::vector<sfw3d::CandHost> cands;
  int pad[3];    // periodic padding (left) per axis of the padded b volume
  int pdims[3];  // padded dims
  int device;
  int mode;      // 0 auto, 1 direct only
  double basis_tol;
  // sfw3d_table_set_option: basis term pruning (-1 = by volume size), fp32
  // shared-term selection tolerance (< 0 = default), refinement item cap
  int prune = -1;
  long long global_voxels = 0;  // > 0: the pruning rule's voxel count (sharded tables)
  double loose_tol = -1.0;
  int refine_cap = 1 << 16;
  int smem_max;  // opt-in shared memory per block of the device
  // shared separable bases (basis.cu), one per storage precision, fitted on
  // first use of that precision (a solve only ever touches one)
  std::vector<sfw3d::BasisCandidate> bcands;
  mutable sfw3d::BasisSet* set32 = nullptr;
  mutable sfw3d::BasisSet* set64 = nullptr;
  void* refcand_dev = nullptr;  // RefCand per candidate (fp64 exact refinement)
  const sfw3d::BasisSet* set(int dtype) const { return dtype == SFW3D_F64 ? set64 : set32; }
};

namespace sfw3d {
namespace {

constexpr int kTY = 32;           // output rows per CTA (one per lane)
constexpr int kJ = 16;            // outputs per thread along z
constexpr int kWarps = 4;         // z-groups per CTA
constexpr int kTZ = kJ * kWarps;  // 64 outputs along z per CTA
constexpr int kThreads = 32 * kWarps;
// folded kernel: outputs per thread along z (fp32 / fp64) and the widest tile
template <typename T>
constexpr int fold_kj() { return sizeof(T) == 4 ? 32 : 16; }
constexpr int kFoldTZMax = 32 * kWarps;

struct CandDev {
  const void* taps;  // dense [la][lb][lc4] of T
  const int2* rows;  // [la][lb]
  int lo_a, lo_b, la, lb, cl, lc4;
};

struct Geo {
  int nx, ny, nz;
  int px, py, pz;      // padding
  long long pys, pxs;  // padded strides (y, x) in elements
  int win[6];          // argmax window (inclusive)
  int ox0, oy0;        // output tile origin (x plane, y row)
  int zbase;           // first z tile origin (multiple of 4)
  int nty, ntz;        // tiles per plane
  int pitch;           // smem row pitch (elements)
  int brows;           // template rows per staged chunk
  double lam;          // eta = sum / lam (certificate.py:160)
  void* accd_g;        // folded kernel: slice sums in global scratch (or NULL: smem)
};

// One 4-tap step with compile-time window rotation R (0..4): the window
// value at relative column u lives in buf[(4R + u) % 20].
// `tc` holds this step's 4 taps; the next step's taps are fetched from
// `tnext` before the FFMAs so the L1 latency is hidden behind them.
template <typename T, int R>
__device__ __forceinline__ void tap_step(T (&acc)[kJ], T (&buf)[20], T (&tc)[4], const T* tnext,
                                         const T* srow) {
  T n0, n1, n2, n3;
  ldg4(tnext, n0, n1, n2, n3);
#pragma unroll
  for (int j = 0; j < kJ; ++j) {
    acc[j] = fma(tc[0], buf[(4 * R + j + 0) % 20], acc[j]);
    acc[j] = fma(tc[1], buf[(4 * R + j + 1) % 20], acc[j]);
    acc[j] = fma(tc[2], buf[(4 * R + j + 2) % 20], acc[j]);
    acc[j] = fma(tc[3], buf[(4 * R + j + 3) % 20], acc[j]);
  }
  // slots of columns 0..3 are free now: load columns 20..23
  ld4(srow + 20, buf[(4 * R) % 20], buf[(4 * R + 1) % 20], buf[(4 * R + 2) % 20],
      buf[(4 * R + 3) % 20]);
  tc[0] = n0;
  tc[1] = n1;
  tc[2] = n2;
  tc[3] = n3;
}

template <typename T>
__device__ __forceinline__ void reduce_store_best(Best best, Best* wbest, Best* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
    for (int w = 1; w < int(blockDim.x / 32); ++w)
      if (better(wbest[w].v, wbest[w].idx, b.v, b.idx)) b = wbest[w];
    *out = b;
  }
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

  T accd[kJ];  // slice partials summed in the storage precision (fp32 error << 1e-5 bar)
#pragma unroll
  for (int j = 0; j < kJ; ++j) accd[j] = T(0);

  for (int ai = 0; ai < cd.la; ++ai) {
    const int a = cd.lo_a + ai;
    const T* plane = bpad + (long long)(x + g.px + a) * g.pxs;
    for (int b0 = 0; b0 < cd.lb; b0 += g.brows) {
      const int nb = min(g.brows, cd.lb - b0);
      bool any = false;  // chunk without taps: skip (uniform over the CTA)
      for (int bi = 0; bi < nb; ++bi) any |= cd.rows[ai * cd.lb + b0 + bi].y > 0;
      if (!any) continue;
      __syncthreads();
      const int nrows = kTY + nb - 1;
      const int nvec = g.pitch / 4;
      const T* src0 = plane + (long long)(y0 + g.py + cd.lo_b + b0) * g.pys + (z0 + g.pz + cd.cl);
      for (int e = threadIdx.x; e < nrows * nvec; e += kThreads) {
        const int r = e / nvec, c4 = e % nvec;
        const T* s = src0 + (long long)r * g.pys + 4 * c4;
        T* d = region + r * g.pitch + 4 * c4;
        cp_async16(d, s);
        if constexpr (sizeof(T) == 8) cp_async16(d + 2, s + 2);
      }
      cp_async_wait_all();
      __syncthreads();
      T acc[kJ];
#pragma unroll
      for (int j = 0; j < kJ; ++j) acc[j] = T(0);
      // software pipeline over template rows: the next row's extent and its
      // first 4 taps are fetched while the current row computes
      const T* trow_base = taps + ((long long)ai * cd.lb + b0) * cd.lc4;
      int2 rr_next = cd.rows[ai * cd.lb + b0];
      T tn[4];
      ldg4(trow_base + 4 * max(rr_next.x, 0), tn[0], tn[1], tn[2], tn[3]);
      for (int bi = 0; bi < nb; ++bi) {
        const int2 rr = rr_next;
        T tc[4] = {tn[0], tn[1], tn[2], tn[3]};
        if (bi + 1 < nb) {
          rr_next = cd.rows[ai * cd.lb + b0 + bi + 1];
          ldg4(trow_base + (long long)(bi + 1) * cd.lc4 + 4 * max(rr_next.x, 0), tn[0], tn[1], tn[2],
               tn[3]);
        }
        if (rr.y <= 0) continue;
        const T* trow = trow_base + (long long)bi * cd.lc4 + 4 * rr.x;
        const T* srow = region + (lane + bi) * g.pitch + warp * kJ + 4 * rr.x;
        T buf[20];
#pragma unroll
        for (int q = 0; q < 5; ++q)
          ld4(srow + 4 * q, buf[4 * q], buf[4 * q + 1], buf[4 * q + 2], buf[4 * q + 3]);
        int s = 0;
        const int ns = rr.y;
        for (; s + 5 <= ns; s += 5) {
          tap_step<T, 0>(acc, buf, tc, trow + 4 * s + 4, srow + 4 * s);
          tap_step<T, 1>(acc, buf, tc, trow + 4 * s + 8, srow + 4 * s + 4);
          tap_step<T, 2>(acc, buf, tc, trow + 4 * s + 12, srow + 4 * s + 8);
          tap_step<T, 3>(acc, buf, tc, trow + 4 * s + 16, srow + 4 * s + 12);
          tap_step<T, 4>(acc, buf, tc, trow + 4 * s + 20, srow + 4 * s + 16);
        }
        const int rem = ns - s;
        if (rem > 0) tap_step<T, 0>(acc, buf, tc, trow + 4 * s + 4, srow + 4 * s);
        if (rem > 1) tap_step<T, 1>(acc, buf, tc, trow + 4 * s + 8, srow + 4 * s + 4);
        if (rem > 2) tap_step<T, 2>(acc, buf, tc, trow + 4 * s + 12, srow + 4 * s + 8);
        if (rem > 3) tap_step<T, 3>(acc, buf, tc, trow + 4 * s + 16, srow + 4 * s + 12);
      }
#pragma unroll
      for (int j = 0; j < kJ; ++j) accd[j] += acc[j];
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
    const double eta = double(accd[j]) / g.lam;
    const long long lin = ((long long)x * g.ny + y) * g.nz + z;
    if (field) field[lin] = T(eta);
    if (row_win && z >= g.win[4] && z <= g.win[5] && better(eta, lin, best.v, best.idx))
      best = {eta, lin};
  }
  reduce_store_best<T>(best, wbest, partial + (long long)blockIdx.y * gridDim.x + blockIdx.x);
}

// ---------------------------------------------------------- direct, folded
// The unit atom is radial: G(a, b, c) = G(+-a, +-b, c). For a box symmetric
// on axes 0 and 1 the four rows (x +- a, y +- b) share one tap row. A CTA owns
// 32 (y) x 4 KJ (z) outputs of one x-plane; per template x-offset a >= 0 it
// stages the SUMMED plane S_a = P(x + a) + P(x - a) once (one smem plane,
// one FADD per staged element), and per b >= 0 the thread sums the rows
// y + b and y - b of S_a (NR = 2) and correlates them with the tap row:
// ~4x fewer FFMA than the unfolded kernel, one LDS.128 + 4 FADD per 4 KJ
// FFMA. lane = output row (pitch = 4 mod 8 words: conflict-free LDS.128);
// each thread slides a (KJ + 4)-register window along z, 4 taps per step:
//   sum the NR rows' next 4 columns (loaded one step earlier) into the slots
//   freed by the previous step, issue the loads for the following step and
//   the next 4 taps, then 4 KJ FFMA (tap-major, KJ independent chains).
// The window rotation is resolved at compile time (no register moves).
// Per-slice fp32 partials are added into a shared-memory accumulator.
// 16-byte vector of 4 fp32 / 2 fp64 (global read-only load, shared store)
template <typename T>
struct V16 {
  using type = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
};
template <typename T>
__device__ __forceinline__ typename V16<T>::type vadd(typename V16<T>::type a,
                                                      typename V16<T>::type b) {
  if constexpr (sizeof(T) == 4)
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  else
    return make_double2(a.x + b.x, a.y + b.y);
}

// S = P(x + a) [+ P(x - a)]: nrows x pitch elements of two padded planes into
// one smem plane. Lanes run over the 16-byte vectors of a row, warps over
// rows; 4 rows per thread in flight.
template <typename T, int NT>
__device__ __forceinline__ void stage_sum(T* __restrict__ S, const T* __restrict__ sp,
                                          const T* __restrict__ sm, int nrows, int pitch,
                                          long long pys) {
  using V = typename V16<T>::type;
  constexpr int kE = 16 / sizeof(T);  // elements per vector
  constexpr int NW = NT / 32;
  const int nvec = pitch / kE;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int v = lane; v < nvec; v += 32) {
    const T* gp = sp + kE * v;
    const T* gm = sm ? sm + kE * v : nullptr;
    T* d = S + kE * v;
#pragma unroll 4
    for (int r = wid; r < nrows; r += NW) {
      const V x = __ldg(reinterpret_cast<const V*>(gp + (long long)r * pys));
      *reinterpret_cast<V*>(d + r * pitch) =
          gm ? vadd<T>(x, __ldg(reinterpret_cast<const V*>(gm + (long long)r * pys))) : x;
    }
  }
}

// resident CTAs per SM the register budget is sized for (fp32 tiles)
template <typename T, int KJ, int NWY, bool AG>
constexpr int fold_min_blocks() {
  return sizeof(T) == 8 ? 1 : (NWY == 2 ? 2 : (KJ == 32 ? (AG ? 4 : 3) : 4));
}

// AG: slice sums in a global scratch slab per CTA instead of shared memory
template <typename T, int KJ, int NWY, bool AG = false>
__global__ void __launch_bounds__(kThreads * NWY, (fold_min_blocks<T, KJ, NWY, AG>())) eta_fold_kernel(const T* __restrict__ bpad, Geo g,
                                                                  CandDev cd, T* __restrict__ field,
                                                                  Best* __restrict__ partial) {
  constexpr int NT = kThreads * NWY, TY = kTY * NWY, TZ = KJ * kWarps;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Best wbest[kWarps * NWY];
  const int nrows = TY + cd.lb - 1;  // rows of the staged plane (whole b range)
  T* accd = AG ? static_cast<T*>(g.accd_g) + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * KJ * NT
               : reinterpret_cast<T*>(smem_raw);  // [KJ][NT] slice sums
  T* stap = AG ? reinterpret_cast<T*>(smem_raw) : accd + KJ * NT;  // [Rb + 1][lc4] tap rows b >= 0 (+8)
  const int ntap = (cd.lb / 2 + 1) * cd.lc4;
  int2* srows = reinterpret_cast<int2*>(stap + ((ntap + 8 + 3) & ~3));  // [Rb + 1] (+pad)
  T* plane = reinterpret_cast<T*>(srows + ((cd.lb / 2 + 1 + 1) & ~1));
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) % kWarps;
  const int ylane = (threadIdx.x >> 5) / kWarps * kTY + lane;  // output row in the tile
  const int ty = blockIdx.x / g.ntz, tz = blockIdx.x % g.ntz;
  const int x = g.ox0 + blockIdx.y;
  const int y0 = g.oy0 + ty * TY;
  const int z0 = g.zbase + tz * TZ;
  const T* taps = static_cast<const T*>(cd.taps);
  const int Ra = cd.la / 2, Rb = cd.lb / 2;  // symmetric boxes: lo = -R
#pragma unroll
  for (int j = 0; j < KJ; ++j) accd[j * NT + threadIdx.x] = T(0);
  const long long corner = (long long)(y0 + g.py + cd.lo_b) * g.pys + (z0 + g.pz + cd.cl);

  for (int a = 0; a <= Ra; ++a) {
    const int ai = a + Ra;  // template slice index of +a (same taps as -a)
    __syncthreads();        // previous slice fully consumed
    // this slice's tap rows b >= 0 and their (first step, nsteps) extents
    {
      const T* tsrc = taps + ((long long)ai * cd.lb + Rb) * cd.lc4;
      for (int e = threadIdx.x; e < ntap + 8; e += NT) stap[e] = e < ntap ? tsrc[e] : T(0);
      for (int e = threadIdx.x; e <= Rb; e += NT) srows[e] = cd.rows[ai * cd.lb + Rb + e];
    }
    __syncthreads();
    bool any = false;
    for (int b = 0; b <= Rb; ++b) any |= srows[b].y > 0;
    if (!any) continue;  // (uniform over the CTA)
    stage_sum<T, NT>(plane, bpad + (long long)(x + g.px + a) * g.pxs + corner,
                     a ? bpad + (long long)(x + g.px - a) * g.pxs + corner : nullptr, nrows,
                     g.pitch, g.pys);
    __syncthreads();
    T acc[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) acc[j] = T(0);
    for (int b = 0; b <= Rb; ++b) {
      const int2 rr = srows[b];
      if (rr.y <= 0) continue;
      const T* trow = stap + b * cd.lc4 + 4 * rr.x;
      const int c0 = warp * KJ + 4 * rr.x;
      const T* pp = plane + (ylane + Rb + b) * g.pitch + c0;
      if (b == 0) {
        const T* const q[1] = {pp};
        Fold<T, KJ, 1>::row(acc, trow, q, rr.y);
      } else {
        const T* const q[2] = {pp, plane + (ylane + Rb - b) * g.pitch + c0};
        Fold<T, KJ, 2>::row(acc, trow, q, rr.y);
      }
    }
#pragma unroll
    for (int j = 0; j < KJ; ++j) accd[j * NT + threadIdx.x] += acc[j];
  }

  const int y = y0 + ylane;
  Best best{-INFINITY, 0x7fffffffffffffffLL};
  const bool row_ok = y < g.ny;
  const bool row_win = x >= g.win[0] && x <= g.win[1] && y >= g.win[2] && y <= g.win[3];
#pragma unroll
  for (int j = 0; j < KJ; ++j) {
    const int z = z0 + warp * KJ + j;
    if (!row_ok || z >= g.nz) continue;
    const double eta = double(accd[j * NT + threadIdx.x]) / g.lam;
    const long long lin = ((long long)x * g.ny + y) * g.nz + z;
    if (field) field[lin] = T(eta);
    if (row_win && z >= g.win[4] && z <= g.win[5] && better(eta, lin, best.v, best.idx))
      best = {eta, lin};
  }
  reduce_store_best<T>(best, wbest, partial + (long long)blockIdx.y * gridDim.x + blockIdx.x);
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
  reduce_store_best<double>(b, sb, out);
}

// ---------------------------------------------------------- exact refinement
// fp64 basis members are approximate (fit error e_c per tap); the voxels
// whose approximate eta is within 2 E_c of the member's approximate maximum
// (E_c = (e_c + 2e-12) ||b||_1 / lam bounds |eta~ - eta| everywhere) are
// re-evaluated exactly here, with the candidate's direct taps on the
// reference box, so the reported maxima and argmaxima are the direct ones.
struct RefCand {
  const double* taps;  // dense [la][lb][lc4]
  const int2* rows;    // [la][lb] (first step, nsteps), step = 4 columns
  int lo_a, lo_b, cl, la, lb, lc4;
};

// sum |b| and max |b| over the volume: per-block partials (fp64), then
// abs_parts_reduce_kernel adds them in block order (run-to-run identical)
template <typename T>
__global__ void abs_sum_kernel(const T* __restrict__ b, long long n, double* __restrict__ parts) {
  __shared__ double red[8];
  __shared__ double redm[8];
  double sacc = 0.0, m = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const double v = fabs(double(b[i]));
    sacc += v;
    m = fmax(m, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = sacc;
    redm[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, mm = 0.0;
    for (int w = 0; w < 8; ++w) {
      t += red[w];
      mm = fmax(mm, redm[w]);
    }
    parts[2 * blockIdx.x] = t;
    parts[2 * blockIdx.x + 1] = mm;
  }
}

__global__ void __launch_bounds__(256) abs_parts_reduce_kernel(const double* __restrict__ parts,
                                                               int nblocks, double* __restrict__ out) {
  __shared__ double st[8], sm[8];
  double t = 0.0, m = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += 256) {  // fixed-order tree
    t += parts[2 * i];
    m = fmax(m, parts[2 * i + 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t += __shfl_down_sync(0xffffffffu, t, o);
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) {
    st[threadIdx.x >> 5] = t;
    sm[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tt = 0.0, mm = 0.0;
    for (int w = 0; w < 8; ++w) {
      tt += st[w];
      mm = fmax(mm, sm[w]);
    }
    out[0] = tt;
    out[1] = mm;
  }
}

// gridDim.y CTAs per item (blockIdx.y = contiguous share of the template
// rows): partial sums of eta * lam = sum_v G_c(v) b(m + v) over the
// candidate's box (periodic indexing), warps over template rows, lanes over
// taps; refine_combine_kernel adds the shares in order (deterministic). The
// split keeps the latency-bound row walk short for the wide boxes (up to
// 171^2 rows).
template <typename T>
__global__ void __launch_bounds__(256) refine_kernel(const T* __restrict__ b, int nx, int ny,
                                                     int nz, int xoff,
                                                     const RefCand* __restrict__ rc,
                                                     const int* __restrict__ item_cand,
                                                     const long long* __restrict__ item_idx,
                                                     double* __restrict__ part) {
  __shared__ double red[8];
  const RefCand c = rc[item_cand[blockIdx.x]];
  const long long lin = item_idx[blockIdx.x];
  // (x-slab: b is the owned planes' window, item x shifted by its halo xoff)
  const int z = int(lin % nz), y = int((lin / nz) % ny), x = int(lin / ((long long)ny * nz)) + xoff;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrows = c.la * c.lb, S = int(gridDim.y);
  const int r0 = int((long long)nrows * blockIdx.y / S), r1 = int((long long)nrows * (blockIdx.y + 1) / S);
  double acc = 0.0;
  for (int r = r0 + warp; r < r1; r += 8) {
    const int2 rr = c.rows[r];
    if (rr.y <= 0) continue;
    const int ai = r / c.lb, bi = r - ai * c.lb;
    int xa = (x + c.lo_a + ai) % nx;
    if (xa < 0) xa += nx;
    int yb = (y + c.lo_b + bi) % ny;
    if (yb < 0) yb += ny;
    const T* brow = b + ((long long)xa * ny + yb) * nz;
    const double* trow = c.taps + (long long)r * c.lc4;
    for (int col = 4 * rr.x + lane; col < 4 * (rr.x + rr.y); col += 32) {
      int zc = (z + c.cl + col) % nz;
      if (zc < 0) zc += nz;
      acc = fma(trow[col], double(brow[zc]), acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[(long long)blockIdx.x * S + blockIdx.y] = t;
  }
}

__global__ void refine_combine_kernel(const double* __restrict__ part, int S, int count,
                                      double lam, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double t = 0.0;
  for (int s = 0; s < S; ++s) t += part[(long long)i * S + s];
  out[i] = t / lam;
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// smem row pitch (elements): >= cols needed, and the 16-byte chunk index of
// consecutive rows advances by an odd number, so the 8 lanes of one LDS.128
// wavefront (lane = row) hit 8 distinct 4-bank groups: fp32 pitch == 4 (mod 8),
// fp64 pitch == 2 (mod 4). (Rows stay 16-byte aligned for cp.async.)
int region_pitch(int lc4, int esize, int tz = kTZ) {
  int p = round_up(lc4 + tz + 8, 4);
  if (esize == 4) {
    if (p % 8 != 4) p += 4;
  } else {
    p += 2;
  }
  return p;
}

}  // namespace

// ------------------------------------------------------------------ table
static int upload(void** dst, const void* src, size_t bytes) {
  SFW3D_CUDA_TRY(cudaMalloc(dst, bytes));
  SFW3D_CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  return SFW3D_OK;
}

// the reference's support box of a unit atom: radius R = ceil(sigma * 36^(1/d)),
// full axis with minimum-image offsets when 2R + 1 >= n (forward.py:97-109)
static void candidate_box(const int dims[3], double sigma, double d, int lo[3], int hi[3]) {
  const int R = int(std::ceil(sigma * std::pow(kTailExponent, 1.0 / d)));
  for (int a = 0; a < 3; ++a) {
    if (2LL * R + 1 >= dims[a]) {
      lo[a] = -(dims[a] / 2);
      hi[a] = lo[a] + dims[a] - 1;
    } else {
      lo[a] = -R;
      hi[a] = R;
    }
  }
}

static int build_candidate(const int dims[3], double sigma, double d, double tap_tol,
                           CandHost& c) {
  c.sigma = sigma;
  c.d = d;
  candidate_box(dims, sigma, d, c.lo, c.hi);
  c.la = c.hi[0] - c.lo[0] + 1;
  c.lb = c.hi[1] - c.lo[1] + 1;
  c.cl = -round_up(-c.lo[2], 4);  // lo[2] rounded down to a multiple of 4
  c.lc4 = round_up(c.hi[2] - c.cl + 1, 4) + 4;
  const double inv2sd = 0.5 / std::pow(sigma, d);
  const double half_d = 0.5 * d;
  const bool d2 = d == 2.0;
  c.rows.assign(size_t(c.la) * c.lb, make_int2(0, 0));
  // +8: the kernel prefetches one 4-tap group past the end of each row
  std::vector<double> t(size_t(c.la) * c.lb * c.lc4 + 8, 0.0);
  c.taps = 0;
  for (int ai = 0; ai < c.la; ++ai) {
    const double a = c.lo[0] + ai;
    for (int bi = 0; bi < c.lb; ++bi) {
      const double b = c.lo[1] + bi;
      int cmin = 1 << 30, cmax = -(1 << 30);
      double* row = &t[(size_t(ai) * c.lb + bi) * c.lc4];
      for (int cc = c.lo[2]; cc <= c.hi[2]; ++cc) {
        const double u2 = (a * a + b * b) + double(cc) * cc;  // forward.py:133
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
  // executed flops of the folded kernel (eta_fold_kernel): per (a >= 0, b >= 0)
  // tap row, 4 FMA per step and (NR - 1) sums per window column, where NR
  // rows (+-a, +-b) share the row; each thread owns KJ outputs and its window
  // spans KJ + 4 * nsteps columns
  if (c.lo[0] == -c.hi[0] && c.lo[1] == -c.hi[1]) {
    const int Ra = c.hi[0], Rb = c.hi[1];
    for (int a = 0; a <= Ra; ++a)
      for (int b = 0; b <= Rb; ++b) {
        const int2 rr = c.rows[size_t(a + Ra) * c.lb + (b + Rb)];
        if (rr.y <= 0) continue;
        const int nr = (a ? 2 : 1) * (b ? 2 : 1);
        for (int k = 0; k < 2; ++k) {
          const double kj = k == 0 ? fold_kj<float>() : fold_kj<double>();
          c.fold_flops[k] += 2.0 * 4.0 * rr.y + double(nr - 1) * (4.0 * rr.y + kj) / kj;
        }
      }
  }
  std::vector<float> t32(t.begin(), t.end());
  SFW3D_TRY(upload(reinterpret_cast<void**>(&c.t64), t.data(), t.size() * sizeof(double)));
  SFW3D_TRY(upload(reinterpret_cast<void**>(&c.t32), t32.data(), t32.size() * sizeof(float)));
  SFW3D_TRY(upload(reinterpret_cast<void**>(&c.rows_dev), c.rows.data(), c.rows.size() * sizeof(int2)));
  return SFW3D_OK;
}

// Fitted bases are shared between tables: the fit (NNLS over the common box
// lattice, greedy pruning: 0.3 s of host time at config 3) depends only on the
// grid geometry, the candidates and the fit options — not on the data — so a
// solver that builds its table for the same grid again (a regularisation
// path, or lambda = c * max eta followed by the solve) reuses it. Entries are
// reference-counted; a few unreferenced ones are kept.
struct BasisCacheEntry {
  std::string key;
  BasisSet* set;
  int refs;
  unsigned long long stamp;
};
static std::mutex g_basis_mu;
static std::vector<BasisCacheEntry> g_basis_cache;
static unsigned long long g_basis_stamp = 0;
constexpr size_t kBasisCacheIdle = 8;

static std::string basis_key(const sfw3d_table* t, int dtype, double tol, bool prune, double loose) {
  std::string k;
  auto put = [&](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
  put(&t->device, sizeof(int));
  put(&dtype, sizeof(int));
  put(t->dims, 3 * sizeof(int));
  put(&tol, sizeof(double));
  put(&prune, sizeof(bool));
  put(&loose, sizeof(double));
  for (const BasisCandidate& c : t->bcands) {
    put(&c.sigma, sizeof(double));
    put(&c.d, sizeof(double));
    put(c.lo, 3 * sizeof(int));
    put(c.hi, 3 * sizeof(int));
    put(&c.direct_taps, sizeof(long long));
    put(&c.tap_tol, sizeof(double));
  }
  return k;
}

static void basis_release(BasisSet* s) {
  if (!s) return;
  std::vector<BasisSet*> dead;
  {
    std::lock_guard<std::mutex> g(g_basis_mu);
    bool found = false;
    for (auto& e : g_basis_cache)
      if (e.set == s) {
        if (e.refs > 0) --e.refs;
        e.stamp = ++g_basis_stamp;
        found = true;
      }
    if (!found) dead.push_back(s);
    // keep the most recently used idle entries only
    for (;;) {
      size_t idle = 0, oldest = g_basis_cache.size();
      for (size_t i = 0; i < g_basis_cache.size(); ++i)
        if (g_basis_cache[i].refs == 0) {
          ++idle;
          if (oldest == g_basis_cache.size() || g_basis_cache[i].stamp < g_basis_cache[oldest].stamp) oldest = i;
        }
      if (idle <= kBasisCacheIdle) break;
      dead.push_back(g_basis_cache[oldest].set);
      g_basis_cache.erase(g_basis_cache.begin() + oldest);
    }
  }
  for (BasisSet* d : dead) basis_set_destroy(d);
}

// builds (or takes from the cache) the shared basis of one storage precision
// on first use (fits accepted at basis_tol; fp64 members with inexact fits
// get their maxima refined exactly, see refine_kernel)
static int ensure_basis(const sfw3d_table* t, int dtype) {
  if (t->mode != 0) return SFW3D_OK;
  BasisSet*& s = dtype == SFW3D_F64 ? t->set64 : t->set32;
  if (s) return SFW3D_OK;
  const double tol = t->basis_tol;
  int dev = 0;
  SFW3D_CUDA_TRY(cudaGetDevice(&dev));
  SFW3D_CUDA_TRY(cudaSetDevice(t->device));
  BasisSet* built = nullptr;
  bool prune = t->prune != 0;
  if (t->prune < 0)
    prune = t->global_voxels > 0 ? basis_prune_voxels(t->global_voxels, dtype)
                                 : basis_prune_rule(t->dims, dtype);
  const double loose = t->loose_tol < 0.0 ? basis_loose_tol(dtype) : t->loose_tol;
  const std::string key = basis_key(t, dtype, tol, prune, loose);
  {
    std::lock_guard<std::mutex> g(g_basis_mu);
    for (auto& e : g_basis_cache)
      if (e.key == key) {
        ++e.refs;
        e.stamp = ++g_basis_stamp;
        s = e.set;
        cudaSetDevice(dev);
        return SFW3D_OK;
      }
  }
  const int st = basis_set_build(t->dims, t->bcands, dtype, tol, &built, true, prune, loose);
  cudaSetDevice(dev);
  if (st != SFW3D_OK) {
    basis_set_destroy(built);
    return st;
  }
  {
    std::lock_guard<std::mutex> g(g_basis_mu);
    g_basis_cache.push_back({key, built, 1, ++g_basis_stamp});
  }
  s = built;
  return SFW3D_OK;
}

// evaluator choice per candidate and storage type (fields: the call keeps
// every eta volume, which signed members cannot certify)
static bool use_basis(const sfw3d_table* t, int ci, int dtype, bool fields = false) {
  return t->mode == 0 && basis_set_member(t->set(dtype), ci, nullptr) &&
         !(fields && basis_set_signed(t->set(dtype), ci));
}

// exact refinement of the maxima: signed members always; in fp64 storage
// also the non-negative members whose fit is not exact
static bool use_refine(const sfw3d_table* t, int ci, int dtype, bool fields = false) {
  if (t->mode != 0) return false;
  const BasisSet* s = t->set(dtype);
  if (basis_set_signed(s, ci)) return !fields;
  double fe = 0.0;
  return dtype == SFW3D_F64 && basis_set_member(s, ci, &fe) && fe > 0.0;
}

// folded kernel tile: outputs per thread along z (fp32 32, fp64 16), one
// 32-row y group per CTA. z extent, smem row pitch, dynamic smem bytes.
static int fold_kj_rt(int esize) { return esize == 8 ? 16 : 32; }
static int fold_nwy_rt(int) { return 1; }
static int fold_tz(int esize) { return fold_kj_rt(esize) * kWarps; }
// fp32 KJ = 32 tiles keep the per-slice sums in a global scratch slab per
// CTA (L2-resident traffic of 2 x 16 KB per slice): the freed 16 KB of shared
// memory and a 128-register budget give 4 resident CTAs instead of 3
static bool fold_accd_global(int esize) { return esize == 4; }
static int fold_smem(const CandHost& c, int esize) {
  const int kj = fold_kj_rt(esize), nwy = fold_nwy_rt(esize);
  if (fold_accd_global(esize)) {
    const int ntap = ((c.lb / 2 + 1) * c.lc4 + 8 + 3) & ~3;
    const int nrow2 = ((c.lb / 2 + 2) & ~1) * (8 / esize);
    return (ntap + nrow2 + (kTY * nwy + c.lb - 1) * region_pitch(c.lc4, esize, fold_tz(esize))) * esize;
  }
  const int ntap = ((c.lb / 2 + 1) * c.lc4 + 8 + 3) & ~3;
  const int nrow2 = ((c.lb / 2 + 2) & ~1) * (8 / esize);  // int2 rows in elements
  return (kj * kThreads * nwy + ntap + nrow2 +
          (kTY * nwy + c.lb - 1) * region_pitch(c.lc4, esize, fold_tz(esize))) * esize;
}

template <typename T, int KJ, int NWY, bool AG = false>
static int launch_fold(sfw3d_ctx* ctx, dim3 grid, int smem, const T* bpad, const Geo& g,
                       const CandDev& cd, T* fld, Best* partial) {
  SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(eta_fold_kernel<T, KJ, NWY, AG>), size_t(smem)));
  eta_fold_kernel<T, KJ, NWY, AG><<<grid, kThreads * NWY, smem, ctx->stream>>>(bpad, g, cd, fld, partial);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

static bool use_sym(const sfw3d_table* t, const CandHost& c, int dtype) {
  const int esize = dtype == SFW3D_F64 ? 8 : 4;
  const bool sym = c.lo[0] == -c.hi[0] && c.lo[1] == -c.hi[1];
  return sym && fold_smem(c, esize) <= std::min(t->smem_max - 2048, 200 * 1024);
}

// executed flops per voxel attributed to one candidate (basis members share
// the term passes equally and each pays its own mix)
static double cand_flops(const sfw3d_table* t, int ci, int dtype) {
  const CandHost& c = t->cands[ci];
  if (use_basis(t, ci, dtype)) {
    const BasisSet* s = t->set(dtype);
    return 2.0 * double(basis_set_taps(s)) / basis_set_n_members(s) + basis_set_member_flops(s);
  }
  return use_sym(t, c, dtype) ? c.fold_flops[dtype == SFW3D_F64 ? 1 : 0] : 2.0 * double(c.taps);
}

}  // namespace sfw3d

using namespace sfw3d;

extern "C" int sfw3d_basis_fit(const int32_t lo[3], const int32_t hi[3], double sigma, double d,
                               int max_terms, double* betas, double* weights, double* w0,
                               int* n_terms, double* fit_err) {
  SFW3D_CHECK_ARG(lo && hi && w0 && n_terms && fit_err, "NULL argument");
  SFW3D_CHECK_ARG(sigma > 0.0 && d > 0.0, "sigma and d must be positive");
  int l[3], h[3];
  for (int a = 0; a < 3; ++a) {
    SFW3D_CHECK_ARG(lo[a] <= 0 && hi[a] >= 0, "box must contain the origin");
    l[a] = lo[a];
    h[a] = hi[a];
  }
  std::vector<std::pair<double, double>> bw;
  bool exact = false;
  fit_profile(l, h, sigma, d, 1e-10, *w0, bw, *fit_err, exact);
  *n_terms = int(bw.size());
  for (int k = 0; k < int(bw.size()) && k < max_terms; ++k) {
    if (betas) betas[k] = bw[k].first;
    if (weights) weights[k] = bw[k].second;
  }
  return SFW3D_OK;
}

extern "C" int sfw3d_basis_set_fit(const int32_t dims[3], int n_sigma, const double* sigmas,
                                   int n_shape, const double* shapes, int dtype, double tol,
                                   int prune, double loose_tol, int max_terms, int* n_terms,
                                   double* betas, double* weights, double* w0, double* fit_err,
                                   int32_t* member) {
  SFW3D_CHECK_ARG(dims && sigmas && shapes && n_terms, "NULL argument");
  SFW3D_CHECK_ARG(n_sigma > 0 && n_shape > 0, "empty candidate grid");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  int dm[3];
  for (int a = 0; a < 3; ++a) {
    SFW3D_CHECK_ARG(dims[a] > 0, "dims must be positive");
    dm[a] = dims[a];
  }
  std::vector<BasisCandidate> bc;
  for (int i = 0; i < n_sigma; ++i)
    for (int j = 0; j < n_shape; ++j) {
      SFW3D_CHECK_ARG(sigmas[i] > 0.0 && shapes[j] > 0.0, "sigma and d must be positive");
      BasisCandidate c{sigmas[i], shapes[j], {0, 0, 0}, {0, 0, 0}, 0};
      candidate_box(dm, c.sigma, c.d, c.lo, c.hi);
      bc.push_back(c);
    }
  BasisSet* s = nullptr;
  const bool pr = prune < 0 ? basis_prune_rule(dm, dtype) : prune != 0;
  const double lo = loose_tol < 0.0 ? basis_loose_tol(dtype) : loose_tol;
  const int st = basis_set_build(dm, bc, dtype, tol, &s, /*on_device=*/false, pr, lo);
  if (st == SFW3D_OK)
    basis_set_export(s, max_terms, n_terms, betas, weights, w0, fit_err, member);
  basis_set_destroy(s);
  return st;
}

extern "C" int sfw3d_table_set_option(sfw3d_table* t, const char* name, double value) {
  SFW3D_CHECK_ARG(t && name, "NULL argument");
  const std::string key(name);
  if (key == "prune") {
    SFW3D_CHECK_ARG(value == -1.0 || value == 0.0 || value == 1.0, "prune must be -1, 0 or 1");
    t->prune = int(value);
  } else if (key == "global_voxels") {
    SFW3D_CHECK_ARG(value >= 0.0 && value < 0x1p62, "global_voxels out of range");
    t->global_voxels = (long long)value;
  } else if (key == "loose_tol") {
    SFW3D_CHECK_ARG(std::isfinite(value), "loose_tol must be finite");
    t->loose_tol = value;
  } else if (key == "refine_cap") {
    SFW3D_CHECK_ARG(value >= 1.0 && value <= double(1 << 24), "refine_cap out of range");
    t->refine_cap = int(value);
    return SFW3D_OK;  // (no basis rebuild)
  } else {
    set_error("unknown table option (prune, global_voxels, loose_tol, refine_cap)");
    return SFW3D_EINVAL;
  }
  // the shared bases depend on prune / loose_tol: refit on next use
  cudaSetDevice(t->device);
  basis_release(t->set32);
  basis_release(t->set64);
  t->set32 = t->set64 = nullptr;
  return SFW3D_OK;
}

extern "C" int sfw3d_table_destroy(sfw3d_table* t) {
  if (!t) return SFW3D_OK;
  cudaSetDevice(t->device);
  for (auto& c : t->cands) {
    if (c.t64) cudaFree(c.t64);
    if (c.t32) cudaFree(c.t32);
    if (c.rows_dev) cudaFree(c.rows_dev);
  }
  basis_release(t->set32);
  basis_release(t->set64);
  if (t->refcand_dev) cudaFree(t->refcand_dev);
  delete t;
  return SFW3D_OK;
}

extern "C" int sfw3d_table_create(sfw3d_ctx* ctx, const sfw3d_psf* psf, int n_sigma,
                                  const double* sigma_host, int n_shape, const double* shape_host,
                                  double tap_tol, int mode, double basis_tol, sfw3d_table** out) {
  SFW3D_CHECK_ARG(ctx && psf && out, "NULL argument");
  SFW3D_CHECK_ARG(n_sigma > 0 && n_shape > 0 && sigma_host && shape_host,
                  "parameter grids must be non-empty");
  SFW3D_CHECK_ARG(mode == 0 || mode == 1, "mode");
  SFW3D_TRY(begin_call(ctx));
  *out = nullptr;
  std::vector<double> sg(sigma_host, sigma_host + n_sigma), dg(shape_host, shape_host + n_shape);
  for (double v : sg) SFW3D_CHECK_ARG(std::isfinite(v) && v > 0.0, "sigma grid values must be > 0");
  for (double v : dg) SFW3D_CHECK_ARG(std::isfinite(v) && v > 0.0, "shape grid values must be > 0");
  std::sort(sg.begin(), sg.end());  // certificate.py:72-73
  std::sort(dg.begin(), dg.end());
  auto* t = new sfw3d_table();
  for (int a = 0; a < 3; ++a) t->dims[a] = psf->dims[a];
  t->n_sigma = n_sigma;
  t->n_shape = n_shape;
  t->psf = psf;
  t->device = ctx->device;
  t->mode = mode;
  t->basis_tol = basis_tol;
  t->smem_max = 48 * 1024;
  cudaDeviceGetAttribute(&t->smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  t->cands.resize(size_t(n_sigma) * n_shape);
  int maxlo[3] = {0, 0, 0}, maxhi[3] = {0, 0, 0}, maxpitch = 0;
  for (int i = 0; i < n_sigma; ++i)
    for (int j = 0; j < n_shape; ++j) {
      CandHost& c = t->cands[size_t(i) * n_shape + j];
      const int s = build_candidate(t->dims, sg[i], dg[j], tap_tol, c);
      if (s != SFW3D_OK) {
        sfw3d_table_destroy(t);
        return s;
      }
      maxlo[0] = std::max(maxlo[0], -c.lo[0]);
      maxhi[0] = std::max(maxhi[0], c.hi[0]);
      maxlo[1] = std::max(maxlo[1], -c.lo[1]);
      maxhi[1] = std::max(maxhi[1], c.hi[1]);
      maxlo[2] = std::max(maxlo[2], -c.cl);
      maxpitch = std::max(maxpitch, std::max(region_pitch(c.lc4, 8, kFoldTZMax),
                                             region_pitch(c.lc4, 4, kFoldTZMax)));
    }
  // padded b: x/y pads cover the template offsets (+ the last partial tile
  // in y), z covers the aligned template start and the widest staged row.
  t->pad[0] = maxlo[0];
  t->pad[1] = maxlo[1];
  t->pad[2] = round_up(maxlo[2], 4);
  t->pdims[0] = t->pad[0] + t->dims[0] + maxhi[0];
  t->pdims[1] = t->pad[1] + round_up(t->dims[1], kTY) + maxhi[1] + kTY;
  t->pdims[2] = round_up(t->pad[2] + round_up(t->dims[2], kFoldTZMax) + 4 + maxpitch, 4);
  for (const auto& c : t->cands)
    t->bcands.push_back(
        {c.sigma, c.d, {c.lo[0], c.lo[1], c.lo[2]}, {c.hi[0], c.hi[1], c.hi[2]}, c.taps, tap_tol});
  {
    std::vector<RefCand> rc;
    for (const auto& c : t->cands) rc.push_back({c.t64, c.rows_dev, c.lo[0], c.lo[1], c.cl, c.la, c.lb, c.lc4});
    const int st = upload(&t->refcand_dev, rc.data(), rc.size() * sizeof(RefCand));
    if (st != SFW3D_OK) {
      sfw3d_table_destroy(t);
      return st;
    }
  }
  *out = t;
  return SFW3D_OK;
}

extern "C" int sfw3d_table_info(const sfw3d_table* t, int dtype, int* n_cand, int* n_direct,
                                int* n_basis, int64_t* direct_taps, int64_t* basis_taps,
                                double* direct_flops, double* basis_flops) {
  SFW3D_CHECK_ARG(t, "table is NULL");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_TRY(ensure_basis(t, dtype));
  int nb = 0;
  long long dt = 0, bt = 0;
  double df = 0.0, bf = 0.0;
  for (int ci = 0; ci < int(t->cands.size()); ++ci) {
    if (use_basis(t, ci, dtype)) {
      ++nb;
    } else {
      dt += t->cands[ci].taps;
      df += cand_flops(t, ci, dtype);
    }
  }
  if (nb) {
    bt = basis_set_taps(t->set(dtype));
    bf = basis_set_flops(t->set(dtype));
  }
  if (n_cand) *n_cand = int(t->cands.size());
  if (n_direct) *n_direct = int(t->cands.size()) - nb;
  if (n_basis) *n_basis = nb;
  if (direct_taps) *direct_taps = dt;
  if (basis_taps) *basis_taps = bt;
  if (direct_flops) *direct_flops = df;
  if (basis_flops) *basis_flops = bf;
  return SFW3D_OK;
}

extern "C" int sfw3d_table_basis_passes(const sfw3d_table* t, int dtype, int cap, int32_t* taps_out,
                                        int* n_out) {
  SFW3D_CHECK_ARG(t && n_out, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_TRY(ensure_basis(t, dtype));
  const int nt = basis_set_n_terms(t->set(dtype));
  *n_out = 3 * nt;
  if (taps_out)
    for (int k = 0; k < nt && 3 * k + 2 < cap; ++k)
      for (int a = 0; a < 3; ++a) taps_out[3 * k + a] = basis_set_pass_taps(t->set(dtype), k, a);
  return SFW3D_OK;
}

extern "C" int sfw3d_table_candidate(const sfw3d_table* t, int dtype, int cand, int* uses_basis,
                                     int* n_terms, double* fit_err, int64_t* direct_taps,
                                     int64_t* basis_taps, double* flops) {
  SFW3D_CHECK_ARG(t && cand >= 0 && cand < int(t->cands.size()), "candidate index");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_TRY(ensure_basis(t, dtype));
  const CandHost& c = t->cands[cand];
  if (uses_basis) *uses_basis = use_basis(t, cand, dtype) ? (use_refine(t, cand, dtype) ? 2 : 1) : 0;
  double fe = INFINITY;
  basis_set_member(t->set(dtype), cand, &fe);
  if (n_terms) *n_terms = basis_set_n_terms(t->set(dtype));  // shared terms of the table
  if (fit_err) *fit_err = fe;
  if (direct_taps) *direct_taps = c.taps;
  if (basis_taps) *basis_taps = basis_set_taps(t->set(dtype));
  if (flops) *flops = cand_flops(t, cand, dtype);
  return SFW3D_OK;
}

namespace {

// voxels the last exact refinement re-evaluated (diagnostics)
int& last_refine_count() {
  static thread_local int c = 0;
  return c;
}

// x-slab evaluation (sfw3d_eta_argmax_slab): the owned planes and the link
struct SlabArgs {
  SlabLink link;
  int n_own;
};

template <typename T>
int eta_typed(sfw3d_ctx* ctx, const sfw3d_table* t, const void* residual, double lam,
              const int32_t win[6], sfw3d_argmax* best_host, sfw3d_argmax* per_cand_host,
              void* fields, const SlabArgs* sl = nullptr) {
  const int dtype = sizeof(T) == 8 ? SFW3D_F64 : SFW3D_F32;
  // evaluation grid: the whole volume, or this rank's owned x-planes
  const int ldims[3] = {sl ? sl->n_own : t->dims[0], t->dims[1], t->dims[2]};
  const int* dims = ldims;
  // local padded geometry for the direct / refinement kernels: on a slab the
  // x padding comes from the neighbours (halo exchange), not from wrapping
  const int pdims0 = sl ? ldims[0] + 2 * t->pad[0] : t->pdims[0];
  const int64_t n = vol_count(dims);
  const size_t vb = size_t(n) * sizeof(T);
  const int nc = int(t->cands.size());
  bool any_direct = false, any_basis = false, any_refine = false;
  const bool fl = fields != nullptr;
  for (int ci = 0; ci < nc; ++ci) {
    (use_basis(t, ci, dtype, fl) ? any_basis : any_direct) = true;
    any_refine |= use_refine(t, ci, dtype, fl);
  }
  // direct evaluation per candidate (refined members fall back to it when
  // their candidate list overflows)
  std::vector<char> direct(nc, 0);
  for (int ci = 0; ci < nc; ++ci) direct[ci] = !use_basis(t, ci, dtype, fl);
  const BasisSet* bset = t->set(dtype);
  const size_t sb = any_basis ? basis_set_scratch(bset, n, dtype, dims) : 0;
  // the padded copy of b feeds the direct kernels only (refinement may fall
  // back to them: the copy is then made on demand)
  const size_t pbytes = size_t(pdims0) * t->pdims[1] * t->pdims[2] * sizeof(T);
  const size_t pb = (any_direct || any_refine) ? pbytes : 0;
  // refinement items per call (a table option: tests shrink it)
  const int kRefCap = t->refine_cap;
  // direct output tiles: the window, or the whole grid when fields are requested
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
  const long long nblocks_direct = (long long)nty * ntz * nxp;
  const long long nblocks = nblocks_direct;
  const int kRefPart = std::max(kRefCap, 4096);  // per-share partial sums
  const size_t rb = any_refine ? size_t(kRefCap) * (4 + 8 + 8) + size_t(kRefPart) * 8 +
                                     size_t(nc) * 12 + 352
                               : 0;
  // folded kernel slice sums in global memory (tuning variant)
  size_t ab = 0;
  if (fold_accd_global(sizeof(T))) {
    const int tzf = fold_tz(sizeof(T));
    const long long nctas = (long long)((ow[3] - ow[2] + 1 + kTY - 1) / kTY) *
                            ((ow[5] - zbase + 1 + tzf - 1) / tzf) * nxp;
    ab = size_t(nctas) * fold_kj_rt(sizeof(T)) * kThreads * sizeof(T);
  }
  // x-slab window buffer: H + owned + H planes, H covering the PSF, every
  // basis term's x pass and the templates' x radius (refinement / direct)
  int H = 0;
  if (sl) {
    // (halos wider than a slab come from several ranks: the transport's job)
    H = std::max({-t->psf->lo[0], t->psf->hi[0], basis_set_max_xhalo(bset), t->pad[0]});
  }
  const size_t wbytes = sl ? size_t(ldims[0] + 2 * H) * t->dims[1] * t->dims[2] * sizeof(T) : 0;
  SFW3D_TRY(ensure_device(ctx, ctx->ws,
                          Carver::need({vb, vb, sb, pb, size_t(nblocks) * sizeof(Best),
                                        size_t(nc) * sizeof(Best), rb, ab, wbytes})));
  Carver cv(ctx->ws.ptr);
  T* b = cv.take<T>(n);
  T* tmp = cv.take<T>(n);
  void* bscratch = sb ? cv.take<char>(sb) : nullptr;
  T* bpad = pb ? cv.take<T>(pb / sizeof(T)) : nullptr;
  Best* partial = cv.take<Best>(nblocks);
  Best* cbest = cv.take<Best>(nc);
  int* ref_cand = any_refine ? cv.take<int>(kRefCap) : nullptr;
  long long* ref_idx = any_refine ? cv.take<long long>(kRefCap) : nullptr;
  double* ref_val = any_refine ? cv.take<double>(kRefCap) : nullptr;
  double* ref_part = any_refine ? cv.take<double>(kRefPart) : nullptr;
  double* ref_thr = any_refine ? cv.take<double>(nc) : nullptr;
  double* ref_l1 = any_refine ? cv.take<double>(2) : nullptr;  // [sum |b|, max |b|]
  int* ref_count = any_refine ? cv.take<int>(1 + nc) : nullptr;  // [total, per member]
  std::vector<Best> refined(nc, Best{NAN, -1});  // exact maxima of refined members
  void* accd_g = ab ? cv.take<char>(ab) : nullptr;
  T* wbuf = sl ? cv.take<T>(wbytes / sizeof(T)) : nullptr;
  // (zeroed once per call: the x passes' padded zero taps also read a few
  // planes past the exchanged halos, which must hold finite values)
  if (sl) SFW3D_CUDA_TRY(cudaMemsetAsync(wbuf, 0, wbytes, ctx->stream));
  const long long plane = (long long)dims[1] * dims[2];
  // b = H^T * r (tmp is pass scratch), then the periodic padding for direct
  if (sl)
    SFW3D_TRY(psf_apply_slab(ctx, t->psf, dtype, residual, b, 1, ldims, wbuf, H, tmp, sl->link));
  else
    SFW3D_TRY(psf_apply_impl(ctx, t->psf, dtype, residual, b, 1, tmp));
  // x-slab: b on the owned planes + the template radius of neighbour planes
  // (refinement and direct kernels read the template box around a voxel)
  const int px = t->pad[0];
  bool bwin_ready = false;
  auto make_bwin = [&]() -> int {
    if (!sl || bwin_ready) return SFW3D_OK;
    T* mid = wbuf + size_t(H) * plane;
    SFW3D_CUDA_TRY(cudaMemcpyAsync(mid, b, vb, cudaMemcpyDeviceToDevice, ctx->stream));
    if (sl->link.halo(sl->link.user, mid - size_t(px) * plane, dtype, dims[0], plane, px, px) != 0) {
      set_error("halo exchange callback failed");
      return SFW3D_ECUDA;
    }
    bwin_ready = true;
    return SFW3D_OK;
  };
  const T* bref = sl ? wbuf + size_t(H - px) * plane : b;  // refinement's view of b
  bool padded = false;
  auto make_pad = [&]() -> int {
    if (padded || !bpad) return SFW3D_OK;
    SFW3D_TRY(make_bwin());
    SFW3D_PROF(ctx, "pad");
    const long long np = (long long)pdims0 * t->pdims[1] * t->pdims[2];
    if (sl)  // the window already holds the x padding: pad y and z only
      pad_kernel<T><<<unsigned((np + 255) / 256), 256, 0, ctx->stream>>>(
          bref, bpad, pdims0, dims[1], dims[2], 0, t->pad[1], t->pad[2], pdims0, t->pdims[1],
          t->pdims[2]);
    else
      pad_kernel<T><<<unsigned((np + 255) / 256), 256, 0, ctx->stream>>>(
          b, bpad, dims[0], dims[1], dims[2], t->pad[0], t->pad[1], t->pad[2], t->pdims[0],
          t->pdims[1], t->pdims[2]);
    SFW3D_LAUNCH_CHECK(ctx);
    padded = true;
    return SFW3D_OK;
  };
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
  g.accd_g = accd_g;
  int smem_max = 0;
  SFW3D_CUDA_TRY(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int budget = std::min(smem_max - 2048, 110 * 1024);
  // every basis member at once: shared separable terms + fused mix/argmax,
  // writing cbest[cand] (and the member fields) directly
  bool abs_done = false;
  SlabEval se;
  if (sl) {
    se.link = sl->link;
    se.win = wbuf;
    se.H = H;
  }
  if (any_basis)
    SFW3D_TRY(basis_set_eval(ctx, bset, dtype, dims, b, lam, win, fields, cbest, bscratch,
                             any_refine ? ref_l1 : nullptr, &abs_done, sl ? &se : nullptr));
  // x-slab: the b window exchange is a collective, so every rank makes it at
  // this fixed point (whatever its own refinement / direct work turns out to be)
  if (sl && (any_refine || any_direct)) SFW3D_TRY(make_bwin());
  if (any_refine) {
    // Every refined member's approximate eta~ is within E_c of its direct
    // value at every voxel: signed members E_c = ebound_c ||b||_inf / lam
    // (basis.cu), fp64 non-negative members E_c = (e_c + 2e-12) ||b||_1 / lam.
    // The true maximum lies among the voxels with eta~ >= max eta~ - 2 E_c.
    SFW3D_PROF(ctx, "eta_refine");
    if (!abs_done) {  // (the mix computes them when it streams b: mix_ring2_kernel)
      const int nab = std::min(4 * ctx->num_sms, kRefPart / 2);  // partials in ref_part
      abs_sum_kernel<T><<<nab, 256, 0, ctx->stream>>>(b, n, ref_part);
      SFW3D_LAUNCH_CHECK(ctx);
      abs_parts_reduce_kernel<<<1, 256, 0, ctx->stream>>>(ref_part, nab, ref_l1);
      SFW3D_LAUNCH_CHECK(ctx);
    }
    std::vector<Best> hb0(nc);
    double l1[2] = {0.0, 0.0};
    SFW3D_TRY(download_sync(ctx, hb0.data(), cbest, size_t(nc) * sizeof(Best)));
    SFW3D_TRY(download_sync(ctx, l1, ref_l1, 2 * sizeof(double)));
    if (sl) {
      // the bounds use the GLOBAL |b| statistics and member maxima (the
      // single-volume thresholds): all-reduce them over the ranks
      std::vector<double> mx(nc + 1);
      for (int ci = 0; ci < nc; ++ci) mx[ci] = std::isfinite(hb0[ci].v) ? hb0[ci].v : -1e308;
      mx[nc] = l1[1];
      if (sl->link.allreduce(sl->link.user, l1, 1, 0) != 0 ||
          sl->link.allreduce(sl->link.user, mx.data(), nc + 1, 1) != 0) {
        set_error("all-reduce callback failed");
        return SFW3D_ECUDA;
      }
      for (int ci = 0; ci < nc; ++ci)
        if (std::isfinite(hb0[ci].v)) hb0[ci].v = mx[ci];
      l1[1] = mx[nc];
    }
    const int nm = basis_set_n_members(bset);
    std::vector<double> thr(nm, INFINITY);
    for (int m = 0; m < nm; ++m) {
      const int ci = basis_set_member_cand(bset, m);
      if (!use_refine(t, ci, dtype, fl) || !std::isfinite(hb0[ci].v)) continue;
      double E;
      if (basis_set_signed(bset, ci)) {
        E = basis_set_ebound(bset, ci) * l1[1] / lam * (1.0 + 1e-6);
      } else {
        double fe = 0.0;
        basis_set_member(bset, ci, &fe);
        E = (fe + 2e-12) * l1[0] / lam;
      }
      thr[m] = hb0[ci].v - 2.0 * E - 1e-12 * std::fabs(hb0[ci].v);
    }
    SFW3D_TRY(stage_upload(ctx, ref_thr, thr.data(), size_t(nm) * sizeof(double)));
    SFW3D_TRY(basis_set_collect(ctx, bset, dtype, dims, b, lam, win, ref_thr, kRefCap, ref_cand,
                                ref_idx, ref_count, bscratch, fl));
    std::vector<int> counts(1 + nm, 0);
    SFW3D_TRY(download_sync(ctx, counts.data(), ref_count, counts.size() * sizeof(int)));
    int count = counts[0];
    if (count > kRefCap) {
      // keep refining the members with the fewest near-maximal voxels (within
      // the cap), evaluate the others directly, and collect again
      std::vector<int> order;
      for (int m = 0; m < nm; ++m)
        if (std::isfinite(thr[m])) order.push_back(m);
      std::sort(order.begin(), order.end(), [&](int x, int y) { return counts[1 + x] < counts[1 + y]; });
      long long used = 0;
      for (int m : order) {
        if (used + counts[1 + m] <= kRefCap) {
          used += counts[1 + m];
        } else {
          thr[m] = INFINITY;
          direct[basis_set_member_cand(bset, m)] = 1;
        }
      }
      SFW3D_TRY(stage_upload(ctx, ref_thr, thr.data(), size_t(nm) * sizeof(double)));
      SFW3D_TRY(basis_set_collect(ctx, bset, dtype, dims, b, lam, win, ref_thr, kRefCap, ref_cand,
                                  ref_idx, ref_count, bscratch, fl));
      SFW3D_TRY(download_sync(ctx, &count, ref_count, sizeof(int)));
    }
    last_refine_count() = count;
    if (count > kRefCap) {  // (cannot happen after the split above; kept as a guard)
      for (int ci = 0; ci < nc; ++ci)
        if (use_refine(t, ci, dtype, fl)) direct[ci] = 1;
      count = 0;
    } else if (count > 0) {
      SFW3D_PROF(ctx, "eta_refine");
      // shares per item: ~4096 CTAs in all, at most 64 per item
      const int S = std::max(1, std::min(64, kRefPart / count));
      SFW3D_TRY(make_bwin());
      refine_kernel<T><<<dim3(unsigned(count), unsigned(S)), 256, 0, ctx->stream>>>(
          bref, sl ? pdims0 : dims[0], dims[1], dims[2], sl ? px : 0,
          static_cast<const RefCand*>(t->refcand_dev), ref_cand, ref_idx, ref_part);
      SFW3D_LAUNCH_CHECK(ctx);
      refine_combine_kernel<<<(count + 255) / 256, 256, 0, ctx->stream>>>(ref_part, S, count, lam,
                                                                          ref_val);
      SFW3D_LAUNCH_CHECK(ctx);
      std::vector<int> hc(count);
      std::vector<long long> hi(count);
      std::vector<double> hv(count);
      SFW3D_TRY(download_sync(ctx, hc.data(), ref_cand, size_t(count) * sizeof(int)));
      SFW3D_TRY(download_sync(ctx, hi.data(), ref_idx, size_t(count) * sizeof(long long)));
      SFW3D_TRY(download_sync(ctx, hv.data(), ref_val, size_t(count) * sizeof(double)));
      for (int i = 0; i < count; ++i) {
        Best& r = refined[hc[i]];
        // larger value wins, ties to the smaller C-order index
        if (std::isnan(r.v) || hv[i] > r.v || (hv[i] == r.v && hi[i] < r.idx)) r = {hv[i], hi[i]};
      }
    }
    // (a refined member always collects its own approximate maximum; if not,
    // evaluate it directly rather than report an uncertified value)
    for (int ci = 0; ci < nc; ++ci)
      if (use_refine(t, ci, dtype, fl) && !direct[ci] && std::isnan(refined[ci].v)) {
        // x-slab: thresholds are the GLOBAL ones, so a member with nothing
        // collected here cannot hold its global maximum on this slab
        if (sl)
          refined[ci] = {-INFINITY, 0x7fffffffffffffffLL};
        else
          direct[ci] = 1;
      }
  }
  for (int ci = 0; ci < nc; ++ci) {
    if (!direct[ci]) continue;
    SFW3D_TRY(make_pad());
    const CandHost& c = t->cands[ci];
    T* fld = fields ? static_cast<T*>(fields) + size_t(ci) * n : nullptr;
    long long nred = 0;
    {
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
      if (use_sym(t, c, dtype)) {
        const int kj = fold_kj_rt(sizeof(T)), nwy = fold_nwy_rt(sizeof(T));
        const int TZ = kj * kWarps, TY = kTY * nwy;
        gc.pitch = region_pitch(c.lc4, sizeof(T), TZ);
        gc.ntz = (ow[5] - zbase + 1 + TZ - 1) / TZ;
        gc.nty = (ow[3] - ow[2] + 1 + TY - 1) / TY;
        gc.brows = c.lb;
        const int smem = fold_smem(c, sizeof(T));
        SFW3D_PROF(ctx, "eta_direct");
        dim3 grid(unsigned(gc.nty * gc.ntz), unsigned(nxp));
        if constexpr (sizeof(T) == 4) {
          SFW3D_TRY((launch_fold<T, 32, 1, true>(ctx, grid, smem, bpad, gc, cd, fld, partial)));
        } else {
          SFW3D_TRY((launch_fold<T, 16, 1>(ctx, grid, smem, bpad, gc, cd, fld, partial)));
        }
        nred = (long long)gc.nty * gc.ntz * nxp;
      } else {
        gc.pitch = region_pitch(c.lc4, sizeof(T));
        const int row_bytes = gc.pitch * int(sizeof(T));
        const int brows = budget / row_bytes - (kTY - 1);
        if (brows < 1) {
          set_error("certificate template too wide for the shared-memory tile");
          return SFW3D_EINVAL;
        }
        gc.brows = std::min(brows, c.lb);
        const int smem = (kTY + gc.brows - 1) * row_bytes;
        SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(eta_direct_kernel<T>), size_t(smem)));
        SFW3D_PROF(ctx, "eta_direct");
        dim3 grid(unsigned(nty * ntz), unsigned(nxp));
        eta_direct_kernel<T><<<grid, kThreads, smem, ctx->stream>>>(bpad, gc, cd, fld, partial);
        SFW3D_LAUNCH_CHECK(ctx);
        nred = nblocks_direct;
      }
    }
    {
      SFW3D_PROF(ctx, "argmax");
      best_reduce_kernel<<<1, 1024, 0, ctx->stream>>>(partial, nred, cbest + ci);
      SFW3D_LAUNCH_CHECK(ctx);
    }
  }
  std::vector<Best> hb(nc);
  SFW3D_TRY(download_sync(ctx, hb.data(), cbest, size_t(nc) * sizeof(Best)));
  for (int ci = 0; ci < nc; ++ci)
    if (!direct[ci] && !std::isnan(refined[ci].v)) hb[ci] = refined[ci];
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
  if (!std::isfinite(bv) && !(sl && bv == -INFINITY)) {
    set_error("non-finite certificate value");
    return SFW3D_ENONFINITE;
  }
  return SFW3D_OK;
}

}  // namespace

extern "C" int sfw3d_last_refine_count(void) { return last_refine_count(); }

extern "C" int sfw3d_eta_argmax_slab(sfw3d_ctx* ctx, const sfw3d_table* t, int dtype,
                                     const void* residual_dev, int n_own, int x0, double lam,
                                     const int32_t window[6], sfw3d_halo_fn halo,
                                     sfw3d_allreduce_fn allreduce, void* user,
                                     sfw3d_argmax* best_host, sfw3d_argmax* per_cand_host) {
  SFW3D_CHECK_ARG(ctx && t && residual_dev && window && halo && allreduce, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(lam > 0.0, "lam must be > 0");
  SFW3D_CHECK_ARG(n_own > 0 && x0 >= 0 && x0 + n_own <= t->dims[0], "slab planes");
  const int ld[3] = {n_own, t->dims[1], t->dims[2]};
  for (int a = 0; a < 3; ++a)
    SFW3D_CHECK_ARG(0 <= window[2 * a] && window[2 * a] <= window[2 * a + 1] &&
                        window[2 * a + 1] < ld[a],
                    "window must be a non-empty box inside the slab (local coordinates)");
  SFW3D_CHECK_ARG(t->mode == 0, "x-slab certificates need the basis evaluator (mode auto)");
  SFW3D_TRY(begin_call(ctx));
  SFW3D_TRY(ensure_basis(t, dtype));
  SlabArgs sa;
  sa.link.halo = halo;
  sa.link.allreduce = allreduce;
  sa.link.user = user;
  sa.n_own = n_own;
  (void)x0;  // (the periodic ring of ranks defines the neighbours)
  if (dtype == SFW3D_F64)
    return eta_typed<double>(ctx, t, residual_dev, lam, window, best_host, per_cand_host, nullptr,
                             &sa);
  return eta_typed<float>(ctx, t, residual_dev, lam, window, best_host, per_cand_host, nullptr,
                          &sa);
}

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
  SFW3D_TRY(ensure_basis(t, dtype));
  if (dtype == SFW3D_F64)
    return eta_typed<double>(ctx, t, residual_dev, lam, window, best_host, per_cand_host, fields_dev);
  return eta_typed<float>(ctx, t, residual_dev, lam, window, best_host, per_cand_host, fields_dev);
}
