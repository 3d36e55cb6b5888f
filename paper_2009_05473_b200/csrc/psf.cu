// K4 — circular 1-D correlation passes: the PSF (convolve / correlate_adjoint,
// forward.py:79-94) and the separable Gaussian-basis certificate terms.
//
// The reference applies the PSF as rfftn -> product -> irfftn. Every
// BASELINE PSF is a box-truncated sampled Gaussian, i.e. exactly separable,
// so here the operator is three 1-D circular passes (one per axis) with
// (hi - lo + 1) taps each; a non-separable kernel falls back to a direct
// 3-D stencil over its non-zero box. Offsets are relative to the kernel
// origin n//2 (forward.py:43-47, ifftshift at :58).
//
// Pass kernels (out = addend_w * addend + w * sum_q taps[q] * in[i + lo + q]):
//  * axes 0/1 (strided): one thread per contiguous inner index (coalesced
//    across the warp) computing J consecutive outputs along the axis with a
//    register window rotated at compile time (1 load + J FFMA per tap),
//    taps broadcast from shared memory;
//  * axis 2 (contiguous): a CTA stages 32 rows x (4J + taps) in shared
//    memory (odd pitch: lane = row, conflict-free), same rotated window.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "window.cuh"

namespace sfw3d {
namespace {

__device__ __forceinline__ int wrap_inc(int i, int n) { return (i + 1 == n) ? 0 : i + 1; }

// a mod n in [0, n) without a division on the common path (|a| < 2n)
__device__ __forceinline__ int pmod_i(int a, int n) {
  if (a < 0) {
    a += n;
    if (a < 0) a = (a % n + n) % n;
  } else if (a >= n) {
    a -= n;
    if (a >= n) a %= n;
  }
  return a;
}

// Taps are zero-padded to a multiple of J in shared memory; each block of J
// taps is read into registers at once, so the inner loop is J x (J FFMA +
// one window load) with no tap-load latency on the critical path.
template <typename T, int J>
__device__ __forceinline__ void load_taps_padded(T* taps, const T* __restrict__ taps_g, int ntaps,
                                                 int npad) {
  for (int q = threadIdx.x; q < npad; q += blockDim.x) taps[q] = q < ntaps ? taps_g[q] : T(0);
}

template <typename T, int J>
__global__ void __launch_bounds__(256) pass_strided_kernel(
    const T* __restrict__ in, T* out, int n_axis, long long stride, const T* __restrict__ taps_g,
    int lo, int ntaps, const T* addend, T aw, T w, int a_begin, int a_end, int out_shift) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* taps = reinterpret_cast<T*>(smem_raw);
  const int npad = (ntaps + J - 1) / J * J;
  load_taps_padded<T, J>(taps, taps_g, ntaps, npad);
  __syncthreads();
  // blockIdx.x runs over the a-blocks so CTAs that share input planes are
  // resident together (L2 reuse of the (J + taps - 1)/J overlap)
  const long long inner = blockIdx.y * (long long)blockDim.x + threadIdx.x;
  if (inner >= stride) return;
  const int a0 = a_begin + blockIdx.x * J;
  const long long base = (long long)blockIdx.z * n_axis * stride + inner;
  T W[J], acc[J];
  int idx = pmod_i(a0 + lo, n_axis);
#pragma unroll
  for (int j = 0; j < J; ++j) {
    W[j] = in[base + idx * stride];
    idx = wrap_inc(idx, n_axis);
    acc[j] = T(0);
  }
  // (taps stay in shared memory here: the strided window loads need the
  // registers more than the broadcast taps do)
  for (int q0 = 0; q0 < npad; q0 += J) {
#pragma unroll
    for (int r = 0; r < J; ++r) {
      const T t = taps[q0 + r];
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma(t, W[(r + j) % J], acc[j]);
      W[r] = in[base + idx * stride];
      idx = wrap_inc(idx, n_axis);
    }
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    if (a0 + j < a_end) {
      const long long o = base + (long long)(a0 + j + out_shift) * stride;
      out[o] = addend ? T(aw * addend[o] + w * acc[j]) : T(w * acc[j]);
    }
  }
}


constexpr int kZRows = 32;   // rows per CTA (one per lane)
constexpr int kZWarps = 4;   // z-groups per CTA

// Contiguous axis: the CTA stages 32 rows x (4J + taps + J) in shared memory
// (odd pitch: lane = row is conflict-free), computes J consecutive outputs
// per thread with the rotated register window, then transposes the results
// through shared memory so the global stores are coalesced along z.
template <typename T, int J>
__global__ void __launch_bounds__(32 * kZWarps) pass_z_kernel(
    const T* __restrict__ in, T* out, int nz, long long nrows, const T* __restrict__ taps_g, int lo,
    int ntaps, int pitch, const T* addend, T aw, T w) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int npad = (ntaps + J - 1) / J * J;
  T* taps = reinterpret_cast<T*>(smem_raw);
  T* tile = taps + npad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long row0 = (long long)blockIdx.y * kZRows;
  const int z0 = blockIdx.x * (J * kZWarps);
  const int width = J * kZWarps + npad;  // staged columns (incl. the padded-tap overrun)
  load_taps_padded<T, J>(taps, taps_g, ntaps, npad);
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    const int zc = pmod_i(z0 + lo + c, nz);
    for (int r = 0; r < kZRows; ++r) {
      const long long row = row0 + r;
      if (row < nrows) {
        if constexpr (sizeof(T) == 8)
          cp_async8(tile + r * pitch + c, in + row * nz + zc);
        else
          cp_async4(tile + r * pitch + c, in + row * nz + zc);
      } else {
        tile[r * pitch + c] = T(0);
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const T* src = tile + lane * pitch + warp * J;
  T W[J], acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    W[j] = src[j];
    acc[j] = T(0);
  }
  for (int q0 = 0; q0 < npad; q0 += J) {
    T tq[J];
#pragma unroll
    for (int r = 0; r < J; ++r) tq[r] = taps[q0 + r];
#pragma unroll
    for (int r = 0; r < J; ++r) {
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma(tq[r], W[(r + j) % J], acc[j]);
      W[r] = src[q0 + r + J];
    }
  }
  __syncthreads();  // every thread is done reading the staged input
  T* res = tile + lane * pitch + warp * J;
#pragma unroll
  for (int j = 0; j < J; ++j) res[j] = acc[j];
  __syncthreads();
  const int ncols = J * kZWarps;
  for (int e = threadIdx.x; e < kZRows * ncols; e += blockDim.x) {
    const int r = e / ncols, c = e % ncols;
    const long long row = row0 + r;
    const int z = z0 + c;
    if (row < nrows && z < nz) {
      const long long o = row * nz + z;
      const T v = tile[r * pitch + c];
      out[o] = addend ? T(aw * addend[o] + w * v) : T(w * v);
    }
  }
}

// Output stores of the contiguous pass: streaming (evict-first) for volumes
// that cannot stay in L2, normal (kept for the next pass) in L2 mode.
template <typename V>
__device__ __forceinline__ void st_out(int l2mode, V* p, V v) {
  if (l2mode) *p = v;
  else __stcs(p, v);
}

// ------------------------------------------------------------ v2 passes
// Register-window passes with ~94% FFMA issue density: taps padded only to a
// multiple of 4 (the window consumes 4 taps per step), the staged tile reused
// by J outputs per thread, incremental wrap arithmetic in the staging loops.

// Strided axes (0, 1): a CTA owns TI consecutive inner (contiguous) indices
// x G groups of J consecutive outputs along the axis. Rows a0 + lo + r
// (wrapped) are staged with 16-byte cp.async; lane = inner index (conflict-
// free scalar smem reads, coalesced 128-byte stores). Per tap: one LDS of the
// next window row + J FFMA (taps read four at a time, broadcast).
template <typename T, int J, int TI, int NT, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) pass_tile2_kernel(
    const T* __restrict__ in, T* __restrict__ out, int n_axis, long long stride,
    const T* __restrict__ taps_g, int lo, int ntaps, const T* addend, T aw, T w, int a_begin,
    int a_end, int out_shift, double* __restrict__ sq_parts, int l2mode) {
  constexpr int G = NT / TI, To = J * G;
  const unsigned long long pol = l2_policy(l2mode);
  constexpr int kVec = 16 / sizeof(T), kRowVecs = TI / kVec;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nt4 = (ntaps + 3) & ~3;
  T* taps = reinterpret_cast<T*>(smem_raw);
  T* tile = taps + nt4;
  const int rows = To + nt4;
  const int a0 = a_begin + blockIdx.x * To;
  const long long base0 = (long long)blockIdx.z * n_axis * stride + (long long)blockIdx.y * TI;
  for (int q = threadIdx.x; q < nt4; q += NT) taps[q] = q < ntaps ? taps_g[q] : T(0);
  {
    static_assert(NT % kRowVecs == 0, "row vectors");
    constexpr int dr = NT / kRowVecs;
    const int c = (threadIdx.x % kRowVecs) * kVec;
    int r = threadIdx.x / kRowVecs;
    int a = (a0 + lo + r) % n_axis;
    if (a < 0) a += n_axis;
    const T* src = in + base0 + c;
    T* dst = tile + r * TI + c;
    if (a0 + lo >= 0 && a0 + lo + rows <= n_axis) {
      // no wrap anywhere in the tile (interior CTAs): one pointer bump per row
      const long long step = (long long)dr * stride;
      const T* p = src + (long long)a * stride;
      for (; r < rows; r += dr, dst += dr * TI, p += step) cp_async16h(dst, p, pol);
    } else if (n_axis >= dr) {  // at most one wrap per step
      for (; r < rows; r += dr, dst += dr * TI) {
        cp_async16h(dst, src + (long long)a * stride, pol);
        a += dr;
        a = a >= n_axis ? a - n_axis : a;
      }
    } else {
      for (; r < rows; r += dr, dst += dr * TI) {
        cp_async16h(dst, src + (long long)a * stride, pol);
        a = (a + dr) % n_axis;
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int il = threadIdx.x % TI, ag = threadIdx.x / TI;
  const T* src = tile + (ag * J) * TI + il;
  T W[J], acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    W[j] = src[j * TI];
    acc[j] = T(0);
  }
  int q0 = 0;
  for (; q0 + J <= nt4; q0 += J) {
#pragma unroll
    for (int r = 0; r < J; r += 4) {
      T t4[4];
      ld4(taps + q0 + r, t4[0], t4[1], t4[2], t4[3]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int j = 0; j < J; ++j) acc[j] = fma(t4[k], W[(r + k + j) % J], acc[j]);
        W[r + k] = src[(q0 + r + k + J) * TI];
      }
    }
  }
  // remaining taps (< J, a multiple of 4): same rotation, guarded 4-tap steps
#pragma unroll
  for (int r = 0; r < J; r += 4) {
    if (q0 + r >= nt4) break;
    T t4[4];
    ld4(taps + q0 + r, t4[0], t4[1], t4[2], t4[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma(t4[k], W[(r + k + j) % J], acc[j]);
      W[r + k] = src[(q0 + r + k + J) * TI];
    }
  }
  {
    const int a1 = a0 + ag * J;
    const long long o0 = base0 + (long long)(a1 + out_shift) * stride + il;
    T* po = out + o0;
    if (!addend && a1 + J <= a_end) {  // full group: unguarded stores
      if (w == T(1)) {
#pragma unroll
        for (int j = 0; j < J; ++j, po += stride) *po = acc[j];
      } else {
#pragma unroll
        for (int j = 0; j < J; ++j, po += stride) *po = T(w * acc[j]);
      }
    } else if (addend) {
      const T* pa = addend + o0;
      double sq = 0.0;  // (fused residual: sum of squares of what is stored)
#pragma unroll
      for (int j = 0; j < J; ++j, po += stride, pa += stride)
        if (a1 + j < a_end) {
          const T v = T(aw * *pa + w * acc[j]);
          *po = v;
          sq += double(v) * double(v);
        }
      if (sq_parts) {  // per-CTA fp64 partial, fixed-order tree
        __shared__ double red[NT / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
          double t = 0.0;
          for (int q = 0; q < NT / 32; ++q) t += red[q];
          sq_parts[blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z)] = t;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < J; ++j, po += stride)
        if (a1 + j < a_end) *po = T(w * acc[j]);
    }
  }
}


// Strided axes, fp32, WIDE filters: pass_tile2_kernel with packed FFMA2.
// Lane l owns the inner pair (2l, 2l + 1) of a 64-wide column block (one
// 8-byte LDS per staged row), so every tap is one FFMA2 per output pair: half
// the FMA issue slots of the scalar tile at the same per-element arithmetic
// (two independent RN FMAs, bit-identical results). 8 groups of J outputs
// along the axis per CTA (To = 8 J); taps stored duplicated (t, t).
template <int J, int MINB, int NT = 256>
__global__ void __launch_bounds__(NT, MINB) pass_tile2x2_kernel(
    const float* __restrict__ in, float* __restrict__ out, int n_axis, long long stride,
    const float* __restrict__ taps_g, int lo, int ntaps, int a_begin, int a_end, int out_shift,
    int l2mode) {
  constexpr int TI = 64, G = NT / 32, To = J * G;
  const unsigned long long pol = l2_policy(l2mode);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nt4 = (ntaps + 3) & ~3;
  f32x2* taps2 = reinterpret_cast<f32x2*>(smem_raw);        // [nt4] (t, t)
  float* tile = reinterpret_cast<float*>(taps2 + nt4);      // [To + nt4][TI]
  const int rows = To + nt4;
  const int a0 = a_begin + blockIdx.x * To;
  const long long base0 = (long long)blockIdx.z * n_axis * stride + (long long)blockIdx.y * TI;
  for (int q = threadIdx.x; q < nt4; q += NT) {
    const float t = q < ntaps ? taps_g[q] : 0.f;
    taps2[q] = pack2(t, t);
  }
  {
    constexpr int kRowVecs = TI / 4, dr = NT / kRowVecs;
    const int c = (threadIdx.x % kRowVecs) * 4;
    int r = threadIdx.x / kRowVecs;
    int a = (a0 + lo + r) % n_axis;
    if (a < 0) a += n_axis;
    const float* src = in + base0 + c;
    float* dst = tile + r * TI + c;
    if (a0 + lo >= 0 && a0 + lo + rows <= n_axis) {
      const long long step = (long long)dr * stride;
      const float* p = src + (long long)a * stride;
      for (; r < rows; r += dr, dst += dr * TI, p += step) cp_async16h(dst, p, pol);
    } else if (n_axis >= dr) {
      for (; r < rows; r += dr, dst += dr * TI) {
        cp_async16h(dst, src + (long long)a * stride, pol);
        a += dr;
        a = a >= n_axis ? a - n_axis : a;
      }
    } else {
      for (; r < rows; r += dr, dst += dr * TI) {
        cp_async16h(dst, src + (long long)a * stride, pol);
        a = (a + dr) % n_axis;
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, ag = threadIdx.x >> 5;
  const f32x2* src = reinterpret_cast<const f32x2*>(tile + (ag * J) * TI) + lane;  // row pitch TI / 2 pairs
  constexpr int P = TI / 2;
  f32x2 W[J], acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    W[j] = src[j * P];
    acc[j] = 0ull;
  }
  int q0 = 0;
  for (; q0 + J <= nt4; q0 += J) {
#pragma unroll
    for (int r = 0; r < J; r += 2) {
      const ulonglong2 t2 = *reinterpret_cast<const ulonglong2*>(taps2 + q0 + r);
      const f32x2 tt[2] = {t2.x, t2.y};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
#pragma unroll
        for (int j = 0; j < J; ++j) acc[j] = fma2(tt[k], W[(r + k + j) % J], acc[j]);
        W[r + k] = src[(q0 + r + k + J) * P];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < J; r += 2) {  // remaining taps (< J, a multiple of 4)
    if (q0 + r >= nt4) break;
    const ulonglong2 t2 = *reinterpret_cast<const ulonglong2*>(taps2 + q0 + r);
    const f32x2 tt[2] = {t2.x, t2.y};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma2(tt[k], W[(r + k + j) % J], acc[j]);
      W[r + k] = src[(q0 + r + k + J) * P];
    }
  }
  const int a1 = a0 + ag * J;
  f32x2* po = reinterpret_cast<f32x2*>(out + base0 + (long long)(a1 + out_shift) * stride) + lane;
  const long long pstep = stride / 2;
  if (a1 + J <= a_end) {
#pragma unroll
    for (int j = 0; j < J; ++j, po += pstep) *po = acc[j];
  } else {
#pragma unroll
    for (int j = 0; j < J; ++j, po += pstep)
      if (a1 + j < a_end) *po = acc[j];
  }
}

// Contiguous axis (2), nz % 4 == 0: a CTA owns 32 rows (lane = row) x 4 J
// outputs (warp = J-column group). The staged row span starts at the aligned
// column floor4(z0 + lo); the misalignment sh = lo mod 4 is absorbed by sh
// leading zero taps, so the window is the shared Fold<T, J, 1> register
// window (LDS.128 per 4 taps, pitch = 4 mod 8 words: conflict-free). Results
// go back through shared memory for coalesced stores.
template <typename T, int J, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) pass_z2_kernel(
    const T* __restrict__ in, T* __restrict__ out, int nz, long long nrows,
    const T* __restrict__ taps_g, int lo, int ntaps, int pitch, const T* addend, T aw, T w,
    int l2mode) {
  constexpr int kVec = 16 / sizeof(T);
  const unsigned long long pol = l2_policy(l2mode);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int sh = ((lo % 4) + 4) % 4;
  const int nt4 = (ntaps + sh + 3) & ~3;
  T* taps = reinterpret_cast<T*>(smem_raw);  // [nt4 + 8]: sh zeros, taps, zeros
  T* tile = taps + nt4 + 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long row0 = (long long)blockIdx.y * 32;
  const int z0 = blockIdx.x * (4 * J);
  for (int q = threadIdx.x; q < nt4 + 8; q += 128)
    taps[q] = (q >= sh && q - sh < ntaps) ? taps_g[q - sh] : T(0);
  // staged columns [zs, zs + width), zs = z0 + lo - sh (aligned), wrapped
  const int width = 4 * J + nt4 + 4;
  const int nv = width / kVec;
  {
    int zs = (z0 + lo - sh) % nz;
    if (zs < 0) zs += nz;
    // lanes over 16-byte vectors of a row (wrapped column per lane is fixed
    // across rows), warps over rows
    if (row0 + 32 <= nrows) {
      // full row group: one wrap test per vector, one pointer bump per row
      const long long step = 4LL * nz;
      for (int v = lane; v < nv; v += 32) {
        int z = zs + v * kVec;
        if (z >= nz) z = z < 2 * nz ? z - nz : z % nz;
        const T* p = in + (row0 + warp) * nz + z;
        T* d = tile + warp * pitch + v * kVec;
#pragma unroll
        for (int i = 0; i < 8; ++i, p += step, d += 4 * pitch) cp_async16h(d, p, pol);
      }
    } else
    for (int v = lane; v < nv; v += 32) {
      int z = (zs + v * kVec) % nz;
      for (int r = warp; r < 32; r += 4) {
        const long long row = row0 + r;
        T* d = tile + r * pitch + v * kVec;
        if (row < nrows)
          cp_async16h(d, in + row * nz + z, pol);
        else
          for (int k = 0; k < kVec; ++k) d[k] = T(0);
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  T acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) acc[j] = T(0);
  {
    const T* const q[1] = {tile + lane * pitch + warp * J};
    Fold<T, J, 1>::row(acc, taps, q, nt4 / 4);
  }
  const long long row = row0 + lane;
  const int zc = z0 + warp * J;
  if (!addend && row0 + 32 <= nrows && z0 + 4 * J <= nz) {
    // narrow filters: transpose through shared memory so every warp store
    // instruction writes whole rows (2 x 256 contiguous bytes)
    __syncthreads();  // every thread is done reading the staged input
    T* res = tile + lane * pitch + warp * J;
#pragma unroll
    for (int j = 0; j < J; j += 4) {
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(res + j) = make_float4(w * acc[j], w * acc[j + 1], w * acc[j + 2], w * acc[j + 3]);
      } else {
        *reinterpret_cast<double2*>(res + j) = make_double2(w * acc[j], w * acc[j + 1]);
        *reinterpret_cast<double2*>(res + j + 2) = make_double2(w * acc[j + 2], w * acc[j + 3]);
      }
    }
    __syncthreads();
    constexpr int vpr = 4 * J / kVec;  // 16-byte vectors per row
#pragma unroll
    for (int e = threadIdx.x; e < 32 * vpr; e += 128) {
      const int r = e / vpr, v = e - r * vpr;
      const T* sv = tile + r * pitch + v * kVec;
      T* dv = out + (row0 + r) * nz + z0 + v * kVec;
      if constexpr (sizeof(T) == 4)
        st_out(l2mode, reinterpret_cast<float4*>(dv), *reinterpret_cast<const float4*>(sv));
      else
        st_out(l2mode, reinterpret_cast<double2*>(dv), *reinterpret_cast<const double2*>(sv));
    }
    return;
  }
  if (!addend) {
    // straight from registers: J consecutive outputs per thread as 16-byte
    // vector stores (the two halves of each 32-byte sector come from the
    // same thread's consecutive stores)
    if (row < nrows) {
      T* po = out + row * nz + zc;
#pragma unroll
      if (w == T(1) && zc + J <= nz) {
#pragma unroll
        for (int j = 0; j < J; j += 4) {
          if constexpr (sizeof(T) == 4) {
            st_out(l2mode, reinterpret_cast<float4*>(po + j), make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
          } else {
            st_out(l2mode, reinterpret_cast<double2*>(po + j), make_double2(acc[j], acc[j + 1]));
            st_out(l2mode, reinterpret_cast<double2*>(po + j + 2), make_double2(acc[j + 2], acc[j + 3]));
          }
        }
        return;
      }
#pragma unroll
      for (int j = 0; j < J; j += 4) {
        if (zc + j >= nz) break;
        if constexpr (sizeof(T) == 4) {
          st_out(l2mode, reinterpret_cast<float4*>(po + j),
                 make_float4(w * acc[j], w * acc[j + 1], w * acc[j + 2], w * acc[j + 3]));
        } else {
          st_out(l2mode, reinterpret_cast<double2*>(po + j), make_double2(w * acc[j], w * acc[j + 1]));
          st_out(l2mode, reinterpret_cast<double2*>(po + j + 2), make_double2(w * acc[j + 2], w * acc[j + 3]));
        }
      }
    }
    return;
  }
  __syncthreads();  // every thread is done reading the staged input
  T* res = tile + lane * pitch + warp * J;
#pragma unroll
  for (int j = 0; j < J; j += 4) {
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float4*>(res + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    } else {
      *reinterpret_cast<double2*>(res + j) = make_double2(acc[j], acc[j + 1]);
      *reinterpret_cast<double2*>(res + j + 2) = make_double2(acc[j + 2], acc[j + 3]);
    }
  }
  __syncthreads();
  const int ncols = 4 * J;
  for (int e = threadIdx.x; e < 32 * ncols; e += 128) {
    const int r = e / ncols, c = e - r * ncols;
    const long long rw = row0 + r;
    const int z = z0 + c;
    if (rw < nrows && z < nz) {
      const long long o = rw * nz + z;
      out[o] = T(aw * addend[o] + w * tile[r * pitch + c]);
    }
  }
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

template <typename T, int J>
int launch_strided(sfw3d_ctx* ctx, const T* in, T* out, const int dims[3], int axis, const T* taps,
                   int lo, int ntaps, const T* addend, double aw, double w, const XRange& xr) {
  long long stride = 1;
  for (int a = axis + 1; a < 3; ++a) stride *= dims[a];
  long long outer = 1;
  for (int a = 0; a < axis; ++a) outer *= dims[a];
  const int n = dims[axis];
  const int ab = xr.begin, ae = xr.end < 0 ? n : xr.end;
  dim3 grid(unsigned((ae - ab + J - 1) / J), unsigned((stride + 255) / 256), unsigned(outer));
  const size_t smem = size_t((ntaps + J - 1) / J * J) * sizeof(T);
  if (smem > 48 * 1024)
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(pass_strided_kernel<T, J>), size_t(int(smem))));
  pass_strided_kernel<T, J><<<grid, 256, smem, ctx->stream>>>(
      in, out, n, stride, taps, lo, ntaps, addend, T(aw), T(w), ab, ae, xr.shift);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}


template <typename T, int J>
int launch_z(sfw3d_ctx* ctx, const T* in, T* out, const int dims[3], const T* taps, int lo,
             int ntaps, const T* addend, double aw, double w) {
  const long long nrows = (long long)dims[0] * dims[1];
  const int npad = (ntaps + J - 1) / J * J;
  const int width = J * kZWarps + npad;
  const int pitch = width | 1;  // odd: 32 lanes on 32 rows hit 32 banks
  const size_t smem = (size_t(npad) + size_t(kZRows) * pitch) * sizeof(T);
  if (smem > 48 * 1024)
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(pass_z_kernel<T, J>), size_t(int(smem))));
  dim3 grid(unsigned((dims[2] + J * kZWarps - 1) / (J * kZWarps)),
            unsigned((nrows + kZRows - 1) / kZRows));
  pass_z_kernel<T, J><<<grid, 32 * kZWarps, smem, ctx->stream>>>(in, out, dims[2], nrows, taps, lo,
                                                                  ntaps, pitch, addend, T(aw), T(w));
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

template <typename T, int J, int MINB = 1, int NT = 256>
int launch_tile2(sfw3d_ctx* ctx, const T* in, T* out, const int dims[3], int axis, const T* taps,
                 int lo, int ntaps, const T* addend, double aw, double w, const XRange& xr) {
  constexpr int TI = 64, To = J * (NT / TI);
  long long stride = 1;
  for (int a = axis + 1; a < 3; ++a) stride *= dims[a];
  long long outer = 1;
  for (int a = 0; a < axis; ++a) outer *= dims[a];
  const int n = dims[axis];
  const int nt4 = (ntaps + 3) & ~3;
  const size_t smem = (size_t(nt4) + size_t(To + nt4) * TI) * sizeof(T);
  if (smem > 48 * 1024)
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(pass_tile2_kernel<T, J, TI, NT, MINB>), size_t(int(smem))));
  const int ab = xr.begin, ae = xr.end < 0 ? n : xr.end;
  dim3 grid(unsigned((ae - ab + To - 1) / To), unsigned(stride / TI), unsigned(outer));
  pass_tile2_kernel<T, J, TI, NT, MINB><<<grid, NT, smem, ctx->stream>>>(
      in, out, n, stride, taps, lo, ntaps, addend, T(aw), T(w), ab, ae, xr.shift, xr.sq, ctx->l2mode);
  xr.nsq = int(grid.x * grid.y * grid.z);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}


template <int J, int MINB, int NT = 256>
int launch_tile2x2(sfw3d_ctx* ctx, const float* in, float* out, const int dims[3], int axis,
                   const float* taps, int lo, int ntaps, const XRange& xr) {
  constexpr int TI = 64, To = J * (NT / 32);
  long long stride = 1;
  for (int a = axis + 1; a < 3; ++a) stride *= dims[a];
  long long outer = 1;
  for (int a = 0; a < axis; ++a) outer *= dims[a];
  const int n = dims[axis];
  const int nt4 = (ntaps + 3) & ~3;
  const size_t smem = size_t(nt4) * 8 + size_t(To + nt4) * TI * sizeof(float);
  if (smem > 48 * 1024)
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(pass_tile2x2_kernel<J, MINB, NT>), size_t(int(smem))));
  const int ab = xr.begin, ae = xr.end < 0 ? n : xr.end;
  dim3 grid(unsigned((ae - ab + To - 1) / To), unsigned(stride / TI), unsigned(outer));
  pass_tile2x2_kernel<J, MINB, NT><<<grid, NT, smem, ctx->stream>>>(in, out, n, stride, taps, lo,
                                                                 ntaps, ab, ae, xr.shift, ctx->l2mode);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

template <typename T, int J, int MINB = 1>
int launch_z2(sfw3d_ctx* ctx, const T* in, T* out, const int dims[3], const T* taps, int lo,
              int ntaps, const T* addend, double aw, double w) {
  const long long nrows = (long long)dims[0] * dims[1];
  const int sh = ((lo % 4) + 4) % 4;
  const int nt4 = (ntaps + sh + 3) & ~3;
  const int width = 4 * J + nt4 + 4;
  // 16-byte rows whose 16-byte chunk index advances by an odd number per row
  int pitch = (width + 3) & ~3;
  if (sizeof(T) == 4) {
    if (pitch % 8 != 4) pitch += 4;
  } else {
    if (pitch % 4 != 2) pitch += 2;
  }
  const size_t smem = (size_t(nt4) + 8 + size_t(32) * pitch) * sizeof(T);
  if (smem > 48 * 1024)
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(pass_z2_kernel<T, J, MINB>), size_t(int(smem))));
  dim3 grid(unsigned((dims[2] + 4 * J - 1) / (4 * J)), unsigned((nrows + 31) / 32));
  pass_z2_kernel<T, J, MINB><<<grid, 128, smem, ctx->stream>>>(in, out, dims[2], nrows, taps, lo, ntaps,
                                                         pitch, addend, T(aw), T(w), ctx->l2mode);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

// Packed strided tile by filter length: up to 64 taps the 128-thread CTA (4
// groups of 16 outputs: 6 resident CTAs per SM instead of 3, so the staging,
// FMA and store phases of different CTAs overlap better — config 4 11.22 ->
// 11.01 ms, 256^3 certificate 2.03 -> 1.90 ms); longer filters keep the
// 256-thread tile, whose halo rows are a smaller share of the staged tile.
inline int launch_x2(sfw3d_ctx* ctx, const float* in, float* out, const int dims[3], int axis,
                     const float* taps, int lo, int ntaps, const XRange& xr) {
  if (ntaps <= 64) return launch_tile2x2<16, 6, 128>(ctx, in, out, dims, axis, taps, lo, ntaps, xr);
  return launch_tile2x2<16, 3>(ctx, in, out, dims, axis, taps, lo, ntaps, xr);
}

// Tile choice. Wide filters (> kNarrowTaps taps) take J = 32 outputs per
// thread; fp32 wide tiles are register-capped for 3 (strided) / 5
// (contiguous) resident CTAs per SM (measured 29.1 -> 27.7 ms over the
// config-4 basis passes). fp64 keeps the unconstrained allocation: with
// twice the registers per value the capped tiles spill (round-1 ptxas log).
// Narrow filters are HBM-bound: the J = 16 tile keeps more CTAs resident.
constexpr int kNarrowTaps = 24;

// A pass chain ping-pongs between two volumes. Up to 72 MiB per volume
// (256^3 fp32) the pair stays L2-resident on B200 when consumed input lines
// are marked evict-first and output lines are stored normally: measured
// 9.0 TB/s against 5.8 TB/s for a copy-shaped pass at 64 MiB
// (tools/micro/l2_pingpong.cu); no gain from 96 MiB on.
inline int l2_mode_for(size_t vol_bytes) {
  return vol_bytes <= (size_t(72) << 20) ? 1 : 0;
}

template <typename T>
int pass_typed(sfw3d_ctx* ctx, const T* in, T* out, const int dims[3], int axis, const T* taps,
               int lo, int ntaps, const T* addend, double aw, double w, const XRange& xr) {
  if (ntaps > 4096) {
    set_error("1-D pass with more than 4096 taps");
    return SFW3D_EINVAL;
  }
  constexpr bool f32 = sizeof(T) == 4;
  const bool wide = ntaps > kNarrowTaps;
  ctx->l2mode = l2_mode_for(size_t(vol_count(dims)) * sizeof(T));
  if (xr.sq && !(axis == 0 && addend && (dims[1] * (long long)dims[2]) % 64 == 0 && ntaps <= 512)) {
    set_error("internal: fused sum of squares needs an axis-0 tiled pass with an addend");
    return SFW3D_EINVAL;
  }
  if (axis != 0 && (xr.begin != 0 || xr.end >= 0 || xr.shift != 0)) {
    set_error("internal: output plane ranges apply to axis-0 passes only");
    return SFW3D_EINVAL;
  }
  if (axis == 2) {
    if (dims[2] % 4 == 0 && ntaps <= 1024) {
      if (dims[2] >= 128 && wide) {
        if constexpr (f32) return launch_z2<T, 32, 5>(ctx, in, out, dims, taps, lo, ntaps, addend, aw, w);
        else return launch_z2<T, 32, 1>(ctx, in, out, dims, taps, lo, ntaps, addend, aw, w);
      }
      if constexpr (f32) return launch_z2<T, 16, 8>(ctx, in, out, dims, taps, lo, ntaps, addend, aw, w);
      else return launch_z2<T, 16>(ctx, in, out, dims, taps, lo, ntaps, addend, aw, w);
    }
    return wide ? launch_z<T, 32>(ctx, in, out, dims, taps, lo, ntaps, addend, aw, w)
                : launch_z<T, 16>(ctx, in, out, dims, taps, lo, ntaps, addend, aw, w);
  }
  long long stride = 1;
  for (int a = axis + 1; a < 3; ++a) stride *= dims[a];
  if (stride % 64 == 0 && ntaps <= 512) {
    // (an x-slab's output range shorter than the 128-plane wide tile takes
    // the 64-plane tile: 2 groups of 32 instead of 4)
    const int range = (xr.end < 0 ? dims[axis] : xr.end) - xr.begin;
    if (dims[axis] >= 128 && wide && range <= 64) {
      if constexpr (f32) {
        // (the 64-output packed tile is exactly an 8-rank slab of 512 planes)
        if (!addend && w == 1.0 && xr.sq == nullptr && ntaps <= 64)
          return launch_tile2x2<16, 6, 128>(ctx, in, out, dims, axis, taps, lo, ntaps, xr);
      }
      if constexpr (f32) return launch_tile2<T, 32, 5, 128>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr);
      else return launch_tile2<T, 32, 1, 128>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr);
    }
    if (dims[axis] >= 128 && wide) {
      if constexpr (f32) {
        if (!addend && w == 1.0 && xr.sq == nullptr)  // packed FFMA2 tile
          return launch_x2(ctx, in, out, dims, axis, taps, lo, ntaps, xr);
        return launch_tile2<T, 32, 3>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr);
      } else {
        return launch_tile2<T, 32, 1>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr);
      }
    }
    if constexpr (f32) {
      // (packed FFMA2 tile also for narrow filters: 512^3 15-tap y/x passes
      // 0.218 -> 0.205 ms, bit-identical)
      if (dims[axis] >= 128 && !addend && w == 1.0 && xr.sq == nullptr)
        return launch_x2(ctx, in, out, dims, axis, taps, lo, ntaps, xr);
      return launch_tile2<T, 16, 5>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr);
    }
    else return launch_tile2<T, 16>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr);
  }
  return wide ? launch_strided<T, 32>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr)
              : launch_strided<T, 8>(ctx, in, out, dims, axis, taps, lo, ntaps, addend, aw, w, xr);
}

}  // namespace

int corr_pass_impl(sfw3d_ctx* ctx, int dtype, const void* in, void* out, const int dims[3], int axis,
                   const void* taps, int lo, int ntaps, const void* addend, double addend_w,
                   double w, const char* family, const XRange* xr) {
  SFW3D_PROF(ctx, family);
  const XRange full{};
  const XRange& r = xr ? *xr : full;
  if (dtype == SFW3D_F64)
    return pass_typed<double>(ctx, static_cast<const double*>(in), static_cast<double*>(out), dims,
                              axis, static_cast<const double*>(taps), lo, ntaps,
                              static_cast<const double*>(addend), addend_w, w, r);
  return pass_typed<float>(ctx, static_cast<const float*>(in), static_cast<float*>(out), dims, axis,
                           static_cast<const float*>(taps), lo, ntaps,
                           static_cast<const float*>(addend), addend_w, w, r);
}

// Separable correlation of an x-slab: `in` holds the rank's n_own owned
// planes (compact), `out` receives the same planes of f_x (x) f_y (x) f_z * in
// of the GLOBAL periodic volume. The z and y passes are plane-local (owned
// planes only, into the middle of `win`); the x pass needs lo_x = -xlo / hi_x
// = xlo + lx - 1 planes of the neighbours' y/z-passed data, which the caller's
// exchange (sfw3d_halo_fn) writes into the halo planes of `win`; the x pass
// then reads the window and writes the owned planes only. win: (H + n_own +
// H) planes with H >= both halos; tmp: one owned-size volume.
int slab_corr_impl(sfw3d_ctx* ctx, int dtype, const void* in, void* out, const int odims[3],
                   const void* const taps[3], const int lo[3], const int nt[3], void* win, int H,
                   void* tmp, const SlabLink& link, const char* family) {
  const size_t es = dtype_size(dtype);
  const long long plane = (long long)odims[1] * odims[2];
  const int lox = std::max(0, -lo[0]), hix = std::max(0, lo[0] + nt[0] - 1);
  if (lox > H || hix > H) {
    set_error("internal: x-slab window narrower than the pass halo");
    return SFW3D_EINVAL;
  }
  char* mid = static_cast<char*>(win) + size_t(H) * plane * es;
  SFW3D_TRY(corr_pass_impl(ctx, dtype, in, tmp, odims, 2, taps[2], lo[2], nt[2], nullptr, 0.0, 1.0,
                           family));
  SFW3D_TRY(corr_pass_impl(ctx, dtype, tmp, mid, odims, 1, taps[1], lo[1], nt[1], nullptr, 0.0,
                           1.0, family));
  if (link.halo) {
    // the exchange sees the window [H - lox, H + n_own + hix)
    char* w0 = mid - size_t(lox) * plane * es;
    if (link.halo(link.user, w0, dtype, odims[0], plane, lox, hix) != 0) {
      set_error("halo exchange callback failed");
      return SFW3D_ECUDA;
    }
  }
  const int wd[3] = {odims[0] + 2 * H, odims[1], odims[2]};
  const XRange xr{H, H + odims[0], -H};
  return corr_pass_impl(ctx, dtype, win, out, wd, 0, taps[0], lo[0], nt[0], nullptr, 0.0, 1.0,
                        family, &xr);
}

// out = H * in - y (the residual, forward.py:249-252) with the x pass's
// epilogue subtracting y and adding up the fp64 squares per CTA into sq_parts
// (returns their count in *nparts); 0 partials = not applicable (the caller
// uses psf_apply_impl + sumsq_diff_impl).
int psf_apply_resid(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                    void* tmp, const void* y, double* sq_parts, int max_parts, int* nparts) {
  *nparts = 0;
  const int* dims = psf->dims;
  const int nt0 = psf->hi[0] - psf->lo[0] + 1;
  if (!psf->separable || (dims[1] * (long long)dims[2]) % 64 != 0 || nt0 > 512) return SFW3D_OK;
  // (the x pass's grid: at most ceil(n / 64) x (ny nz / 64) CTAs)
  const long long ctas = (long long)((dims[0] + 63) / 64) * (dims[1] * (long long)dims[2] / 64);
  if (ctas > max_parts) return SFW3D_OK;
  int lo[3], nt[3];
  const void* tp[3];
  for (int a = 0; a < 3; ++a) {
    nt[a] = psf->hi[a] - psf->lo[a] + 1;
    lo[a] = -psf->hi[a];
    tp[a] = dtype == SFW3D_F64 ? static_cast<const void*>(psf->taps64[a] + nt[a])
                               : static_cast<const void*>(psf->taps32[a] + nt[a]);
  }
  SFW3D_TRY(corr_pass_impl(ctx, dtype, in, out, dims, 2, tp[2], lo[2], nt[2], nullptr, 0.0, 1.0,
                           "psf_pass"));
  SFW3D_TRY(corr_pass_impl(ctx, dtype, out, tmp, dims, 1, tp[1], lo[1], nt[1], nullptr, 0.0, 1.0,
                           "psf_pass"));
  XRange xr;
  xr.sq = sq_parts;
  SFW3D_TRY(corr_pass_impl(ctx, dtype, tmp, out, dims, 0, tp[0], lo[0], nt[0], y, -1.0, 1.0,
                           "psf_pass", &xr));
  *nparts = xr.nsq;
  return SFW3D_OK;
}

int psf_apply_slab(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                   int adjoint, const int odims[3], void* win, int H, void* tmp,
                   const SlabLink& link) {
  if (!psf->separable) {
    set_error("x-slab sharding needs a separable PSF");
    return SFW3D_EINVAL;
  }
  int lo[3], nt[3];
  const void* tp[3];
  for (int a = 0; a < 3; ++a) {
    nt[a] = psf->hi[a] - psf->lo[a] + 1;
    lo[a] = adjoint ? psf->lo[a] : -psf->hi[a];
    if (dtype == SFW3D_F64)
      tp[a] = adjoint ? psf->taps64[a] : psf->taps64[a] + nt[a];
    else
      tp[a] = adjoint ? psf->taps32[a] : psf->taps32[a] + nt[a];
  }
  return slab_corr_impl(ctx, dtype, in, out, odims, tp, lo, nt, win, H, tmp, link, "psf_pass");
}


int psf_apply_impl(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* in, void* out,
                   int adjoint, void* tmp) {
  const int* dims = psf->dims;
  if (psf->separable) {
    // adjoint: correlation with taps over [lo, hi]; forward: convolution =
    // correlation with reversed taps over [-hi, -lo] (stored after the
    // forward taps, see sfw3d_psf_create).
    int lo[3], nt[3];
    const void* tp[3];
    for (int a = 0; a < 3; ++a) {
      nt[a] = psf->hi[a] - psf->lo[a] + 1;
      lo[a] = adjoint ? psf->lo[a] : -psf->hi[a];
      if (dtype == SFW3D_F64)
        tp[a] = adjoint ? psf->taps64[a] : psf->taps64[a] + nt[a];
      else
        tp[a] = adjoint ? psf->taps32[a] : psf->taps32[a] + nt[a];
    }
    SFW3D_TRY(corr_pass_impl(ctx, dtype, in, out, dims, 2, tp[2], lo[2], nt[2], nullptr, 0.0,
                             1.0, "psf_pass"));
    SFW3D_TRY(corr_pass_impl(ctx, dtype, out, tmp, dims, 1, tp[1], lo[1], nt[1], nullptr, 0.0,
                             1.0, "psf_pass"));
    SFW3D_TRY(corr_pass_impl(ctx, dtype, tmp, out, dims, 0, tp[0], lo[0], nt[0], nullptr, 0.0, 1.0,
                             "psf_pass"));
    return SFW3D_OK;
  }
  if (psf_use_fft(psf)) return psf_fft_apply(ctx, psf, dtype, in, out, adjoint);
  const long long n = vol_count(dims);
  const int l0 = psf->hi[0] - psf->lo[0] + 1, l1 = psf->hi[1] - psf->lo[1] + 1,
            l2 = psf->hi[2] - psf->lo[2] + 1;
  SFW3D_PROF(ctx, "psf_pass");
  if (dtype == SFW3D_F64)
    stencil3d_kernel<double><<<unsigned((n + 255) / 256), 256, 0, ctx->stream>>>(
        static_cast<const double*>(in), static_cast<double*>(out), dims[0], dims[1], dims[2],
        psf->box64, psf->lo[0], psf->lo[1], psf->lo[2], l0, l1, l2, adjoint ? 1 : -1);
  else
    stencil3d_kernel<float><<<unsigned((n + 255) / 256), 256, 0, ctx->stream>>>(
        static_cast<const float*>(in), static_cast<float*>(out), dims[0], dims[1], dims[2],
        psf->box32, psf->lo[0], psf->lo[1], psf->lo[2], l0, l1, l2, adjoint ? 1 : -1);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

}  // namespace sfw3d
