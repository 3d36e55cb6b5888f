// K3 / K6 / K7 — generalized-Gaussian atoms on their support boxes.
//
// Restates _unit_atom (forward.py:119-152), _accumulate_atoms
// (forward.py:165-174) and the per-atom inner products of _gradient_rows
// (forward.py:209-229) / neg_eta (certificate.py:201-209).
//
//  * render: deterministic GATHER. One CTA owns a 4x8x16 brick, compacts
//    (in row order) the atoms whose wrapped box meets the brick, tabulates
//    each listed atom's per-axis offsets for the brick's 4 + 8 + 16
//    coordinates once in shared memory, and each thread sums w*G for its
//    voxel in atom order — the reference's per-voxel summation order
//    (acc[box] += w*values, atom by atom), no float atomics.
//  * atom sums: each atom box is cut into fixed 4096-voxel chunks; a CTA
//    tabulates the atom's per-axis (wrapped index, offset) once, then reduces
//    the six products <P_c, field> over its chunk (fp64 across threads); a
//    second kernel adds the chunk partials of each atom in chunk order.
// fp64 volumes use fp64 math with products/sums rounded exactly as numpy
// does (no FMA contraction where the reference rounds twice); fp32 volumes
// use fp32 math on the MUFU (ex2/lg2/rcp) with fp64 accumulation.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <type_traits>

#include "internal.cuh"

namespace sfw3d {
namespace {

constexpr int kChunk = 4096;               // atom-sum chunk (voxels)
constexpr int kSumThreads = 256;

constexpr int kMaxAxis = 1024;             // tabulated axis length in atom sums
constexpr int kMaxRows = 512;              // rows per chunk (fp64)
// fp32: 4x larger chunks (amortise the row table and the fp64 block
// reduction over 64 voxels per thread)
constexpr int kChunk32 = 16384, kMaxRows32 = 2048;
template <typename T>
constexpr int max_rows() { return sizeof(T) == 8 ? kMaxRows : kMaxRows32; }
static int chunk32() { return kChunk32; }

// a mod n in [0, n) without a division on the common path (|a| < 2n)
__device__ __forceinline__ int pmod(int a, int n) {
  if (a < 0) {
    a += n;
    if (a < 0) a = (a % n + n) % n;
  } else if (a >= n) {
    a -= n;
    if (a >= n) a %= n;
  }
  return a;
}

// Minimum-image offset of voxel i from centre m on a full axis
// (forward.py:109): np.remainder(i - m + n/2, n) - n/2 with numpy's
// fmod-then-adjust remainder.
__device__ __forceinline__ double min_image(int i, double m, int n) {
  double x = __dadd_rn(__dsub_rn(double(i), m), double(n) * 0.5);
  double r = fmod(x, double(n));
  if (r != 0.0 && r < 0.0) r = __dadd_rn(r, double(n));
  return __dsub_rn(r, double(n) * 0.5);
}

// Offset of global voxel index g from the atom centre along one axis, or
// false when g is outside the atom's box (forward.py:102-116).
__device__ __forceinline__ bool axis_offset(const AtomGeo& a, int axis, int g, int n, double& off) {
  if (a.full[axis]) {
    off = min_image(g, a.m[axis], n);
    return true;
  }
  int il = pmod(g - a.start[axis], n);
  if (il >= a.len[axis]) return false;
  off = __dsub_rn(double(a.start[axis] + il), a.m[axis]);
  return true;
}

__device__ __forceinline__ bool box_meets(const AtomGeo& a, int axis, int b0, int b1, int n) {
  if (a.full[axis]) return true;
  int s = pmod(a.start[axis], n);
  int e = s + a.len[axis] - 1;
  if (e < n) return !(e < b0 || s > b1);
  return (b1 >= s) || (b0 <= e - n);
}

__device__ __forceinline__ double u2_exact(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// unit profile, fp64 (forward.py:133-137)
__device__ __forceinline__ double profile64(const AtomGeo& a, double u2, double& t) {
  const double p = a.d2 ? u2 : pow(u2, a.half_d);
  t = __dmul_rn(a.inv2sd, p);
  return exp(-t);
}

// single-instruction MUFU transcendentals (flush-to-zero approximations;
// the fp32 storage path's own rounding dominates their error)
// register-pair forms of the packed f32x2 helpers (a pair is two adjacent
// registers: these moves are usually free)
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ void upk2(f32x2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// small non-negative int -> float and small unsigned division without the
// XU (MUFU / conversion) pipe, which bounds the fp32 atom kernels
__device__ __forceinline__ float i2f_small(int i) {  // 0 <= i < 2^23
  return __int_as_float(0x4B000000 + i) - 8388608.f;
}
__device__ __forceinline__ unsigned div_magic(int d) {  // ceil(2^32 / d); 0 stands for d == 1
  return d <= 1 ? 0u : 0xFFFFFFFFu / unsigned(d) + 1u;
}
__device__ __forceinline__ int div_small(int a, unsigned magic) {  // a / d for a * d < 2^32
  return magic ? int(__umulhi(unsigned(a), magic)) : a;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// unit profile, fp32 on the MUFU; lg2u2 returns log2(u2) for reuse
// (u2 = 0: lg2 = -inf, ex2(-inf) = 0, so p = 0 and the profile is 1)
__device__ __forceinline__ float profile32(float inv2sd, float half_d, bool d2, float u2, float& t,
                                           float& lg2u2) {
  lg2u2 = lg2_approx(u2);
  const float p = d2 ? u2 : ex2_approx(half_d * lg2u2);
  t = inv2sd * p;
  return ex2_approx(-1.4426950408889634f * t);
}

// ------------------------------------------------------------------ render
// One CTA per 16 (x) x 16 (y) x 32 (z) superbrick; thread (y, z) owns the
// 16-voxel column along x. The CTA scans the atoms in row order (512 per
// pass), ballot-compacts those whose wrapped box meets the superbrick, and
// per group of kGroup listed atoms tabulates each atom's per-axis offsets
// over the superbrick (inf = outside the box) and its profile parameters in
// shared memory. Threads skip atoms missing their (y, z) at once; the x loop
// accumulates w * G in the reference's per-voxel atom order.
constexpr int kSX = 16, kSY = 16, kSZ = 32, kGroup = 32;

template <typename T>
__global__ void __launch_bounds__(512) render_kernel(const AtomGeo* __restrict__ atoms, int k,
                                                     int nx, int ny, int nz, T* __restrict__ out) {
  using Off = T;  // offsets tabulated in the storage precision (exact for fp64)
  __shared__ int list[512];
  __shared__ int warp_cnt[16];
  __shared__ int list_n;
  __shared__ Off tx[kGroup][kSX], ty[kGroup][kSY], tz[kGroup][kSZ];
  __shared__ float pw[kGroup], pinv[kGroup], phd[kGroup];
  __shared__ int pd2[kGroup];

  const int nbz = (nz + kSZ - 1) / kSZ, nby = (ny + kSY - 1) / kSY;
  const int bz = blockIdx.x % nbz, by = (blockIdx.x / nbz) % nby, bx = blockIdx.x / (nbz * nby);
  const int x0 = bx * kSX, y0 = by * kSY, z0 = bz * kSZ;
  const int x1 = min(x0 + kSX, nx) - 1, y1 = min(y0 + kSY, ny) - 1, z1 = min(z0 + kSZ, nz) - 1;
  const int tid = threadIdx.x;
  // a warp covers a 4 (y) x 8 (z) patch: atoms meeting part of a warp's
  // columns waste fewer lanes than with 32 consecutive z (the per-voxel
  // profile's MUFU ops dominate); stores stay 32-byte sectors
  const int lz = (tid & 7) + 8 * ((tid >> 5) & 3), ly = ((tid >> 3) & 3) + 4 * (tid >> 7);
  const int gy = y0 + ly, gz = z0 + lz;
  const bool live = gy < ny && gz < nz;
  const int lane = tid & 31, warp = tid >> 5;
  const Off kOut = Off(INFINITY);

  // fp64 storage: fp64 sums with the reference's rounding; fp32 storage:
  // fp32 sums (the result is stored in fp32)
  using Acc = typename std::conditional<sizeof(T) == 8, double, float>::type;
  Acc acc[kSX];
#pragma unroll
  for (int i = 0; i < kSX; ++i) acc[i] = Acc(0);
  for (int base = 0; base < k; base += 512) {
    const int ai = base + tid;
    bool hit = false;
    if (ai < k) {
      const AtomGeo& a = atoms[ai];
      hit = box_meets(a, 0, x0, x1, nx) && box_meets(a, 1, y0, y1, ny) &&
            box_meets(a, 2, z0, z1, nz);
    }
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) warp_cnt[warp] = __popc(mask);
    __syncthreads();
    if (tid == 0) {
      int sacc = 0;
      for (int w = 0; w < 16; ++w) {
        const int c = warp_cnt[w];
        warp_cnt[w] = sacc;
        sacc += c;
      }
      list_n = sacc;
    }
    __syncthreads();
    if (hit) list[warp_cnt[warp] + __popc(mask & ((1u << lane) - 1u))] = ai;
    __syncthreads();
    const int cnt = list_n;
    for (int q0 = 0; q0 < cnt; q0 += kGroup) {
      const int nq = min(kGroup, cnt - q0);
      // tabulate the group's offsets over the superbrick (inf = outside)
      for (int e = tid; e < nq * (kSX + kSY + kSZ); e += 512) {
        const int q = e / (kSX + kSY + kSZ), r = e % (kSX + kSY + kSZ);
        const AtomGeo& a = atoms[list[q0 + q]];
        int axis, li, g, n;
        if (r < kSX) { axis = 0; li = r; g = x0 + r; n = nx; }
        else if (r < kSX + kSY) { axis = 1; li = r - kSX; g = y0 + li; n = ny; }
        else { axis = 2; li = r - kSX - kSY; g = z0 + li; n = nz; }
        double off = 0.0;
        const bool in = g < n && axis_offset(a, axis, g, n, off);
        const Off v = in ? Off(off) : kOut;
        if (axis == 0) tx[q][li] = v; else if (axis == 1) ty[q][li] = v; else tz[q][li] = v;
      }
      if (tid < nq) {
        const AtomGeo& a = atoms[list[q0 + tid]];
        pw[tid] = float(a.w);
        pinv[tid] = float(a.inv2sd);
        phd[tid] = float(a.half_d);
        pd2[tid] = a.d2;
      }
      __syncthreads();
      if (live) {
        for (int q = 0; q < nq; ++q) {
          const Off oy = ty[q][ly], oz = tz[q][lz];
          if (oy == kOut || oz == kOut) continue;
          if constexpr (sizeof(T) == 8) {
            const AtomGeo& a = atoms[list[q0 + q]];
#pragma unroll
            for (int i = 0; i < kSX; ++i) {
              const Off ox = tx[q][i];
              if (ox == kOut) continue;
              double t;
              const double v = profile64(a, u2_exact(ox, oy, oz), t);
              acc[i] = __dadd_rn(acc[i], __dmul_rn(a.w, v));
            }
          } else {
            const float yz = oy * oy + oz * oz;
            const float inv = pinv[q], hd = phd[q], w = pw[q];
            const bool d2 = pd2[q] != 0;
#pragma unroll
            for (int i = 0; i < kSX; ++i) {
              const Off ox = tx[q][i];
              if (ox == kOut) continue;
              float t, lg;
              const float v = profile32(inv, hd, d2, ox * ox + yz, t, lg);
              acc[i] = fmaf(w, v, acc[i]);
            }
          }
        }
      }
      __syncthreads();
    }
  }
  if (live) {
#pragma unroll
    for (int i = 0; i < kSX; ++i)
      if (x0 + i < nx) out[((long long)(x0 + i) * ny + gy) * nz + gz] = T(acc[i]);
  }
}

// -------------------------------------------------------------- atom sums
// A chunk is a run of whole z-rows (a, b) of one atom box, ~4096 voxels.
// Warps take rows; lanes run along z (coalesced field loads, tabulated
// per-axis wrapped index / offset, one integer division per row).
struct Chunk {
  int atom;
  int row0;   // first row (a * len[1] + b)
  int nrows;
};

template <typename T>
__device__ __forceinline__ void atom_terms(const AtomGeo& a, T ox, T oy, T oz, T b, double (&s)[6],
                                           float (&sf)[6], float inv2sd, float half_d, float dd,
                                           float dos, float lsig) {
  if constexpr (sizeof(T) == 8) {
    const double u2 = u2_exact(ox, oy, oz);
    double t;
    const double val = profile64(a, u2, t);
    double ampl = 0.0, lr = 0.0;
    if (u2 > 0.0) {
      ampl = __ddiv_rn(__dmul_rn(__dmul_rn(a.d, val), t), u2);
      lr = __dsub_rn(__dmul_rn(0.5, log(u2)), a.log_sigma);
    }
    const double vt = __dmul_rn(val, t);
    s[0] += val * b;
    s[1] += __dmul_rn(ampl, ox) * b;
    s[2] += __dmul_rn(ampl, oy) * b;
    s[3] += __dmul_rn(ampl, oz) * b;
    s[4] += __dmul_rn(vt, a.d_over_sigma) * b;
    s[5] += __dmul_rn(-vt, lr) * b;
  } else {
    const float u2 = ox * ox + oy * oy + oz * oz;
    float t, lg;
    const float val = profile32(inv2sd, half_d, a.d2, u2, t, lg);
    float ampl = 0.f, lr = 0.f;
    if (u2 > 0.f) {
      ampl = __fdividef(dd * val * t, u2);
      lr = 0.34657359027997264f * lg - lsig;  // 0.5 ln(u2) = 0.5 ln2 log2(u2)
    }
    const float vt = val * t;
    const float ab = ampl * b;
    sf[0] += val * b;
    sf[1] += ab * ox;
    sf[2] += ab * oy;
    sf[3] += ab * oz;
    sf[4] += vt * dos * b;
    sf[5] -= vt * lr * b;
  }
}

// per-row record of a chunk: offsets (x, y) from the atom centre and the
// linear offset of the row's first z in the volume (int32: < 2^31 voxels)
template <typename T>
struct RowRec {
  T ox, oy;
  int lin;
};

template <typename T>
__global__ void __launch_bounds__(kSumThreads) atom_sums_kernel(
    const AtomGeo* __restrict__ atoms, const Chunk* __restrict__ chunks, int nx, int ny, int nz,
    const T* __restrict__ field, double* __restrict__ partials) {
  __shared__ RowRec<T> rows[max_rows<T>()];
  __shared__ T tzo[kMaxAxis];   // z offsets (full z axes only)
  const Chunk ch = chunks[blockIdx.x];
  const AtomGeo& a = atoms[ch.atom];
  const int l1 = a.len[1], l2 = a.len[2];
  for (int q = threadIdx.x; q < ch.nrows; q += kSumThreads) {
    const int r = ch.row0 + q;
    const int il[2] = {r / l1, r - (r / l1) * l1};
    const int dims2[2] = {nx, ny};
    int g[2];
    T o[2];
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      if (a.full[ax]) {
        g[ax] = il[ax];
        o[ax] = T(min_image(il[ax], a.m[ax], dims2[ax]));
      } else {
        const int p = a.start[ax] + il[ax];
        g[ax] = pmod(p, dims2[ax]);
        o[ax] = T(__dsub_rn(double(p), a.m[ax]));
      }
    }
    rows[q] = {o[0], o[1], (g[0] * ny + g[1]) * nz};
  }
  const bool zfull = a.full[2] != 0;
  if (zfull)
    for (int ic = threadIdx.x; ic < l2; ic += kSumThreads) tzo[ic] = T(min_image(ic, a.m[2], nz));
  __syncthreads();

  double s[6] = {0, 0, 0, 0, 0, 0};
  float sf[6] = {0, 0, 0, 0, 0, 0};
  const float inv2sd = float(a.inv2sd), half_d = float(a.half_d), dd = float(a.d),
              dos = float(a.d_over_sigma), lsig = float(a.log_sigma);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // z of box column ic: volume index zs + ic (wrapped once), offset oz0 + ic
  const int zs = zfull ? 0 : pmod(a.start[2], nz);
  const T oz0 = zfull ? T(0) : T(__dsub_rn(double(a.start[2]), a.m[2]));
  // flat voxels of the chunk (z fastest), one per thread per kSumThreads step
  const int nv = ch.nrows * l2;
  int ic = threadIdx.x % l2, q = threadIdx.x / l2;
  const int dq = kSumThreads / l2, dc = kSumThreads % l2;
  for (int v = threadIdx.x; v < nv; v += kSumThreads) {
    const RowRec<T> rr = rows[q];
    int gz;
    T oz;
    if (zfull) {
      gz = ic;
      oz = tzo[ic];
    } else {
      gz = zs + ic;
      gz = gz >= nz ? gz - nz : gz;
      if constexpr (sizeof(T) == 8)
        oz = __dsub_rn(double(a.start[2] + ic), a.m[2]);  // the reference's span - m
      else
        oz = oz0 + float(ic);
    }
    atom_terms<T>(a, rr.ox, rr.oy, oz, field[rr.lin + gz], s, sf, inv2sd, half_d, dd, dos, lsig);
    ic += dc;
    q += dq;
    if (ic >= l2) {
      ic -= l2;
      ++q;
    }
  }
  if constexpr (sizeof(T) != 8) {
#pragma unroll
    for (int c = 0; c < 6; ++c) s[c] = double(sf[c]);
  }
  // block reduction in fp64 (fixed order: warp tree, then warps in order)
  __shared__ double red[6][kSumThreads / 32];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x = s[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[c][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double x = 0.0;
    for (int w = 0; w < kSumThreads / 32; ++w) x += red[threadIdx.x][w];
    partials[(long long)blockIdx.x * 6 + threadIdx.x] = x;
  }
}

// Boxes with an axis longer than kMaxAxis (huge sigma on a huge grid): one
// voxel per thread with the offsets computed on the fly (rare fallback).
template <typename T>
__global__ void __launch_bounds__(kSumThreads) atom_sums_big_kernel(
    const AtomGeo* __restrict__ atoms, const Chunk* __restrict__ chunks, int nx, int ny, int nz,
    const T* __restrict__ field, double* __restrict__ partials) {
  const Chunk ch = chunks[blockIdx.x];
  const AtomGeo& a = atoms[ch.atom];
  const int dims[3] = {nx, ny, nz};
  const int l1 = a.len[1], l2 = a.len[2];
  double s[6] = {0, 0, 0, 0, 0, 0};
  float sf[6] = {0, 0, 0, 0, 0, 0};
  const float inv2sd = float(a.inv2sd), half_d = float(a.half_d), dd = float(a.d),
              dos = float(a.d_over_sigma), lsig = float(a.log_sigma);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = ch.row0 + warp; r < ch.row0 + ch.nrows; r += kSumThreads / 32) {
    const int il[2] = {r / l1, r - (r / l1) * l1};
    int g[2];
    T o[2];
    for (int ax = 0; ax < 2; ++ax) {
      if (a.full[ax]) {
        g[ax] = il[ax];
        o[ax] = T(min_image(il[ax], a.m[ax], dims[ax]));
      } else {
        const int p = a.start[ax] + il[ax];
        g[ax] = pmod(p, dims[ax]);
        o[ax] = T(__dsub_rn(double(p), a.m[ax]));
      }
    }
    const T* frow = field + ((long long)g[0] * ny + g[1]) * nz;
    for (int ic = lane; ic < l2; ic += 32) {
      int gz;
      T oz;
      if (a.full[2]) {
        gz = ic;
        oz = T(min_image(ic, a.m[2], nz));
      } else {
        const int p = a.start[2] + ic;
        gz = pmod(p, nz);
        oz = T(__dsub_rn(double(p), a.m[2]));
      }
      atom_terms<T>(a, o[0], o[1], oz, frow[gz], s, sf, inv2sd, half_d, dd, dos, lsig);
    }
  }
  if constexpr (sizeof(T) != 8) {
#pragma unroll
    for (int c = 0; c < 6; ++c) s[c] = double(sf[c]);
  }
  __shared__ double red[6][kSumThreads / 32];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x = s[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[c][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double x = 0.0;
    for (int w = 0; w < kSumThreads / 32; ++w) x += red[threadIdx.x][w];
    partials[(long long)blockIdx.x * 6 + threadIdx.x] = x;
  }
}

// ---------------------------------------------- one atom, for the ascent
// neg_eta of the certificate ascent (certificate.py:201-209): the six inner
// products of ONE unit atom with the device field, once per L-BFGS-B
// evaluation. Built for latency: the atom's geometry arrives as a kernel
// parameter (no upload), the voxels of its box are spread flat over the grid
// with the offsets computed on the fly, fp64 profile math for fp32 and fp64
// storage alike (the ascent's gtol = 1e-8 needs a smooth objective), CTA
// partials combined in CTA order by the last CTA to finish (fixed order:
// bit-reproducible), which writes the result and a sequence flag straight
// into mapped pinned host memory, where the calling thread is spinning.
constexpr int kOneThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kOneThreads) refine_sums_kernel(
    const __grid_constant__ AtomGeo a, int nx, int ny, int nz, const T* __restrict__ field,
    double* __restrict__ partials, unsigned* __restrict__ ticket,
    volatile double* __restrict__ out_host, volatile unsigned long long* __restrict__ flag_host,
    unsigned long long seq) {
  const int l1 = a.len[1], l2 = a.len[2];
  const long long nv = (long long)a.len[0] * l1 * l2;
  double s[6] = {0, 0, 0, 0, 0, 0};
  float sf[6];
  const long long stride = (long long)gridDim.x * kOneThreads;
  for (long long v = (long long)blockIdx.x * kOneThreads + threadIdx.x; v < nv; v += stride) {
    const int q = int(v / l2), ic = int(v - (long long)q * l2);
    const int il[3] = {q / l1, q - (q / l1) * l1, ic};
    const int dims[3] = {nx, ny, nz};
    int g[3];
    double o[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (a.full[ax]) {
        g[ax] = il[ax];
        o[ax] = min_image(il[ax], a.m[ax], dims[ax]);
      } else {
        const int p = a.start[ax] + il[ax];
        g[ax] = pmod(p, dims[ax]);
        o[ax] = __dsub_rn(double(p), a.m[ax]);
      }
    }
    const double b = double(field[((long long)g[0] * ny + g[1]) * nz + g[2]]);
    atom_terms<double>(a, o[0], o[1], o[2], b, s, sf, 0.f, 0.f, 0.f, 0.f, 0.f);
  }
  __shared__ double red[6][kOneThreads / 32];
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x = s[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[c][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double x = 0.0;
    for (int w = 0; w < kOneThreads / 32; ++w) x += red[threadIdx.x][w];
    partials[(long long)blockIdx.x * 6 + threadIdx.x] = x;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 6) {
    double x = 0.0;
    for (unsigned bI = 0; bI < gridDim.x; ++bI) x += __ldcg(partials + (long long)bI * 6 + threadIdx.x);
    out_host[threadIdx.x] = x;
    __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *ticket = 0u;  // ready for the next evaluation (stream order)
    *flag_host = seq;
    __threadfence_system();
  }
}

// ------------------------------------------------ render, fp32 interval path
// fp32 storage when every atom box is a product of three unwrapped intervals
// that meet a brick in ONE run per axis (no full axis, len <= n - brick):
// then box ∩ brick is an interval per axis and every offset is linear,
// o(i) = o0 + i. A CTA owns a 16 x 16 x 32 brick with its accumulator in
// shared memory (row pitch 33), compacts the atoms meeting it in row order
// (256 per pass) and prepares each listed atom's intersection record in
// parallel (one thread per atom). Warp w owns x-planes 2w, 2w + 1 and walks
// the list on its own: the voxels of (its planes ∩ atom) are spread over the
// lanes (4 x-y rows at one z per lane: lanes along z), then __syncwarp — so
// every voxel still sums its atoms in the reference's row order, with no
// CTA-wide barrier per atom.
constexpr int kFX = 16, kFY = 16, kFZ = 32, kFP = kFZ + 1, kFT = 256, kFW = kFX / (kFT / 32);

struct FAtom {
  float o0x, o0y, o0z;
  int lo, cnt;       // brick-local start / count per axis: byte a = axis
  float w, hd, inv2sd;  // inv2sd: -log2(e) / (2 sigma^d)
  int d2;
  unsigned ngz_magic;  // div_magic(ceil(cz / 4))
};

// run of the unwrapped box [s, s + l) meeting brick coords [b0, b0 + B)
// (l <= n - B: one run); returns the count (0 = none)
__device__ __forceinline__ int brick_run(int s, int l, double m, int b0, int B, int n, int& lo,
                                         float& o0) {
  const int d = pmod(b0 - s, n);
  if (d < l) {  // brick start inside the box
    lo = 0;
    o0 = float(double(s + d) - m);
    return min(l - d, B);
  }
  const int e = pmod(s - b0, n);  // box start inside the brick?
  if (e < B) {
    lo = e;
    o0 = float(double(s) - m);
    return min(l, B - e);
  }
  lo = 0;
  o0 = 0.f;
  return 0;
}

// exact small-integer division a / b (a < 2^21) through a float reciprocal
__device__ __forceinline__ int fdiv_small(int a, int, float inv_b) {
  return __float2int_rz((float(a) + 0.5f) * inv_b);
}

__global__ void __launch_bounds__(kFT) render_f32_kernel(const AtomGeo* __restrict__ atoms,
                                                         const int4* __restrict__ boxes, int k,
                                                         int nx, int ny, int nz,
                                                         float* __restrict__ out) {
  __shared__ float acc[kFX * kFY * kFP];
  __shared__ FAtom fa[kFT];
  __shared__ int warp_cnt[kFT / 32];
  __shared__ int list_n;
  const int nbz = (nz + kFZ - 1) / kFZ, nby = (ny + kFY - 1) / kFY;
  const int bz = blockIdx.x % nbz, by = (blockIdx.x / nbz) % nby, bx = blockIdx.x / (nbz * nby);
  const int x0 = bx * kFX, y0 = by * kFY, z0 = bz * kFZ;
  const int BX = min(kFX, nx - x0), BY = min(kFY, ny - y0), BZ = min(kFZ, nz - z0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < kFX * kFY * kFP; e += kFT) acc[e] = 0.f;
  const int wx0 = warp * kFW;  // this warp's first x-plane
  for (int base = 0; base < k; base += kFT) {
    const int ai = base + tid;
    FAtom f;
    bool hit = false;
    if (ai < k) {
      const int4 bx4 = boxes[ai];  // start x, y, z; lengths (10 bits each)
      const int l[3] = {bx4.w & 1023, (bx4.w >> 10) & 1023, bx4.w >> 20};
      const int st[3] = {bx4.x, bx4.y, bx4.z};
      const int b0[3] = {x0, y0, z0}, B[3] = {BX, BY, BZ}, n[3] = {nx, ny, nz};
      int lo[3], c[3];
      float o0[3];
      hit = true;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        // (offsets need the centre: read only for atoms that meet the brick)
        c[ax] = brick_run(st[ax], l[ax], 0.0, b0[ax], B[ax], n[ax], lo[ax], o0[ax]);
        hit &= c[ax] > 0;
      }
      if (hit) {
        const AtomGeo& a = atoms[ai];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
          brick_run(st[ax], l[ax], a.m[ax], b0[ax], B[ax], n[ax], lo[ax], o0[ax]);
        f.o0x = o0[0];
        f.o0y = o0[1];
        f.o0z = o0[2];
        f.lo = lo[0] | (lo[1] << 8) | (lo[2] << 16);
        f.cnt = c[0] | (c[1] << 8) | (c[2] << 16);
        f.w = float(a.w);
        f.hd = float(a.half_d);
        f.inv2sd = float(-1.4426950408889634 * a.inv2sd);  // (-log2 e) / (2 sigma^d)
        f.d2 = a.d2;
        f.ngz_magic = div_magic((c[2] + 3) >> 2);
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) warp_cnt[warp] = __popc(mask);
    __syncthreads();  // (also: the previous pass's warps are done with fa)
    if (tid == 0) {
      int sacc = 0;
      for (int w = 0; w < kFT / 32; ++w) {
        const int c = warp_cnt[w];
        warp_cnt[w] = sacc;
        sacc += c;
      }
      list_n = sacc;
    }
    __syncthreads();
    if (hit) fa[warp_cnt[warp] + __popc(mask & ((1u << lane) - 1u))] = f;
    __syncthreads();
    const int cnt = list_n;
    for (int q = 0; q < cnt; ++q) {
      const FAtom g = fa[q];
      const int lo0 = g.lo & 255, lo1 = (g.lo >> 8) & 255, lo2 = g.lo >> 16;
      const int cx = g.cnt & 255, cy = (g.cnt >> 8) & 255, cz = g.cnt >> 16;
      const int px0 = max(wx0, lo0), px1 = min(wx0 + kFW, lo0 + cx);
      const int rows = (px1 - px0) * cy;
      if (rows <= 0) continue;
      const int ngz = (cz + 3) >> 2;
      const int units = rows * ngz;
      const float ox0 = g.o0x + float(px0 - lo0);
      const bool d2 = g.d2 != 0;
      // unit = one x-y row x 4 consecutive z (lanes along z groups)
      for (int u = lane; u < units; u += 32) {
        const int row = div_small(u, g.ngz_magic);
        const int gz = u - row * ngz;
        const int ix = row >= cy ? 1 : 0;  // (kFW = 2 planes per warp)
        const int iy = row - ix * cy;
        const float ox = ox0 + i2f_small(ix), oy = g.o0y + i2f_small(iy);
        const float oxy2 = fmaf(ox, ox, oy * oy);
        float oz = g.o0z + i2f_small(4 * gz);
        float* pa = acc + ((px0 + ix) * kFY + lo1 + iy) * kFP + lo2 + 4 * gz;
        const int nz4 = cz - 4 * gz;  // valid voxels of this group (>= 1)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float u2 = fmaf(oz, oz, oxy2);
          const float p = d2 ? u2 : ex2_approx(g.hd * lg2_approx(u2));
          const float v = ex2_approx(g.inv2sd * p);  // exp(-u2^(d/2) / (2 sigma^d))
          if (j < nz4) pa[j] = fmaf(g.w, v, pa[j]);
          oz += 1.f;
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < kFX * kFY * kFZ; e += kFT) {
    const int z = e & (kFZ - 1), y = (e >> 5) & (kFY - 1), x = e >> 9;
    if (x < BX && y < BY && z < BZ)
      out[((long long)(x0 + x) * ny + y0 + y) * nz + z0 + z] = acc[(x * kFY + y) * kFP + z];
  }
}

// ------------------------------------------- atom sums, fp32 interval path
// Same chunks as atom_sums_kernel (runs of whole rows of one box). A thread
// unit is 4 consecutive rows at one z (lanes along z: coalesced field loads);
// offsets are linear in the box indices, so per voxel the work is the profile
// (lg2, ex2, ex2 on the MUFU), one reciprocal and the accumulations:
//   s0 += v b, s4 += v t b (x d/sigma at the end), s5 += v t b log2(u2)
//   (-> -(ln2/2 s5 - ln sigma s4)), and with ab = d v t b / u2:
//   s1 += ab ox, s2 += ab oy, s3 += oz sum_rows ab.
struct RowF {
  float ox, oy, oxy2;
  int lin;  // volume offset of the row's z = 0
};

__global__ void __launch_bounds__(kSumThreads) atom_sums_f32_kernel(
    const AtomGeo* __restrict__ atoms, const Chunk* __restrict__ chunks, int nx, int ny, int nz,
    const float* __restrict__ field, double* __restrict__ partials) {
  __shared__ RowF rows[kMaxRows32 + 4];
  const Chunk ch = chunks[blockIdx.x];
  const AtomGeo& a = atoms[ch.atom];
  const int l1 = a.len[1], l2 = a.len[2];
  const float inv2sd = float(a.inv2sd), hd = float(a.half_d);
  const bool d2 = a.d2 != 0;
  const float o0z = float(double(a.start[2]) - a.m[2]);
  const int zs = pmod(a.start[2], nz);
  // per-row record: offsets and the wrapped row base (padding rows: b = 0)
  for (int q = threadIdx.x; q < ch.nrows; q += kSumThreads) {
    RowF rr;
    {
      const int r = ch.row0 + q;
      const int ix = r / l1, iy = r - ix * l1;
      const int px = a.start[0] + ix, py = a.start[1] + iy;
      rr.ox = float(double(px) - a.m[0]);
      rr.oy = float(double(py) - a.m[1]);
      rr.oxy2 = fmaf(rr.ox, rr.ox, rr.oy * rr.oy);
      rr.lin = (pmod(px, nx) * ny + pmod(py, ny)) * nz;
    }
    rows[q] = rr;
  }
  __syncthreads();
  // unit = one x-y row x 8 consecutive z, as 4 voxel PAIRS on the packed
  // f32x2 pipe (fma / mul / add of both voxels in one instruction; the MUFU
  // ops lg2, ex2, ex2, rcp stay per voxel): the arithmetic around the four
  // MUFU ops was what bound this kernel (issue slots, not the MUFU pipe)
  // Units are ALIGNED groups of 8 consecutive volume z (two 16-byte loads per
  // lane: the scalar loads' 32 sector look-ups per instruction were what
  // bound this kernel, L1/TEX at 85%); voxels of a group outside the box's z
  // span are masked (b = 0). nz % 4 == 0 (dispatch), so a 16-byte vector
  // never straddles the periodic wrap.
  constexpr int ZG = 8;
  const int za = zs & 3;                       // the box starts za voxels into its first vector
  const int ngz = (za + l2 + ZG - 1) / ZG;
  const unsigned ngz_magic = div_magic(ngz);
  const int units = ch.nrows * ngz;
  const int zbase = zs - za;                   // aligned volume z of group 0
  const float ozbase = o0z - i2f_small(za);    // its offset from the centre
  f32x2 S0 = 0ull, S3 = 0ull, S4 = 0ull, S5 = 0ull;
  float s1 = 0.f, s2 = 0.f;
  const f32x2 hd2 = pk2(hd, hd), inv2 = pk2(inv2sd, inv2sd),
              nl2e = pk2(-1.4426950408889634f, -1.4426950408889634f), two2 = pk2(2.f, 2.f);
  for (int u = threadIdx.x; u < units; u += kSumThreads) {
    const int q = div_small(u, ngz_magic);
    const int g8 = ZG * (u - q * ngz);          // group start, in voxels from zbase
    const RowF rr = rows[q];
    const int i0 = g8 - za;                     // box-local z index of the group's first voxel
    float b[ZG];
#pragma unroll
    for (int h = 0; h < ZG / 4; ++h) {
      int z4 = zbase + g8 + 4 * h;
      z4 = z4 >= nz ? z4 - nz : z4;
      float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i0 + 4 * h + 3 >= 0 && i0 + 4 * h < l2)
        v4 = __ldg(reinterpret_cast<const float4*>(field + rr.lin + z4));
      const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + 4 * h + j;
        b[4 * h + j] = (i >= 0 && i < l2) ? vv[j] : 0.f;
      }
    }
    const float ozs = ozbase + i2f_small(g8);
    f32x2 oz2 = pk2(ozs, ozs + 1.f);
    const f32x2 oxy2 = pk2(rr.oxy2, rr.oxy2);
    f32x2 SAB = 0ull;
#pragma unroll
    for (int jp = 0; jp < ZG / 2; ++jp) {
      const f32x2 u2 = fma2(oz2, oz2, oxy2);
      float ua, ub;
      upk2(u2, ua, ub);
      const float lga = lg2_approx(ua), lgb = lg2_approx(ub);
      f32x2 p2 = u2;
      if (!d2) {
        const f32x2 e2 = mul2(hd2, pk2(lga, lgb));
        float ea, eb;
        upk2(e2, ea, eb);
        p2 = pk2(ex2_approx(ea), ex2_approx(eb));
      }
      const f32x2 t2 = mul2(inv2, p2);
      float xa, xb;
      upk2(mul2(nl2e, t2), xa, xb);
      const f32x2 v2 = pk2(ex2_approx(xa), ex2_approx(xb));
      const f32x2 vb = mul2(v2, pk2(b[2 * jp], b[2 * jp + 1]));
      const f32x2 vtb = mul2(vb, t2);
      S0 = add2(S0, vb);
      S4 = add2(S4, vtb);
      S5 = fma2(vtb, pk2(fmaxf(lga, -126.f), fmaxf(lgb, -126.f)), S5);  // (u2 = 0: vtb = 0)
      const f32x2 ab = mul2(vtb, pk2(rcp_approx(fmaxf(ua, 1e-30f)), rcp_approx(fmaxf(ub, 1e-30f))));
      SAB = add2(SAB, ab);
      S3 = fma2(ab, oz2, S3);
      oz2 = add2(oz2, two2);
    }
    float sa, sb;
    upk2(SAB, sa, sb);
    const float sab = sa + sb;
    s1 = fmaf(sab, rr.ox, s1);
    s2 = fmaf(sab, rr.oy, s2);
  }
  float s0, s3, s4, s5;
  {
    float x, y;
    upk2(S0, x, y); s0 = x + y;
    upk2(S3, x, y); s3 = x + y;
    upk2(S4, x, y); s4 = x + y;
    upk2(S5, x, y); s5 = x + y;
  }
  const float dd = float(a.d);
  double s[6] = {double(s0), double(dd * s1), double(dd * s2), double(dd * s3),
                 double(s4) * a.d_over_sigma,
                 -(0.34657359027997264 * double(s5) - a.log_sigma * double(s4))};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double red[6][kSumThreads / 32];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x = s[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[c][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double x = 0.0;
    for (int w = 0; w < kSumThreads / 32; ++w) x += red[threadIdx.x][w];
    partials[(long long)blockIdx.x * 6 + threadIdx.x] = x;
  }
}

__global__ void chunk_combine_kernel(const int* __restrict__ first_chunk, int k,
                                     const double* __restrict__ partials, double* __restrict__ sums) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k * 6) return;
  const int atom = i / 6, c = i % 6;
  double x = 0.0;
  for (int ch = first_chunk[atom]; ch < first_chunk[atom + 1]; ++ch) x += partials[ch * 6 + c];
  sums[i] = x;
}

// --------------------------------------------------------------- sumsq
constexpr int kRedThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kRedThreads) sumsq_diff_kernel(const T* __restrict__ a,
                                                                 const T* __restrict__ b,
                                                                 T* __restrict__ diff, long long n,
                                                                 double* __restrict__ partials) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kRedThreads) {
    T d = b ? T(a[i] - b[i]) : a[i];
    if (diff) diff[i] = d;
    const double dd = double(d);
    s += dd * dd;
  }
  __shared__ double red[kRedThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) x += red[w];
    partials[blockIdx.x] = x;
  }
}

__global__ void final_sum_kernel(const double* __restrict__ partials, int n, double* __restrict__ out) {
  __shared__ double red[kRedThreads / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kRedThreads) s += partials[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) x += red[w];
    *out = x;
  }
}

}  // namespace

// every box a product of unwrapped intervals meeting any brick of size B in
// one run per axis (the fp32 interval kernels' precondition)
static bool interval_boxes(const std::vector<AtomGeo>& atoms, const int dims[3], const int B[3]) {
  if ((long long)dims[0] * dims[1] * dims[2] >= (1LL << 31)) return false;
  for (const auto& a : atoms)
    for (int ax = 0; ax < 3; ++ax)
      if (a.full[ax] || a.len[ax] > dims[ax] - B[ax] || a.len[ax] >= 1024) return false;
  return true;
}

int render_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const std::vector<AtomGeo>& atoms,
                const AtomGeo* atoms_dev, int k, void* out) {
  SFW3D_PROF(ctx, "render");
  static const int kFB[3] = {kFX, kFY, kFZ};
  if (dtype == SFW3D_F32 && interval_boxes(atoms, dims, kFB)) {
    const int nbf = ((dims[0] + kFX - 1) / kFX) * ((dims[1] + kFY - 1) / kFY) *
                    ((dims[2] + kFZ - 1) / kFZ);
    // compact boxes for the per-brick culling: start x, y, z; lengths
    std::vector<int4> bx(std::max(k, 1));
    for (int i = 0; i < k; ++i)
      bx[i] = make_int4(atoms[i].start[0], atoms[i].start[1], atoms[i].start[2],
                        atoms[i].len[0] | (atoms[i].len[1] << 10) | (atoms[i].len[2] << 20));
    SFW3D_TRY(ensure_device(ctx, ctx->ws_aux, bx.size() * sizeof(int4)));
    int4* bx_dev = static_cast<int4*>(ctx->ws_aux.ptr);
    SFW3D_TRY(stage_upload(ctx, bx_dev, bx.data(), bx.size() * sizeof(int4)));
    render_f32_kernel<<<nbf, kFT, 0, ctx->stream>>>(atoms_dev, bx_dev, k, dims[0], dims[1],
                                                    dims[2], static_cast<float*>(out));
    SFW3D_LAUNCH_CHECK(ctx);
    return SFW3D_OK;
  }
  const int nb = ((dims[0] + kSX - 1) / kSX) * ((dims[1] + kSY - 1) / kSY) *
                 ((dims[2] + kSZ - 1) / kSZ);
  if (dtype == SFW3D_F64)
    render_kernel<double><<<nb, 512, 0, ctx->stream>>>(atoms_dev, k, dims[0], dims[1], dims[2],
                                                        static_cast<double*>(out));
  else
    render_kernel<float><<<nb, 512, 0, ctx->stream>>>(atoms_dev, k, dims[0], dims[1], dims[2],
                                                       static_cast<float*>(out));
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

// Row chunks (~kChunk voxels of whole z-rows) per atom, in atom order; the
// atom's chunks are contiguous and first[i]..first[i+1] delimits them.
static void chunk_plan(const std::vector<AtomGeo>& atoms, std::vector<Chunk>& chunks,
                       std::vector<int>& first, int chunk = kChunk, int max_rows = kMaxRows) {
  chunks.clear();
  first.assign(atoms.size() + 1, 0);
  for (size_t i = 0; i < atoms.size(); ++i) {
    first[i] = int(chunks.size());
    const AtomGeo& a = atoms[i];
    const int rows = a.len[0] * a.len[1];
    const int per = std::min(max_rows, std::max(1, chunk / std::max(1, a.len[2])));
    for (int r = 0; r < rows; r += per) chunks.push_back({int(i), r, std::min(per, rows - r)});
  }
  first[atoms.size()] = int(chunks.size());
}

static bool small_boxes(const std::vector<AtomGeo>& atoms, const int dims[3]) {
  if ((long long)dims[0] * dims[1] * dims[2] >= (1LL << 31)) return false;  // int32 offsets
  for (const auto& a : atoms)
    if (a.len[0] > kMaxAxis || a.len[1] > kMaxAxis || a.len[2] > kMaxAxis) return false;
  return true;
}

// The chunk plan is made here, on the host, typically while the device is
// still rendering / convolving (the callers enqueue those first); its device
// copy and the chunk partials live in the context's own ws_plan arena.
int atom_sums_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* field,
                   const std::vector<AtomGeo>& atoms, const AtomGeo* atoms_dev, double* sums_dev) {
  const int k = int(atoms.size());
  if (k == 0) return SFW3D_OK;
  std::vector<Chunk> chunks;
  std::vector<int> first;
  // chunk size: the defaults amortise the per-chunk row table over many
  // voxels, but a few atoms (the certificate refine's single atom) would then
  // fill only a fraction of the SMs: aim at >= 4 chunks per SM
  long long total = 0;
  for (const auto& a : atoms) total += (long long)a.len[0] * a.len[1] * a.len[2];
  const int fill = int(std::max<long long>(512, total / (4LL * ctx->num_sms)));
  if (dtype == SFW3D_F64 || !small_boxes(atoms, dims))
    chunk_plan(atoms, chunks, first, std::min(kChunk, fill));
  else
    chunk_plan(atoms, chunks, first, std::min(std::max(kChunk, chunk32()), fill), kMaxRows32);
  SFW3D_TRY(ensure_device(ctx, ctx->ws_plan,
                          Carver::need({chunks.size() * sizeof(Chunk), first.size() * sizeof(int),
                                        chunks.size() * 6 * sizeof(double)})));
  Carver cv(ctx->ws_plan.ptr);
  Chunk* ch_dev = cv.take<Chunk>(chunks.size());
  int* first_dev = cv.take<int>(first.size());
  double* part = cv.take<double>(chunks.size() * 6);
  SFW3D_TRY(stage_upload(ctx, ch_dev, chunks.data(), chunks.size() * sizeof(Chunk)));
  SFW3D_TRY(stage_upload(ctx, first_dev, first.data(), first.size() * sizeof(int)));
  const unsigned nch = unsigned(chunks.size());
  SFW3D_PROF(ctx, "atom_sums");
  const bool small = small_boxes(atoms, dims);
  if (dtype == SFW3D_F64) {
    if (small)
      atom_sums_kernel<double><<<nch, kSumThreads, 0, ctx->stream>>>(
          atoms_dev, ch_dev, dims[0], dims[1], dims[2], static_cast<const double*>(field), part);
    else
      atom_sums_big_kernel<double><<<nch, kSumThreads, 0, ctx->stream>>>(
          atoms_dev, ch_dev, dims[0], dims[1], dims[2], static_cast<const double*>(field), part);
  } else {
    static const int kOne[3] = {1, 1, 1};
    if (interval_boxes(atoms, dims, kOne) && dims[2] % 4 == 0)  // (16-byte field loads)
      atom_sums_f32_kernel<<<nch, kSumThreads, 0, ctx->stream>>>(
          atoms_dev, ch_dev, dims[0], dims[1], dims[2], static_cast<const float*>(field), part);
    else if (small)
      atom_sums_kernel<float><<<nch, kSumThreads, 0, ctx->stream>>>(
          atoms_dev, ch_dev, dims[0], dims[1], dims[2], static_cast<const float*>(field), part);
    else
      atom_sums_big_kernel<float><<<nch, kSumThreads, 0, ctx->stream>>>(
          atoms_dev, ch_dev, dims[0], dims[1], dims[2], static_cast<const float*>(field), part);
  }
  SFW3D_LAUNCH_CHECK(ctx);
  chunk_combine_kernel<<<(k * 6 + 255) / 256, 256, 0, ctx->stream>>>(first_dev, k, part, sums_dev);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

int refine_sums_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* field,
                     const AtomGeo& atom, double out[6]) {
  if (!ctx->one_host) {
    SFW3D_CUDA_TRY(cudaHostAlloc(&ctx->one_host, 8 * sizeof(double), cudaHostAllocMapped));
    std::memset(ctx->one_host, 0, 8 * sizeof(double));
    SFW3D_CUDA_TRY(cudaHostGetDevicePointer(&ctx->one_host_dev, ctx->one_host, 0));
  }
  const long long nv = (long long)atom.len[0] * atom.len[1] * atom.len[2];
  const int maxg = 4 * ctx->num_sms;
  const int grid = int(std::min<long long>(maxg, std::max<long long>(1, (nv + 2 * kOneThreads - 1) / (2 * kOneThreads))));
  const size_t need = size_t(maxg) * 6 * sizeof(double) + 256;
  if (ctx->ws_one.bytes < need) {
    SFW3D_TRY(ensure_device(ctx, ctx->ws_one, need));
    SFW3D_CUDA_TRY(cudaMemsetAsync(ctx->ws_one.ptr, 0, need, ctx->stream));
  }
  unsigned* ticket = static_cast<unsigned*>(ctx->ws_one.ptr);
  double* partials = reinterpret_cast<double*>(static_cast<char*>(ctx->ws_one.ptr) + 256);
  volatile double* host = static_cast<volatile double*>(ctx->one_host);
  volatile unsigned long long* flag = reinterpret_cast<volatile unsigned long long*>(host + 7);
  volatile double* host_dev = static_cast<volatile double*>(ctx->one_host_dev);
  const unsigned long long seq = ++ctx->one_seq;
  {
    SFW3D_PROF(ctx, "atom_sums");
    if (dtype == SFW3D_F64)
      refine_sums_kernel<double><<<grid, kOneThreads, 0, ctx->stream>>>(
          atom, dims[0], dims[1], dims[2], static_cast<const double*>(field), partials, ticket, host_dev,
          reinterpret_cast<volatile unsigned long long*>(host_dev + 7), seq);
    else
      refine_sums_kernel<float><<<grid, kOneThreads, 0, ctx->stream>>>(
          atom, dims[0], dims[1], dims[2], static_cast<const float*>(field), partials, ticket, host_dev,
          reinterpret_cast<volatile unsigned long long*>(host_dev + 7), seq);
    SFW3D_LAUNCH_CHECK(ctx);
  }
  // spin on the mapped flag (a stream synchronise costs more than the kernel);
  // the stream is polled now and then so that a failed launch cannot hang us
  for (unsigned spins = 1; *flag != seq; ++spins) {
    if ((spins & 0x3fff) == 0) {
      const cudaError_t e = cudaStreamQuery(ctx->stream);
      if (e == cudaSuccess) {
        if (*flag == seq) break;
        set_error("ascent kernel finished without publishing its result");
        return SFW3D_ECUDA;
      }
      if (e != cudaErrorNotReady) SFW3D_CUDA_TRY(e);
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  for (int c = 0; c < 6; ++c) out[c] = host[c];
  return SFW3D_OK;
}

int sum_parts_impl(sfw3d_ctx* ctx, const double* parts, int n, double* out) {
  final_sum_kernel<<<1, kRedThreads, 0, ctx->stream>>>(parts, n, out);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

int sumsq_diff_impl(sfw3d_ctx* ctx, int dtype, int64_t n, const void* a, const void* b,
                    void* diff_out, double* partials, double* result_dev) {
  const int nblk = 4 * ctx->num_sms;
  SFW3D_PROF(ctx, "sumsq");
  if (dtype == SFW3D_F64)
    sumsq_diff_kernel<double><<<nblk, kRedThreads, 0, ctx->stream>>>(
        static_cast<const double*>(a), static_cast<const double*>(b),
        static_cast<double*>(diff_out), n, partials);
  else
    sumsq_diff_kernel<float><<<nblk, kRedThreads, 0, ctx->stream>>>(
        static_cast<const float*>(a), static_cast<const float*>(b), static_cast<float*>(diff_out),
        n, partials);
  SFW3D_LAUNCH_CHECK(ctx);
  final_sum_kernel<<<1, kRedThreads, 0, ctx->stream>>>(partials, nblk, result_dev);
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

}  // namespace sfw3d
