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
#include "internal.cuh"

namespace sfw3d {
namespace {

constexpr int kBX = 4, kBY = 8, kBZ = 16;  // render brick (512 voxels)
constexpr int kSub = 16;                   // listed atoms tabulated per pass
constexpr int kChunk = 4096;               // atom-sum chunk (voxels)
constexpr int kSumThreads = 256;
constexpr int kMaxAxis = 1024;             // tabulated axis length in atom sums

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

// unit profile, fp32 on the MUFU; lg2u2 returns log2(u2) for reuse
__device__ __forceinline__ float profile32(float inv2sd, float half_d, bool d2, float u2, float& t,
                                           float& lg2u2) {
  lg2u2 = __log2f(u2);
  const float p = d2 ? u2 : exp2f(half_d * lg2u2);
  t = inv2sd * p;
  return __expf(-t);
}

// ------------------------------------------------------------------ render
template <typename T>
__global__ void __launch_bounds__(512) render_kernel(const AtomGeo* __restrict__ atoms, int k,
                                                     int nx, int ny, int nz, T* __restrict__ out) {
  using Off = T;  // offsets tabulated in the storage precision (exact for fp64)
  __shared__ int list[512];
  __shared__ int warp_cnt[16];
  __shared__ int list_n;
  __shared__ Off tx[kSub][kBX], ty[kSub][kBY], tz[kSub][kBZ];

  const int nbz = (nz + kBZ - 1) / kBZ, nby = (ny + kBY - 1) / kBY;
  const int bz = blockIdx.x % nbz, by = (blockIdx.x / nbz) % nby, bx = blockIdx.x / (nbz * nby);
  const int x0 = bx * kBX, y0 = by * kBY, z0 = bz * kBZ;
  const int x1 = min(x0 + kBX, nx) - 1, y1 = min(y0 + kBY, ny) - 1, z1 = min(z0 + kBZ, nz) - 1;
  const int tid = threadIdx.x;
  const int lz = tid % kBZ, ly = (tid / kBZ) % kBY, lx = tid / (kBZ * kBY);
  const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
  const bool live = gx < nx && gy < ny && gz < nz;
  const int lane = tid & 31, warp = tid >> 5;
  const Off kOut = Off(INFINITY);

  double acc = 0.0;
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
      int s = 0;
      for (int w = 0; w < 16; ++w) {
        int c = warp_cnt[w];
        warp_cnt[w] = s;
        s += c;
      }
      list_n = s;
    }
    __syncthreads();
    if (hit) list[warp_cnt[warp] + __popc(mask & ((1u << lane) - 1u))] = ai;
    __syncthreads();
    const int cnt = list_n;
    for (int q0 = 0; q0 < cnt; q0 += kSub) {
      const int nq = min(kSub, cnt - q0);
      // tabulate offsets of the brick coordinates (inf = outside the box)
      if (tid < nq * (kBX + kBY + kBZ)) {
        const int q = tid / (kBX + kBY + kBZ), e = tid % (kBX + kBY + kBZ);
        const AtomGeo& a = atoms[list[q0 + q]];
        int axis, li, g, n;
        if (e < kBX) { axis = 0; li = e; g = x0 + e; n = nx; }
        else if (e < kBX + kBY) { axis = 1; li = e - kBX; g = y0 + li; n = ny; }
        else { axis = 2; li = e - kBX - kBY; g = z0 + li; n = nz; }
        double off = 0.0;
        const bool in = g < n && axis_offset(a, axis, g, n, off);
        const Off v = in ? Off(off) : kOut;
        if (axis == 0) tx[q][li] = v; else if (axis == 1) ty[q][li] = v; else tz[q][li] = v;
      }
      __syncthreads();
      if (live) {
        for (int q = 0; q < nq; ++q) {
          const Off ox = tx[q][lx], oy = ty[q][ly], oz = tz[q][lz];
          if (ox == kOut || oy == kOut || oz == kOut) continue;
          const AtomGeo& a = atoms[list[q0 + q]];
          if constexpr (sizeof(T) == 8) {
            double t;
            const double v = profile64(a, u2_exact(ox, oy, oz), t);
            acc = __dadd_rn(acc, __dmul_rn(a.w, v));
          } else {
            float t, lg;
            const float v = profile32(float(a.inv2sd), float(a.half_d), a.d2, ox * ox + oy * oy + oz * oz,
                                      t, lg);
            acc += a.w * double(v);
          }
        }
      }
      __syncthreads();
    }
  }
  if (live) out[((long long)gx * ny + gy) * nz + gz] = T(acc);
}

// -------------------------------------------------------------- atom sums
struct Chunk {
  int atom;
  int first;  // first voxel (linear in the atom box, z fastest)
};

template <typename T>
__global__ void __launch_bounds__(kSumThreads) atom_sums_kernel(
    const AtomGeo* __restrict__ atoms, const Chunk* __restrict__ chunks, int nx, int ny, int nz,
    const T* __restrict__ field, double* __restrict__ partials) {
  using Off = T;
  __shared__ Off toff[3][kMaxAxis];
  __shared__ int tidx[3][kMaxAxis];
  const Chunk ch = chunks[blockIdx.x];
  const AtomGeo& a = atoms[ch.atom];
  const int dims[3] = {nx, ny, nz};
  const int vend = int(min((long long)ch.first + kChunk, a.nvox));
  const int l2 = a.len[2], l1 = a.len[1];
  const bool tab = a.len[0] <= kMaxAxis && l1 <= kMaxAxis && l2 <= kMaxAxis;
  if (tab) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
      for (int il = threadIdx.x; il < a.len[ax]; il += kSumThreads) {
        if (a.full[ax]) {
          tidx[ax][il] = il;
          toff[ax][il] = Off(min_image(il, a.m[ax], dims[ax]));
        } else {
          const int p = a.start[ax] + il;
          tidx[ax][il] = pmod(p, dims[ax]);
          toff[ax][il] = Off(__dsub_rn(double(p), a.m[ax]));
        }
      }
  }
  __syncthreads();

  double s[6] = {0, 0, 0, 0, 0, 0};
  float sf[6] = {0, 0, 0, 0, 0, 0};
  const float inv2sd = float(a.inv2sd), half_d = float(a.half_d), dd = float(a.d),
              dos = float(a.d_over_sigma), lsig = float(a.log_sigma);
  for (int v = ch.first + threadIdx.x; v < vend; v += kSumThreads) {
    const int rest = v / l2;  // 32-bit index math (boxes hold < 2^31 voxels)
    const int ic = v - rest * l2;
    const int ia = rest / l1;
    const int ib = rest - ia * l1;
    int g[3];
    Off off[3];
    const int il[3] = {ia, ib, ic};
    if (tab) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        g[ax] = tidx[ax][il[ax]];
        off[ax] = toff[ax][il[ax]];
      }
    } else {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        if (a.full[ax]) {
          g[ax] = il[ax];
          off[ax] = Off(min_image(il[ax], a.m[ax], dims[ax]));
        } else {
          const int p = a.start[ax] + il[ax];
          g[ax] = pmod(p, dims[ax]);
          off[ax] = Off(__dsub_rn(double(p), a.m[ax]));
        }
      }
    }
    const T b = field[((long long)g[0] * ny + g[1]) * nz + g[2]];
    if constexpr (sizeof(T) == 8) {
      const double u2 = u2_exact(off[0], off[1], off[2]);
      double t;
      const double val = profile64(a, u2, t);
      double ampl = 0.0, lr = 0.0;
      if (u2 > 0.0) {
        ampl = __ddiv_rn(__dmul_rn(__dmul_rn(a.d, val), t), u2);
        lr = __dsub_rn(__dmul_rn(0.5, log(u2)), a.log_sigma);
      }
      const double vt = __dmul_rn(val, t);
      s[0] += val * b;
      s[1] += __dmul_rn(ampl, off[0]) * b;
      s[2] += __dmul_rn(ampl, off[1]) * b;
      s[3] += __dmul_rn(ampl, off[2]) * b;
      s[4] += __dmul_rn(vt, a.d_over_sigma) * b;
      s[5] += __dmul_rn(-vt, lr) * b;
    } else {
      const float fx = off[0], fy = off[1], fz = off[2];
      const float u2 = fx * fx + fy * fy + fz * fz;
      float t, lg;
      const float val = profile32(inv2sd, half_d, a.d2, u2, t, lg);
      float ampl = 0.f, lr = 0.f;
      if (u2 > 0.f) {
        ampl = dd * val * t * __frcp_rn(u2);
        lr = 0.34657359027997264f * lg - lsig;  // 0.5 ln(u2) = 0.5 ln2 log2(u2)
      }
      const float vt = val * t;
      const float bf = float(b);
      const float ab = ampl * bf;
      sf[0] += val * bf;
      sf[1] += ab * fx;
      sf[2] += ab * fy;
      sf[3] += ab * fz;
      sf[4] += vt * dos * bf;
      sf[5] -= vt * lr * bf;
    }
  }
  if constexpr (sizeof(T) != 8) {
#pragma unroll
    for (int c = 0; c < 6; ++c) s[c] = double(sf[c]);
  }
  // block reduction in fp64 (fixed order: warp tree, then warps in order)
  __shared__ double red[6][kSumThreads / 32];
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

int render_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const AtomGeo* atoms_dev, int k,
                void* out) {
  const int nb = ((dims[0] + kBX - 1) / kBX) * ((dims[1] + kBY - 1) / kBY) *
                 ((dims[2] + kBZ - 1) / kBZ);
  SFW3D_PROF(ctx, "render");
  if (dtype == SFW3D_F64)
    render_kernel<double><<<nb, 512, 0, ctx->stream>>>(atoms_dev, k, dims[0], dims[1], dims[2],
                                                        static_cast<double*>(out));
  else
    render_kernel<float><<<nb, 512, 0, ctx->stream>>>(atoms_dev, k, dims[0], dims[1], dims[2],
                                                       static_cast<float*>(out));
  SFW3D_LAUNCH_CHECK(ctx);
  return SFW3D_OK;
}

static void chunk_plan(const std::vector<AtomGeo>& atoms, std::vector<Chunk>& chunks,
                       std::vector<int>& first) {
  chunks.clear();
  first.assign(atoms.size() + 1, 0);
  for (size_t i = 0; i < atoms.size(); ++i) {
    first[i] = int(chunks.size());
    for (long long v = 0; v < atoms[i].nvox; v += kChunk) chunks.push_back({int(i), int(v)});
  }
  first[atoms.size()] = int(chunks.size());
}

size_t atom_sums_scratch(const std::vector<AtomGeo>& atoms) {
  size_t nch = 0;
  for (auto& a : atoms) nch += size_t((a.nvox + kChunk - 1) / kChunk);
  return Carver::need({nch * sizeof(Chunk), (atoms.size() + 1) * sizeof(int), nch * 6 * sizeof(double)});
}

int atom_sums_impl(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* field,
                   const std::vector<AtomGeo>& atoms, const AtomGeo* atoms_dev, double* sums_dev,
                   void* scratch, size_t scratch_bytes) {
  const int k = int(atoms.size());
  if (k == 0) return SFW3D_OK;
  std::vector<Chunk> chunks;
  std::vector<int> first;
  chunk_plan(atoms, chunks, first);
  Carver cv(scratch);
  Chunk* ch_dev = cv.take<Chunk>(chunks.size());
  int* first_dev = cv.take<int>(first.size());
  double* part = cv.take<double>(chunks.size() * 6);
  if (cv.off > scratch_bytes) {
    set_error("atom_sums scratch too small");
    return SFW3D_ECUDA;
  }
  SFW3D_TRY(stage_upload(ctx, ch_dev, chunks.data(), chunks.size() * sizeof(Chunk)));
  SFW3D_TRY(stage_upload(ctx, first_dev, first.data(), first.size() * sizeof(int)));
  const unsigned nch = unsigned(chunks.size());
  SFW3D_PROF(ctx, "atom_sums");
  if (dtype == SFW3D_F64)
    atom_sums_kernel<double><<<nch, kSumThreads, 0, ctx->stream>>>(
        atoms_dev, ch_dev, dims[0], dims[1], dims[2], static_cast<const double*>(field), part);
  else
    atom_sums_kernel<float><<<nch, kSumThreads, 0, ctx->stream>>>(
        atoms_dev, ch_dev, dims[0], dims[1], dims[2], static_cast<const float*>(field), part);
  SFW3D_LAUNCH_CHECK(ctx);
  chunk_combine_kernel<<<(k * 6 + 255) / 256, 256, 0, ctx->stream>>>(first_dev, k, part, sums_dev);
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
