// Shared separable Gaussian basis for the certificate (see basis.cu).
#pragma once

#include <cstdlib>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace sfw3d {

// argmax record shared by the certificate kernels: larger value wins, ties
// go to the smaller C-order index (first maximum, certificate.py:161-163)
struct Best {
  double v;
  long long idx;
};

__device__ __forceinline__ bool better(double v, long long i, double bv, long long bi) {
  return (v > bv) || (v == bv && i < bi);
}

struct BasisCandidate {
  double sigma, d;
  int lo[3], hi[3];   // the candidate's reference support box (offsets)
  long long direct_taps;
  double tap_tol = 0.0;  // direct taps below this are dropped (eta.cu build_candidate)
};

struct BasisSet;

// Fits every candidate on one shared dictionary of Gaussians (see basis.cu)
// and keeps those whose max abs error on the common box is <= tol.
// on_device = false fits on the host only (no device buffers; eval unusable);
// prune = greedily drop shared terms while every member stays within tol.
int basis_set_build(const int dims[3], const std::vector<BasisCandidate>& cands, int dtype,
                    double tol, BasisSet** out, bool on_device = true, bool prune = false,
                    double loose = 0.0);
// storage-dependent looser selection tolerance for the shared terms (fp32:
// 1e-5; fp64: none)
double basis_loose_tol(int dtype);
// host copy of the fit: betas[n_terms], weights[n_cand][max_terms] (member rows,
// zero elsewhere), w0[n_cand], fit_err[n_cand], member[n_cand]; NULLs skipped
void basis_set_export(const BasisSet* s, int max_terms, int* n_terms, double* betas,
                      double* weights, double* w0, double* fit_err, int32_t* member);
void basis_set_destroy(BasisSet* s);
// tables prune their shared terms for volumes of >= 2^26 voxels (~406^3;
// fp32 storage: >= 2^24, 256^3): there a term's three full-volume passes per
// certificate outweigh the seconds of host NNLS refits the pruning costs
// once per table (config 3: 48 -> 18 terms). The table option "prune"
// overrides (sfw3d_table_set_option); sharded tables pass the GLOBAL dims.
inline bool basis_prune_voxels(long long voxels, int dtype) {
  return voxels >= (dtype == SFW3D_F32 ? (1LL << 24) : (1LL << 26));
}
inline bool basis_prune_rule(const int dims[3], int dtype) {
  return basis_prune_voxels((long long)dims[0] * dims[1] * dims[2], dtype);
}
// candidate -> (is member, fit error of its shared-dictionary fit)
bool basis_set_member(const BasisSet* s, int cand, double* fit_err);
// Signed members: candidates outside the non-negative pool (d > 2, or d <= 2
// fits missing tol) fitted by weighted-ridge least squares on the SHARED terms.
// Their eta is only certified to within ebound * ||b||_inf / lam at every
// voxel (fit + rounding, see basis.cu), so they are used for argmax-only
// evaluations and always refined exactly (eta.cu); never for fields.
bool basis_set_signed(const BasisSet* s, int cand);
// per-candidate bound factor E (0 for non-signed): |eta~ - eta| <= E ||b||_inf / lam
double basis_set_ebound(const BasisSet* s, int cand);
int basis_set_n_terms(const BasisSet* s);
int basis_set_n_members(const BasisSet* s);
long long basis_set_taps(const BasisSet* s);        // per voxel, all shared terms
int basis_set_pass_taps(const BasisSet* s, int term, int axis);  // taps of one 1-D pass
// 1-D filters longer than this are FP32-bound (wide tiles), the others HBM-bound
// (psf.cu: kNarrowTaps; the profile families "eta_basis_wide" / "eta_basis")
constexpr int kBasisNarrowTaps = 24;
double basis_set_flops(const BasisSet* s);          // executed flops per voxel (all members)
double basis_set_member_flops(const BasisSet* s);   // mix flops per voxel per member

// Scratch (bytes) basis_set_eval needs for a volume of n elements.
size_t basis_set_scratch(const BasisSet* s, long long n, int dtype, const int dims[3]);
// eta for all members: best_dev[cand] receives each member's windowed
// argmax; fields (n_cand volumes, candidate-major) are written when non-NULL
// (then the signed members are skipped: their values are not certified).
// abs_dev (optional, device [2]): receives [sum |b|, max |b|] when the mix
// computed them on the way (*abs_done = true), saving a separate pass over b.
// x-slab evaluation (sfw3d_eta_argmax_slab): dims are the OWNED planes, every
// term's x pass runs through slab_corr_impl (window `win` of H + owned + H
// planes, H >= basis_set_max_xhalo, exchanged through `link`).
struct SlabEval {
  SlabLink link;
  void* win = nullptr;
  int H = 0;
};
int basis_set_max_xhalo(const BasisSet* s);
int basis_set_eval(sfw3d_ctx* ctx, const BasisSet* s, int dtype, const int dims[3], const void* b,
                   double lam, const int32_t win[6], void* fields, Best* best_dev, void* scratch,
                   double* abs_dev = nullptr, bool* abs_done = nullptr,
                   const SlabEval* se = nullptr);

// Refinement support (inexact / signed members): re-runs the fused mix over
// the terms basis_set_eval left in `scratch` (same `fields` flag; only the
// CTAs whose evaluation-pass maxima reach a threshold) and appends every windowed
// voxel whose approximate eta >= thr_dev[member] (member-indexed) to
// (cand_dev = candidate id, idx_dev = voxel); count_dev[0] receives the total
// (may exceed cap: then the list is incomplete), count_dev[1 + m] member m's.
int basis_set_collect(sfw3d_ctx* ctx, const BasisSet* s, int dtype, const int dims[3],
                      const void* b, double lam, const int32_t win[6], const double* thr_dev,
                      int cap, int* cand_dev, long long* idx_dev, int* count_dev, void* scratch,
                      bool fields);
int basis_set_member_index(const BasisSet* s, int cand);  // -1 when not a member
int basis_set_member_cand(const BasisSet* s, int member);

// Host-only single-candidate fit (the sfw3d_basis_fit ABI helper).
void fit_profile(const int lo[3], const int hi[3], double sigma, double d, double target,
                 double& w0, std::vector<std::pair<double, double>>& terms, double& err,
                 bool& exact);

}  // namespace sfw3d
