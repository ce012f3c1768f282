// assign.cuh — kernel (b): bit-exact nearest-centroid assignment.
//
// Replaces assign / nearest_row (proj/src/quantizer.cpp:113-145) and the
// driver's serial loop over realisations (driver.cpp:206-210):
//   eta_k = sqrt(lambda_k) * xi_k           (Scale map, T2Map::to_quant :50-55)
//   d_p   = ((0 + t_0^2) + t_1^2) + ...     t_k = eta_k - c_pk, no FMA
//   label = argmin_p d_p, smallest p on ties (strict <)
// Every product/sum uses __dmul_rn/__dsub_rn/__dadd_rn so the fp64 values are
// the reference's bit for bit; the argmin over a lane group combines
// (d, p) lexicographically with warp shuffles, which equals the serial
// strict-< scan. Grid and sign-grid codebooks measure in latent space
// (quantizer.cpp:139-141): pass root == nullptr and the latent sites.
// Non-finite xi -> label -1 ("invalid-latent").
//
// SPLIT lanes cooperate on one sample (lane q scans p = q, q+SPLIT, ...), so
// small batches still fill the machine; the codebook streams through shared
// memory in tiles with a padded row stride (conflict-free strided reads).
#pragma once
#include "common.cuh"

namespace vqpc {

constexpr int AS_THREADS = 128;
constexpr int AS_TILE_DOUBLES = 6144;  // 48 KB of centroids per tile

struct AssignParams {
  const double* xi;     // B x ld
  int64_t ld;
  int64_t B;
  const double* root;   // m (Scale map) or nullptr (latent / pre-mapped)
  const double* sites;  // P x m
  int P, m;
  int32_t* labels;      // B
  double* best;         // B (nullable): the winning distance
  const int* only_if;   // nullable: run only when *only_if != 0 (fallback after assign_mma_kernel)
};

template <int M, int SPLIT>
__global__ void __launch_bounds__(AS_THREADS) assign_kernel(const AssignParams prm) {
  if (prm.only_if && *prm.only_if == 0) return;
  extern __shared__ double sc[];
  constexpr int SLD = M + 1;  // padded stride
  const int tid = threadIdx.x, lane = tid & 31;
  const int q = lane % SPLIT;
  const int64_t b = (static_cast<int64_t>(blockIdx.x) * AS_THREADS + tid) / SPLIT;
  const bool active = b < prm.B;

  double eta[M];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double v = active ? prm.xi[b * prm.ld + k] : 0.0;
    bad |= !isfinite(v);
    eta[k] = prm.root ? __dmul_rn(prm.root[k], v) : v;
  }

  const int tileP = AS_TILE_DOUBLES / SLD;
  double best_d = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int best = 0x7fffffff;
  for (int p0 = 0; p0 < prm.P; p0 += tileP) {
    const int np = min(tileP, prm.P - p0);
    __syncthreads();
    for (int e = tid; e < np * M; e += AS_THREADS) {
      const int pp = e / M, k = e % M;
      sc[pp * SLD + k] = prm.sites[static_cast<size_t>(p0 + pp) * M + k];
    }
    __syncthreads();
    for (int pp = q; pp < np; pp += SPLIT) {
      const double* c = sc + pp * SLD;
      double d = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double t = __dsub_rn(eta[k], c[k]);
        d = __dadd_rn(d, __dmul_rn(t, t));
      }
      if (d < best_d) {  // strict: within this lane's increasing p, smallest wins
        best_d = d;
        best = p0 + pp;
      }
    }
  }
  // lexicographic (d, p) min across the SPLIT lanes of a sample
#pragma unroll
  for (int off = 1; off < SPLIT; off <<= 1) {
    const double od = shfl_xor(best_d, off);
    const int op = __shfl_xor_sync(VQPC_FULL_MASK, best, off);
    if (od < best_d || (od == best_d && op < best)) {
      best_d = od;
      best = op;
    }
  }
  if (active && q == 0) {
    prm.labels[b] = bad ? -1 : (best == 0x7fffffff ? 0 : best);
    if (prm.best) prm.best[b] = best_d;
  }
}

// Generic m (eta staged in local memory), used when no specialisation exists.
template <int SPLIT>
__global__ void __launch_bounds__(AS_THREADS) assign_kernel_generic(const AssignParams prm) {
  if (prm.only_if && *prm.only_if == 0) return;
  extern __shared__ double sc[];
  const int M = prm.m, SLD = M + 1;
  const int tid = threadIdx.x, lane = tid & 31;
  const int q = lane % SPLIT;
  const int64_t b = (static_cast<int64_t>(blockIdx.x) * AS_THREADS + tid) / SPLIT;
  const bool active = b < prm.B;
  double eta[256];
  bool bad = false;
  for (int k = 0; k < M; ++k) {
    const double v = active ? prm.xi[b * prm.ld + k] : 0.0;
    bad |= !isfinite(v);
    eta[k] = prm.root ? __dmul_rn(prm.root[k], v) : v;
  }
  const int tileP = AS_TILE_DOUBLES / SLD;
  double best_d = __longlong_as_double(0x7ff0000000000000ll);
  int best = 0x7fffffff;
  for (int p0 = 0; p0 < prm.P; p0 += tileP) {
    const int np = min(tileP, prm.P - p0);
    __syncthreads();
    for (int e = tid; e < np * M; e += AS_THREADS) {
      const int pp = e / M, k = e % M;
      sc[pp * SLD + k] = prm.sites[static_cast<size_t>(p0 + pp) * M + k];
    }
    __syncthreads();
    for (int pp = q; pp < np; pp += SPLIT) {
      const double* c = sc + pp * SLD;
      double d = 0.0;
      for (int k = 0; k < M; ++k) {
        const double t = __dsub_rn(eta[k], c[k]);
        d = __dadd_rn(d, __dmul_rn(t, t));
      }
      if (d < best_d) {
        best_d = d;
        best = p0 + pp;
      }
    }
  }
#pragma unroll
  for (int off = 1; off < SPLIT; off <<= 1) {
    const double od = shfl_xor(best_d, off);
    const int op = __shfl_xor_sync(VQPC_FULL_MASK, best, off);
    if (od < best_d || (od == best_d && op < best)) {
      best_d = od;
      best = op;
    }
  }
  if (active && q == 0) {
    prm.labels[b] = bad ? -1 : (best == 0x7fffffff ? 0 : best);
    if (prm.best) prm.best[b] = best_d;
  }
}

// ---- minmax (farthest point) seeding helpers (quantizer.cpp:181-213) --------
// min_d[i] = min(min_d[i], |x_i - c|^2) with the reference's exact arithmetic;
// init = true writes the first distances.
static __global__ void minmax_update_kernel(const double* pts, int n, int m, const double* centroids, int p_src,
                                     double* min_d, bool init) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* x = pts + static_cast<size_t>(i) * m;
  const double* c = centroids + static_cast<size_t>(p_src) * m;
  double d = 0.0;
  for (int k = 0; k < m; ++k) {
    const double t = __dsub_rn(x[k], c[k]);
    d = __dadd_rn(d, __dmul_rn(t, t));
  }
  min_d[i] = init ? d : (d < min_d[i] ? d : min_d[i]);  // std::min keeps the first on ties
}

// block-level (max value, smallest index) of min_d
static __global__ void argmax_first_kernel(const double* v, int n, double* part_v, int* part_i) {
  __shared__ double sv[32];
  __shared__ int si[32];
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = v[i];
    if (x > bv) {  // increasing i within a thread: keeps the first maximum
      bv = x;
      bi = i;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = shfl_xor(bv, off);
    const int oi = __shfl_xor_sync(VQPC_FULL_MASK, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = bv;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k)
      if (sv[k] > bv || (sv[k] == bv && si[k] < bi)) {
        bv = sv[k];
        bi = si[k];
      }
    part_v[blockIdx.x] = bv;
    part_i[blockIdx.x] = bi;
  }
}

// final reduction + copy of the chosen point into centroid slot p; flags a
// non-positive maximum ("insufficient-samples").
static __global__ void minmax_pick_kernel(const double* part_v, const int* part_i, int nparts, const double* pts,
                                   int m, double* centroids, int p, int* err) {
  __shared__ int s_far;
  if (threadIdx.x == 0) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int k = 0; k < nparts; ++k)
      if (part_v[k] > bv || (part_v[k] == bv && part_i[k] < bi)) {
        bv = part_v[k];
        bi = part_i[k];
      }
    if (!(bv > 0.0)) *err = 1;
    s_far = bi;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < m; k += blockDim.x)
    centroids[static_cast<size_t>(p) * m + k] = pts[static_cast<size_t>(s_far) * m + k];
}

}  // namespace vqpc
