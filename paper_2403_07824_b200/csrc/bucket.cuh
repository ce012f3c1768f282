// bucket.cuh — kernel (c): stable counting sort of sample ids by label.
//
// Replaces the grouping loop of run_campaign_with (proj/src/driver.cpp:221-226):
// groups[p] = {i : a_i = p} in index order. Output perm[] lists the samples
// bucket by bucket, increasing index inside a bucket; offsets[p] is bucket p's
// start (P+2 entries: bucket P collects invalid samples, label -1).
// Three passes, all HBM/L2-bound integer work:
//   1. per-tile histograms  (tile = BK_TILE samples, shared-memory atomics)
//   2. exclusive scan of the (bin-major, tile-minor) count matrix (one CTA)
//   3. per-tile stable scatter: one warp walks its tile in order 32 samples at
//      a time; __match_any_sync groups equal labels, popc ranks them.
#pragma once
#include "common.cuh"

namespace vqpc {

constexpr int BK_TILE = 1024;

static __global__ void bucket_hist_kernel(const int32_t* labels, const int32_t* ids, int64_t B, int P, int ntiles,
                                          int32_t* counts) {
  extern __shared__ int32_t sh[];  // P + 1 bins
  const int tile = blockIdx.x;
  for (int p = threadIdx.x; p <= P; p += blockDim.x) sh[p] = 0;
  __syncthreads();
  const int64_t lo = static_cast<int64_t>(tile) * BK_TILE;
  const int64_t hi = min64(B, lo + BK_TILE);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    int l = labels[ids ? ids[i] : i];
    if (l < 0 || l >= P) l = P;
    atomicAdd(&sh[l], 1);
  }
  __syncthreads();
  for (int p = threadIdx.x; p <= P; p += blockDim.x) counts[static_cast<size_t>(p) * ntiles + tile] = sh[p];
}

// exclusive scan of counts[(P+1) * ntiles] in place; offsets[p] = start of bin p
static __global__ void __launch_bounds__(1024) bucket_scan_kernel(int32_t* counts, int64_t total, int P, int ntiles,
                                                           int64_t* offsets) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (total + 1023) / 1024;
  const int64_t lo = min64(total, t * per), hi = min64(total, lo + per);
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += counts[i];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = t > 0 ? part[t - 1] : 0;
  for (int64_t i = lo; i < hi; ++i) {
    const int32_t c = counts[i];
    counts[i] = static_cast<int32_t>(run);
    run += c;
  }
  __syncthreads();
  for (int p = t; p <= P; p += 1024) offsets[p] = counts[static_cast<size_t>(p) * ntiles];
  if (t == 0) offsets[P + 1] = part[1023];
}

static __global__ void bucket_scatter_kernel(const int32_t* labels, const int32_t* ids, int64_t B, int P, int ntiles,
                                             const int32_t* starts, int32_t* perm) {
  extern __shared__ int32_t cnt[];  // P + 1 running positions
  const int tile = blockIdx.x, lane = threadIdx.x;
  for (int p = lane; p <= P; p += 32) cnt[p] = starts[static_cast<size_t>(p) * ntiles + tile];
  __syncwarp();
  const int64_t lo = static_cast<int64_t>(tile) * BK_TILE;
  const int64_t hi = min64(B, lo + BK_TILE);
  for (int64_t base = lo; base < hi; base += 32) {
    const int64_t i = base + lane;
    const bool valid = i < hi;
    const int32_t id = valid ? (ids ? ids[i] : static_cast<int32_t>(i)) : 0;
    int l = valid ? labels[id] : -2;
    if (valid && (l < 0 || l >= P)) l = P;
    const unsigned peers = __match_any_sync(VQPC_FULL_MASK, l);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int pos = 0;
    if (valid) pos = cnt[l] + rank;
    __syncwarp();
    if (valid) {
      perm[pos] = id;
      if (rank == 0) cnt[l] += __popc(peers);
    }
    __syncwarp();
  }
}

// Work-queue order (longest predicted solve first). The PCG work per sample is
// heavy-tailed (C2: 11 % of the samples take 78 % of the iterations), so a
// bucket-ordered queue leaves a tail of a few long solves on otherwise idle SMs.
// Predictor: the KL-weighted distance between the sample and its centroid's
// field, |log kappa - log kappa_c|^2 in M-norm = sum_k lambda_k (xi_k - c_k)^2
// (c_k = the centroid's latent coordinates for k < m, 0 beyond). Keys are
// descending eighth-octave bins of it; a stable second counting-sort pass over
// the label buckets keeps samples of one preconditioner together inside a bin.
// (Pure scheduling: per-sample results do not depend on the order.)
constexpr int COST_BINS = 128;
static __global__ void cost_key_kernel(const double* xi, int64_t ld, int64_t B, int K, int m, const int32_t* labels,
                                       const double* sqrt_lam, const double* sites, const double* root,
                                       int32_t* keys) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const int l = labels[i];
  if (l < 0) {
    keys[i] = COST_BINS - 1;
    return;
  }
  const double* x = xi + i * ld;
  const double* c = sites + static_cast<size_t>(l) * m;
  double s = 0.0;
  for (int k = 0; k < K; ++k) {
    double v = x[k];
    if (k < m) v -= root ? c[k] / root[k] : c[k];  // centroid in latent coordinates
    const double d = sqrt_lam[k] * v;
    s = fma(d, d, s);
  }
  int bin = s > 0.0 ? static_cast<int>(floor(8.0 * log2(s))) + COST_BINS / 2 : 0;
  bin = bin < 0 ? 0 : (bin >= COST_BINS ? COST_BINS - 1 : bin);
  keys[i] = COST_BINS - 1 - bin;
}

}  // namespace vqpc
