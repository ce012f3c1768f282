// assign_mma.cuh — kernel (b) for large codebooks: the distance step as a DMMA
// contraction plus an exact re-check, still bit-exact against the reference.
//
// nearest_row (proj/src/quantizer.cpp:113-130) evaluates d_p = sum_k (eta_k - c_pk)^2
// serially (products and sums rounded, no FMA) and keeps the first p with the
// smallest d_p. For P = 4096 centroids in m = 64 dimensions (BASELINE C5) that is a
// 2^20 x 64 x 4096 distance table. Here the table is formed as a contraction on the
// fp64 tensor pipe,
//     d~_p = (|eta|^2 + |c_p|^2) - 2 eta . c_p      (mma.sync.m8n8k4.f64),
// whose error against the exact real distance is below ~3e-14 (|eta|^2 + |c_p|^2)
// for m <= 64 (dot, norms and the two final roundings), and the reference's own
// rounded d_p is within m u d_p of it. With the bound
//     e_p = AM_EPS (|eta|^2 + |c_p|^2),   AM_EPS = 1e-12 (a 30x margin),
// the reference's argmin p* satisfies d~_{p*} - e_{p*} <= U := min_q (d~_q + e_q):
// pass 1 computes U per sample, pass 2 recomputes the table and evaluates the exact
// reference distance (same operations as nearest_row) for every p with
// d~_p - e_p <= U — typically the winner alone — keeping the smallest exact d and,
// among equal ones, the smallest p. The labels are the reference's bit for bit;
// only the candidate filter is approximate. A CTA whose candidate list overflows
// (pathological near-ties, non-finite distances) reports it and the batch is redone
// with the direct kernel (assign.cuh).
//
// Tiling: a CTA owns 64 samples (eta resident in shared memory) and streams the
// codebook in tiles of 128 centroids (L2-resident), 8 warps as 2 x 4 with a 32 x 32
// warp tile = 4 x 4 DMMA tiles; the same layout as the realisation kernel.
#pragma once
#include "common.cuh"

namespace vqpc {

constexpr int AM_BM = 64, AM_BN = 128, AM_THREADS = 256, AM_CAND = 256;
constexpr double AM_EPS = 1e-12;

struct AssignMmaParams {
  const double* xi;     // B x ld
  int64_t ld;
  int64_t B;
  const double* root;   // m (Scale map) or nullptr (latent sites)
  const double* sites;  // P x m
  const double* cnorm;  // P: |c_p|^2 (any summation order; covered by the bound)
  int P;
  int32_t* labels;
  double* best;         // nullable: the winning exact distance
  int* overflow;        // set when a CTA's candidate list overflows (batch redone directly)
};

__device__ __forceinline__ void am_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// order-preserving map of doubles to u64 (key(x) < key(y) iff x < y)
__device__ __forceinline__ unsigned long long am_key(double x) {
  const unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(x));
  return (v >> 63) ? ~v : (v | 0x8000000000000000ull);
}
__device__ __forceinline__ double am_val(unsigned long long k) {
  return __longlong_as_double(static_cast<long long>((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

template <int M>
constexpr size_t assign_mma_smem() {
  return sizeof(double) * (AM_BM * (M + 1) + AM_BN * (M + 1) + AM_BM + AM_CAND) +
         sizeof(unsigned long long) * 2 * AM_BM + sizeof(int) * (3 * AM_BM + 2 * AM_CAND + 1);
}

template <int M>
__global__ void __launch_bounds__(AM_THREADS) assign_mma_kernel(const AssignMmaParams prm) {
  static_assert(M % 4 == 0 && M <= 64, "k steps of 4");
  constexpr int LD = M + 1;
  extern __shared__ __align__(16) unsigned char am_raw[];
  double* sA = reinterpret_cast<double*>(am_raw);  // [64][LD] eta
  double* sB = sA + AM_BM * LD;                     // [128][LD] centroid tile
  double* sN = sB + AM_BN * LD;                     // [64] |eta|^2
  double* cD = sN + AM_BM;                          // [AM_CAND] exact distances of candidates
  unsigned long long* sU = reinterpret_cast<unsigned long long*>(cD + AM_CAND);  // [64] key of U_b
  unsigned long long* sBK = sU + AM_BM;                                          // [64] key of best exact d
  int* sBP = reinterpret_cast<int*>(sBK + AM_BM);  // [64] best p
  int* sBad = sBP + AM_BM;                         // [64] non-finite eta
  int* sValid = sBad + AM_BM;                      // [64]
  int* cB = sValid + AM_BM;                        // [AM_CAND] candidate row
  int* cP = cB + AM_CAND;                          // [AM_CAND] candidate p
  int* cN = cP + AM_CAND;                          // candidate count

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * AM_BM;
  const int P = prm.P;

  if (tid < AM_BM) {
    sBad[tid] = 0;
    sValid[tid] = b0 + tid < prm.B;
    sU[tid] = am_key(__longlong_as_double(0x7ff0000000000000ll));
    sBK[tid] = am_key(__longlong_as_double(0x7ff0000000000000ll));
    sBP[tid] = 0x7fffffff;
  }
  if (tid == 0) *cN = 0;
  __syncthreads();
  // eta tile: the reference's T2Map product (quantizer.cpp:50-55), exact
  for (int e = tid; e < AM_BM * M; e += AM_THREADS) {
    const int rb = e / M, k = e % M;
    const int64_t b = b0 + rb;
    double v = 0.0;
    if (b < prm.B) {
      v = prm.xi[b * prm.ld + k];
      if (!isfinite(v)) atomicOr(&sBad[rb], 1);
      v = prm.root ? __dmul_rn(prm.root[k], v) : v;
    }
    sA[rb * LD + k] = v;
  }
  __syncthreads();
  if (tid < AM_BM) {
    double s = 0.0;
    for (int k = 0; k < M; ++k) s = fma(sA[tid * LD + k], sA[tid * LD + k], s);
    sN[tid] = s;
  }
  for (int pass = 0; pass < 2; ++pass) {
    for (int p0 = 0; p0 < P; p0 += AM_BN) {
      __syncthreads();
      for (int e = tid; e < AM_BN * M; e += AM_THREADS) {
        const int pp = e / M, k = e % M;
        sB[pp * LD + k] = p0 + pp < P ? prm.sites[static_cast<size_t>(p0 + pp) * M + k] : 0.0;
      }
      __syncthreads();
      double acc[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < M; ks += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) af[a] = sA[(wm * 32 + a * 8 + (lane >> 2)) * LD + ks + (lane & 3)];
#pragma unroll
        for (int c = 0; c < 4; ++c) bf[c] = sB[(wn * 32 + c * 8 + (lane >> 2)) * LD + ks + (lane & 3)];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) am_dmma(acc[a][c][0], acc[a][c][1], af[a], bf[c]);
      }
      // epilogue: C (8x8) element (row lane/4, cols 2 (lane%4) + {0,1}) of tile (a, c)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int rb = wm * 32 + a * 8 + (lane >> 2);
        const double ne = sN[rb];
        const double U = pass == 1 ? am_val(sU[rb]) : 0.0;
        double umin = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int pp = wn * 32 + c * 8 + 2 * (lane & 3) + e;
            const int p = p0 + pp;
            if (p >= P || !sValid[rb] || sBad[rb]) continue;  // non-finite eta: label -1 below
            const double s = ne + prm.cnorm[p];
            const double dt = s - 2.0 * acc[a][c][e];
            const double bnd = AM_EPS * s;
            if (pass == 0) {
              umin = fmin(umin, dt + bnd);
            } else if (!(dt - bnd > U)) {  // candidate (NaN-safe: NaN is a candidate)
              // the reference's distance, operation for operation (quantizer.cpp:118-123)
              double d = 0.0;
              for (int k = 0; k < M; ++k) {
                const double t = __dsub_rn(sA[rb * LD + k], sB[pp * LD + k]);
                d = __dadd_rn(d, __dmul_rn(t, t));
              }
              const int slot = atomicAdd(cN, 1);
              if (slot < AM_CAND) {
                cB[slot] = rb;
                cP[slot] = p;
                cD[slot] = d;
              }
              atomicMin(&sBK[rb], am_key(d));
            }
          }
        if (pass == 0) {  // rows are shared by the 4 lanes of a quad and the 4 warps wn
          umin = fmin(umin, shfl_xor(umin, 1));
          umin = fmin(umin, shfl_xor(umin, 2));
          if ((lane & 3) == 0) atomicMin(&sU[rb], am_key(umin));
        }
      }
    }
    __syncthreads();
  }
  // among the candidates at the smallest exact distance, the smallest p (strict <)
  const int nc = *cN;
  if (nc > AM_CAND) {
    if (tid == 0) atomicExch(prm.overflow, 1);
    return;
  }
  for (int i = tid; i < nc; i += AM_THREADS)
    if (am_key(cD[i]) == sBK[cB[i]]) atomicMin(&sBP[cB[i]], cP[i]);
  __syncthreads();
  if (tid < AM_BM && sValid[tid]) {
    const int64_t b = b0 + tid;
    const int p = sBP[tid];
    prm.labels[b] = sBad[tid] ? -1 : (p == 0x7fffffff ? 0 : p);
    if (prm.best) prm.best[b] = am_val(sBK[tid]);
  }
}

// |c_p|^2 for the contraction form (once per context)
static __global__ void centroid_norms_kernel(const double* sites, int P, int m, double* cnorm) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double s = 0.0;
  for (int k = 0; k < m; ++k) s = fma(sites[static_cast<size_t>(p) * m + k], sites[static_cast<size_t>(p) * m + k], s);
  cnorm[p] = s;
}

}  // namespace vqpc
