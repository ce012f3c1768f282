// realise.cuh — kernel (a): KL realisation kappa = exp(W Phi), W = sqrt(Lambda) .* Xi.
//
// Replaces lift (proj/src/field.cpp:113-125) + transport (:138-145) for a batch
// of samples: log kappa (B x N) = W (B x K) * Phi (K x N) with
// W_bk = sqrt(lambda_k) * xi_bk (the reference's `w`, same IEEE product) and
// Phi mode-major (field.hpp:25). The contraction runs on the FP64 tensor pipe
// (DMMA, mma.sync.m8n8k4.f64 — tcgen05 has no f64 kind); the exp epilogue
// writes kappa (the only per-element quantity the matrix-free solvers need)
// and flags samples with a non-finite value ("coefficient-overflow").
// Summation order differs from the reference's k-outer AXPY: kappa agrees to
// rounding (~1e-15 relative), checked in tests.
//
// Tiling: CTA = 64 samples x 128 points, 8 warps as 2 (samples) x 4 (points),
// warp tile 32 x 32 = 4 x 4 DMMA tiles (32 fp64 accumulators per lane).
// K is staged through shared memory in blocks of 16 (zero padded).
#pragma once
#include "common.cuh"

namespace vqpc {

constexpr int RL_BM = 64, RL_BN = 128, RL_BK = 16, RL_THREADS = 256;
constexpr int RL_WLD = RL_BK + 1;   // padded row stride of the W tile
constexpr int RL_PLD = RL_BN + 4;   // padded row stride of the Phi tile

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct RealiseParams {
  const double* xi;        // B x ld (rows), first K_use columns used
  int64_t ld;
  int64_t B;
  const double* sqrt_lam;  // >= K_use
  const double* phi;       // n_kl x n_nodes mode-major
  int n_nodes;
  int K_use;               // modes lifted (m)
  double* kappa;           // B x ldk
  int64_t ldk;
  uint8_t* flag;           // per sample, ORed: 1 non-finite kappa (transport's coefficient-overflow),
                           // 2 kappa == 0 (assembly's invalid-coefficient); nullable
};

// dynamic shared memory of realise_kernel: two stages of {W tile, Phi tile}
constexpr int RL_STAGE = RL_BM * RL_WLD + RL_BK * RL_PLD;  // doubles per stage
constexpr size_t RL_SMEM = sizeof(double) * 2 * RL_STAGE;

static __global__ void __launch_bounds__(RL_THREADS) realise_kernel(const RealiseParams prm) {
  // K blocks are double-buffered: the global loads of block k + 1 are issued into
  // registers before the DMMA loop of block k and stored to the other stage after it,
  // so their latency hides behind the tensor work and one barrier per block suffices.
  // The accumulation order over k is unchanged (kappa bits as the single-stage kernel).
  extern __shared__ __align__(16) double rl_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  const int64_t b0 = static_cast<int64_t>(blockIdx.y) * RL_BM;
  const int i0 = blockIdx.x * RL_BN;
  constexpr int NWE = RL_BM * RL_BK / RL_THREADS;  // W elements per thread (4)
  constexpr int NPE = RL_BK * RL_BN / RL_THREADS;  // Phi elements per thread (8)

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;

  double rw[NWE], rp[NPE];
  auto load_block = [&](int k0) {
#pragma unroll
    for (int u = 0; u < NWE; ++u) {  // W tile: 64 x 16, w = sqrt(lambda_k) * xi (no contraction)
      const int e = tid + u * RL_THREADS, rb = e / RL_BK, kk = e % RL_BK;
      const int64_t b = b0 + rb;
      const int k = k0 + kk;
      rw[u] = (b < prm.B && k < prm.K_use) ? __dmul_rn(prm.sqrt_lam[k], prm.xi[b * prm.ld + k]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < NPE; ++u) {  // Phi tile: 16 x 128 (coalesced along points)
      const int e = tid + u * RL_THREADS, kk = e / RL_BN, ii = e % RL_BN;
      const int k = k0 + kk, i = i0 + ii;
      rp[u] = (k < prm.K_use && i < prm.n_nodes) ? prm.phi[static_cast<size_t>(k) * prm.n_nodes + i] : 0.0;
    }
  };
  auto store_block = [&](int stage) {
    double* sW = rl_smem + stage * RL_STAGE;
    double* sP = sW + RL_BM * RL_WLD;
#pragma unroll
    for (int u = 0; u < NWE; ++u) {
      const int e = tid + u * RL_THREADS;
      sW[(e / RL_BK) * RL_WLD + e % RL_BK] = rw[u];
    }
#pragma unroll
    for (int u = 0; u < NPE; ++u) {
      const int e = tid + u * RL_THREADS;
      sP[(e / RL_BN) * RL_PLD + e % RL_BN] = rp[u];
    }
  };
  load_block(0);
  store_block(0);
  __syncthreads();
  int stage = 0;
  for (int k0 = 0; k0 < prm.K_use; k0 += RL_BK, stage ^= 1) {
    const bool more = k0 + RL_BK < prm.K_use;
    if (more) load_block(k0 + RL_BK);
    const double* sW = rl_smem + stage * RL_STAGE;
    const double* sP = sW + RL_BM * RL_WLD;
#pragma unroll
    for (int ks = 0; ks < RL_BK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a)  // A (8x4 row): row = lane/4, col = lane%4
        af[a] = sW[(wm * 32 + a * 8 + (lane >> 2)) * RL_WLD + ks + (lane & 3)];
#pragma unroll
      for (int c = 0; c < 4; ++c)  // B (4x8 col): k = lane%4, n = lane/4
        bf[c] = sP[(ks + (lane & 3)) * RL_PLD + wn * 32 + c * 8 + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma_8x8x4(acc[a][c][0], acc[a][c][1], af[a], bf[c]);
    }
    if (more) store_block(stage ^ 1);  // last read two blocks ago, before the previous barrier
    __syncthreads();
  }
  // epilogue: C (8x8): row = lane/4, cols = 2*(lane%4) + {0,1}
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t b = b0 + wm * 32 + a * 8 + (lane >> 2);
    if (b >= prm.B) continue;
    unsigned bad = 0;  // bit 0: non-finite kappa (transport), bit 1: kappa == 0 (assembly)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + wn * 32 + c * 8 + 2 * (lane & 3);
      const double k0v = exp(acc[a][c][0]);
      const double k1v = exp(acc[a][c][1]);
      double* dst = prm.kappa + b * prm.ldk + i;
      if (i + 1 < prm.n_nodes) {
        bad |= (!isfinite(k0v) || !isfinite(k1v) ? 1u : 0u) | (k0v == 0.0 || k1v == 0.0 ? 2u : 0u);
        if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          *reinterpret_cast<double2*>(dst) = make_double2(k0v, k1v);
        } else {
          dst[0] = k0v;
          dst[1] = k1v;
        }
      } else if (i < prm.n_nodes) {
        bad |= (!isfinite(k0v) ? 1u : 0u) | (k0v == 0.0 ? 2u : 0u);
        dst[0] = k0v;
      }
    }
    if (bad && prm.flag) {  // several lanes / CTAs flag one sample: OR into the byte atomically
      uint8_t* fp = prm.flag + b;
      const uintptr_t a = reinterpret_cast<uintptr_t>(fp);
      atomicOr(reinterpret_cast<unsigned*>(a & ~static_cast<uintptr_t>(3)), bad << (8 * (a & 3)));
    }
  }
}

// Reference-order realisation (vqpc_set_exact_reductions): h = lift(xi) as the
// reference's k-outer AXPY (field.cpp:113-125) — h_i = 0; for each k with
// w_k = sqrt(lambda_k) xi_k != 0: h_i += w_k * phi_ki, product and sum rounded
// separately — on the CUDA cores, then kappa = exp(h) as in the DMMA kernel. h is
// bit-identical to the reference's lift; kappa differs from a glibc exp by at most
// CUDA exp's 1-ulp error. Same tiling as realise_kernel (64 samples x 128 points
// per CTA); each thread owns 4 samples x 8 points.
static __global__ void __launch_bounds__(RL_THREADS) realise_exact_kernel(const RealiseParams prm) {
  __shared__ double sW[RL_BM * RL_WLD];
  __shared__ double sP[RL_BK * RL_PLD];
  const int tid = threadIdx.x;
  const int ts = tid >> 4, tp = tid & 15;  // 16 x 16 threads: samples ts*4.., points tp + 16 c
  const int64_t b0 = static_cast<int64_t>(blockIdx.y) * RL_BM;
  const int i0 = blockIdx.x * RL_BN;
  double acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[a][c] = 0.0;
  for (int k0 = 0; k0 < prm.K_use; k0 += RL_BK) {
    __syncthreads();
    for (int e = tid; e < RL_BM * RL_BK; e += RL_THREADS) {
      const int rb = e / RL_BK, kk = e % RL_BK;
      const int64_t b = b0 + rb;
      const int k = k0 + kk;
      double v = 0.0;
      if (b < prm.B && k < prm.K_use) v = __dmul_rn(prm.sqrt_lam[k], prm.xi[b * prm.ld + k]);
      sW[rb * RL_WLD + kk] = v;
    }
    for (int e = tid; e < RL_BK * RL_BN; e += RL_THREADS) {
      const int kk = e / RL_BN, ii = e % RL_BN;
      const int k = k0 + kk, i = i0 + ii;
      sP[kk * RL_PLD + ii] = (k < prm.K_use && i < prm.n_nodes) ? prm.phi[static_cast<size_t>(k) * prm.n_nodes + i]
                                                                 : 0.0;
    }
    __syncthreads();
    const int kend = prm.K_use - k0 < RL_BK ? prm.K_use - k0 : RL_BK;
    for (int kk = 0; kk < kend; ++kk) {
      double ph[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) ph[c] = sP[kk * RL_PLD + tp + 16 * c];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double w = sW[(ts * 4 + a) * RL_WLD + kk];
        if (w != 0.0) {  // the reference skips w == 0 (field.cpp:120)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[a][c] = __dadd_rn(acc[a][c], __dmul_rn(w, ph[c]));
        }
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t b = b0 + ts * 4 + a;
    if (b >= prm.B) continue;
    unsigned bad = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = i0 + tp + 16 * c;
      if (i >= prm.n_nodes) continue;
      const double kv = exp(acc[a][c]);
      bad |= (!isfinite(kv) ? 1u : 0u) | (kv == 0.0 ? 2u : 0u);
      prm.kappa[b * prm.ldk + i] = kv;
    }
    if (bad && prm.flag) {
      uint8_t* fp = prm.flag + b;
      const uintptr_t ad = reinterpret_cast<uintptr_t>(fp);
      atomicOr(reinterpret_cast<unsigned*>(ad & ~static_cast<uintptr_t>(3)), bad << (8 * (ad & 3)));
    }
  }
}

}  // namespace vqpc
