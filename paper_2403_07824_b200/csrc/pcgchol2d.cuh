// pcgchol2d.cuh — 2-D campaigns with the reference's own `cholesky` preconditioner
// (proj/src/solver.cpp:72-111, kind "cholesky", driver.hpp:13): every centroid
// matrix is reordered by reverse Cuthill-McKee (solver.cpp:32-70, computed once
// on the host: the pattern is the same for every centroid), factored as LL^T over
// its envelope, and each sample's PCG applies z = P^T L^-T L^-1 P r.
//
// (e) cholfactor2d_kernel — one CTA per centroid, the factor BIT-IDENTICAL to the
//     oracle's restatement of SimplicialLLT's up-looking rows (oracle/src/
//     vqp_oracle.cpp CholeskyPreconditioner): row k of the permuted matrix is
//     L_kl = (B_kl - sum_j L_kj L_lj) / L_ll (j ascending, rounded products, no
//     contraction), L_kk = sqrt(B_kk - sum_l L_kl^2). Rows are dealt round-robin to
//     the 256 threads; a thread computing L_kl waits on a shared-memory flag until
//     row l is final, so up to 256 rows advance as a pipelined wavefront.
//     cholinv_kernel then inverts the 32 x 32 diagonal blocks of L (per centroid,
//     once) so the in-block part of each triangular solve is a small GEMV.
// (d) pcgchol2d_kernel<S> — one CTA per group of S samples that share a label
//     (multi right-hand side: every byte of the factor streamed from HBM serves S
//     solves). All vectors live in HBM in the RCM order, so the preconditioner's
//     permutation is free and the stencil product gathers through a neighbour
//     table. The triangular solves walk the envelope in blocks of 32 rows: a
//     block's rows are contiguous in L, so one cp.async.bulk (TMA) copy per block
//     lands them in shared memory, double-buffered on transaction mbarriers.
//       forward  y_B = Linv_B (r_B - L_{B,<B} y)       (left-looking, warp per row)
//       backward z_B = Linv_B^T w_B; w_j -= L_{B,j}^T z_B  (right-looking, thread per column)
//     with y / w in a shared-memory ring of the last PC_RING rows (>= W + 32, W the
//     envelope width). Dot products are block-tree sums (the throughput mode of
//     pcg2d); the control flow and the update arithmetic follow solver.cpp:186-245.
#pragma once
#include "pcg2d.cuh"

namespace vqpc {

#ifndef PC_PF
#define PC_PF 1   // batches ahead the vector passes pull their streamed operands into L2 (0: off)
#endif
__device__ __forceinline__ void pc_prefetch(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

constexpr int PC_T = 256;     // threads per CTA
constexpr int PC_BS = 32;     // rows per block of the triangular solves
constexpr int PC_RING = 1024; // y / w ring (rows)
constexpr int PC_NV = 12;     // per sample slot: D, cS, cW, cE, cN, b, x, r, p, Ap, z, x'
constexpr int PC_MAXS = 8;
#ifndef VQPC_PC_U
#define VQPC_PC_U 4
#endif
#ifndef VQPC_PC_U2
#define VQPC_PC_U2 2
#endif
constexpr int PC_U = VQPC_PC_U;    // rows per thread per batch of the elementwise vector passes
constexpr int PC_U2 = VQPC_PC_U2;  // ... and of the stencil passes (Ap, b - Ax)
// y / w ring rows for S slots: 1024 up to S = 4; 512 beyond, so that the ring and two
// stages still fit 227 KB (W <= PC_WIN keeps W + 3 PC_BS <= 512)
constexpr int pc_ring(int S) { return S > 4 ? 512 : PC_RING; }
constexpr int PC_WIN = 256;   // columns left of a block the products cover (>= the envelope width W)
// per block of a centroid's Linv array and of a stage (doubles): Linv_B [1024] |
// block metadata [32: first[32], offset of row i's column 0 in the staged rows[32]];
// a stage then holds the block's envelope rows
constexpr int PC_STG_META = PC_BS * PC_BS;
constexpr int PC_LIB = PC_STG_META + PC_BS;
constexpr int PC_STG_R = PC_LIB;

struct CholLayout {
  int n;                 // unknowns
  int W;                 // envelope width max_k (k - first[k])
  int nblk;              // ceil(n / PC_BS)
  const int* cperm;      // permuted row -> natural interior id (iy * m + ix)
  const int* first;      // envelope start of each permuted row
  const int64_t* start;  // offset of row k (entries first[k] .. k) in L; n + 1 entries
  const int4* nbr;       // permuted rows of the S, W, E, N neighbours (-1: none)
};

// ---- (e) factor -----------------------------------------------------------------
__global__ void __launch_bounds__(PC_T) cholfactor2d_kernel(const double* kappa_c, int64_t ldk, int P,
                                                            const Grid2D g, const CholLayout lay, double* L,
                                                            int64_t ldL, int* err) {
  __shared__ int done[PC_T];  // 1 + the last row finished by thread t (its rows ascend)
  const int p = blockIdx.x, t = threadIdx.x;
  if (p >= P) return;
  const double* kap = kappa_c + static_cast<size_t>(p) * ldk;
  double* Lp = L + static_cast<size_t>(p) * ldL;
  done[t] = 0;
  __syncthreads();
  volatile int* vdone = done;
  bool ok = true;
  for (int k = t; k < lay.n; k += PC_T) {
    const int f = lay.first[k];
    double* Lk = Lp + lay.start[k] - f;  // Lk[l] = L(k, l)
    for (int l = f; l <= k; ++l) Lk[l] = 0.0;
    const int id = lay.cperm[k];
    const RowCoef rc = assemble_row(kap, g, id % g.m, id / g.m);
    const int4 nb = lay.nbr[k];
    if (nb.x >= 0 && nb.x < k) Lk[nb.x] = rc.s;
    if (nb.y >= 0 && nb.y < k) Lk[nb.y] = rc.w;
    if (nb.z >= 0 && nb.z < k) Lk[nb.z] = rc.e;
    if (nb.w >= 0 && nb.w < k) Lk[nb.w] = rc.nn;
    double d = rc.d;
    for (int l = f; l < k; ++l) {
      const int owner = l % PC_T;
      while (vdone[owner] <= l) {
      }
      __threadfence_block();
      const int fl = lay.first[l];
      const double* Ll = Lp + lay.start[l] - fl;
      double s = Lk[l];
      for (int j = f > fl ? f : fl; j < l; ++j) s = __dsub_rn(s, __dmul_rn(Lk[j], Ll[j]));
      const double lkl = __ddiv_rn(s, Ll[l]);
      Lk[l] = lkl;
      d = __dsub_rn(d, __dmul_rn(lkl, lkl));
    }
    if (!(d > 0.0)) ok = false;
    Lk[k] = __dsqrt_rn(d);
    __threadfence_block();
    vdone[t] = k + 1;
  }
  if (!ok) atomicExch(err, 1);
}

// inverse of every 32 x 32 diagonal block of L (row-major [i][c], zero above the
// diagonal; rows past n are identity rows), into the first 1024 doubles of the
// block's PC_LIB-double record. One thread per (centroid, block, column).
__global__ void cholinv_kernel(const double* L, int64_t ldL, const CholLayout lay, int P, double* Linv,
                               int64_t ldLi) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = static_cast<int>(idx & 31);
  const int64_t bp = idx >> 5;
  if (bp >= static_cast<int64_t>(P) * lay.nblk) return;
  const int p = static_cast<int>(bp / lay.nblk), blk = static_cast<int>(bp % lay.nblk);
  const int r0 = blk * PC_BS;
  const double* Lp = L + static_cast<size_t>(p) * ldL;
  double* out = Linv + static_cast<size_t>(p) * ldLi + static_cast<size_t>(blk) * (PC_BS * PC_BS + PC_BS);
  double x[PC_BS];
  for (int i = 0; i < PC_BS; ++i) {
    const int k = r0 + i;
    if (k >= lay.n) {
      x[i] = i == c ? 1.0 : 0.0;
    } else if (i < c) {
      x[i] = 0.0;
    } else {
      const int f = lay.first[k];
      const double* Lk = Lp + lay.start[k] - f;
      double s = i == c ? 1.0 : 0.0;
      for (int q = (f - r0 > c ? f - r0 : c); q < i; ++q) s = fma(-Lk[r0 + q], x[q], s);
      x[i] = s / Lk[k];
    }
  }
  for (int i = 0; i < PC_BS; ++i) out[i * PC_BS + c] = x[i];
}

// Work groups: up to S consecutive entries of a label bucket (perm is label-major,
// predicted-cost-descending inside a bucket). Emitted q-major — the q-th group of
// every label before any (q+1)-th — so every factor's heaviest samples go first.
// One CTA: per round q, the labels whose bucket still has a q-th group are
// compacted by a block-wide exclusive scan over the P + 1 buckets (O(P / CG_T)
// per round instead of a serial O(P) loop).
constexpr int CG_T = 1024;
constexpr int CG_PER = 8;  // buckets per thread per scan (P + 1 <= CG_T * CG_PER handled per chunk)
__global__ void __launch_bounds__(CG_T) chol_groups_kernel(const int64_t* offsets, int P, int S, int2* groups,
                                                           int* ngroups) {
  __shared__ int wsum[CG_T / 32];
  __shared__ int s_base, s_any;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_base = 0;
  __syncthreads();
  for (int64_t q = 0;; ++q) {
    if (t == 0) s_any = 0;
    __syncthreads();
    for (int c0 = 0; c0 <= P; c0 += CG_T * CG_PER) {
      int cnt = 0;
      bool has[CG_PER];
#pragma unroll
      for (int u = 0; u < CG_PER; ++u) {
        const int p = c0 + t * CG_PER + u;
        has[u] = p <= P && offsets[p] + q * S < offsets[p + 1];
        cnt += has[u];
      }
      int incl = cnt;  // inclusive scan of cnt over the block
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        int w = lane < CG_T / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, w, off);
          if (lane >= off) w += v;
        }
        if (lane < CG_T / 32) wsum[lane] = w;  // inclusive over warps
      }
      __syncthreads();
      int pos = s_base + (warp > 0 ? wsum[warp - 1] : 0) + incl - cnt;
#pragma unroll
      for (int u = 0; u < CG_PER; ++u) {
        const int p = c0 + t * CG_PER + u;
        if (has[u]) {
          const int64_t lo = offsets[p] + q * S, hi = offsets[p + 1];
          groups[pos++] = make_int2(static_cast<int>(lo), static_cast<int>(hi - lo < S ? hi - lo : S));
        }
      }
      const int total = wsum[CG_T / 32 - 1];
      __syncthreads();
      if (t == 0) {
        s_base += total;
        if (total) s_any = 1;
      }
      __syncthreads();
    }
    if (!s_any) break;
  }
  if (t == 0) *ngroups = s_base;
}

struct PcholParams {
  Grid2D g;
  CholLayout lay;
  const double* kappa;  // samples x ldk nodal kappa
  int64_t ldk;
  const uint8_t* kflag;
  const int32_t* perm;  // label-major order
  const int32_t* labels;
  const int2* groups;
  const int* ngroups;
  const double* L;      // P x ldL envelope factors
  int64_t ldL;
  const double* Linv;   // P x ldLi inverted diagonal blocks
  int64_t ldLi;
  int cap;              // doubles per staged block (max over blocks, 16-byte padded)
  const int64_t* blk_a0;     // per block: first staged L index (even)
  const unsigned* blk_bytes; // per block: staged bytes (multiple of 16)
  int ldv;              // per-slot vector stride (multiple of 32)
  double* work;         // per CTA: S * PC_NV * ldv doubles
  int64_t B, out_base, solve_limit;
  double eps;
  int max_iter;
  const int32_t* max_iter_arr;
  int* counter;
  int32_t* iters;
  double* rel;
  uint8_t* status;
  double* x_out;        // nullable, natural interior order
};

__device__ __forceinline__ void pc_bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void pc_mbar_init(unsigned bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void pc_mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pc_mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n PC_WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PC_WAIT;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void pc_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int S>
__device__ __forceinline__ void pc_block_sums(double (&v)[S], double (*red)[PC_T / 32], int warp, int lane) {
#pragma unroll
  for (int s = 0; s < S; ++s) v[s] = warp_allsum(v[s]);
  if (lane == 0)
#pragma unroll
    for (int s = 0; s < S; ++s) red[s][warp] = v[s];
  __syncthreads();
#pragma unroll
  for (int s = 0; s < S; ++s) {
    double a[PC_T / 32];
#pragma unroll
    for (int i = 0; i < PC_T / 32; ++i) a[i] = red[s][i];
#pragma unroll
    for (int w = 1; w < PC_T / 32; w <<= 1)
#pragma unroll
      for (int i = 0; i + w < PC_T / 32; i += 2 * w) a[i] += a[i + w];
    v[s] = a[0];
  }
  __syncthreads();
}

template <int S>
__global__ void __launch_bounds__(PC_T, 1) pcgchol2d_kernel(const PcholParams prm) {
  extern __shared__ __align__(128) double dsm[];
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ double red[S][PC_T / 32];
  __shared__ double tv[S][PC_BS];
  __shared__ double red2[(PC_T / 32) * PC_BS * S];  // per-warp partial products (forward)
  __shared__ int s_first[PC_BS];
  __shared__ int64_t s_start[PC_BS];
  __shared__ int s_grp;
  const Grid2D g = prm.g;
  const CholLayout lay = prm.lay;
  const int n = lay.n, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int stage_len = PC_LIB + prm.cap;
  constexpr int RING = pc_ring(S);
  double* ring = dsm + 2 * stage_len;  // [S][RING]
  const unsigned bar0 = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[0]));
  if (t == 0) {
    pc_mbar_init(bar0);
    pc_mbar_init(bar0 + 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ldv = prm.ldv;  // vector stride: n rounded up to whole 32-row blocks (TMA-aligned)
  double* base = prm.work + static_cast<size_t>(blockIdx.x) * S * PC_NV * ldv;
  auto vec = [&](int s, int v) { return base + (static_cast<size_t>(s) * PC_NV + v) * ldv; };
  enum { VD = 0, VS, VW, VE, VN, VB, VX, VR, VP, VAP, VZ, VX2 };
  int64_t vg = 0;  // staged-block visits issued by this CTA (mbarrier phases)
  const int nvis = 2 * lay.nblk;

  for (;;) {
    if (t == 0) s_grp = atomicAdd(prm.counter, 1);
    __syncthreads();
    const int grp = s_grp;
    __syncthreads();
    if (grp >= *prm.ngroups) break;
    const int2 gr = prm.groups[grp];
    int sid[S];
    int64_t gsv[S];
    bool act[S];
    int J[S], mit[S];
    double rel_rec[S], norm_b[S], rz[S], beta[S], alpha[S];
    uint8_t st[S];
    int label = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      act[s] = false;
      J[s] = 0;
      rel_rec[s] = 0.0;
      st[s] = VQPC_S_MAX_ITER;
      sid[s] = -1;
      gsv[s] = 0;
      if (s < gr.y) {
        const int sm = prm.perm[gr.x + s];
        sid[s] = sm;
        gsv[s] = prm.out_base + sm;
        const int lb = prm.labels[sm];
        if (lb < 0 || prm.kflag[sm] || gsv[s] >= prm.solve_limit) {
          st[s] = gsv[s] >= prm.solve_limit ? VQPC_S_NOT_SOLVED
                  : lb < 0                  ? VQPC_S_INVALID_LATENT
                                            : (prm.kflag[sm] & 1) ? VQPC_S_COEFF_OVERFLOW : VQPC_S_INVALID_COEFF;
        } else {
          act[s] = true;
          label = lb;  // a group shares one label (bucketed)
        }
        mit[s] = prm.max_iter_arr ? prm.max_iter_arr[gsv[s]] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);
      }
    }
    const double* Lp = prm.L + static_cast<size_t>(label) * prm.ldL;
    const double* Lip = prm.Linv + static_cast<size_t>(label) * prm.ldLi;

    // ---- setup: rows of every sample in RCM order; x = 0, r = b ---------------------
    double part[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      part[s] = 0.0;
      if (!act[s]) continue;
      const double* kap = prm.kappa + static_cast<size_t>(sid[s]) * prm.ldk;
      for (int k = t; k < n; k += PC_T) {
        const int id = lay.cperm[k];
        const RowCoef rc = assemble_row(kap, g, id % g.m, id / g.m);
        vec(s, VD)[k] = rc.d;
        vec(s, VS)[k] = rc.s;
        vec(s, VW)[k] = rc.w;
        vec(s, VE)[k] = rc.e;
        vec(s, VN)[k] = rc.nn;
        vec(s, VB)[k] = rc.b;
        vec(s, VX)[k] = 0.0;
        vec(s, VR)[k] = rc.b;
        part[s] = fma(rc.b, rc.b, part[s]);
      }
    }
    pc_block_sums<S>(part, red, warp, lane);
#pragma unroll
    for (int s = 0; s < S; ++s) norm_b[s] = sqrt(part[s]);

    // ---- z = M^{-1} r for every slot of the group; returns the r.z partials --------
    // Visit v = 0 .. 2 nblk - 1 walks the blocks forward then backward. Everything a
    // visit reads from HBM arrives by TMA one visit ahead on the stage's mbarrier:
    // Linv_B, the block's metadata (first[], offsets), r_B of every slot, the block's
    // envelope rows, and (backward) the y block entering the w window.
    const int WB = (lay.W + PC_BS - 1) / PC_BS;
    // issued by warp 0, one copy per lane (lane 0 arms the barrier first)
    auto issue = [&](int v, int64_t a0, unsigned cbytes) {
      if (warp != 0 || v >= nvis) return;
      const bool fwd = v < lay.nblk;
      const int blk = fwd ? v : nvis - 1 - v;
      const int stg = static_cast<int>((vg + v) & 1);
      double* sp = dsm + stg * stage_len;
      const unsigned bar = bar0 + 8u * stg;
      const int e = blk - WB;  // backward: y block entering the window (not left in the ring by the forward sweep)
      const bool zin = !fwd && e >= 0 && e < lay.nblk - RING / PC_BS;
      if (lane == 0) pc_mbar_expect(bar, PC_LIB * 8u + cbytes + (zin ? S * 256u : 0u));
      __syncwarp();
      auto sa = [](const void* q) { return static_cast<unsigned>(__cvta_generic_to_shared(q)); };
      VQPC_DCHECK(cbytes <= 8u * static_cast<unsigned>(prm.cap) && (cbytes & 15u) == 0 && (a0 & 1) == 0);
      if (lane == 0) {
        pc_bulk_g2s(sa(sp + PC_LIB), Lp + a0, cbytes, bar);
      } else if (lane == 1) {
        pc_bulk_g2s(sa(sp), Lip + static_cast<size_t>(blk) * PC_LIB, PC_LIB * 8u, bar);
      } else if (zin && lane >= 8 && lane < 8 + S) {
        const int s = lane - 8;
        pc_bulk_g2s(sa(ring + s * RING + ((e * PC_BS) & (RING - 1))), vec(s, VZ) + e * PC_BS, 256u, bar);
      }
    };
    auto blk_of = [&](int v) { return v < lay.nblk ? v : nvis - 1 - v; };
    auto solve = [&](double (&rzp)[S]) {
      P2_TIC(t_solve);
#pragma unroll
      for (int s = 0; s < S; ++s) rzp[s] = 0.0;
      __syncthreads();
      if (warp == 0) {
        issue(0, prm.blk_a0[blk_of(0)], prm.blk_bytes[blk_of(0)]);
        if (nvis > 1) issue(1, prm.blk_a0[blk_of(1)], prm.blk_bytes[blk_of(1)]);
      }
      for (int v = 0; v < nvis; ++v) {
        const bool fwd = v < lay.nblk;
        const int blk = blk_of(v);
        const int r0 = blk * PC_BS, r1 = min(n, r0 + PC_BS);
        const int64_t gv = vg + v;
        const int stg = static_cast<int>(gv & 1);
        const double* Li = dsm + stg * stage_len;
        const int* meta = reinterpret_cast<const int*>(Li + PC_STG_META);  // first[32], off[32]
        const double* ch = Li + PC_LIB;  // L(r0 + i, j) = ch[off[i] + j]
        VQPC_DCHECK(r1 - r0 <= PC_BS && lay.W + 3 * PC_BS <= RING);
        int64_t na0 = 0;
        unsigned nby = 0;
        if (warp == 0 && v + 2 < nvis) {  // next issue's source range, loaded while this visit computes
          na0 = prm.blk_a0[blk_of(v + 2)];
          nby = prm.blk_bytes[blk_of(v + 2)];
        }
        // r of the rows this thread finishes (forward: row t >> 3 for q < S; backward:
        // row t >> 3 of slot q), loaded before the wait so the latency hides behind it
        double rv = 0.0;
        {
          const int ii = t >> 3, q = t & 7;
          if (q < S && r0 + ii < r1) rv = vec(q, VR)[r0 + ii];
        }
        P2_TIC(t_wait);
        pc_mbar_wait(bar0 + 8u * stg, static_cast<unsigned>((gv >> 1) & 1));
        P2_TOC(2, t_wait);
        P2_TIC(t_fwd);
        if (fwd) {
          {
            // T = L_{B,window} Y on the fp64 tensor pipe (mma.sync.m8n8k4.f64): 32 rows
            // (4 m-tiles) x the PC_WIN columns left of the block (8 k-steps per warp) x
            // the S slots (N = 8, zero-padded); entries left of first[] are zeros
            const int cofs = static_cast<int>(ch - dsm);
            const int ra = lane >> 2, ka = lane & 3;
            const int jw = r0 - PC_WIN + 32 * warp;
            int fr[4], of[4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
              fr[mt] = meta[8 * mt + ra];
              of[mt] = cofs + meta[PC_BS + 8 * mt + ra];
            }
            double c[4][2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) c[mt][0] = c[mt][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const int j = jw + 4 * ks + ka;
              const double b = (ra < S && j >= 0) ? ring[ra * RING + (j & (RING - 1))] : 0.0;
#pragma unroll
              for (int mt = 0; mt < 4; ++mt) {
                const double a = j >= fr[mt] ? dsm[of[mt] + j] : 0.0;
                pc_dmma(c[mt][0], c[mt][1], a, b);
              }
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                if (2 * ka + e < S) red2[(warp * PC_BS + 8 * mt + ra) * S + 2 * ka + e] = c[mt][e];
          }
          __syncthreads();
          {
            const int ii = t >> 3, q = t & 7;
            if (q < S) {
              double a = 0.0;
#pragma unroll
              for (int w = 0; w < PC_T / 32; ++w) a += red2[(w * PC_BS + ii) * S + q];
              tv[q][ii] = r0 + ii < r1 ? rv - a : 0.0;
            }
          }
          __syncthreads();
          if (warp < 4) {
            // y_B = Linv_B T on DMMA: warp = m-tile (8 rows), K = the 32 block columns,
            // N = the S slots (zero-padded to 8)
            const int ra = lane >> 2, ka = lane & 3, i = 8 * warp + ra;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const int k = 4 * ks + ka;
              pc_dmma(c0, c1, Li[i * PC_BS + k], ra < S ? tv[ra][k] : 0.0);
            }
            // y into the ring and to HBM straight from the fragments (the backward sweep
            // re-reads HBM blocks by TMA); 8 consecutive rows per slot per warp store
            if (r0 + i < r1) {
              if (2 * ka < S) {
                ring[(2 * ka) * RING + ((r0 + i) & (RING - 1))] = c0;
                vec(2 * ka, VZ)[r0 + i] = c0;
              }
              if (2 * ka + 1 < S) {
                ring[(2 * ka + 1) * RING + ((r0 + i) & (RING - 1))] = c1;
                vec(2 * ka + 1, VZ)[r0 + i] = c1;
              }
            }
          }
          // y goes back to HBM; the backward sweep re-reads blocks of it by TMA, the
          // first of them WB + 1 visits after the sweep turns (fence below)
          __syncthreads();
          P2_TOC(3, t_fwd);
        } else {
          if (v == lay.nblk) asm volatile("fence.proxy.async;" ::: "memory");  // this thread's y stores
          if (warp < 4) {
            // z_B = Linv_B^T w_B on DMMA: warp = m-tile (8 columns c), K = the 32 block
            // rows, N = the S slots (zero-padded to 8)
            const int ra = lane >> 2, ka = lane & 3, c = 8 * warp + ra;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const int i = 4 * ks + ka;
              const double w = ra < S && r0 + i < r1 ? ring[ra * RING + ((r0 + i) & (RING - 1))] : 0.0;
              pc_dmma(c0, c1, Li[i * PC_BS + c], w);
            }
            if (2 * ka < S) tv[2 * ka][c] = r0 + c < r1 ? c0 : 0.0;
            if (2 * ka + 1 < S) tv[2 * ka + 1][c] = r0 + c < r1 ? c1 : 0.0;
          }
          __syncthreads();
          {
            const int c = t >> 3, q = t & 7;
            if (q < S && r0 + c < r1) {
              const double z = tv[q][c];
              vec(q, VZ)[r0 + c] = z;
#pragma unroll
              for (int s = 0; s < S; ++s)
                if (q == s) rzp[s] = fma(rv, z, rzp[s]);
            }
          }
          const int lo = r0 - lay.W > 0 ? r0 - lay.W : 0;
          {
            // w_j -= sum_i L(r0 + i, j) z_i for the PC_WIN columns left of the block, as
            // DMMA tiles: M = columns (4 m-tiles of 8 per warp), K = the 32 block rows
            // (8 k-steps), N = the S slots
            const int cofs = static_cast<int>(ch - dsm);
            const int ra = lane >> 2, ka = lane & 3;
            int fi[8], oi[8];
            double bz[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const int i = 4 * ks + ka;
              fi[ks] = meta[i];
              oi[ks] = cofs + meta[PC_BS + i];
              bz[ks] = ra < S ? tv[ra][i] : 0.0;
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
              const int j = r0 - PC_WIN + 32 * warp + 8 * mt + ra;
              double c0 = 0.0, c1 = 0.0;
#pragma unroll
              for (int ks = 0; ks < 8; ++ks) {
                const double a = j >= fi[ks] ? dsm[oi[ks] + j] : 0.0;
                pc_dmma(c0, c1, a, bz[ks]);
              }
              if (j >= lo) {
                if (2 * ka < S) ring[(2 * ka) * RING + (j & (RING - 1))] -= c0;
                if (2 * ka + 1 < S) ring[(2 * ka + 1) * RING + (j & (RING - 1))] -= c1;
              }
            }
          }
          // these generic-proxy writes to the ring precede later cp.async.bulk writes of
          // the same rows (the zin reloads): order them for the async proxy before the
          // barrier that releases the next issue
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
        }
        P2_TIC(t_iss);
        issue(v + 2, na0, nby);
        P2_TOC(0, t_iss);
      }
      vg += nvis;
      pc_block_sums<S>(rzp, red, warp, lane);
      P2_TOC(1, t_solve);
    };

    bool any0 = false;
#pragma unroll
    for (int s = 0; s < S; ++s) any0 |= act[s];
    double rzp[S];
    if (any0) solve(rzp);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      rz[s] = rzp[s];
      beta[s] = 0.0;
      if (!act[s]) continue;
      if (norm_b[s] == 0.0) {
        st[s] = VQPC_S_CONVERGED;
        act[s] = false;
      } else if (!(rz[s] > 0.0)) {
        st[s] = VQPC_S_BREAKDOWN;
        act[s] = false;
      } else if (mit[s] < 1) {
        act[s] = false;
      }
    }
    for (int j = 1;; ++j) {
      bool any = false;
#pragma unroll
      for (int s = 0; s < S; ++s) any |= act[s];
      if (!any) break;
      // p = z + beta p (p = z on the first iteration), solver.cpp:241
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (!act[s]) continue;
        double* P = vec(s, VP);
        const double* Z = vec(s, VZ);
        // the vector passes batch PC_U rows per thread (loads first, then the same
        // per-row operations and accumulation order): 8 warps per SM need the MLP
        for (int k0 = t; k0 < n; k0 += PC_U * PC_T) {
          double zv[PC_U], pv[PC_U];
          if (PC_PF > 0) {
#pragma unroll
            for (int u = 0; u < PC_U; ++u) {
              const int kp = k0 + (PC_PF * PC_U + u) * PC_T;
              if (kp < n) {
                pc_prefetch(Z + kp);
                if (j != 1) pc_prefetch(P + kp);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < PC_U; ++u) {
            const int k = k0 + u * PC_T;
            zv[u] = k < n ? Z[k] : 0.0;
            pv[u] = k < n && j != 1 ? P[k] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < PC_U; ++u) {
            const int k = k0 + u * PC_T;
            if (k < n) P[k] = j == 1 ? zv[u] : __dadd_rn(zv[u], __dmul_rn(beta[s], pv[u]));
          }
        }
      }
      __syncthreads();
      // Ap and p.Ap (CSR column order S, W, diag, E, N; no contraction)
#pragma unroll
      for (int s = 0; s < S; ++s) {
        part[s] = 0.0;
        if (!act[s]) continue;
        const double* P = vec(s, VP);
        double* AP = vec(s, VAP);
        for (int k0 = t; k0 < n; k0 += PC_U2 * PC_T) {
          double ap[PC_U2], pk[PC_U2];
          if (PC_PF > 0) {
#pragma unroll
            for (int u = 0; u < PC_U2; ++u) {
              const int kp = k0 + (PC_PF * PC_U2 + u) * PC_T;
              if (kp < n) {
                pc_prefetch(lay.nbr + kp);
                pc_prefetch(P + kp);
                pc_prefetch(vec(s, VS) + kp);
                pc_prefetch(vec(s, VW) + kp);
                pc_prefetch(vec(s, VD) + kp);
                pc_prefetch(vec(s, VE) + kp);
                pc_prefetch(vec(s, VN) + kp);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < PC_U2; ++u) {
            const int k = k0 + u * PC_T;
            ap[u] = pk[u] = 0.0;
            if (k < n) {
              const int4 nb = lay.nbr[k];
              pk[u] = P[k];
              ap[u] = row_apply(vec(s, VS)[k], vec(s, VW)[k], vec(s, VD)[k], vec(s, VE)[k], vec(s, VN)[k],
                                nb.x >= 0 ? P[nb.x] : 0.0, nb.y >= 0 ? P[nb.y] : 0.0, pk[u],
                                nb.z >= 0 ? P[nb.z] : 0.0, nb.w >= 0 ? P[nb.w] : 0.0);
            }
          }
#pragma unroll
          for (int u = 0; u < PC_U2; ++u) {
            const int k = k0 + u * PC_T;
            if (k < n) {
              AP[k] = ap[u];
              part[s] = fma(pk[u], ap[u], part[s]);
            }
          }
        }
      }
      pc_block_sums<S>(part, red, warp, lane);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (!act[s]) continue;
        if (!(part[s] > 0.0)) {
          st[s] = VQPC_S_BREAKDOWN;
          act[s] = false;
          continue;
        }
        alpha[s] = rz[s] / part[s];
      }
      // x, r updates fused with the true residual b - A x (solver.cpp:220-222): x_new at
      // the stencil's points is recomputed from the old x and p with the same two
      // operations and stored into the other x buffer (iteration j writes buffer j & 1),
      // so no barrier separates the update from the residual sweep
#pragma unroll
      for (int s = 0; s < S; ++s) {
        part[s] = 0.0;
        if (!act[s]) continue;
        const double a = alpha[s];
        const double* Xo = vec(s, (j & 1) ? VX : VX2);
        double* Xn = vec(s, (j & 1) ? VX2 : VX);
        double* R = vec(s, VR);
        const double* P = vec(s, VP);
        const double* AP = vec(s, VAP);
        auto xnew = [&](int i) { return __dadd_rn(Xo[i], __dmul_rn(a, P[i])); };
        for (int k0 = t; k0 < n; k0 += PC_U2 * PC_T) {
          double rt[PC_U2];
          if (PC_PF > 0) {
#pragma unroll
            for (int u = 0; u < PC_U2; ++u) {
              const int kp = k0 + (PC_PF * PC_U2 + u) * PC_T;
              if (kp < n) {
                pc_prefetch(lay.nbr + kp);
                pc_prefetch(Xo + kp);
                pc_prefetch(P + kp);
                pc_prefetch(AP + kp);
                pc_prefetch(R + kp);
                pc_prefetch(vec(s, VB) + kp);
                pc_prefetch(vec(s, VS) + kp);
                pc_prefetch(vec(s, VW) + kp);
                pc_prefetch(vec(s, VD) + kp);
                pc_prefetch(vec(s, VE) + kp);
                pc_prefetch(vec(s, VN) + kp);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < PC_U2; ++u) {
            const int k = k0 + u * PC_T;
            rt[u] = 0.0;
            if (k < n) {
              const int4 nb = lay.nbr[k];
              const double xk = xnew(k);
              const double ax = row_apply(vec(s, VS)[k], vec(s, VW)[k], vec(s, VD)[k], vec(s, VE)[k], vec(s, VN)[k],
                                          nb.x >= 0 ? xnew(nb.x) : 0.0, nb.y >= 0 ? xnew(nb.y) : 0.0, xk,
                                          nb.z >= 0 ? xnew(nb.z) : 0.0, nb.w >= 0 ? xnew(nb.w) : 0.0);
              rt[u] = __dsub_rn(vec(s, VB)[k], ax);
              Xn[k] = xk;
              R[k] = __dsub_rn(R[k], __dmul_rn(a, AP[k]));
            }
          }
#pragma unroll
          for (int u = 0; u < PC_U2; ++u)
            if (k0 + u * PC_T < n) part[s] = fma(rt[u], rt[u], part[s]);
        }
      }
      pc_block_sums<S>(part, red, warp, lane);
      bool need = false;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (!act[s]) continue;
        const double rel = sqrt(part[s]) / norm_b[s];
        J[s] = j;
        rel_rec[s] = rel;
        if (rel < prm.eps) {
          st[s] = VQPC_S_CONVERGED;
          act[s] = false;
        } else {
          need = true;
        }
      }
      if (!need) break;
      solve(rzp);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (!act[s]) continue;
        if (!(rzp[s] > 0.0)) {
          st[s] = VQPC_S_BREAKDOWN;
          act[s] = false;
          continue;
        }
        beta[s] = rzp[s] / rz[s];
        rz[s] = rzp[s];
        if (j >= mit[s]) act[s] = false;  // loop exhausted: MAX_ITER
      }
    }
    // ---- outputs -------------------------------------------------------------------
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (s >= gr.y) continue;
      if (t == 0) {
        prm.iters[gsv[s]] = J[s];
        prm.rel[gsv[s]] = rel_rec[s];
        prm.status[gsv[s]] = st[s];
      }
      const bool solved = st[s] == VQPC_S_CONVERGED || st[s] == VQPC_S_MAX_ITER || st[s] == VQPC_S_BREAKDOWN;
      if (prm.x_out && solved) {
        double* xo = prm.x_out + static_cast<size_t>(gsv[s]) * n;
        const double* X = vec(s, (J[s] & 1) ? VX2 : VX);  // iteration J wrote buffer J & 1
        for (int k = t; k < n; k += PC_T) xo[lay.cperm[k]] = J[s] > 0 ? X[k] : 0.0;
      }
    }
    __syncthreads();
  }
}

// Preconditioner::apply for one centroid in the reference's serial order:
// Eigen's SimplicialLLT solve (solver.cpp:99-105; SimplicialCholeskyBase::_solve_impl)
// on the RCM-permuted vector. Forward: the column-major lower factor, every y_k
// receiving its column contributions in increasing column order. Backward:
// matrixU() = L.adjoint(), a row-major upper view, solved row by row from the
// bottom, z_i = (y_i - L(j1,i) z_j1 - L(j2,i) z_j2 - ...) / L(i,i) with j
// ascending over column i's stored rows (first[j] <= i, j - first[j] <= W).
// y is overwritten by z; one thread (the instrument, not the throughput path).
__device__ void chol_serial_solve(const double* Lp, const CholLayout& lay, double* y) {
  const int n = lay.n;
  for (int k = 0; k < n; ++k) {
    const int f = lay.first[k];
    const double* Lk = Lp + lay.start[k] - f;
    double s = y[k];
    for (int j = f; j < k; ++j) s = __dsub_rn(s, __dmul_rn(y[j], Lk[j]));
    y[k] = __ddiv_rn(s, Lk[k]);
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    const int jmax = min(n - 1, i + lay.W);
    for (int j = i + 1; j <= jmax; ++j) {
      const int fj = lay.first[j];
      if (fj > i) continue;
      s = __dsub_rn(s, __dmul_rn(Lp[lay.start[j] - fj + i], y[j]));
    }
    y[i] = __ddiv_rn(s, Lp[lay.start[i] - lay.first[i] + i]);
  }
}

__global__ void cholapply_serial_kernel(const double* L, int64_t ldL, const CholLayout lay, int p,
                                        const double* r, double* y, double* z) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* Lp = L + static_cast<size_t>(p) * ldL;
  const int n = lay.n;
  for (int k = 0; k < n; ++k) y[k] = r[lay.cperm[k]];
  chol_serial_solve(Lp, lay, y);
  for (int k = 0; k < n; ++k) z[lay.cperm[k]] = y[k];
}

// Reference-order mode of the 2-D cholesky kind (vqpc_set_exact_reductions): one CTA
// per sample; the vector passes are the throughput kernel's (same operations), the
// dot products are summed serially in NATURAL order (solver.cpp:176-180) from
// products stored at their natural index, and the preconditioner is
// chol_serial_solve. Given the same coefficient bits the whole solve (J, status,
// residual record, x) is bit-identical to the oracle. A parity instrument: the
// serial triangular solves cost ~n W dependent operations per application.
constexpr int PCX_NV = 13;  // D, cS, cW, cE, cN, b, x, r, p, Ap, z, prod, (spare)
__global__ void __launch_bounds__(PC_T) pcgchol2d_exact_kernel(const PcholParams prm) {
  __shared__ double s_val;
  __shared__ int64_t s_item;
  const Grid2D g = prm.g;
  const CholLayout lay = prm.lay;
  const int n = lay.n, t = threadIdx.x;
  double* base = prm.work + static_cast<size_t>(blockIdx.x) * PCX_NV * prm.ldv;
  auto vec = [&](int v) { return base + static_cast<size_t>(v) * prm.ldv; };
  double *D = vec(0), *CS = vec(1), *CW = vec(2), *CE = vec(3), *CN = vec(4), *Bv = vec(5), *X = vec(6), *R = vec(7),
         *Pv = vec(8), *AP = vec(9), *Z = vec(10), *Prod = vec(11);
  auto serial = [&]() {  // s = 0; s += prod_i, natural order
    __syncthreads();
    if (t == 0) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, Prod[i]);
      s_val = acc;
    }
    __syncthreads();
    const double v = s_val;
    __syncthreads();
    return v;
  };
  for (;;) {
    if (t == 0) s_item = atomicAdd(prm.counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    __syncthreads();
    if (item >= prm.B) break;
    const int sm = prm.perm[item];
    const int64_t gs = prm.out_base + sm;
    const int label = prm.labels[sm];
    if (label < 0 || prm.kflag[sm] || gs >= prm.solve_limit) {
      if (t == 0) {
        prm.iters[gs] = 0;
        prm.rel[gs] = 0.0;
        prm.status[gs] = gs >= prm.solve_limit ? VQPC_S_NOT_SOLVED
                         : label < 0           ? VQPC_S_INVALID_LATENT
                                               : (prm.kflag[sm] & 1) ? VQPC_S_COEFF_OVERFLOW : VQPC_S_INVALID_COEFF;
      }
      continue;
    }
    const double* Lp = prm.L + static_cast<size_t>(label) * prm.ldL;
    const double* kap = prm.kappa + static_cast<size_t>(sm) * prm.ldk;
    const int max_iter = prm.max_iter_arr ? prm.max_iter_arr[gs] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);
    for (int k = t; k < n; k += PC_T) {
      const int id = lay.cperm[k];
      const RowCoef rc = assemble_row(kap, g, id % g.m, id / g.m);
      D[k] = rc.d;
      CS[k] = rc.s;
      CW[k] = rc.w;
      CE[k] = rc.e;
      CN[k] = rc.nn;
      Bv[k] = rc.b;
      X[k] = 0.0;
      R[k] = rc.b;
      Z[k] = rc.b;
      Prod[id] = __dmul_rn(rc.b, rc.b);
    }
    const double norm_b = sqrt(serial());
    if (t == 0) chol_serial_solve(Lp, lay, Z);
    __syncthreads();
    for (int k = t; k < n; k += PC_T) {
      Pv[k] = Z[k];
      Prod[lay.cperm[k]] = __dmul_rn(R[k], Z[k]);
    }
    double rz = serial();
    int J = 0;
    double rel_rec = 0.0;
    uint8_t st = VQPC_S_MAX_ITER;
    if (norm_b == 0.0) st = VQPC_S_CONVERGED;
    else if (!(rz > 0.0)) st = VQPC_S_BREAKDOWN;
    else {
      for (int j = 1; j <= max_iter; ++j) {
        for (int k = t; k < n; k += PC_T) {
          const int4 nb = lay.nbr[k];
          const double ap = row_apply(CS[k], CW[k], D[k], CE[k], CN[k], nb.x >= 0 ? Pv[nb.x] : 0.0,
                                      nb.y >= 0 ? Pv[nb.y] : 0.0, Pv[k], nb.z >= 0 ? Pv[nb.z] : 0.0,
                                      nb.w >= 0 ? Pv[nb.w] : 0.0);
          AP[k] = ap;
          Prod[lay.cperm[k]] = __dmul_rn(Pv[k], ap);
        }
        const double pAp = serial();
        if (!(pAp > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        const double alpha = rz / pAp;
        for (int k = t; k < n; k += PC_T) {
          X[k] = __dadd_rn(X[k], __dmul_rn(alpha, Pv[k]));
          R[k] = __dsub_rn(R[k], __dmul_rn(alpha, AP[k]));
        }
        __syncthreads();
        for (int k = t; k < n; k += PC_T) {
          const int4 nb = lay.nbr[k];
          const double ax = row_apply(CS[k], CW[k], D[k], CE[k], CN[k], nb.x >= 0 ? X[nb.x] : 0.0,
                                      nb.y >= 0 ? X[nb.y] : 0.0, X[k], nb.z >= 0 ? X[nb.z] : 0.0,
                                      nb.w >= 0 ? X[nb.w] : 0.0);
          const double rt = __dsub_rn(Bv[k], ax);
          Prod[lay.cperm[k]] = __dmul_rn(rt, rt);
          Z[k] = R[k];
        }
        const double rel = sqrt(serial()) / norm_b;
        J = j;
        rel_rec = rel;
        if (rel < prm.eps) {
          st = VQPC_S_CONVERGED;
          break;
        }
        if (t == 0) chol_serial_solve(Lp, lay, Z);
        __syncthreads();
        for (int k = t; k < n; k += PC_T) Prod[lay.cperm[k]] = __dmul_rn(R[k], Z[k]);
        const double rz_next = serial();
        if (!(rz_next > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        const double beta = rz_next / rz;
        rz = rz_next;
        for (int k = t; k < n; k += PC_T) Pv[k] = __dadd_rn(Z[k], __dmul_rn(beta, Pv[k]));
        __syncthreads();
      }
    }
    if (t == 0) {
      prm.iters[gs] = J;
      prm.rel[gs] = rel_rec;
      prm.status[gs] = st;
    }
    if (prm.x_out) {
      double* xo = prm.x_out + static_cast<size_t>(gs) * n;
      for (int k = t; k < n; k += PC_T) xo[lay.cperm[k]] = X[k];
    }
    __syncthreads();
  }
}

}  // namespace vqpc
