// pcg1d.cuh — kernel (d), 1-D: batched PCG, one CTA per sample, persistent grid.
//
// Replaces, for every sample of a bucket, the reference's per-sample loop body
// (proj/src/driver.cpp:228-239): transport(lift) -> assemble -> pcg with the
// centroid's Cholesky preconditioner (proj/src/solver.cpp:186-245, :80-111).
//
// Layout. One CTA of T threads owns one sample at a time; thread t owns the R
// consecutive rows [tR, tR+R) of the n unknowns (n <= R*T; padding rows are
// dead and provably inert, see below). Registers per thread: x, r, p (R each),
// the preconditioner couplings n_j and the transient w/z (or A p). Shared
// memory is thread-major ([i*T + t] holds row tR+i, so warp accesses are
// bank-conflict free, 8 bytes per row and array): the sample's element
// conductances c_j = kappa_j/h (the diagonal c_j + c_{j+1} is re-formed with the
// same IEEE add wherever it is needed), the centroid factor's n_j and 1/u_j^2
// and per-thread scan constants, reloaded only when the bucket (label) changes.
//
// Operator: A_jj = c_j + c_{j+1}, A_{j,j+1} = -c_{j+1}
// with c_j = kappa_j / h — the same IEEE values the oracle's CSR holds; b_j = h.
// Matrix-free: (A v)_j = -c_j v_{j-1} + d_j v_j - c_{j+1} v_{j+1}, evaluated in the
// reference's CSR row order without contraction (see VQPC_AP_CSR/VQPC_RESID_CSR).
//
// Preconditioner: the exact factor of the centroid matrix, M = U U^T with U the
// upper-bidiagonal Cholesky factor of the reference's RCM (= reversed) order
// (solver.cpp:32-70 on a path graph), stored as U = (I+N) D:
//   sweep 1 (descending)  y_j = r_j - n_j y_{j+1};   y_j <- y_j / u_j^2
//   sweep 2 (ascending)   z_j = y_j - n_{j-1} z_{j-1}
// Each sweep is a first-order linear recurrence, solved as a chunked scan:
// four interleaved serial chains over the quarters of a thread's rows, an
// affine scan over lanes with shuffles whose multipliers are per-centroid
// constants (one SHFL pair + one FMA per level), one barrier for the warp
// aggregates, a short fold over warps, and a fix-up pass.
//
// Per iteration, in the reference's operation order (solver.cpp:211-242):
//   Ap = A p; pAp = p.Ap               -> barrier 1 (reduction)
//   alpha; x += alpha p; r -= alpha Ap
//   r_true = b - A x; rr = |r_true|^2   (rides barrier 2)
//   sweep 1                             -> barrier 2 (warp aggregates + rr)
//   rel = sqrt(rr)/|b|
//   sweep 2                             -> barrier 3 (warp aggregates)
//   record; rel < eps -> converged (the exit waits for sweep 2: off the critical path)
//   rz' = r.z                            -> barrier 4 (reduction + z halos)
//   beta = rz'/rz; p = z + beta p
// Halo values of x and p are never exchanged: each thread updates its copy of
// the neighbours' boundary entries with the same FMA the neighbour executes,
// so they stay bit-identical; only z boundary values travel (barrier 4).
// Block reductions: 4 split accumulators per thread, a butterfly inside the
// warp, then every thread sums the NW warp partials with the same fixed tree —
// all threads hold identical bits and the order never depends on scheduling.
// Breakdown checks use !(v > 0) exactly like the reference (NaN-safe).
//
// Cluster variant (CL = 2, n up to 2 R T): a sample spans the two CTAs of a
// thread-block cluster (one per SM); warp aggregates, reduction partials and
// the CTA-boundary z halos are written into the peer's shared memory with
// st.async, each carrying its byte count to the peer's per-exchange mbarrier,
// so every per-iteration barrier is a local __syncthreads plus an mbarrier
// phase wait instead of a cluster barrier (C5: 109k -> 139k samples/s). Every
// CTA still folds the same NWT = CL * NW warp values in the same order, so
// results are identical to a single-CTA run of the same rows.
//
// Dead rows j >= n: n_j = 1/u_j^2 = 0 (so z_j = p_j = x_j = 0) and n_{n-1} = 0.
// Shared memory holds the conductances c_j for j <= n (c_n is the true right
// conductance of row n-1, so d_{n-1} = c_{n-1} + c_n needs no special case;
// its coupling term multiplies the dead p_n = 0) and 0 beyond. Warps that own
// dead rows (the last one for n = 2^k - 1; up to all but the first for other n)
// take a masked code path for A p and b - A x behind a warp-uniform branch (row
// n would otherwise see c_n, and every dead row would add b_j = h to |b - A x|).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace vqpc {

struct Pcg1dParams {
  int n;                      // unknowns
  int N;                      // elements (= n + 1)
  double h;                   // 1 / N
  const double* kappa;        // samples x N (row stride ldk), natural sample order
  int64_t ldk;
  const uint8_t* kflag;       // per sample: nonzero -> coefficient overflow
  const int32_t* perm;        // bucket order -> local sample index
  const int32_t* labels;      // per local sample
  const double2* factors;     // P x NP {n_j, 1/u_j^2}
  int NP;                     // padded rows per factor (= R*T)
  int64_t B;                  // samples in this batch
  int64_t out_base;           // global index of local sample 0 (outputs)
  int64_t solve_limit;        // samples with global index >= this are not solved
  double eps;
  int max_iter;               // < 0 -> 10 n
  const int32_t* max_iter_arr;  // nullable, indexed by global sample
  int* counter;               // work queue head
  int32_t* iters;
  double* rel;
  uint8_t* status;
  double* x_out;              // nullable, (global sample) x n
  unsigned long long* t_span;  // nullable diagnostics: per CTA {start, end} %globaltimer (ns)
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

#ifdef VQPC_PHASE_TIMING
__device__ unsigned long long g_pcg1d_phase[4];  // cycles from each barrier to the next (thread 0)
#define P1D_MARK(i)                                                                         \
  if (tid == 0 && rank == 0) {                                                              \
    const long long now_ = clock64();                                                       \
    if (ph_last >= 0) atomicAdd(&g_pcg1d_phase[i], static_cast<unsigned long long>(now_ - ph_last)); \
    ph_last = now_;                                                                         \
  }
#else
#define P1D_MARK(i)
#endif

template <int R, int T, int CL>
struct Pcg1dShared {
  static constexpr int NW = T / 32;
  static constexpr int NWT = CL * NW;  // warps per sample (whole cluster)
  double fn[R * T];       // factor couplings n_j, thread-major
  double fu[R * T];       // factor pivots 1/u_j^2, thread-major
  double c[R * T];        // element conductances c_j = kappa_j / h for j <= n (0 beyond), thread-major;
                          // the diagonal d_j = c_j + c_{j+1} is formed on the fly (same IEEE add)
  double cs_end;          // c_{R*T}: right conductance of the last thread's last row (0 beyond n)
  double lev[12 * T];     // per-thread lane-scan multipliers: L1[5], Q1, L2[5], Q2
  double qa[8 * T];       // per-thread quarter products: sweep 1 [0..3], sweep 2 [4..7]
  double2 f1[NWT], f2[NWT];   // per warp {product of the sweep multipliers (per centroid),
                              //           aggregate of this iteration}, sweeps 1 and 2 (all CTAs)
  double red[4][NWT];         // reduction partials: pAp, rr, rz, |b|^2 (all CTAs)
  double zf[T], zl[T];      // first / last z of every thread
  double zf_peer, zl_peer;  // CL == 2: the peer CTA's boundary z (rank 0 gets rank 1's first, rank 1 rank 0's last)
  unsigned long long mbar[4];  // CL == 2: per-exchange transaction barriers (barriers 1..4)
  int64_t item;
};

// The true residual b - A x decides J (rel < eps), so it is evaluated in the
// reference's exact CSR order without contraction: given the same x it is
// bit-identical to the CPU's, which measurably tightens iteration-count parity
// (C1: |dJ| <= 2, mean J equal to 2 decimals). A p only shapes
// the trajectory, yet evaluating it in the same CSR order also keeps the GPU
// trajectory measurably closer to the CPU's (C1 A/B: frac(|dJ|>1) 0.68 % vs 1.1 %,
// max |dJ| 2 vs 6) for ~15 % more time; VQPC_AP_CSR=0 selects the 3-op FMA form.
#ifndef VQPC_RESID_CSR
#define VQPC_RESID_CSR 1
#endif
#ifndef VQPC_AP_CSR
#define VQPC_AP_CSR 1
#endif

// One CSR row product in the reference's order without contraction
// (fem.cpp:142-148: s = 0; s += a_{j,j-1} v_{j-1}; s += a_jj v_j; s += a_{j,j+1} v_{j+1}).
__device__ __forceinline__ double csr_row(double c_lo, double d, double c_hi, double vl, double v, double vr) {
  double sacc = __dmul_rn(-c_lo, vl);
  sacc = __dadd_rn(sacc, __dmul_rn(d, v));
  return __dadd_rn(sacc, __dmul_rn(-c_hi, vr));
}

// The same row with FMA contraction (3 fp64 operations; different rounding).
__device__ __forceinline__ double fused_row(double c_lo, double d, double c_hi, double vl, double v, double vr) {
  return fma(d, v, -fma(c_hi, vr, c_lo * vl));
}

// |b - A x|^2 over a thread's rows (4 split accumulators)
template <int R, int T, bool MASK>
__device__ __forceinline__ double true_residual(const double (&x)[R], double x_left, double x_right,
                                                const double* ct, const double* c_halo, double h, int j0, int n) {
  constexpr int Q = R / 4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double c_lo = ct[0];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const double c_hi = i + 1 < R ? ct[(i + 1) * T] : *c_halo;
    const double d = __dadd_rn(c_lo, c_hi);
    const double xl = i == 0 ? x_left : x[i - 1];
    const double xr = i + 1 < R ? x[i + 1] : x_right;
#if VQPC_RESID_CSR
    double rt = __dsub_rn(h, csr_row(c_lo, d, c_hi, xl, x[i], xr));
#else
    double rt = h - fused_row(c_lo, d, c_hi, xl, x[i], xr);
#endif
    if (MASK && j0 + i >= n) rt = 0.0;
    acc[i / Q] = fma(rt, rt, acc[i / Q]);
    c_lo = c_hi;
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// A p over a thread's rows into wz, and the p.Ap partial (4 split accumulators).
// Dead rows (j >= n, last warp only) are masked: row n's c_j is the true c_n.
template <int R, int T, bool MASK>
__device__ __forceinline__ double apply_rows(const double (&p)[R], double p_left, double p_right, const double* ct,
                                             const double* c_halo, int j0, int n, double (&wz)[R]) {
  constexpr int Q = R / 4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double c_lo = ct[0];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const double c_hi = i + 1 < R ? ct[(i + 1) * T] : *c_halo;
    const double d = __dadd_rn(c_lo, c_hi);
    const double pl = i == 0 ? p_left : p[i - 1];
    const double pr = i + 1 < R ? p[i + 1] : p_right;
#if VQPC_AP_CSR
    double v = csr_row(c_lo, d, c_hi, pl, p[i], pr);
#else
    double v = fused_row(c_lo, d, c_hi, pl, p[i], pr);
#endif
    if (MASK && j0 + i >= n) v = 0.0;
    wz[i] = v;
    acc[i / Q] = fma(p[i], v, acc[i / Q]);
    c_lo = c_hi;
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}


// ---- CL == 2 exchanges without cluster barriers --------------------------------
// Each of the four per-iteration cross-warp exchanges writes the peer CTA's copy
// with st.async (DSMEM) carrying a byte count to the peer's mbarrier; a CTA then
// needs only its own __syncthreads plus a wait on its mbarrier phase, instead of
// a cluster-wide barrier (~380 cycles + L1 invalidation each).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa_peer(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(unsigned bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void st_async_f64(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}

// pairwise sum of NW smem partials in a fixed tree (every thread: same bits)
template <int NW>
__device__ __forceinline__ double tree_sum(const double* part) {
  double v[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) v[i] = part[i];
#pragma unroll
  for (int w = 1; w < NW; w <<= 1)
#pragma unroll
    for (int i = 0; i + w < NW; i += 2 * w) v[i] += v[i + w];
  return v[0];
}

template <int R, int T, int CL, int MINB = 1>
__global__ void __launch_bounds__(T, MINB) pcg1d_kernel(const Pcg1dParams prm) {
  using Sh = Pcg1dShared<R, T, CL>;
  constexpr int NW = Sh::NW;
  constexpr int NWT = Sh::NWT;
  constexpr int Q = R / 4;  // rows per quarter chain
  static_assert(R % 4 == 0 && R >= 4, "four quarter-chains per thread");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sh& S = *reinterpret_cast<Sh*>(smem_raw);

  namespace cg = cooperative_groups;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = CL == 1 ? 0 : static_cast<int>(cg::this_cluster().block_rank());
  const int gwarp = rank * NW + warp;  // warp index within the sample
  const int j0 = (rank * T + tid) * R;  // first row of this thread
  // this warp owns rows >= n (warp-uniform): only then the masked row paths run
  const bool dead_warp = (gwarp + 1) * 32 * R > prm.n;
  // peer CTA's shared struct (CL == 2); same layout at the same offset
  Sh* peer = &S;
  if constexpr (CL == 2) peer = cg::this_cluster().map_shared_rank(&S, rank ^ 1);
  auto bar = [&]() {
    if constexpr (CL == 1)
      __syncthreads();
    else
      cg::this_cluster().sync();
  };
  // write a cross-warp value into every CTA of the cluster (label-change path:
  // plain DSMEM stores, followed by a cluster barrier)
  auto publish = [&](double* local_arr, int idx, double v) {
    local_arr[idx] = v;
    if constexpr (CL == 2) reinterpret_cast<double*>(reinterpret_cast<char*>(peer) +
                                                     (reinterpret_cast<char*>(local_arr) - reinterpret_cast<char*>(&S)))[idx] = v;
  };
  // per-iteration exchanges (CL == 2): st.async into the peer + transaction mbarriers
  const unsigned s_base = smem_u32(&S);
  const unsigned p_base = CL == 2 ? mapa_peer(s_base, rank ^ 1) : 0u;
  unsigned ph = 0;  // bit k: phase parity of exchange k
  if constexpr (CL == 2) {
    if (tid == 0) {
      for (int k = 0; k < 4; ++k) mbar_init(smem_u32(&S.mbar[k]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();
  }
  // value v into local_arr[idx] here and in the peer, counted on the peer's barrier k
  auto send = [&](double* local_arr, int idx, double v, int k) {
    local_arr[idx] = v;
    if constexpr (CL == 2) {
      const unsigned off = smem_u32(&local_arr[idx]) - s_base;
      st_async_f64(p_base + off, v, p_base + (smem_u32(&S.mbar[k]) - s_base));
    }
  };
  // exchange k complete: own warps (__syncthreads) and the peer's bytes (mbarrier)
  auto xchg = [&](int k, unsigned bytes) {
    __syncthreads();
    if constexpr (CL == 2) {
      const unsigned mb = smem_u32(&S.mbar[k]);
      if (tid == 0) mbar_expect_tx(mb, bytes);
      const unsigned par = (ph >> k) & 1u;
      while (!mbar_try_wait(mb, par)) {
      }
      ph ^= 1u << k;
    }
  };
  const int n = prm.n;
  const double* ct = S.c + tid;        // ct[i*T] = c_{j0+i}
  const double* levt = S.lev + tid;    // levt[k*T]
  const double* qat = S.qa + tid;      // qat[q*T]
  const double* fut = S.fu + tid;      // fut[i*T] = 1/u_{j0+i}^2
  const double* c_halo = tid + 1 < T ? &S.c[tid + 1] : &S.cs_end;  // c_{j0+R}

  if (prm.t_span && tid == 0) prm.t_span[2 * blockIdx.x] = globaltimer_ns();
  int cur_label = -1;
#ifdef VQPC_PHASE_TIMING
  long long ph_last = -1;
#endif
  double nc[R];         // n_j of own rows
  double n_left = 0.0;  // n_{j0-1}

  for (;;) {
    if (rank == 0 && tid == 0) {
      const int64_t it = atomicAdd(prm.counter, 1);
      S.item = it;
      if constexpr (CL == 2) peer->item = it;
    }
    bar();
    const int64_t item = S.item;
    bar();
    if (item >= prm.B) break;
    const int s = prm.perm[item];
    const int64_t gs = prm.out_base + s;
    const int label = prm.labels[s];
    if (label < 0 || prm.kflag[s] || gs >= prm.solve_limit) {
      if (rank == 0 && tid == 0) {
        prm.iters[gs] = 0;
        prm.rel[gs] = 0.0;
        prm.status[gs] = gs >= prm.solve_limit ? VQPC_S_NOT_SOLVED
                         : label < 0           ? VQPC_S_INVALID_LATENT
                                               : (prm.kflag[s] & 1) ? VQPC_S_COEFF_OVERFLOW : VQPC_S_INVALID_COEFF;
      }
      continue;
    }
    if (label != cur_label) {
      // ---- new bucket: factor to smem, per-thread / per-lane scan constants ----
      const double2* src = prm.factors + static_cast<size_t>(label) * prm.NP + static_cast<size_t>(rank) * R * T;
      for (int e = tid; e < R * T; e += T) {  // coalesced read
        const double2 f = src[e];
        S.fn[(e % R) * T + e / R] = f.x;
        S.fu[(e % R) * T + e / R] = f.y;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < R; ++i) nc[i] = S.fn[i * T + tid];
      n_left = tid > 0 ? S.fn[(R - 1) * T + tid - 1] : (j0 > 0 ? src[-1].x : 0.0);
      double P1 = 1.0, P2 = 1.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double a1 = 1.0, a2 = 1.0;
#pragma unroll
        for (int i = q * Q; i < q * Q + Q; ++i) {
          a1 *= -nc[i];
          a2 *= i == 0 ? -n_left : -nc[i - 1];
        }
        S.qa[q * T + tid] = a1;
        S.qa[(4 + q) * T + tid] = a2;
        P1 *= a1;
        P2 *= a2;
      }
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int off = 1 << k;
        S.lev[k * T + tid] = lane + off < 32 ? P1 : 0.0;    // suffix-scan multiplier
        S.lev[(6 + k) * T + tid] = lane >= off ? P2 : 0.0;  // prefix-scan multiplier
        const double o1 = shfl_down(P1, off), o2 = shfl_up(P2, off);
        if (lane + off < 32) P1 *= o1;
        if (lane >= off) P2 *= o2;
      }
      // now P1 = prod over lanes [lane, 31], P2 = prod over lanes [0, lane]
      const double q1 = shfl_down(P1, 1), q2 = shfl_up(P2, 1);
      S.lev[5 * T + tid] = lane < 31 ? q1 : 1.0;
      S.lev[11 * T + tid] = lane > 0 ? q2 : 1.0;
      if (lane == 0) publish(&S.f1[0].x, 2 * gwarp, P1);
      if (lane == 31) publish(&S.f2[0].x, 2 * gwarp, P2);
      cur_label = label;
      bar();  // the per-centroid multipliers (f1/f2 .x) reach the peer before any use
    }

    // ---- sample setup: c_j = kappa_j / h, b = h, x = 0, r = b --------------
    const double* kap = prm.kappa + static_cast<size_t>(s) * prm.ldk;
    {
      // IEEE division: the oracle's kappa/h; d_j = c_j + c_{j+1} like its CSR diagonal
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int j = j0 + i;
        S.c[i * T + tid] = j <= n ? kap[j] / prm.h : 0.0;
      }
      // right conductance of this CTA's last row: c_{j0+R} (0 beyond element n)
      if (tid == T - 1) S.cs_end = j0 + R <= n ? kap[j0 + R] / prm.h : 0.0;
    }
    double x[R], r[R], p[R], wz[R];
    double bbq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < R; ++i) {
      x[i] = 0.0;
      r[i] = j0 + i < n ? prm.h : 0.0;
      bbq[i / Q] = fma(r[i], r[i], bbq[i / Q]);
    }
    const double bb = (bbq[0] + bbq[1]) + (bbq[2] + bbq[3]);
    const int max_iter = prm.max_iter_arr ? prm.max_iter_arr[gs] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);

    double rz = 0.0, norm_b = 0.0;
    double rz_inv = 0.0;  // RN(1 / rz): beta = rz_next / rz by Markstein's correction (exact quotient)
    double rr_hi = 0.0;   // rr above this => rel >= eps for certain (see below)
    double rr_rec = 0.0;  // |b - A x|^2 of the last completed iteration (J of them)
    int J = 0;
    uint8_t st = VQPC_S_MAX_ITER;
    double rr_loc = 0.0;
    double p_left = 0.0, p_right = 0.0, x_left = 0.0, x_right = 0.0;
    int j = 0;  // 0: setup pass (z = M^{-1} b); >= 1: iteration j
    for (;;) {
      // ================= sweep 1 (descending) + rr: barrier 2 ===============
      {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = 0.0;
#pragma unroll
        for (int i = Q - 1; i >= 0; --i)
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = fma(-nc[q * Q + i], v[q], r[q * Q + i]);
        const double a0 = qat[0], a1 = qat[T], a2 = qat[2 * T], a3 = qat[3 * T];
        double W = fma(a2, v[3], v[2]);
        W = fma(a1, W, v[1]);
        W = fma(a0, W, v[0]);
#pragma unroll
        for (int k = 0; k < 5; ++k) W = fma(levt[k * T], shfl_down(W, 1 << k), W);
        const double rrw = warp_allsum(rr_loc);
        if (lane == 0) {
          send(&S.f1[0].x, 2 * gwarp + 1, W, 1);
          send(S.red[1], gwarp, rrw, 1);
        }
        xchg(1, 2 * NW * 8);  // barrier 2
        P1D_MARK(1);  // alpha, x/r update, true residual, sweep 1
        double vw = 0.0;
#pragma unroll
        for (int w2 = NWT - 1; w2 > 0; --w2)
          if (w2 > gwarp) {
            const double2 f = S.f1[w2];
            vw = fma(f.x, vw, f.y);
          }
        const double Wn = shfl_down(W, 1);
        double in[4];
        in[3] = fma(levt[5 * T], vw, lane == 31 ? 0.0 : Wn);
        in[2] = fma(a3, in[3], v[3]);
        in[1] = fma(a2, in[2], v[2]);
        in[0] = fma(a1, in[1], v[1]);
        // fix-up chains written straight into wz (no register copies)
#pragma unroll
        for (int q = 0; q < 4; ++q) wz[q * Q + Q - 1] = fma(-nc[q * Q + Q - 1], in[q], r[q * Q + Q - 1]);
#pragma unroll
        for (int i = Q - 2; i >= 0; --i)
#pragma unroll
          for (int q = 0; q < 4; ++q) wz[q * Q + i] = fma(-nc[q * Q + i], wz[q * Q + i + 1], r[q * Q + i]);
#pragma unroll
        for (int i = 0; i < R; ++i) wz[i] *= fut[i * T];
      }
      // the relative true residual decides convergence; its sqrt and division
      // overlap sweep 2, and the (warp-uniform) exit is taken after it
      // |b - A x|^2 of this iteration; the exact rel = sqrt(rr)/|b| (solver.cpp:229) is
      // only evaluated when rr is within 1e-9 of the threshold (eps |b|)^2 or at the
      // exit, so its sqrt/division chain leaves the critical path of most iterations
      const double rr = tree_sum<NWT>(S.red[1]);
      // ================= sweep 2 (ascending): barrier 3 =====================
      {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = wz[q * Q];  // incoming 0
#pragma unroll
        for (int i = 1; i < Q; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = fma(-nc[q * Q + i - 1], v[q], wz[q * Q + i]);
        const double b0 = qat[4 * T], b1 = qat[5 * T], b2 = qat[6 * T], b3 = qat[7 * T];
        double W = fma(b1, v[0], v[1]);
        W = fma(b2, W, v[2]);
        W = fma(b3, W, v[3]);
#pragma unroll
        for (int k = 0; k < 5; ++k) W = fma(levt[(6 + k) * T], shfl_up(W, 1 << k), W);
        if (lane == 31) send(&S.f2[0].x, 2 * gwarp + 1, W, 2);
        xchg(2, NW * 8);  // barrier 3
        P1D_MARK(2);  // fold + fix-up of sweep 1, sweep 2
        double vw = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < NWT - 1; ++w2)
          if (w2 < gwarp) {
            const double2 f = S.f2[w2];
            vw = fma(f.x, vw, f.y);
          }
        const double Wp = shfl_up(W, 1);
        double in[4];
        in[0] = fma(levt[11 * T], vw, lane == 0 ? 0.0 : Wp);
        in[1] = fma(b0, in[0], v[0]);
        in[2] = fma(b1, in[1], v[1]);
        in[3] = fma(b2, in[2], v[2]);
        // fix-up chains in place (z overwrites y row by row; no register copies)
        wz[0] = fma(-n_left, in[0], wz[0]);
#pragma unroll
        for (int q = 1; q < 4; ++q) wz[q * Q] = fma(-nc[q * Q - 1], in[q], wz[q * Q]);
#pragma unroll
        for (int i = 1; i < Q; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) wz[q * Q + i] = fma(-nc[q * Q + i - 1], wz[q * Q + i - 1], wz[q * Q + i]);
      }
      if (j > 0) {
        J = j;
        rr_rec = rr;
        // rr > rr_hi >= (eps |b|)^2 (1 + 0.9e-9) implies RN(RN(sqrt(rr)) / |b|) >= eps:
        // the comparison's outcome is decided without evaluating rel (NaN takes the exact path)
        if (!(rr > rr_hi) && sqrt(rr) / norm_b < prm.eps) {
          st = VQPC_S_CONVERGED;
          break;
        }
      }
      // ================= rz (+|b|^2 at setup), z halos: barrier 4 ===========
      {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < R; ++i) acc[i / Q] = fma(r[i], wz[i], acc[i / Q]);
        const double a = warp_allsum((acc[0] + acc[1]) + (acc[2] + acc[3]));
        const double b2 = j == 0 ? warp_allsum(bb) : 0.0;
        if (lane == 0) {
          send(S.red[2], gwarp, a, 3);
          send(S.red[3], gwarp, b2, 3);
        }
        S.zf[tid] = wz[0];
        S.zl[tid] = wz[R - 1];
        if constexpr (CL == 2) {  // the CTA-boundary z travels with this exchange
          if (rank == 1 && tid == 0) st_async_f64(p_base + (smem_u32(&S.zf_peer) - s_base), wz[0],
                                                  p_base + (smem_u32(&S.mbar[3]) - s_base));
          if (rank == 0 && tid == T - 1) st_async_f64(p_base + (smem_u32(&S.zl_peer) - s_base), wz[R - 1],
                                                      p_base + (smem_u32(&S.mbar[3]) - s_base));
        }
        xchg(3, 2 * NW * 8 + 8);  // barrier 4
        P1D_MARK(3);  // fold + fix-up of sweep 2, r.z
      }
      const double rz_next = tree_sum<NWT>(S.red[2]);
      // z halos; across the CTA boundary they are read from the peer (DSMEM)
      const double zl_left = tid > 0 ? S.zl[tid - 1] : (CL == 2 && rank == 1 ? S.zl_peer : 0.0);
      const double zf_right = tid < T - 1 ? S.zf[tid + 1] : (CL == 2 && rank == 0 ? S.zf_peer : 0.0);
      if (j == 0) {
        norm_b = sqrt(tree_sum<NWT>(S.red[3]));
        if (norm_b == 0.0) {
          st = VQPC_S_CONVERGED;
          break;
        }
        if (!(rz_next > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        rz = rz_next;
        rr_hi = (prm.eps * norm_b) * (prm.eps * norm_b) * (1.0 + 1e-9);
#pragma unroll
        for (int i = 0; i < R; ++i) p[i] = wz[i];
        p_left = zl_left;
        p_right = zf_right;
      } else {
        if (!(rz_next > 0.0)) {
          st = VQPC_S_BREAKDOWN;
          break;
        }
        // beta = RN(rz_next / rz): q0 = RN(a y), e = a - b q0 (exact), RN(q0 + e y) with
        // y = RN(1/b) is the correctly rounded quotient (Markstein) as long as nothing
        // under- or overflows; y was formed off the critical path, so only three dependent
        // operations remain here. Stagnating samples drive rz towards the subnormal range:
        // there (warp-uniform, rare) the IEEE division is used directly.
        double beta;
        if (rz > 1e-150 && rz < 1e150 && rz_next > 1e-150 && rz_next < 1e150) {
          const double q0 = rz_next * rz_inv;
          beta = fma(fma(-rz, q0, rz_next), rz_inv, q0);
        } else {
          beta = rz_next / rz;
        }
        rz = rz_next;
#pragma unroll
        for (int i = 0; i < R; ++i) p[i] = fma(beta, p[i], wz[i]);
        p_left = fma(beta, p_left, zl_left);
        p_right = fma(beta, p_right, zf_right);
      }
      // ================= next iteration: Ap, pAp -> barrier 1 ===============
      ++j;
      if (j > max_iter) {
        st = VQPC_S_MAX_ITER;
        break;
      }
      {
        // dead rows (j >= n) take a warp-uniform masked path (row n would see c_n)
        const double part = dead_warp ? apply_rows<R, T, true>(p, p_left, p_right, ct, c_halo, j0, n, wz)
                                             : apply_rows<R, T, false>(p, p_left, p_right, ct, c_halo, j0, n, wz);
        const double a = warp_allsum(part);
        rz_inv = __drcp_rn(rz);  // overlaps the reduction chain (used by next iteration's beta)
        if (lane == 0) send(S.red[0], gwarp, a, 0);
        xchg(0, NW * 8);  // barrier 1
        P1D_MARK(0);  // p update, A p, p.Ap
      }
      const double pAp = tree_sum<NWT>(S.red[0]);
      if (!(pAp > 0.0)) {
        st = VQPC_S_BREAKDOWN;
        break;
      }
      const double alpha = rz / pAp;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        x[i] = fma(alpha, p[i], x[i]);
        r[i] = fma(-alpha, wz[i], r[i]);
      }
      x_left = fma(alpha, p_left, x_left);
      x_right = fma(alpha, p_right, x_right);
      // true residual b - A x; dead rows (b_j = 0) are masked
      rr_loc = dead_warp ? true_residual<R, T, true>(x, x_left, x_right, ct, c_halo, prm.h, j0, n)
                              : true_residual<R, T, false>(x, x_left, x_right, ct, c_halo, prm.h, j0, n);
    }

    if (rank == 0 && tid == 0) {
      prm.iters[gs] = J;
      prm.rel[gs] = J > 0 ? sqrt(rr_rec) / norm_b : 0.0;  // the record of iteration J
      prm.status[gs] = st;
    }
    if (prm.x_out) {
      double* xo = prm.x_out + static_cast<size_t>(gs) * n;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (j0 + i < n) xo[j0 + i] = x[i];
    }
  }
  if (prm.t_span && tid == 0) prm.t_span[2 * blockIdx.x + 1] = globaltimer_ns();
  if constexpr (CL == 2) cg::this_cluster().sync();  // no CTA exits while its peer may read its smem
}

template <int R, int T, int CL>
constexpr size_t pcg1d_smem_bytes() {
  return sizeof(Pcg1dShared<R, T, CL>);
}

}  // namespace vqpc
