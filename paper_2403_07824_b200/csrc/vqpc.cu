// vqpc.cu — context, device memory and the C-ABI entry points (include/vqpc.h).
//
// Host orchestration of the hot path, restating run_campaign_with
// (proj/src/driver.cpp:193-281) over device kernels:
//   assign (b) -> bucket (c) -> realise (a) -> pcg (d) -> per-centroid stats,
// chunk by chunk, after the one-time centroid factorisation (e).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <thread>

#include "amg_setup.cuh"
#include "assign.cuh"
#include "assign_mma.cuh"
#include "bucket.cuh"
#include "common.cuh"
#include "factor.cuh"
#include "pcg1d.cuh"
#include "pcg1d_exact.cuh"
#include "pcg2d.cuh"
#include "pcgamg2d.cuh"
#include "pcgchol2d.cuh"
#include "realise.cuh"
#include "vqpc.h"

using namespace vqpc;

namespace {

struct CudaError {
  int code;
  std::string msg;
};

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw CudaError{e_ == cudaErrorMemoryAllocation ? VQPC_OUT_OF_MEMORY : VQPC_CUDA_ERROR,     \
                      std::string(#call) + ": " + cudaGetErrorString(e_)};                        \
  } while (0)

struct ApiError {
  int code;
  std::string msg;
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

int check_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0) return VQPC_NO_DEVICE;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return VQPC_NO_DEVICE;
  if (prop.major < 10) return VQPC_NO_DEVICE;  // built for sm_100a only
  return VQPC_OK;
}

}  // namespace

struct vqpc_ctx {
  vqpc_problem pb{};
  int n = 0;        // unknowns per sample system
  int NP = 0;       // padded rows per factor (R*T of the pcg variant)
  int pcgR = 0, pcgT = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool factored = false;
  int64_t launches = 0;
  std::string last_error;
  std::vector<double> h_lambdas;
  // device-resident problem data
  DBuf<double> phi, sqrt_lam, root, sites, kappa_c;
  DBuf<double2> fac;
  // 2-D path: grid, IC(0) factors (P x 3n, wavefront order), per-CTA PCG scratch
  Grid2D g2{};
  DBuf<double> fac2, work2;
  DBuf<int> gmap;
  DBuf<double> bvec2;  // per-node right-hand side when it is not uniform (see pcg2d.cuh)
  DBuf<double> cnorm;  // |c_p|^2 for the contraction form of the assignment (assign_mma.cuh)
  // 2-D `cholesky` preconditioner (pcgchol2d.cuh): RCM envelope, factors, groups
  bool chol2d = false;
  CholLayout clay{};
  DBuf<int> ch_cperm, ch_first, ch_ngroups;
  DBuf<int64_t> ch_start, ch_off, ch_a0;
  DBuf<int> ch_bmeta;
  DBuf<unsigned> ch_bytes;
  DBuf<int4> ch_nbr;
  DBuf<int2> ch_groups;
  DBuf<int32_t> ch_perm;
  DBuf<double> ch_L, ch_Linv, ch_work;
  int64_t ch_ldL = 0, ch_ldLi = 0, ch_nnz = 0;
  int ch_cap = 0;
  int ch_S = 8;
  // 2-D SA-AMG kind (pcgamg2d.cuh): host hierarchies (kept for vqpc_amg_level) and their device copy
  bool amg = false;
  std::vector<amg::Hierarchy> amg_h;
  DBuf<int> amg_i;
  DBuf<double> amg_d, amg_work;
  DBuf<AmgHierD> amg_hd;
  int amg_cv = 0;           // doubles of coarse-level scratch per CTA and slot (max over centroids)
  int amg_dense_max = 0;    // largest coarsest dense size over the centroids
  int64_t amg_entries = 0;  // stored hierarchy entries per centroid (mean), roofline accounting
  cudaStream_t aux = nullptr;              // chunks beyond the solve subset (overlap with the PCG)
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  DBuf<int> aflag;     // assign_mma candidate-list overflow flag
  bool b2_checked = false, b2_uniform = true;
  int exact = 0;  // reference-order mode: serial dot products (2-D); 1-D: pcg1d_exact_kernel
  DBuf<double2> fac_lu;  // 1-D reference-order mode: P x NP {l_j, u_j}, built on first use
  bool have_lu = false;
  const double* lu_src = nullptr;  // the coefficients the current factors were built from (factor_coefficients)
  int64_t lu_ld = 0;
  int lu_count = 0;
  DBuf<double> work1x;
  // work buffers
  DBuf<double> xi, kappa, best, dvec;
  DBuf<uint8_t> kflag, status;
  DBuf<int32_t> labels, perm, counts, iters, mia, keys, perm2;
  DBuf<int64_t> offsets, stats, offsets2;
  bool no_cost_order = getenv("VQPC_BUCKET_ORDER") != nullptr;  // diagnostics: label order only
  DBuf<double> rel, x;
  DBuf<int> counter, err;
  // optional per-kernel CUDA-event timing (bench roofline)
  bool prof = false;
  struct Rec {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double prof_ms[VQPC_NKINDS] = {};
  int64_t prof_n[VQPC_NKINDS] = {};
};

namespace {

double h_of(const vqpc_problem& pb) { return 1.0 / pb.size; }

void launch_check(vqpc_ctx* c) {
  ++c->launches;
  CK(cudaGetLastError());
}

cudaEvent_t take_event(vqpc_ctx* c) {
  if (c->pool.empty()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = c->pool.back();
  c->pool.pop_back();
  return e;
}

// RAII bracket: records CUDA events around a launch on the context's stream
struct Timed {
  vqpc_ctx* c;
  int kind;
  cudaEvent_t a = nullptr;
  Timed(vqpc_ctx* c_, int kind_) : c(c_), kind(kind_) {
    if (c->prof) {
      a = take_event(c);
      CK(cudaEventRecord(a, c->stream));
    }
  }
  ~Timed() {
    if (c->prof && a) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, c->stream);
      c->recs.push_back({kind, a, b});
    }
  }
};

// Diagnostics / determinism tests: VQPC_MAX_GROUPS=k caps the
// persistent PCG grids at k concurrently resident samples (CTAs or clusters).
int64_t cap_groups(int64_t g) {
  const char* env = std::getenv("VQPC_MAX_GROUPS");  // read per launch (tests set it mid-process)
  const int64_t cap = env ? std::atoll(env) : 0;
  return cap > 0 ? std::min(g, cap) : g;
}

// Per row pattern of the structured 2-D mesh (neighbours W, E, S, N present),
// the order in which the reference's SparseBuilder (fem.cpp:177-211) sums the six
// diagonal contributions: the row's insertion sequence (triangles in mesh order,
// vertices j = 0..2 each; assemble, fem.cpp:226-245) is ordered with the same
// std::sort on the column, and the diagonal's terms are read off in sorted order.
// Keys are column ranks SW < S < W < C < E < N < NE (the order of the true interior
// indices for m >= 2), which std::sort treats exactly like the true columns.
void diag_orders(unsigned char out[16][6]) {
  enum { SW, S, W, C, E, N, NE };
  // node C's six triangles in mesh order: T1, T2 of cell (X-1, Y-1), T2 of (X, Y-1),
  // T1 of (X-1, Y), T1, T2 of (X, Y); their vertices in local order
  static const int seq[18] = {SW, S, C, SW, C, W, S, E, C, W, C, N, C, E, NE, C, NE, N};
  for (int pat = 0; pat < 16; ++pat) {
    const bool hw = pat & 1, he = pat & 2, hs = pat & 4, hn = pat & 8;
    const bool has[7] = {hw && hs, hs, hw, true, he, hn, he && hn};
    std::vector<std::pair<int, double>> row;  // the reference's element type
    int tag = 0;
    for (int q = 0; q < 18; ++q)
      if (has[seq[q]]) row.emplace_back(seq[q], seq[q] == C ? static_cast<double>(tag++) : -1.0);
    std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    int k = 0;
    for (const auto& e : row)
      if (e.first == C) out[pat][k++] = static_cast<unsigned char>(e.second);
  }
}

// ---- pcg variant table: rows per thread R, threads T (n <= R*T) ------------
using PcgFn = void (*)(const Pcg1dParams);
struct PcgVariant {
  int R, T, CL;
  PcgFn fn;
  size_t smem;
};

template <int R, int T, int CL, int MINB = 1>
PcgVariant make_variant() {
  return PcgVariant{R, T, CL, &pcg1d_kernel<R, T, CL, MINB>, pcg1d_smem_bytes<R, T, CL>()};
}

// smallest variant whose R*T*CL rows hold the n unknowns; n <= 4096 fits one SM's
// register file (one CTA per sample), n <= 8192 uses a 2-CTA cluster
const PcgVariant* pick_pcg(int n) {
  // n <= 1024: 8 rows x 128 threads (4 warps beat 2 warps of 16 rows: C1 667k -> 735k samples/s);
  // larger n: 16 rows per thread (C3 676k vs 475k, C2 190k vs 125k with 8 rows)
  static const PcgVariant table[] = {make_variant<8, 128, 1>(), make_variant<16, 128, 1>(),
                                     make_variant<16, 256, 1>(), make_variant<16, 256, 2>()};
  // experiments: VQPC_PCG_R=8 selects the 8-rows-per-thread layout (twice the warps)
  static const PcgVariant table8[] = {make_variant<8, 128, 1>(), make_variant<8, 256, 1>(),
                                      make_variant<8, 512, 1>(), make_variant<8, 512, 2>()};
  // experiments: VQPC_PCG_SPLIT=1 spreads n in (2048, 4096] over a 2-CTA cluster of 128-thread
  // CTAs (two half-samples per SM; same warp layout, so results are bit-identical)
  static const PcgVariant split2 = make_variant<16, 128, 2>();
  // n <= 1024 runs the 8 x 128 layout capped at 128 registers, so four CTAs (16 warps) share an SM
  // instead of three: C1 3.34M -> 4.37M samples/s, records bit-identical (profiles/r02w_*).
  // VQPC_PCG_OCC4=0 selects the uncapped build (A/B runs).
  static const PcgVariant occ4 = make_variant<8, 128, 1, 4>();
  const char* o4 = std::getenv("VQPC_PCG_OCC4");
  if (!(o4 && std::atoi(o4) == 0) && n <= 1024) return &occ4;
  const char* env = std::getenv("VQPC_PCG_R");
  const bool r8 = env && std::atoi(env) == 8;
  const char* sp = std::getenv("VQPC_PCG_SPLIT");
  if (sp && std::atoi(sp) == 1 && n > 2048 && n <= 4096) return &split2;
  for (const auto& v : (r8 ? table8 : table))
    if (n <= v.R * v.T * v.CL) return &v;
  return nullptr;
}

// ---- assign dispatch ---------------------------------------------------------
using AssignFn = void (*)(const AssignParams);
template <int M>
AssignFn assign_fn(int split) {
  return split == 1 ? &assign_kernel<M, 1> : split == 4 ? &assign_kernel<M, 4> : &assign_kernel<M, 8>;
}
AssignFn pick_assign(int m, int split) {
  switch (m) {
#define VQPC_M(k) \
  case k: return assign_fn<k>(split);
    VQPC_M(1) VQPC_M(2) VQPC_M(3) VQPC_M(4) VQPC_M(5) VQPC_M(6) VQPC_M(7) VQPC_M(8) VQPC_M(9) VQPC_M(10)
    VQPC_M(11) VQPC_M(12) VQPC_M(13) VQPC_M(14) VQPC_M(15) VQPC_M(16) VQPC_M(32) VQPC_M(64)
#undef VQPC_M
    default:
      return split == 1 ? &assign_kernel_generic<1> : split == 4 ? &assign_kernel_generic<4> : &assign_kernel_generic<8>;
  }
}

void run_assign(vqpc_ctx* c, const double* d_xi, int64_t B, int64_t ld, const double* d_root, const double* d_sites,
                int P, int m, int32_t* d_labels, double* d_best) {
  if (B <= 0) return;
  if (m > 256) throw ApiError{VQPC_INVALID_ARGUMENT, "m > 256 not supported"};
  const int64_t target = static_cast<int64_t>(c->sm_count) * 1024;
  int split = 1;
  if (B * 1 < target && P >= 32) split = 8;
  else if (B < 2 * target && P >= 16) split = 4;
  AssignParams prm{d_xi, ld, B, d_root, d_sites, P, m, d_labels, d_best, nullptr};
  const int64_t threads = B * split;
  const int blocks = static_cast<int>(ceil_div(threads, AS_THREADS));
  AssignFn fn = pick_assign(m, split);
  const size_t smem = AS_TILE_DOUBLES * sizeof(double);
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  Timed tm(c, VQPC_K_ASSIGN);
  // large codebooks (C5: m = 64, P = 4096): the distance table as a DMMA contraction with an
  // exact re-check of the candidates (assign_mma.cuh); the direct kernel then runs only if a
  // candidate list overflowed (device-side flag, no host synchronisation)
  static const bool direct_only = std::getenv("VQPC_ASSIGN_DIRECT") != nullptr;
  if (!direct_only && d_sites == c->sites.p && (m == 32 || m == 64) && P >= 256) {
    if (!c->cnorm.p) {
      c->cnorm.ensure(P);
      centroid_norms_kernel<<<static_cast<unsigned>(ceil_div(P, 128)), 128, 0, c->stream>>>(d_sites, P, m,
                                                                                             c->cnorm.p);
      launch_check(c);
    }
    c->aflag.ensure(1);
    CK(cudaMemsetAsync(c->aflag.p, 0, sizeof(int), c->stream));
    AssignMmaParams am{d_xi, ld, B, d_root, d_sites, c->cnorm.p, P, d_labels, d_best, c->aflag.p};
    const unsigned gb = static_cast<unsigned>(ceil_div(B, AM_BM));
    if (m == 64) {
      CK(cudaFuncSetAttribute(assign_mma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(assign_mma_smem<64>())));
      assign_mma_kernel<64><<<gb, AM_THREADS, assign_mma_smem<64>(), c->stream>>>(am);
    } else {
      CK(cudaFuncSetAttribute(assign_mma_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(assign_mma_smem<32>())));
      assign_mma_kernel<32><<<gb, AM_THREADS, assign_mma_smem<32>(), c->stream>>>(am);
    }
    launch_check(c);
    prm.only_if = c->aflag.p;
  }
  fn<<<blocks, AS_THREADS, smem, c->stream>>>(prm);
  launch_check(c);
}

void run_realise(vqpc_ctx* c, const double* d_xi, int64_t B, int64_t ld, int K_use, double* d_kappa, int64_t ldk,
                 uint8_t* d_flag) {
  if (B <= 0) return;
  RealiseParams prm{d_xi, ld, B, c->sqrt_lam.p, c->phi.p, c->pb.n_nodes, K_use, d_kappa, ldk, d_flag};
  dim3 grid(static_cast<unsigned>(ceil_div(c->pb.n_nodes, RL_BN)), static_cast<unsigned>(ceil_div(B, RL_BM)));
  Timed tm(c, VQPC_K_REALISE);
  if (c->exact) {  // reference-order mode: the reference's k-outer AXPY on the CUDA cores
    realise_exact_kernel<<<grid, RL_THREADS, 0, c->stream>>>(prm);
  } else {
    CK(cudaFuncSetAttribute(realise_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(RL_SMEM)));
    realise_kernel<<<grid, RL_THREADS, RL_SMEM, c->stream>>>(prm);
  }
  launch_check(c);
}

// stable counting sort of ids (identity when d_ids is null) by keys[id] in [0, P) (P: invalid)
void counting_sort(vqpc_ctx* c, const int32_t* d_keys, const int32_t* d_ids, int64_t B, int P, int32_t* d_perm,
                   int64_t* d_offsets) {
  const int ntiles = static_cast<int>(ceil_div(B, BK_TILE));
  c->counts.ensure(static_cast<size_t>(P + 1) * ntiles);
  const size_t sm = sizeof(int32_t) * (P + 1);
  if (sm > 48 * 1024) {
    CK(cudaFuncSetAttribute(bucket_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    CK(cudaFuncSetAttribute(bucket_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  }
  bucket_hist_kernel<<<ntiles, 256, sm, c->stream>>>(d_keys, d_ids, B, P, ntiles, c->counts.p);
  launch_check(c);
  bucket_scan_kernel<<<1, 1024, 0, c->stream>>>(c->counts.p, static_cast<int64_t>(P + 1) * ntiles, P, ntiles,
                                                d_offsets);
  launch_check(c);
  bucket_scatter_kernel<<<ntiles, 32, sm, c->stream>>>(d_keys, d_ids, B, P, ntiles, c->counts.p, d_perm);
  launch_check(c);
}

void run_bucket(vqpc_ctx* c, const int32_t* d_labels, int64_t B, int32_t* d_perm, int64_t* d_offsets) {
  const int P = c->pb.P;
  if (B <= 0) {
    CK(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t) * (P + 2), c->stream));
    return;
  }
  Timed tm(c, VQPC_K_BUCKET);
  counting_sort(c, d_labels, nullptr, B, P, d_perm, d_offsets);
}

// Solve order for the PCG work queue: label buckets (run_bucket), then a stable
// pass by descending predicted cost (cost_key_kernel in bucket.cuh).
void run_schedule(vqpc_ctx* c, const double* d_xi, int64_t ld, const int32_t* d_labels, int64_t B,
                  const double* d_root) {
  const int P = c->pb.P;
  run_bucket(c, d_labels, B, c->perm.p, c->offsets.p);
  if (B <= 0 || c->no_cost_order) return;
  c->keys.ensure(B);
  c->perm2.ensure(B);
  c->offsets2.ensure(COST_BINS + 2);
  Timed tm(c, VQPC_K_BUCKET);
  cost_key_kernel<<<static_cast<unsigned>(ceil_div(B, 256)), 256, 0, c->stream>>>(
      d_xi, ld, B, c->pb.n_kl, c->pb.m, d_labels, c->sqrt_lam.p, c->sites.p, d_root, c->keys.p);
  launch_check(c);
  counting_sort(c, c->keys.p, c->perm.p, B, COST_BINS, c->perm2.p, c->offsets2.p);
  std::swap(c->perm, c->perm2);
  (void)P;
}

size_t pchol_smem(const vqpc_ctx* c, int S) {
  return sizeof(double) * (2 * (static_cast<size_t>(c->ch_cap) + PC_LIB) + static_cast<size_t>(S) * pc_ring(S));
}

// 2-D `cholesky` kind: label-major order (stable over the cost-ordered queue), work
// groups of up to S same-label samples, then one CTA per SM over the groups.
void run_pcgchol2d(vqpc_ctx* c, const double* d_kappa, int64_t ldk, const uint8_t* d_kflag, const int32_t* d_perm,
                   const int32_t* d_labels, int64_t B, int64_t out_base, double eps, int max_iter,
                   const int32_t* d_mia, int32_t* d_iters, double* d_rel, uint8_t* d_status, double* d_x,
                   int64_t solve_limit) {
  const int P = c->pb.P, S = c->ch_S, n = c->n;
  if (c->exact) {  // reference-order instrument: one CTA per sample, serial solves and dots
    const int ldv = static_cast<int>(ceil_div(n, PC_BS) * PC_BS);
    const int64_t blocks = cap_groups(std::min<int64_t>(B, 2LL * c->sm_count));
    c->ch_work.ensure(static_cast<size_t>(blocks) * PCX_NV * ldv);
    c->counter.ensure(1);
    CK(cudaMemsetAsync(c->counter.p, 0, sizeof(int), c->stream));
    PcholParams prm{};
    prm.g = c->g2;
    prm.lay = c->clay;
    prm.kappa = d_kappa;
    prm.ldk = ldk;
    prm.kflag = d_kflag;
    prm.perm = d_perm;
    prm.labels = d_labels;
    prm.L = c->ch_L.p;
    prm.ldL = c->ch_ldL;
    prm.ldv = ldv;
    prm.work = c->ch_work.p;
    prm.B = B;
    prm.out_base = out_base;
    prm.solve_limit = solve_limit;
    prm.eps = eps;
    prm.max_iter = max_iter;
    prm.max_iter_arr = d_mia;
    prm.counter = c->counter.p;
    prm.iters = d_iters;
    prm.rel = d_rel;
    prm.status = d_status;
    prm.x_out = d_x;
    Timed tm(c, VQPC_K_PCG);
    pcgchol2d_exact_kernel<<<static_cast<unsigned>(blocks), PC_T, 0, c->stream>>>(prm);
    launch_check(c);
    return;
  }
  c->ch_perm.ensure(B);
  c->ch_off.ensure(P + 2);
  c->ch_groups.ensure(B + P + 1);
  c->ch_ngroups.ensure(1);
  {
    Timed tm(c, VQPC_K_BUCKET);
    counting_sort(c, d_labels, d_perm, B, P, c->ch_perm.p, c->ch_off.p);
    chol_groups_kernel<<<1, CG_T, 0, c->stream>>>(c->ch_off.p, P, S, c->ch_groups.p, c->ch_ngroups.p);
    launch_check(c);
  }
  void (*const kerns[PC_MAXS])(const PcholParams) = {
      pcgchol2d_kernel<1>, pcgchol2d_kernel<2>, pcgchol2d_kernel<3>, pcgchol2d_kernel<4>,
      pcgchol2d_kernel<5>, pcgchol2d_kernel<6>, pcgchol2d_kernel<7>, pcgchol2d_kernel<8>};
  void (*kern)(const PcholParams) = kerns[S - 1];
  const size_t smem = pchol_smem(c, S);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PC_T, smem));
  if (per_sm < 1) throw ApiError{VQPC_CUDA_ERROR, "pcgchol2d kernel does not fit on an SM"};
  const int64_t blocks = cap_groups(std::min<int64_t>(ceil_div(B, S) + P + 1, static_cast<int64_t>(per_sm) * c->sm_count));
  const int ldv = static_cast<int>(ceil_div(n, PC_BS) * PC_BS);
  c->ch_work.ensure(static_cast<size_t>(blocks) * S * PC_NV * ldv);
  c->counter.ensure(1);
  CK(cudaMemsetAsync(c->counter.p, 0, sizeof(int), c->stream));
  PcholParams prm{};
  prm.g = c->g2;
  prm.lay = c->clay;
  prm.kappa = d_kappa;
  prm.ldk = ldk;
  prm.kflag = d_kflag;
  prm.perm = c->ch_perm.p;
  prm.labels = d_labels;
  prm.groups = c->ch_groups.p;
  prm.ngroups = c->ch_ngroups.p;
  prm.L = c->ch_L.p;
  prm.ldL = c->ch_ldL;
  prm.Linv = c->ch_Linv.p;
  prm.ldLi = c->ch_ldLi;
  prm.cap = c->ch_cap;
  prm.blk_a0 = c->ch_a0.p;
  prm.blk_bytes = c->ch_bytes.p;
  prm.ldv = ldv;
  prm.work = c->ch_work.p;
  prm.B = B;
  prm.out_base = out_base;
  prm.solve_limit = solve_limit;
  prm.eps = eps;
  prm.max_iter = max_iter;
  prm.max_iter_arr = d_mia;
  prm.counter = c->counter.p;
  prm.iters = d_iters;
  prm.rel = d_rel;
  prm.status = d_status;
  prm.x_out = d_x;
  Timed tm(c, VQPC_K_PCG);
  kern<<<static_cast<unsigned>(blocks), PC_T, smem, c->stream>>>(prm);
  launch_check(c);
}

// SA-AMG kind: label-major order (stable over the cost-ordered queue), groups of up
// to S same-label samples (the centroid's hierarchy is streamed once per group),
// one persistent CTA per group.
template <int S>
void launch_pcgamg2d(vqpc_ctx* c, PcgAmgParams& prm, int64_t ngroups_max) {
  const size_t smem = sizeof(double) * static_cast<size_t>(std::max(c->amg_dense_max, 1)) * S;
  CK(cudaFuncSetAttribute(pcgamg2d_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcgamg2d_kernel<S>, AMG_T, smem));
  if (per_sm < 1) throw ApiError{VQPC_CUDA_ERROR, "pcgamg2d kernel does not fit on an SM"};
  const int64_t blocks = cap_groups(std::min<int64_t>(ngroups_max, static_cast<int64_t>(per_sm) * c->sm_count));
  prm.cv_off = static_cast<int64_t>(AMG_WORK) * c->n * S;
  prm.cta_stride = prm.cv_off + static_cast<int64_t>(c->amg_cv) * S + 2;
  c->amg_work.ensure(static_cast<size_t>(blocks) * prm.cta_stride);
  prm.work = c->amg_work.p;
  Timed tm(c, VQPC_K_PCG);
  pcgamg2d_kernel<S><<<static_cast<unsigned>(blocks), AMG_T, smem, c->stream>>>(prm);
  launch_check(c);
}

void run_pcgamg2d(vqpc_ctx* c, const double* d_kappa, int64_t ldk, const uint8_t* d_kflag, const int32_t* d_perm,
                  const int32_t* d_labels, int64_t B, int64_t out_base, double eps, int max_iter, const int32_t* d_mia,
                  int32_t* d_iters, double* d_rel, uint8_t* d_status, double* d_x, int64_t solve_limit) {
  const int P = c->pb.P;
  // samples per CTA (same label: the centroid's hierarchy is loaded once for all of them).
  // VQPC_AMG_S overrides: 1, 2, 4, 8. On 5,328 C4amg samples (final round-2 kernel) 2 gives
  // 1,262 samples/s, 1 gives 1,134, 4 gives 952 (profiles/r02u_ab_amg_s*.log); records identical
  int S = 2;
  if (const char* e = getenv("VQPC_AMG_S")) S = atoi(e);
  S = S >= 8 ? 8 : S >= 4 ? 4 : S >= 2 ? 2 : 1;
  c->ch_perm.ensure(B);
  c->ch_off.ensure(P + 2);
  c->ch_groups.ensure(B + P + 1);
  c->ch_ngroups.ensure(1);
  {
    Timed tm(c, VQPC_K_BUCKET);
    counting_sort(c, d_labels, d_perm, B, P, c->ch_perm.p, c->ch_off.p);
    chol_groups_kernel<<<1, CG_T, 0, c->stream>>>(c->ch_off.p, P, S, c->ch_groups.p, c->ch_ngroups.p);
    launch_check(c);
  }
  c->counter.ensure(1);
  CK(cudaMemsetAsync(c->counter.p, 0, sizeof(int), c->stream));
  PcgAmgParams prm{};
  prm.g = c->g2;
  prm.kappa = d_kappa;
  prm.ldk = ldk;
  prm.kflag = d_kflag;
  prm.perm = c->ch_perm.p;
  prm.labels = d_labels;
  prm.groups = c->ch_groups.p;
  prm.ngroups = c->ch_ngroups.p;
  prm.hier = c->amg_hd.p;
  prm.omega = 2.0 / 3.0;  // AmgOptions::jacobi_weight (solver.hpp:37)
  prm.B = B;
  prm.out_base = out_base;
  prm.solve_limit = solve_limit;
  prm.eps = eps;
  prm.max_iter = max_iter;
  prm.max_iter_arr = d_mia;
  prm.counter = c->counter.p;
  prm.iters = d_iters;
  prm.rel = d_rel;
  prm.status = d_status;
  prm.x_out = d_x;
  prm.exact = c->exact;
  const int64_t ng = ceil_div(B, S) + P + 1;
  switch (S) {
    case 8: launch_pcgamg2d<8>(c, prm, ng); break;
    case 4: launch_pcgamg2d<4>(c, prm, ng); break;
    case 2: launch_pcgamg2d<2>(c, prm, ng); break;
    default: launch_pcgamg2d<1>(c, prm, ng); break;
  }
}

// the per-grid wavefront map (level | row << 16) and, when the mesh's b is not
// uniform, the per-node right-hand side (shared by every sample)
void ensure_gmap_bvec(vqpc_ctx* c, const double* d_kappa) {
  if (!c->gmap.p) {
    c->gmap.ensure(c->n);
    build_gmap_kernel<<<64, P2_T, 0, c->stream>>>(c->g2, c->gmap.p);
    launch_check(c);
  }
  if (!c->b2_checked) {  // is b_i = area_sum_i / 3 the same for every node? (yes when h = 1/r is exact)
    c->bvec2.ensure(c->n);
    // b does not depend on kappa; any coefficient row serves the assembly call
    build_bvec_kernel<<<64, P2_T, 0, c->stream>>>(c->g2, c->kappa_c.p ? c->kappa_c.p : d_kappa, c->gmap.p,
                                                  c->bvec2.p);
    launch_check(c);
    std::vector<double> hb(c->n);
    CK(cudaMemcpyAsync(hb.data(), c->bvec2.p, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->b2_uniform = std::all_of(hb.begin(), hb.end(), [&](double v) { return v == hb[0]; });
    c->b2_checked = true;
  }
}

void run_pcg2d(vqpc_ctx* c, const double* d_kappa, int64_t ldk, const uint8_t* d_kflag, const int32_t* d_perm,
               const int32_t* d_labels, int64_t B, int64_t out_base, double eps, int max_iter, const int32_t* d_mia,
               int32_t* d_iters, double* d_rel, uint8_t* d_status, double* d_x, int64_t solve_limit) {
  if (c->chol2d) {
    run_pcgchol2d(c, d_kappa, ldk, d_kflag, d_perm, d_labels, B, out_base, eps, max_iter, d_mia, d_iters, d_rel,
                  d_status, d_x, solve_limit);
    return;
  }
  if (c->amg) {
    run_pcgamg2d(c, d_kappa, ldk, d_kflag, d_perm, d_labels, B, out_base, eps, max_iter, d_mia, d_iters, d_rel,
                 d_status, d_x, solve_limit);
    return;
  }
  int per_sm = 0;
  // C4's mesh (m = 255) has a specialised instantiation; other sizes take the generic one.
  // Meshes with more than 256 interior rows run the same kernel with 512 threads (one
  // thread per grid row, one CTA per SM).
  const char* ge = getenv("VQPC_P2_GENERIC");  // tests: the generic instantiation on C4's mesh
  const bool spec = c->g2.m == 255 && !(ge && atoi(ge));
  const bool big = c->g2.m > P2_T;
  const int TT = big ? P2_TBIG : P2_T;
  void (*kern)(const Pcg2dParams) = big ? pcg2d_kernel<0, P2_TBIG> : spec ? pcg2d_kernel<255, P2_T> : pcg2d_kernel<0, P2_T>;
  const size_t P2_DSMEM = p2_dsmem(TT);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P2_DSMEM)));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TT, P2_DSMEM));
  if (per_sm < 1) throw ApiError{VQPC_CUDA_ERROR, "pcg2d kernel does not fit on an SM"};
  const int64_t blocks = cap_groups(std::min<int64_t>(B, static_cast<int64_t>(per_sm) * c->sm_count));
  c->work2.ensure(static_cast<size_t>(blocks) * P2_WORK * c->n);
  c->counter.ensure(1);
  CK(cudaMemsetAsync(c->counter.p, 0, sizeof(int), c->stream));
  Pcg2dParams prm{};
  prm.g = c->g2;
  prm.kappa = d_kappa;
  prm.ldk = ldk;
  prm.kflag = d_kflag;
  prm.perm = d_perm;
  prm.labels = d_labels;
  prm.fac = c->fac2.p;
  prm.work = c->work2.p;
  prm.B = B;
  prm.out_base = out_base;
  prm.solve_limit = solve_limit;
  prm.eps = eps;
  prm.max_iter = max_iter;
  prm.max_iter_arr = d_mia;
  prm.counter = c->counter.p;
  prm.iters = d_iters;
  prm.rel = d_rel;
  prm.status = d_status;
  prm.x_out = d_x;
  prm.exact = c->exact;
  ensure_gmap_bvec(c, d_kappa);
  prm.gmap = c->gmap.p;
  prm.bvec = c->b2_uniform ? nullptr : c->bvec2.p;
  Timed tm(c, VQPC_K_PCG);
  kern<<<static_cast<unsigned>(blocks), TT, P2_DSMEM, c->stream>>>(prm);
  launch_check(c);
}

// 1-D reference-order mode (vqpc_set_exact_reductions): the serial-arithmetic
// instrument kernel; the factor's pass-1 values {l_j, u_j} are produced by the
// same factor1d_kernel on first use.
void run_pcg1d_exact(vqpc_ctx* c, const double* d_kappa, int64_t ldk, const uint8_t* d_kflag, const int32_t* d_perm,
                     const int32_t* d_labels, int64_t B, int64_t out_base, double eps, int max_iter,
                     const int32_t* d_mia, int32_t* d_iters, double* d_rel, uint8_t* d_status, double* d_x,
                     int64_t solve_limit) {
  const int P = c->lu_count, n = c->n;
  if (!c->have_lu) {
    c->fac_lu.ensure(static_cast<size_t>(P) * c->NP);
    CK(cudaMemsetAsync(c->err.p, 0, sizeof(int), c->stream));
    Timed tm(c, VQPC_K_OTHER);
    factor1d_kernel<<<static_cast<unsigned>(ceil_div(P, 64)), 64, 0, c->stream>>>(
        c->lu_src, c->lu_ld, P, n, h_of(c->pb), c->fac.p, c->NP, c->err.p, c->fac_lu.p);
    launch_check(c);
    c->have_lu = true;
  }
  int per_sm = 0;
  const size_t smem = sizeof(double) * n;
  CK(cudaFuncSetAttribute(pcg1d_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg1d_exact_kernel, PX_T, smem));
  const int64_t blocks = std::max<int64_t>(1, cap_groups(std::min<int64_t>(B, static_cast<int64_t>(per_sm) * c->sm_count)));
  c->work1x.ensure(static_cast<size_t>(blocks) * (6 * static_cast<size_t>(n) + 1));
  c->counter.ensure(1);
  CK(cudaMemsetAsync(c->counter.p, 0, sizeof(int), c->stream));
  Pcg1dExactParams prm{};
  prm.n = n;
  prm.h = h_of(c->pb);
  prm.kappa = d_kappa;
  prm.ldk = ldk;
  prm.kflag = d_kflag;
  prm.perm = d_perm;
  prm.labels = d_labels;
  prm.lu = c->fac_lu.p;
  prm.NP = c->NP;
  prm.B = B;
  prm.out_base = out_base;
  prm.solve_limit = solve_limit;
  prm.eps = eps;
  prm.max_iter = max_iter;
  prm.max_iter_arr = d_mia;
  prm.counter = c->counter.p;
  prm.iters = d_iters;
  prm.rel = d_rel;
  prm.status = d_status;
  prm.x_out = d_x;
  prm.work = c->work1x.p;
  Timed tm(c, VQPC_K_PCG);
  pcg1d_exact_kernel<<<static_cast<unsigned>(blocks), PX_T, smem, c->stream>>>(prm);
  launch_check(c);
}

void run_pcg(vqpc_ctx* c, const double* d_kappa, int64_t ldk, const uint8_t* d_kflag, const int32_t* d_perm,
             const int32_t* d_labels, int64_t B, int64_t out_base, double eps, int max_iter, const int32_t* d_mia,
             int32_t* d_iters, double* d_rel, uint8_t* d_status, double* d_x,
             int64_t solve_limit = INT64_MAX) {
  if (B <= 0) return;
  if (c->pb.dim == 2) {
    run_pcg2d(c, d_kappa, ldk, d_kflag, d_perm, d_labels, B, out_base, eps, max_iter, d_mia, d_iters, d_rel,
              d_status, d_x, solve_limit);
    return;
  }
  if (c->exact) {
    run_pcg1d_exact(c, d_kappa, ldk, d_kflag, d_perm, d_labels, B, out_base, eps, max_iter, d_mia, d_iters, d_rel,
                    d_status, d_x, solve_limit);
    return;
  }
  const PcgVariant* v = pick_pcg(c->n);
  c->counter.ensure(1);
  CK(cudaMemsetAsync(c->counter.p, 0, sizeof(int), c->stream));
  Pcg1dParams prm{};
  prm.n = c->n;
  prm.N = c->pb.size;
  prm.h = h_of(c->pb);
  prm.kappa = d_kappa;
  prm.ldk = ldk;
  prm.kflag = d_kflag;
  prm.perm = d_perm;
  prm.labels = d_labels;
  prm.factors = c->fac.p;
  prm.NP = c->NP;
  prm.B = B;
  prm.out_base = out_base;
  prm.solve_limit = solve_limit;
  prm.eps = eps;
  prm.max_iter = max_iter;
  prm.max_iter_arr = d_mia;
  prm.counter = c->counter.p;
  prm.iters = d_iters;
  prm.rel = d_rel;
  prm.status = d_status;
  prm.x_out = d_x;
  CK(cudaFuncSetAttribute(v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(v->smem)));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(v->T);
  cfg.dynamicSmemBytes = v->smem;
  cfg.stream = c->stream;
  int64_t groups = 0;  // concurrently resident samples (CTAs or clusters)
  if (v->CL == 1) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v->fn, v->T, v->smem));
    groups = static_cast<int64_t>(per_sm) * c->sm_count;
  } else {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = v->CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(v->CL * c->sm_count));
    int clusters = 0;
    CK(cudaOccupancyMaxActiveClusters(&clusters, v->fn, &cfg));
    groups = clusters;
  }
  if (groups < 1) throw ApiError{VQPC_CUDA_ERROR, "pcg kernel does not fit on the device"};
  groups = cap_groups(std::min<int64_t>(B, groups));
  cfg.gridDim = dim3(static_cast<unsigned>(groups * v->CL));
  // diagnostics (VQPC_TAIL=1): per-CTA busy span, to size the work-queue tail
  static const bool tail = getenv("VQPC_TAIL") != nullptr;
  unsigned long long* d_span = nullptr;
  const unsigned nblk = cfg.gridDim.x;
  if (tail) {
    CK(cudaMallocAsync(&d_span, 2 * sizeof(unsigned long long) * nblk, c->stream));
    prm.t_span = d_span;
  }
  {
    Timed tm(c, VQPC_K_PCG);
    CK(cudaLaunchKernelEx(&cfg, v->fn, prm));
    launch_check(c);
  }
  if (tail) {
    std::vector<unsigned long long> h(2 * nblk);
    CK(cudaMemcpyAsync(h.data(), d_span, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaFreeAsync(d_span, c->stream));
    unsigned long long t0 = ~0ull, t1 = 0;
    std::vector<double> ends;
    for (unsigned b = 0; b < nblk; ++b) {
      t0 = std::min(t0, h[2 * b]);
      t1 = std::max(t1, h[2 * b + 1]);
    }
    for (unsigned b = 0; b < nblk; ++b) ends.push_back(1e-6 * static_cast<double>(h[2 * b + 1] - t0));
    std::sort(ends.begin(), ends.end());
    fprintf(stderr, "[vqpc tail] pcg1d B=%lld ctas=%u span %.3f ms; CTA end ms: min %.3f p10 %.3f median %.3f p90 %.3f max %.3f\n",
            static_cast<long long>(B), nblk, 1e-6 * static_cast<double>(t1 - t0), ends.front(), ends[nblk / 10],
            ends[nblk / 2], ends[9 * nblk / 10], ends.back());
  }
}

__global__ void stats_kernel(const int32_t* labels, const int32_t* iters, const uint8_t* status, int64_t B, int P,
                             unsigned long long* stats, unsigned long long* summary) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const int l = labels[i];
  if (status[i] == VQPC_S_NOT_SOLVED) return;
  const unsigned long long J = static_cast<unsigned long long>(iters[i]);
  const bool conv = status[i] == VQPC_S_CONVERGED;
  atomicAdd(&summary[0], J);
  atomicAdd(&summary[conv ? 2 : 1], 1ull);
  if (conv) atomicAdd(&summary[3], J);
  if (l < 0 || l >= P) return;
  atomicAdd(&stats[l], 1ull);
  atomicAdd(&stats[P + l], J);
  if (conv) {
    atomicAdd(&stats[2 * P + l], 1ull);
    atomicAdd(&stats[3 * P + l], J);
  }
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[i] = static_cast<int32_t>(i);
}

__global__ void mark_unsolved_kernel(int32_t* iters, double* rel, uint8_t* status, int64_t B) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= B) return;
  iters[i] = 0;
  rel[i] = 0.0;
  status[i] = VQPC_S_NOT_SOLVED;
}

template <class F>
int guard(vqpc_ctx* c, F&& f) {
  try {
    if (c) CK(cudaSetDevice(c->pb.device));
    f();
    return VQPC_OK;
  } catch (const CudaError& e) {
    if (c) c->last_error = e.msg;
    return e.code;
  } catch (const ApiError& e) {
    if (c) c->last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (c) c->last_error = "host allocation failed";
    return VQPC_OUT_OF_MEMORY;
  }
}

template <class T>
void h2d(vqpc_ctx* c, T* dst, const T* src, size_t count) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
}
template <class T>
void d2h(vqpc_ctx* c, T* dst, const T* src, size_t count) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
}

int64_t kappa_ld(const vqpc_ctx* c) { return (c->pb.n_nodes + 1) & ~1; }

// 2-D `cholesky` kind: the symbolic part, once per context (the pattern is the same
// for every centroid and sample). Interior node id = iy * m + ix (fem.cpp:28-42);
// its stored columns, ascending, are SW, S, W, itself, E, N, NE (the a-d diagonal of
// every cell couples SW/NE with an exact zero the reference still stores, so they
// count for the degrees and the envelope). Reverse Cuthill-McKee as in
// solver.cpp:32-70: start every component at the unvisited node of least (degree,
// id), breadth-first, each node's unvisited neighbours enqueued by (degree, id),
// then the order reversed. Then the envelope of the permuted matrix (first[k] =
// smallest permuted column of row k), its row offsets, and the staging capacity of
// the blocked solves.
void setup_chol2d(vqpc_ctx* c) {
  const int m = c->g2.m, n = m * m;
  auto cols = [&](int id, int* out) {  // ascending stored columns of row id
    const int ix = id % m, iy = id / m;
    int k = 0;
    if (iy > 0 && ix > 0) out[k++] = id - m - 1;
    if (iy > 0) out[k++] = id - m;
    if (ix > 0) out[k++] = id - 1;
    out[k++] = id;
    if (ix < m - 1) out[k++] = id + 1;
    if (iy < m - 1) out[k++] = id + m;
    if (iy < m - 1 && ix < m - 1) out[k++] = id + m + 1;
    return k;
  };
  std::vector<int> deg(n);
  int buf[7];
  for (int i = 0; i < n; ++i) deg[i] = cols(i, buf);
  auto before = [&](int a, int b) { return deg[a] < deg[b] || (deg[a] == deg[b] && a < b); };
  std::vector<int> seeds(n);
  for (int i = 0; i < n; ++i) seeds[i] = i;
  std::sort(seeds.begin(), seeds.end(), before);
  std::vector<int> order;
  order.reserve(n);
  std::vector<char> visited(n, 0);
  for (int s0 : seeds) {
    if (visited[s0]) continue;
    visited[s0] = 1;
    size_t head = order.size();
    order.push_back(s0);
    while (head < order.size()) {
      const int u = order[head++];
      int nb[7], cnt = 0;
      const int kk = cols(u, buf);
      for (int e = 0; e < kk; ++e)
        if (buf[e] != u && !visited[buf[e]]) {
          visited[buf[e]] = 1;
          nb[cnt++] = buf[e];
        }
      std::sort(nb, nb + cnt, before);
      for (int e = 0; e < cnt; ++e) order.push_back(nb[e]);
    }
  }
  std::reverse(order.begin(), order.end());  // order[k] = natural id of permuted row k
  std::vector<int> inv(n), first(n);
  for (int k = 0; k < n; ++k) inv[order[k]] = k;
  std::vector<int64_t> start(n + 1, 0);
  std::vector<int4> nbr(n);
  int W = 0;
  for (int k = 0; k < n; ++k) {
    const int id = order[k], kk = cols(id, buf);
    int f = k;
    for (int e = 0; e < kk; ++e) f = std::min(f, inv[buf[e]]);
    first[k] = f;
    W = std::max(W, k - f);
    start[k + 1] = start[k] + (k - f + 1);
    const int ix = id % m, iy = id / m;
    nbr[k] = make_int4(iy > 0 ? inv[id - m] : -1, ix > 0 ? inv[id - 1] : -1, ix < m - 1 ? inv[id + 1] : -1,
                       iy < m - 1 ? inv[id + m] : -1);
  }
  const int nblk = static_cast<int>(ceil_div(n, PC_BS));
  // per 32-row block: the staged range of L (16-byte aligned) and, per row, first[]
  // and the offset of its column 0 inside the staged range (rows past n: empty)
  int64_t cap = 0;
  std::vector<int64_t> a0s(nblk);
  std::vector<unsigned> bytes(nblk);
  std::vector<int> bmeta(static_cast<size_t>(nblk) * 2 * PC_BS);
  for (int b = 0; b < nblk; ++b) {
    const int r0 = b * PC_BS, r1 = std::min(n, r0 + PC_BS);
    const int64_t a0 = start[r0] & ~int64_t{1}, a1 = (start[r1] + 1) & ~int64_t{1};
    cap = std::max(cap, a1 - a0);
    a0s[b] = a0;
    bytes[b] = static_cast<unsigned>((a1 - a0) * 8);
    for (int i = 0; i < PC_BS; ++i) {
      const int k = r0 + i;
      bmeta[static_cast<size_t>(b) * 2 * PC_BS + i] = k < n ? first[k] : k;
      bmeta[static_cast<size_t>(b) * 2 * PC_BS + PC_BS + i] = k < n ? static_cast<int>(start[k] - first[k] - a0) : 0;
    }
  }
  c->ch_a0.ensure(nblk);
  c->ch_bytes.ensure(nblk);
  c->ch_bmeta.ensure(bmeta.size());
  h2d(c, c->ch_a0.p, a0s.data(), nblk);
  h2d(c, c->ch_bytes.p, bytes.data(), nblk);
  h2d(c, c->ch_bmeta.p, bmeta.data(), bmeta.size());
  if (W > PC_WIN || W + 3 * PC_BS > pc_ring(PC_MAXS)) throw ApiError{VQPC_INVALID_CONFIG, "cholesky envelope wider than the solve ring"};
  c->ch_cperm.ensure(n);
  c->ch_first.ensure(n);
  c->ch_start.ensure(n + 1);
  c->ch_nbr.ensure(n);
  h2d(c, c->ch_cperm.p, order.data(), n);
  h2d(c, c->ch_first.p, first.data(), n);
  h2d(c, c->ch_start.p, start.data(), n + 1);
  h2d(c, c->ch_nbr.p, nbr.data(), n);
  c->clay.n = n;
  c->clay.W = W;
  c->clay.nblk = nblk;
  c->clay.cperm = c->ch_cperm.p;
  c->clay.first = c->ch_first.p;
  c->clay.start = c->ch_start.p;
  c->clay.nbr = c->ch_nbr.p;
  c->ch_ldL = (start[n] + 1) & ~int64_t{1};
  c->ch_nnz = start[n];
  c->ch_ldLi = static_cast<int64_t>(nblk) * PC_LIB;
  c->ch_cap = static_cast<int>(cap);
  c->chol2d = true;
  if (const char* e = getenv("VQPC_CHOL_S")) c->ch_S = std::max(1, std::min(PC_MAXS, atoi(e)));
  CK(cudaStreamSynchronize(c->stream));
}

// 2-D SA-AMG kind: the centroid matrices' CSR rows are assembled on the device with
// the oracle's operations (amg_centroid_rows_kernel), the P hierarchies are built on
// host threads (amg_setup.cuh; independent per centroid, as the reference builds
// each AmgPreconditioner, driver.cpp:212-219) and packed as sliced ELL.
void setup_amg(vqpc_ctx* c, const double* d_kc, int64_t ldk, int P) {
  const int n = c->n;
  DBuf<double> rows;
  rows.ensure(static_cast<size_t>(P) * n * 7);
  amg_centroid_rows_kernel<<<4 * c->sm_count, 256, 0, c->stream>>>(d_kc, ldk, P, c->g2, rows.p);
  launch_check(c);
  std::vector<double> hv(static_cast<size_t>(P) * n * 7);
  d2h(c, hv.data(), rows.p, hv.size());
  CK(cudaStreamSynchronize(c->stream));
  rows.release();
  c->amg_h.assign(P, {});
  std::vector<int> failed(P, 0);
  const int m = c->g2.m;
  const int offs[7] = {-m - 1, -m, -1, 0, 1, m, m + 1};
  auto work = [&](int p) {
    amg::Csr A;
    A.rows = A.cols = n;
    A.ptr.assign(n + 1, 0);
    A.idx.reserve(static_cast<size_t>(n) * 7);
    A.val.reserve(static_cast<size_t>(n) * 7);
    for (int i = 0; i < n; ++i) {
      const double* v = hv.data() + (static_cast<size_t>(p) * n + i) * 7;
      for (int k = 0; k < 7; ++k)
        if (!std::isnan(v[k])) {
          A.idx.push_back(i + offs[k]);
          A.val.push_back(v[k]);
        }
      A.ptr[i + 1] = static_cast<int>(A.idx.size());
    }
    try {
      c->amg_h[p] = amg::build(A);
    } catch (const amg::NotSpd&) {
      failed[p] = 1;
    }
  };
  {
    const int nt = std::max(1, std::min<int>(P, static_cast<int>(std::thread::hardware_concurrency())));
    std::vector<std::thread> pool;
    std::atomic<int> next{0};
    for (int w = 0; w < nt; ++w)
      pool.emplace_back([&] {
        for (int p = next++; p < P; p = next++) work(p);
      });
    for (auto& th : pool) th.join();
  }
  for (int p = 0; p < P; ++p)
    if (failed[p]) throw ApiError{VQPC_NOT_SPD, "not-spd (AMG hierarchy of centroid " + std::to_string(p) + ")"};
  // pack: ints (slice offsets + columns) and doubles (values, inverse diagonals, dense L)
  std::vector<int> hi;
  std::vector<double> hd;
  struct EllOff { size_t row, rec; };
  auto pack_ell = [&](const amg::Csr& M) {
    EllOff o{};
    const int ns = (M.rows + 31) / 32;
    std::vector<int> soff(ns + 1, 0);
    for (int s = 0; s < ns; ++s) {
      int w = 0;
      for (int i = 32 * s; i < std::min(M.rows, 32 * s + 32); ++i) w = std::max(w, M.ptr[i + 1] - M.ptr[i]);
      soff[s + 1] = soff[s] + 32 * w;
    }
    if (hi.size() & 1) hi.push_back(0);  // int2 alignment of the per-row {first record, length}
    o.row = hi.size();
    for (int i = 0; i < M.rows; ++i) {
      hi.push_back(soff[i >> 5] + (i & 31));
      hi.push_back(M.ptr[i + 1] - M.ptr[i]);
    }
    if (hd.size() & 1) hd.push_back(0.0);  // 16-byte alignment of the records
    o.rec = hd.size();
    hd.resize(hd.size() + 2 * static_cast<size_t>(soff[ns]), 0.0);
    for (size_t e = 0; e < static_cast<size_t>(soff[ns]); ++e) {  // padding records: value 0, column -1
      const long long pad = -1;
      std::memcpy(&hd[o.rec + 2 * e + 1], &pad, sizeof(double));
    }
    for (int i = 0; i < M.rows; ++i)
      for (int k = 0; k < M.ptr[i + 1] - M.ptr[i]; ++k) {
        const size_t e = soff[i >> 5] + 32 * static_cast<size_t>(k) + (i & 31);
        hd[o.rec + 2 * e] = M.val[M.ptr[i] + k];
        const long long col = M.idx[M.ptr[i] + k];
        std::memcpy(&hd[o.rec + 2 * e + 1], &col, sizeof(double));
      }
    return o;
  };
  struct LevOff { EllOff A, P, Pt; size_t inv, st; };
  std::vector<std::vector<LevOff>> lo(P);
  std::vector<size_t> loff(P);
  std::vector<AmgHierD> hh(P);
  int cv_max = 0;
  int64_t entries = 0;
  for (int p = 0; p < P; ++p) {
    const amg::Hierarchy& H = c->amg_h[p];
    if (H.lv.size() > static_cast<size_t>(AMG_MAXLEV))
      throw ApiError{VQPC_INVALID_CONFIG, "AMG hierarchy deeper than the device limit"};
    if (H.dense_n > AMG_MAXDENSE) throw ApiError{VQPC_INVALID_CONFIG, "AMG coarsest level too large for the dense solve"};
    int cv = 0;
    for (size_t l = 0; l < H.lv.size(); ++l) {
      const amg::Level& L = H.lv[l];
      LevOff o{};
      o.A = pack_ell(L.A);
      if (L.P.rows) {
        o.P = pack_ell(L.P);
        o.Pt = pack_ell(L.Pt);
      }
      o.inv = hd.size();
      hd.insert(hd.end(), L.inv_diag.begin(), L.inv_diag.end());
      o.st = SIZE_MAX;
      if (l == 0) {  // the centroid matrix's stencil: S, W, diagonal per row (zeros where absent)
        o.st = hd.size();
        hd.resize(hd.size() + 3 * static_cast<size_t>(n), 0.0);
        double* st = hd.data() + o.st;
        for (int i = 0; i < n; ++i)
          for (int e = L.A.ptr[i]; e < L.A.ptr[i + 1]; ++e) {
            const int j = L.A.idx[e];
            if (j == i - m) st[i] = L.A.val[e];
            else if (j == i - 1) st[n + i] = L.A.val[e];
            else if (j == i) st[2 * static_cast<size_t>(n) + i] = L.A.val[e];
          }
      }
      lo[p].push_back(o);
      AmgLevelD& d = hh[p].lv[l];
      d.n = L.A.rows;
      d.nc = L.P.rows ? L.P.cols : 0;
      d.voff = l == 0 ? 0 : cv;
      if (l > 0) cv += 3 * d.n;
      entries += L.A.nnz() + L.P.nnz() + L.Pt.nnz();
    }
    cv_max = std::max(cv_max, cv);
    loff[p] = hd.size();
    hd.insert(hd.end(), H.L.begin(), H.L.end());
    hh[p].nlev = static_cast<int>(H.lv.size());
    hh[p].dense_n = H.dense_n;
  }
  c->amg_i.ensure(hi.size());
  c->amg_d.ensure(hd.size());
  h2d(c, c->amg_i.p, hi.data(), hi.size());
  h2d(c, c->amg_d.p, hd.data(), hd.size());
  auto ell_ptr = [&](const EllOff& o, int rows, int cols) {
    return AmgEll{reinterpret_cast<const int2*>(c->amg_i.p + o.row), reinterpret_cast<const double2*>(c->amg_d.p + o.rec),
                  rows, cols};
  };
  for (int p = 0; p < P; ++p) {
    for (int l = 0; l < hh[p].nlev; ++l) {
      AmgLevelD& d = hh[p].lv[l];
      d.A = ell_ptr(lo[p][l].A, d.n, d.n);
      if (d.nc) {
        d.P = ell_ptr(lo[p][l].P, d.n, d.nc);
        d.Pt = ell_ptr(lo[p][l].Pt, d.nc, d.n);
      }
      d.inv_diag = c->amg_d.p + lo[p][l].inv;
      d.st_s = d.st_w = d.st_c = nullptr;
      d.st_m = m;
      if (lo[p][l].st != SIZE_MAX) {
        d.st_s = c->amg_d.p + lo[p][l].st;
        d.st_w = d.st_s + n;
        d.st_c = d.st_w + n;
      }
    }
    hh[p].L = c->amg_d.p + loff[p];
  }
  c->amg_hd.ensure(P);
  h2d(c, c->amg_hd.p, hh.data(), P);
  CK(cudaStreamSynchronize(c->stream));
  c->amg_cv = (cv_max + 1) & ~1;
  c->amg_entries = entries / P;
  c->amg_dense_max = 0;
  for (int p = 0; p < P; ++p) c->amg_dense_max = std::max(c->amg_dense_max, hh[p].dense_n);
}

// Factor P coefficient fields (d_kc: P rows of ldk nodal/elemental values) into the
// context's factor buffers, indexed by label 0..P-1: the per-centroid step of
// run_campaign_with (driver.cpp:212-219), also used by the ideal sweep with one
// factor per realisation (driver.cpp:317-320). Throws not-spd.
void factor_coefficients(vqpc_ctx* c, const double* d_kc, int64_t ldk, int P) {
  const vqpc_problem& pb = c->pb;
  c->lu_src = d_kc;  // the 1-D reference-order mode rebuilds its {l_j, u_j} from these on first use
  c->lu_ld = ldk;
  c->lu_count = P;
  c->have_lu = false;
    c->err.ensure(1);
    CK(cudaMemsetAsync(c->err.p, 0, sizeof(int), c->stream));
    if (pb.dim == 2 && c->chol2d) {
      c->ch_L.ensure(static_cast<size_t>(P) * c->ch_ldL);
      c->ch_Linv.ensure(static_cast<size_t>(P) * c->ch_ldLi);
      Timed tm(c, VQPC_K_OTHER);
      cholfactor2d_kernel<<<P, PC_T, 0, c->stream>>>(d_kc, ldk, P, c->g2, c->clay, c->ch_L.p, c->ch_ldL,
                                                     c->err.p);
      launch_check(c);
      const int64_t th = static_cast<int64_t>(P) * c->clay.nblk * PC_BS;
      cholinv_kernel<<<static_cast<unsigned>(ceil_div(th, 128)), 128, 0, c->stream>>>(c->ch_L.p, c->ch_ldL, c->clay,
                                                                                      P, c->ch_Linv.p, c->ch_ldLi);
      launch_check(c);
      for (int p = 0; p < P; ++p)  // each block record's metadata tail (one TMA copy per block)
        CK(cudaMemcpy2DAsync(c->ch_Linv.p + static_cast<size_t>(p) * c->ch_ldLi + PC_STG_META, PC_LIB * sizeof(double),
                             c->ch_bmeta.p, 2 * PC_BS * sizeof(int), 2 * PC_BS * sizeof(int), c->clay.nblk,
                             cudaMemcpyDeviceToDevice, c->stream));
    } else if (pb.dim == 2 && c->amg) {
      setup_amg(c, d_kc, ldk, P);
    } else if (pb.dim == 2) {
      c->fac2.ensure(static_cast<size_t>(P) * P2_FAC * c->n);
      Timed tm(c, VQPC_K_OTHER);
      if (c->g2.m > P2_T)
        factor2d_kernel<P2_TBIG><<<P, P2_TBIG, 0, c->stream>>>(d_kc, ldk, P, c->g2, c->fac2.p, c->err.p);
      else
        factor2d_kernel<P2_T><<<P, P2_T, 0, c->stream>>>(d_kc, ldk, P, c->g2, c->fac2.p, c->err.p);
      launch_check(c);
    } else {
      c->fac.ensure(static_cast<size_t>(P) * c->NP);
      Timed tm(c, VQPC_K_OTHER);
      factor1d_kernel<<<static_cast<unsigned>(ceil_div(P, 64)), 64, 0, c->stream>>>(d_kc, ldk, P, c->n,
                                                                                      h_of(pb), c->fac.p, c->NP,
                                                                                      c->err.p);
      launch_check(c);
    }
  int err = 0;
  d2h(c, &err, c->err.p, 1);
  CK(cudaStreamSynchronize(c->stream));
  if (err) throw ApiError{VQPC_NOT_SPD, "not-spd"};
}

// The full campaign on device-resident arrays (run_campaign_with semantics).
void campaign_device(vqpc_ctx* c, const double* d_xi, int64_t B, int ld, double eps, int max_iter, int64_t chunk,
                     int32_t* d_labels, int32_t* d_iters, double* d_rel, uint8_t* d_status, int64_t* d_stats,
                     int64_t* d_summary, int64_t solve_limit = INT64_MAX, double* d_x = nullptr) {
  if (!(eps > 0.0) || eps >= 1.0) throw ApiError{VQPC_INVALID_TOLERANCE, "invalid-tolerance"};
  if (ld < c->pb.n_kl) throw ApiError{VQPC_INVALID_ARGUMENT, "ld < n_kl"};
  if (!c->factored) throw ApiError{VQPC_INVALID_CONFIG, "vqpc_factor_centroids must precede solves"};
  const int P = c->pb.P;
  if (chunk <= 0 || chunk > B) chunk = B;
  const int64_t ldk = kappa_ld(c);
  const double* root = c->pb.method == VQPC_GRID || c->pb.method == VQPC_SIGN_GRID ? nullptr : c->root.p;
  // Samples [0, nsolve) are solved. When that range spans several chunks, their
  // kappa rows are kept and solved by ONE PCG launch after the chunk loop (one
  // work-queue tail instead of one per chunk; C5: 4 launches -> 1) as long as the
  // rows fit a fixed budget; otherwise every chunk is solved as it is realised.
  const int64_t nsolve = std::min<int64_t>(B, std::max<int64_t>(solve_limit, 0));
  constexpr double kMergeBudget = 16e9;  // bytes of kept kappa rows
  const bool merge = chunk < B && nsolve > chunk &&
                     static_cast<double>(nsolve) * static_cast<double>(ldk) * 8.0 <= kMergeBudget;
  const int64_t keep = merge ? nsolve : 0;  // kept rows (merged solve)
  c->kappa.ensure(static_cast<size_t>(std::max<int64_t>(keep + chunk, 1)) * ldk);
  c->kflag.ensure(static_cast<size_t>(std::max<int64_t>(keep + chunk, 1)) + 4);  // + 4: word-wide atomicOr flags
  c->perm.ensure(std::max<int64_t>(std::max(keep, chunk), 1));
  c->offsets.ensure(P + 2);
  double* const kappa_scratch = c->kappa.p + static_cast<size_t>(keep) * ldk;  // rows of unsolved chunks
  uint8_t* const kflag_scratch = c->kflag.p + keep;
  if (merge) CK(cudaMemsetAsync(c->kflag.p, 0, keep, c->stream));
  // Merged solve with chunks entirely beyond the solve subset (C5: 60 of 64 chunks are
  // realised and assigned only): those chunks run on a second stream after the merged
  // PCG launch, so their kernels fill the SMs the PCG's work-queue tail leaves idle
  // instead of preceding the solve. They touch only the scratch rows and their own
  // labels/records; the stats kernel waits for them.
  // (not while per-launch events are recorded: profiled steps run serially so that the
  // kernel times do not overlap)
  const bool overlap = merge && nsolve < B && !c->prof && std::getenv("VQPC_NO_OVERLAP") == nullptr;
  const int64_t split_c0 = overlap ? std::min<int64_t>(B, ceil_div(nsolve, chunk) * chunk) : B;
  auto realise_assign_only = [&](int64_t c0) {  // a chunk beyond the solve subset
    const int64_t nb = std::min(chunk, B - c0);
    const double* xi = d_xi + c0 * ld;
    run_assign(c, xi, nb, ld, root, c->sites.p, P, c->pb.m, d_labels + c0, nullptr);
    CK(cudaMemsetAsync(kflag_scratch, 0, nb, c->stream));
    run_realise(c, xi, nb, ld, c->pb.n_kl, kappa_scratch, ldk, kflag_scratch);
    mark_unsolved_kernel<<<static_cast<unsigned>(ceil_div(nb, 256)), 256, 0, c->stream>>>(
        d_iters + c0, d_rel + c0, d_status + c0, nb);
    launch_check(c);
  };
  for (int64_t c0 = 0; c0 < split_c0; c0 += chunk) {
    const int64_t nb = std::min(chunk, B - c0);
    const double* xi = d_xi + c0 * ld;
    run_assign(c, xi, nb, ld, root, c->sites.p, P, c->pb.m, d_labels + c0, nullptr);
    const bool kept = merge && c0 < nsolve;  // rows [c0, c0 + nb) land in the kept buffer
    double* kap = kept ? c->kappa.p + static_cast<size_t>(c0) * ldk : kappa_scratch;
    uint8_t* kfl = kept ? c->kflag.p + c0 : kflag_scratch;
    if (!kept) CK(cudaMemsetAsync(kfl, 0, nb, c->stream));
    run_realise(c, xi, nb, ld, c->pb.n_kl, kap, ldk, kfl);
    if (merge) {
      // beyond the solve subset: mark here; solved rows wait for the merged launch
      const int64_t u0 = std::max(c0, nsolve), u1 = c0 + nb;
      if (u1 > u0) {
        mark_unsolved_kernel<<<static_cast<unsigned>(ceil_div(u1 - u0, 256)), 256, 0, c->stream>>>(
            d_iters + u0, d_rel + u0, d_status + u0, u1 - u0);
        launch_check(c);
      }
      continue;
    }
    if (c0 >= solve_limit) {  // whole chunk beyond the solve subset: mark, skip the solver
      mark_unsolved_kernel<<<static_cast<unsigned>(ceil_div(nb, 256)), 256, 0, c->stream>>>(
          d_iters + c0, d_rel + c0, d_status + c0, nb);
      launch_check(c);
      continue;
    }
    run_schedule(c, xi, ld, d_labels + c0, nb, root);
    run_pcg(c, kap, ldk, kfl, c->perm.p, d_labels + c0, nb, c0, eps, max_iter, nullptr, d_iters, d_rel, d_status,
            d_x, solve_limit);
  }
  if (overlap && split_c0 < B) {
    if (!c->aux) CK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    if (!c->ev_a) CK(cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming));
    if (!c->ev_b) CK(cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming));
    CK(cudaEventRecord(c->ev_a, c->stream));  // the solve subset is assigned and realised
  }
  if (merge) {
    run_schedule(c, d_xi, ld, d_labels, nsolve, root);
    run_pcg(c, c->kappa.p, ldk, c->kflag.p, c->perm.p, d_labels, nsolve, 0, eps, max_iter, nullptr, d_iters,
            d_rel, d_status, d_x, solve_limit);
  }
  if (overlap && split_c0 < B) {
    CK(cudaStreamWaitEvent(c->aux, c->ev_a, 0));
    std::swap(c->stream, c->aux);  // every launch helper (and its event timing) uses c->stream
    try {
      for (int64_t c0 = split_c0; c0 < B; c0 += chunk) realise_assign_only(c0);
    } catch (...) {
      std::swap(c->stream, c->aux);
      throw;
    }
    std::swap(c->stream, c->aux);
    CK(cudaEventRecord(c->ev_b, c->aux));
    CK(cudaStreamWaitEvent(c->stream, c->ev_b, 0));
  }
  CK(cudaMemsetAsync(d_stats, 0, sizeof(int64_t) * 4 * P, c->stream));
  CK(cudaMemsetAsync(d_summary, 0, sizeof(int64_t) * 4, c->stream));
  if (B <= 0) return;  // empty batch: zero statistics
  Timed tm(c, VQPC_K_OTHER);
  stats_kernel<<<static_cast<unsigned>(ceil_div(B, 256)), 256, 0, c->stream>>>(
      d_labels, d_iters, d_status, B, P, reinterpret_cast<unsigned long long*>(d_stats),
      reinterpret_cast<unsigned long long*>(d_summary));
  launch_check(c);
}

}  // namespace

// =============================================================================
extern "C" {

const char* vqpc_error_string(int code) {
  switch (code) {
    case VQPC_OK: return "ok";
    case VQPC_INVALID_LATENT: return "invalid-latent";
    case VQPC_INVALID_COEFFICIENT: return "invalid-coefficient";
    case VQPC_COEFFICIENT_OVERFLOW: return "coefficient-overflow";
    case VQPC_NOT_SPD: return "not-spd";
    case VQPC_PCG_BREAKDOWN: return "pcg-breakdown";
    case VQPC_INVALID_TOLERANCE: return "invalid-tolerance";
    case VQPC_MODE_COUNT_OUT_OF_RANGE: return "mode-count-out-of-range";
    case VQPC_INVALID_CODEBOOK: return "invalid-codebook";
    case VQPC_INSUFFICIENT_SAMPLES: return "insufficient-samples";
    case VQPC_INVALID_CONFIG: return "invalid-config";
    case VQPC_INVALID_ARGUMENT: return "invalid-argument";
    case VQPC_CUDA_ERROR: return "cuda-error";
    case VQPC_NO_DEVICE: return "no-device";
    case VQPC_OUT_OF_MEMORY: return "out-of-memory";
    default: return "unknown";
  }
}

const char* vqpc_last_error(const vqpc_ctx* c) { return c ? c->last_error.c_str() : ""; }
int vqpc_unknowns(const vqpc_ctx* c) { return c ? c->n : 0; }
int64_t vqpc_factor_entries(const vqpc_ctx* c) {
  if (!c) return 0;
  if (c->chol2d) return c->ch_nnz;
  if (c->amg) return c->amg_entries;
  return c->pb.dim == 2 ? 3 * static_cast<int64_t>(c->n) : 2 * static_cast<int64_t>(c->n) - 1;
}
int64_t vqpc_launch_count(const vqpc_ctx* c) { return c ? c->launches : 0; }

int vqpc_ctx_create(const vqpc_problem* pb, vqpc_ctx** out) {
  if (!pb || !out) return VQPC_INVALID_ARGUMENT;
  *out = nullptr;
  const int dev_ok = check_device(pb->device);
  if (dev_ok != VQPC_OK) return dev_ok;
  if (pb->dim != 1 && pb->dim != 2) return VQPC_INVALID_CONFIG;
  if (pb->size < 2 || pb->n_kl < 1 || pb->P < 1 || pb->m < 0) return VQPC_INVALID_CONFIG;
  const int n_nodes = pb->dim == 1 ? pb->size : (pb->size + 1) * (pb->size + 1);
  if (pb->n_nodes != n_nodes) return VQPC_INVALID_CONFIG;
  if (pb->m > pb->n_kl) return VQPC_MODE_COUNT_OUT_OF_RANGE;
  const bool grid = pb->method == VQPC_GRID || pb->method == VQPC_SIGN_GRID;
  if (grid && !pb->latent) return VQPC_INVALID_CODEBOOK;
  if (pb->dim == 1 && pb->precond != VQPC_PC_CHOLESKY) return VQPC_INVALID_CONFIG;
  // IC(0)'s level sweeps put one thread on each grid row (r - 1 <= 512: 256-thread CTAs up
  // to r = 257, 512-thread CTAs beyond); the cholesky kind checks its envelope width at
  // setup; the AMG kind has no mesh-size limit
  if (pb->dim == 2 && ((pb->precond != VQPC_PC_IC0 && pb->precond != VQPC_PC_CHOLESKY && pb->precond != VQPC_PC_AMG) ||
                       (pb->precond == VQPC_PC_IC0 && pb->size - 1 > P2_TBIG)))
    return VQPC_INVALID_CONFIG;
  auto* c = new vqpc_ctx();
  c->pb = *pb;
  c->n = pb->dim == 1 ? pb->size - 1 : (pb->size - 1) * (pb->size - 1);
  const int rc = guard(c, [&] {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, pb->device));
    c->sm_count = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    if (pb->dim == 2) {
      c->g2.r = pb->size;
      c->g2.m = pb->size - 1;
      c->g2.n = c->g2.m * c->g2.m;
      c->g2.L = 2 * c->g2.m - 1;
      c->g2.h = 1.0 / pb->size;
      unsigned char dp[16][6];
      diag_orders(dp);
      CK(cudaMemcpyToSymbol(vqpc_dperm, dp, sizeof(dp)));
      if (pb->precond == VQPC_PC_CHOLESKY) setup_chol2d(c);
      c->amg = pb->precond == VQPC_PC_AMG;
    }
    if (pb->dim == 1) {
      const PcgVariant* v = pick_pcg(c->n);
      if (!v) throw ApiError{VQPC_INVALID_CONFIG, "1-D system larger than the largest pcg variant"};
      c->pcgR = v->R;
      c->pcgT = v->T;
      c->NP = v->R * v->T * v->CL;
    }
    const size_t K = pb->n_kl, nn = pb->n_nodes;
    std::vector<double> sl(K);
    for (size_t k = 0; k < K; ++k) {
      if (!(pb->eigenvalues[k] >= 0.0)) throw ApiError{VQPC_INVALID_CONFIG, "negative eigenvalue"};
      sl[k] = std::sqrt(pb->eigenvalues[k]);  // the reference's std::sqrt(lambda_k)
    }
    c->phi.ensure(K * nn);
    c->sqrt_lam.ensure(K);
    h2d(c, c->phi.p, pb->eigenvectors, K * nn);
    h2d(c, c->sqrt_lam.p, sl.data(), K);
    const size_t Pm = static_cast<size_t>(pb->P) * pb->m;
    c->sites.ensure(std::max<size_t>(Pm, 1));
    h2d(c, c->sites.p, grid ? pb->latent : pb->centroids, Pm);
    c->h_lambdas.assign(pb->lambdas, pb->lambdas + pb->m);
    std::vector<double> root(std::max(pb->m, 1));
    for (int k = 0; k < pb->m; ++k) root[k] = std::sqrt(pb->lambdas[k]);  // T2Map::to_quant root
    c->root.ensure(root.size());
    h2d(c, c->root.p, root.data(), root.size());
    if (pb->map == VQPC_CDF && !grid) throw ApiError{VQPC_INVALID_CONFIG, "ScaledCdf map: not on the GPU path"};
    CK(cudaStreamSynchronize(c->stream));
  });
  if (rc != VQPC_OK) {
    vqpc_ctx_destroy(c);
    return rc;
  }
  *out = c;
  return VQPC_OK;
}

void vqpc_ctx_destroy(vqpc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->pb.device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto* b : {&c->phi, &c->sqrt_lam, &c->root, &c->sites, &c->kappa_c, &c->xi, &c->kappa, &c->best, &c->dvec,
                  &c->rel, &c->x, &c->fac2, &c->work2})
    b->release();
  c->fac.release();
  c->fac_lu.release();
  c->work1x.release();
  c->kflag.release();
  c->status.release();
  for (auto* b : {&c->labels, &c->perm, &c->counts, &c->iters, &c->mia, &c->keys, &c->perm2}) b->release();
  c->offsets.release();
  c->offsets2.release();
  c->stats.release();
  c->counter.release();
  c->err.release();
  c->gmap.release();
  c->bvec2.release();
  c->cnorm.release();
  for (auto* b : {&c->ch_cperm, &c->ch_first, &c->ch_ngroups, &c->ch_bmeta}) b->release();
  c->ch_a0.release();
  c->ch_bytes.release();
  c->ch_start.release();
  c->ch_off.release();
  c->ch_nbr.release();
  c->ch_groups.release();
  c->ch_perm.release();
  for (auto* b : {&c->ch_L, &c->ch_Linv, &c->ch_work}) b->release();
  c->amg_i.release();
  c->amg_d.release();
  c->amg_work.release();
  c->amg_hd.release();
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  c->aflag.release();
  for (auto& r : c->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int vqpc_set_stream(vqpc_ctx* c, void* stream) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (c->own_stream && c->stream) {
      CK(cudaStreamSynchronize(c->stream));
      CK(cudaStreamDestroy(c->stream));
    }
    c->own_stream = stream == nullptr;
    if (stream)
      c->stream = static_cast<cudaStream_t>(stream);
    else
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  });
}

int vqpc_set_exact_reductions(vqpc_ctx* c, int enable) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  c->exact = enable != 0;
  return VQPC_OK;
}

int vqpc_synchronize(vqpc_ctx* c) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] { CK(cudaStreamSynchronize(c->stream)); });
}

// (e): centroid coefficients (realise over the first m modes of the latent
// centroid chi_p, quantizer.cpp:465-476) then the per-centroid factor.
int vqpc_factor_centroids(vqpc_ctx* c) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    const vqpc_problem& pb = c->pb;
    const int P = pb.P, m = pb.m;
    // chi_p: latent sites for grids, T2(centroid) = eta / sqrt(lambda) for Scale
    std::vector<double> chi(static_cast<size_t>(P) * std::max(m, 1), 0.0);
    const bool grid = pb.method == VQPC_GRID || pb.method == VQPC_SIGN_GRID;
    for (int p = 0; p < P; ++p)
      for (int k = 0; k < m; ++k) {
        const size_t e = static_cast<size_t>(p) * m + k;
        chi[e] = grid ? pb.latent[e] : pb.centroids[e] / std::sqrt(pb.lambdas[k]);
      }
    c->xi.ensure(chi.size());
    h2d(c, c->xi.p, chi.data(), chi.size());
    const int64_t ldk = kappa_ld(c);
    c->kappa_c.ensure(static_cast<size_t>(P) * ldk);
    c->kflag.ensure(static_cast<size_t>(P) + 4);  // + 4: word-wide atomicOr flags
    CK(cudaMemsetAsync(c->kflag.p, 0, P, c->stream));
    run_realise(c, c->xi.p, P, std::max(m, 1), m, c->kappa_c.p, ldk, c->kflag.p);
    factor_coefficients(c, c->kappa_c.p, ldk, P);
    int err = 0;
    std::vector<uint8_t> flags(P);
    d2h(c, &err, c->err.p, 1);
    d2h(c, flags.data(), c->kflag.p, P);
    CK(cudaStreamSynchronize(c->stream));
    for (uint8_t f : flags) {
      if (f & 1) throw ApiError{VQPC_COEFFICIENT_OVERFLOW, "coefficient-overflow in a centroid coefficient"};
      if (f) throw ApiError{VQPC_INVALID_COEFFICIENT, "invalid-coefficient (kappa underflow) in a centroid coefficient"};
    }
    if (err) throw ApiError{VQPC_NOT_SPD, "not-spd"};
    c->factored = true;
    c->have_lu = false;  // reference-order 1-D factor values are rebuilt on first use
  });
}

int vqpc_centroid_coefficients(vqpc_ctx* c, double* kappa_out) {
  if (!c || !kappa_out) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (!c->kappa_c.p) throw ApiError{VQPC_INVALID_CONFIG, "call vqpc_factor_centroids first"};
    const int64_t ldk = kappa_ld(c);
    CK(cudaMemcpy2DAsync(kappa_out, sizeof(double) * c->pb.n_nodes, c->kappa_c.p, sizeof(double) * ldk,
                         sizeof(double) * c->pb.n_nodes, c->pb.P, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int vqpc_precond_apply(vqpc_ctx* c, int p, const double* r, double* z) {
  if (!c || !r || !z) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (!c->factored) throw ApiError{VQPC_INVALID_CONFIG, "not factored"};
    if (p < 0 || p >= c->pb.P) throw ApiError{VQPC_INVALID_ARGUMENT, "p out of range"};
    c->dvec.ensure(3 * static_cast<size_t>(c->n));
    h2d(c, c->dvec.p, r, c->n);
    if (c->amg) {
      c->dvec.ensure(5 * static_cast<size_t>(c->n) + c->amg_cv);
      h2d(c, c->dvec.p, r, c->n);
      amg_apply_kernel<<<1, AMG_T, sizeof(double) * std::max(c->amg_dense_max, 1), c->stream>>>(
          c->amg_hd.p, p, 2.0 / 3.0, c->dvec.p, c->dvec.p + c->n,
                                                   c->dvec.p + 2 * c->n, c->dvec.p + 3 * c->n, c->dvec.p + 5 * c->n);
    } else if (c->chol2d)
      cholapply_serial_kernel<<<1, 1, 0, c->stream>>>(c->ch_L.p, c->ch_ldL, c->clay, p, c->dvec.p,
                                                      c->dvec.p + 2 * c->n, c->dvec.p + c->n);
    else if (c->pb.dim == 2)
      if (c->g2.m > P2_T)
        precond2d_apply_kernel<P2_TBIG><<<1, P2_TBIG, 0, c->stream>>>(c->fac2.p, p, c->g2, c->dvec.p, c->dvec.p + c->n,
                                                                      c->dvec.p + 2 * c->n);
      else
        precond2d_apply_kernel<P2_T><<<1, P2_T, 0, c->stream>>>(c->fac2.p, p, c->g2, c->dvec.p, c->dvec.p + c->n,
                                                                c->dvec.p + 2 * c->n);
    else
      precond1d_apply_kernel<<<1, 1, 0, c->stream>>>(c->fac.p, c->NP, p, c->n, c->dvec.p, c->dvec.p + c->n);
    launch_check(c);
    d2h(c, z, c->dvec.p + c->n, c->n);
    CK(cudaStreamSynchronize(c->stream));
  });
}

// SA-AMG hierarchy of centroid p (AmgOptions::level_sizes_out, solver.hpp:42, and
// the operators, for bit-level checks against the oracle's setup)
int vqpc_amg_info(const vqpc_ctx* c, int p, int max_levels, int64_t* info, int* nlev, int* dense_n) {
  if (!c || !info || !nlev || !dense_n) return VQPC_INVALID_ARGUMENT;
  if (!c->amg || c->amg_h.empty()) return VQPC_INVALID_CONFIG;
  if (p < 0 || p >= c->pb.P) return VQPC_INVALID_ARGUMENT;
  const amg::Hierarchy& H = c->amg_h[p];
  *nlev = static_cast<int>(H.lv.size());
  *dense_n = H.dense_n;
  for (int l = 0; l < *nlev && l < max_levels; ++l) {
    info[4 * l] = H.lv[l].A.rows;
    info[4 * l + 1] = H.lv[l].A.nnz();
    info[4 * l + 2] = H.lv[l].P.nnz();
    info[4 * l + 3] = H.lv[l].P.rows ? H.lv[l].P.cols : 0;
  }
  return VQPC_OK;
}

int vqpc_amg_level(const vqpc_ctx* c, int p, int l, int* a_rp, int* a_col, double* a_val, double* inv_diag,
                   int* p_rp, int* p_col, double* p_val, double* L) {
  if (!c || !c->amg || c->amg_h.empty()) return VQPC_INVALID_CONFIG;
  if (p < 0 || p >= c->pb.P || l < 0 || l >= static_cast<int>(c->amg_h[p].lv.size())) return VQPC_INVALID_ARGUMENT;
  const amg::Hierarchy& H = c->amg_h[p];
  const amg::Level& lv = H.lv[l];
  std::copy(lv.A.ptr.begin(), lv.A.ptr.end(), a_rp);
  std::copy(lv.A.idx.begin(), lv.A.idx.end(), a_col);
  std::copy(lv.A.val.begin(), lv.A.val.end(), a_val);
  std::copy(lv.inv_diag.begin(), lv.inv_diag.end(), inv_diag);
  if (lv.P.rows) {
    std::copy(lv.P.ptr.begin(), lv.P.ptr.end(), p_rp);
    std::copy(lv.P.idx.begin(), lv.P.idx.end(), p_col);
    std::copy(lv.P.val.begin(), lv.P.val.end(), p_val);
  }
  if (L && l + 1 == static_cast<int>(H.lv.size())) std::copy(H.L.begin(), H.L.end(), L);
  return VQPC_OK;
}

int vqpc_assign_d(vqpc_ctx* c, const double* d_xi, int64_t B, int ld, int32_t* d_labels) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (ld < c->pb.m) throw ApiError{VQPC_INVALID_ARGUMENT, "ld < m"};
    const bool grid = c->pb.method == VQPC_GRID || c->pb.method == VQPC_SIGN_GRID;
    run_assign(c, d_xi, B, ld, grid ? nullptr : c->root.p, c->sites.p, c->pb.P, c->pb.m, d_labels, nullptr);
  });
}

int vqpc_assign(vqpc_ctx* c, const double* xi, int64_t B, int ld, int32_t* labels) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (ld < c->pb.m) throw ApiError{VQPC_INVALID_ARGUMENT, "ld < m"};
    c->xi.ensure(static_cast<size_t>(std::max<int64_t>(B, 1)) * ld);
    c->labels.ensure(std::max<int64_t>(B, 1));
    h2d(c, c->xi.p, xi, static_cast<size_t>(B) * ld);
    const bool grid = c->pb.method == VQPC_GRID || c->pb.method == VQPC_SIGN_GRID;
    run_assign(c, c->xi.p, B, ld, grid ? nullptr : c->root.p, c->sites.p, c->pb.P, c->pb.m, c->labels.p, nullptr);
    d2h(c, labels, c->labels.p, B);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int vqpc_bucket_d(vqpc_ctx* c, const int32_t* d_labels, int64_t B, int32_t* d_perm, int64_t* d_offsets) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] { run_bucket(c, d_labels, B, d_perm, d_offsets); });
}

int vqpc_realise(vqpc_ctx* c, const double* xi, int64_t B, int ld, int m, double* kappa_out, uint8_t* status_out) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (m < 0 || m > c->pb.n_kl) throw ApiError{VQPC_MODE_COUNT_OUT_OF_RANGE, "mode-count-out-of-range"};
    if (ld < m) throw ApiError{VQPC_INVALID_ARGUMENT, "ld < m"};
    const int64_t ldk = kappa_ld(c);
    c->xi.ensure(static_cast<size_t>(std::max<int64_t>(B, 1)) * ld);
    c->kappa.ensure(static_cast<size_t>(std::max<int64_t>(B, 1)) * ldk);
    c->kflag.ensure(static_cast<size_t>(std::max<int64_t>(B, 1)) + 4);  // + 4: word-wide atomicOr flags
    h2d(c, c->xi.p, xi, static_cast<size_t>(B) * ld);
    CK(cudaMemsetAsync(c->kflag.p, 0, std::max<int64_t>(B, 1), c->stream));
    run_realise(c, c->xi.p, B, ld, m, c->kappa.p, ldk, c->kflag.p);
    CK(cudaMemcpy2DAsync(kappa_out, sizeof(double) * c->pb.n_nodes, c->kappa.p, sizeof(double) * ldk,
                         sizeof(double) * c->pb.n_nodes, B, cudaMemcpyDeviceToHost, c->stream));
    if (status_out) {
      d2h(c, status_out, c->kflag.p, B);
      CK(cudaStreamSynchronize(c->stream));
      for (int64_t i = 0; i < B; ++i)
        status_out[i] = (status_out[i] & 1) ? VQPC_S_COEFF_OVERFLOW : status_out[i] ? VQPC_S_INVALID_COEFF : 0;
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int vqpc_solve_batch(vqpc_ctx* c, const double* xi, int64_t B, int ld, const int32_t* labels, double eps,
                     int max_iter, const int32_t* max_iter_arr, int32_t* iters, double* final_rel, uint8_t* status,
                     double* x_out) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (!(eps > 0.0) || eps >= 1.0) throw ApiError{VQPC_INVALID_TOLERANCE, "invalid-tolerance"};
    if (!c->factored) throw ApiError{VQPC_INVALID_CONFIG, "vqpc_factor_centroids must precede solves"};
    if (ld < c->pb.n_kl) throw ApiError{VQPC_INVALID_ARGUMENT, "ld < n_kl"};
    const int P = c->pb.P;
    for (int64_t i = 0; i < B; ++i)
      if (labels[i] < -1 || labels[i] >= P) throw ApiError{VQPC_INVALID_ARGUMENT, "label out of range"};
    const int64_t Bm = std::max<int64_t>(B, 1);
    const int64_t ldk = kappa_ld(c);
    c->xi.ensure(static_cast<size_t>(Bm) * ld);
    c->labels.ensure(Bm);
    c->perm.ensure(Bm);
    c->offsets.ensure(P + 2);
    c->kappa.ensure(static_cast<size_t>(Bm) * ldk);
    c->kflag.ensure(static_cast<size_t>(Bm) + 4);  // + 4: word-wide atomicOr flags
    c->iters.ensure(Bm);
    c->rel.ensure(Bm);
    c->status.ensure(Bm);
    if (x_out) c->x.ensure(static_cast<size_t>(Bm) * c->n);
    if (max_iter_arr) {
      c->mia.ensure(Bm);
      h2d(c, c->mia.p, max_iter_arr, B);
    }
    h2d(c, c->xi.p, xi, static_cast<size_t>(B) * ld);
    h2d(c, c->labels.p, labels, B);
    run_bucket(c, c->labels.p, B, c->perm.p, c->offsets.p);
    CK(cudaMemsetAsync(c->kflag.p, 0, Bm, c->stream));
    run_realise(c, c->xi.p, B, ld, c->pb.n_kl, c->kappa.p, ldk, c->kflag.p);
    run_pcg(c, c->kappa.p, ldk, c->kflag.p, c->perm.p, c->labels.p, B, 0, eps, max_iter,
            max_iter_arr ? c->mia.p : nullptr, c->iters.p, c->rel.p, c->status.p, x_out ? c->x.p : nullptr);
    d2h(c, iters, c->iters.p, B);
    d2h(c, final_rel, c->rel.p, B);
    d2h(c, status, c->status.p, B);
    if (x_out) d2h(c, x_out, c->x.p, static_cast<size_t>(B) * c->n);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int vqpc_profile(vqpc_ctx* c, int enable) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  c->prof = enable != 0;
  return VQPC_OK;
}

int vqpc_profile_read(vqpc_ctx* c, double* ms, int64_t* counts, int reset) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    CK(cudaStreamSynchronize(c->stream));
    for (auto& r : c->recs) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, r.a, r.b));
      c->prof_ms[r.kind] += t;
      c->prof_n[r.kind] += 1;
      c->pool.push_back(r.a);
      c->pool.push_back(r.b);
    }
    c->recs.clear();
    for (int k = 0; k < VQPC_NKINDS; ++k) {
      if (ms) ms[k] = c->prof_ms[k];
      if (counts) counts[k] = c->prof_n[k];
      if (reset) {
        c->prof_ms[k] = 0.0;
        c->prof_n[k] = 0;
      }
    }
  });
}

int vqpc_run_campaign_ex_d(vqpc_ctx* c, const double* d_xi, int64_t B, int ld, double eps, int max_iter,
                           int64_t chunk, int64_t solve_limit, int32_t* d_labels, int32_t* d_iters, double* d_rel,
                           uint8_t* d_status, int64_t* d_stats, int64_t* d_summary) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    campaign_device(c, d_xi, B, ld, eps, max_iter, chunk, d_labels, d_iters, d_rel, d_status, d_stats, d_summary,
                    solve_limit < 0 ? INT64_MAX : solve_limit);
  });
}

int vqpc_run_campaign_d(vqpc_ctx* c, const double* d_xi, int64_t B, int ld, double eps, int max_iter, int64_t chunk,
                        int32_t* d_labels, int32_t* d_iters, double* d_rel, uint8_t* d_status, int64_t* d_stats,
                        int64_t* d_summary) {
  return vqpc_run_campaign_ex_d(c, d_xi, B, ld, eps, max_iter, chunk, -1, d_labels, d_iters, d_rel, d_status,
                                d_stats, d_summary);
}

namespace {
int campaign_host(vqpc_ctx* c, const double* xi, int64_t B, int ld, double eps, int max_iter, int64_t chunk,
                  int64_t solve_limit, int32_t* labels, int32_t* iters, double* final_rel, uint8_t* status,
                  int64_t* stats, int64_t* summary, bool sync) {
  if (!c) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    const int P = c->pb.P;
    const int64_t Bm = std::max<int64_t>(B, 1);
    c->xi.ensure(static_cast<size_t>(Bm) * ld);
    c->labels.ensure(Bm);
    c->iters.ensure(Bm);
    c->rel.ensure(Bm);
    c->status.ensure(Bm);
    c->stats.ensure(4 * static_cast<size_t>(P) + 4);
    h2d(c, c->xi.p, xi, static_cast<size_t>(B) * ld);
    campaign_device(c, c->xi.p, B, ld, eps, max_iter, chunk, c->labels.p, c->iters.p, c->rel.p, c->status.p,
                    c->stats.p, c->stats.p + 4 * P, solve_limit < 0 ? INT64_MAX : solve_limit);
    d2h(c, labels, c->labels.p, B);
    d2h(c, iters, c->iters.p, B);
    d2h(c, final_rel, c->rel.p, B);
    d2h(c, status, c->status.p, B);
    d2h(c, stats, c->stats.p, 4 * static_cast<size_t>(P));
    d2h(c, summary, c->stats.p + 4 * P, 4);
    if (sync) CK(cudaStreamSynchronize(c->stream));
  });
}
}  // namespace

int vqpc_run_campaign_ex(vqpc_ctx* c, const double* xi, int64_t B, int ld, double eps, int max_iter, int64_t chunk,
                         int64_t solve_limit, int32_t* labels, int32_t* iters, double* final_rel, uint8_t* status,
                         int64_t* stats, int64_t* summary) {
  return campaign_host(c, xi, B, ld, eps, max_iter, chunk, solve_limit, labels, iters, final_rel, status, stats,
                       summary, true);
}

int vqpc_run_campaign_async(vqpc_ctx* c, const double* xi, int64_t B, int ld, double eps, int max_iter,
                            int64_t chunk, int64_t solve_limit, int32_t* labels, int32_t* iters, double* final_rel,
                            uint8_t* status, int64_t* stats, int64_t* summary) {
  return campaign_host(c, xi, B, ld, eps, max_iter, chunk, solve_limit, labels, iters, final_rel, status, stats,
                       summary, false);
}

// run_campaign_with plus the solutions the reference computes and discards
// (driver.cpp:236-237): x_out row i = x of realisation i (n doubles; rows of
// unsolved samples are left untouched).
int vqpc_run_campaign_x(vqpc_ctx* c, const double* xi, int64_t B, int ld, double eps, int max_iter, int64_t chunk,
                        int64_t solve_limit, int32_t* labels, int32_t* iters, double* final_rel, uint8_t* status,
                        int64_t* stats, int64_t* summary, double* x_out) {
  if (!c || !x_out) return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    const int P = c->pb.P;
    const int64_t Bm = std::max<int64_t>(B, 1);
    c->xi.ensure(static_cast<size_t>(Bm) * ld);
    c->labels.ensure(Bm);
    c->iters.ensure(Bm);
    c->rel.ensure(Bm);
    c->status.ensure(Bm);
    c->stats.ensure(4 * static_cast<size_t>(P) + 4);
    c->x.ensure(static_cast<size_t>(Bm) * c->n);
    h2d(c, c->xi.p, xi, static_cast<size_t>(B) * ld);
    h2d(c, c->x.p, x_out, static_cast<size_t>(B) * c->n);  // untouched rows keep the caller's values
    campaign_device(c, c->xi.p, B, ld, eps, max_iter, chunk, c->labels.p, c->iters.p, c->rel.p, c->status.p,
                    c->stats.p, c->stats.p + 4 * P, solve_limit < 0 ? INT64_MAX : solve_limit, c->x.p);
    d2h(c, labels, c->labels.p, B);
    d2h(c, iters, c->iters.p, B);
    d2h(c, final_rel, c->rel.p, B);
    d2h(c, status, c->status.p, B);
    d2h(c, stats, c->stats.p, 4 * static_cast<size_t>(P));
    d2h(c, summary, c->stats.p + 4 * P, 4);
    d2h(c, x_out, c->x.p, static_cast<size_t>(B) * c->n);
    CK(cudaStreamSynchronize(c->stream));
  });
}

// ideal_sweep (driver.cpp:290-340) on the device: for every m of m_list, the
// realisations are taken in chunks; each chunk's m-truncated coefficients are
// realised and factored as if they were centroids (one preconditioner per
// realisation, label i -> factor i), and the chunk's full-coefficient systems are
// solved with them by the campaign's own PCG kernels. The context's centroid
// factors are set aside for the sweep and restored after it.
int vqpc_ideal_sweep(vqpc_ctx* c, const double* xi, int64_t B, int ld, const int* m_list, int n_m, double eps,
                     int max_iter, int32_t* iters, double* final_rel, uint8_t* status) {
  if (!c || (B > 0 && (!xi || !iters || !final_rel || !status)) || n_m < 0 || (n_m > 0 && !m_list))
    return VQPC_INVALID_ARGUMENT;
  return guard(c, [&] {
    if (!(eps > 0.0) || eps >= 1.0) throw ApiError{VQPC_INVALID_TOLERANCE, "invalid-tolerance"};
    if (ld < c->pb.n_kl) throw ApiError{VQPC_INVALID_ARGUMENT, "ld < n_kl"};
    for (int im = 0; im < n_m; ++im)
      if (m_list[im] < 0 || m_list[im] > c->pb.n_kl)
        throw ApiError{VQPC_MODE_COUNT_OUT_OF_RANGE, "mode-count-out-of-range"};
    if (B <= 0 || n_m == 0) return;
    const int64_t ldk = kappa_ld(c);
    c->xi.ensure(static_cast<size_t>(B) * ld);
    h2d(c, c->xi.p, xi, static_cast<size_t>(B) * ld);
    c->kappa.ensure(static_cast<size_t>(B) * ldk);
    c->kflag.ensure(static_cast<size_t>(B) + 4);
    CK(cudaMemsetAsync(c->kflag.p, 0, B, c->stream));
    run_realise(c, c->xi.p, B, ld, c->pb.n_kl, c->kappa.p, ldk, c->kflag.p);
    // per-realisation factors: how many fit at once (1-D 2n doubles each; 2-D IC(0) 4n;
    // cholesky nnz(L); AMG a hierarchy built on the host)
    // (the cholesky kind's group builder buckets labels into pb.P bins: at most P per chunk)
    const int64_t nc = std::min<int64_t>(B, c->pb.dim == 1 ? 8192
                                            : c->chol2d  ? std::min(32, c->pb.P)
                                            : c->amg     ? 256
                                                         : 1024);
    DBuf<double> kc;
    DBuf<uint8_t> kcf;
    DBuf<int32_t> ids, d_it;
    DBuf<double> d_rel;
    DBuf<uint8_t> d_st;
    kc.ensure(static_cast<size_t>(nc) * ldk);
    kcf.ensure(static_cast<size_t>(nc) + 4);
    ids.ensure(nc);
    d_it.ensure(B);
    d_rel.ensure(B);
    d_st.ensure(B);
    iota_kernel<<<static_cast<unsigned>(ceil_div(nc, 256)), 256, 0, c->stream>>>(ids.p, nc);
    launch_check(c);
    // set the centroid factors aside
    auto swap_factors = [&](vqpc_ctx& o) {
      std::swap(c->fac, o.fac);
      std::swap(c->fac2, o.fac2);
      std::swap(c->ch_L, o.ch_L);
      std::swap(c->ch_Linv, o.ch_Linv);
      std::swap(c->amg_i, o.amg_i);
      std::swap(c->amg_d, o.amg_d);
      std::swap(c->amg_hd, o.amg_hd);
      std::swap(c->amg_h, o.amg_h);
      std::swap(c->amg_cv, o.amg_cv);
      std::swap(c->amg_entries, o.amg_entries);
      std::swap(c->amg_dense_max, o.amg_dense_max);
      std::swap(c->fac_lu, o.fac_lu);
      std::swap(c->have_lu, o.have_lu);
      std::swap(c->lu_src, o.lu_src);
      std::swap(c->lu_ld, o.lu_ld);
      std::swap(c->lu_count, o.lu_count);
    };
    vqpc_ctx saved;
    swap_factors(saved);
    auto release = [&](vqpc_ctx& o) {
      for (auto* b : {&o.fac2, &o.ch_L, &o.ch_Linv, &o.amg_d}) b->release();
      o.fac.release();
      o.fac_lu.release();
      o.amg_i.release();
      o.amg_hd.release();
    };
    std::vector<int32_t> h_it(B);
    std::vector<double> h_rel(B);
    std::vector<uint8_t> h_st(B);
    try {
      for (int im = 0; im < n_m; ++im) {
        for (int64_t c0 = 0; c0 < B; c0 += nc) {
          const int64_t nb = std::min(nc, B - c0);
          CK(cudaMemsetAsync(kcf.p, 0, nb, c->stream));
          run_realise(c, c->xi.p + c0 * ld, nb, ld, m_list[im], kc.p, ldk, kcf.p);
          std::vector<uint8_t> f(nb);
          d2h(c, f.data(), kcf.p, nb);
          CK(cudaStreamSynchronize(c->stream));
          for (uint8_t v : f)
            if (v) throw ApiError{v & 1 ? VQPC_COEFFICIENT_OVERFLOW : VQPC_INVALID_COEFFICIENT,
                                  "truncated coefficient of the ideal sweep is not finite / positive"};
          c->have_lu = false;
          factor_coefficients(c, kc.p, ldk, static_cast<int>(nb));
          run_pcg(c, c->kappa.p + c0 * ldk, ldk, c->kflag.p + c0, ids.p, ids.p, nb, c0, eps, max_iter, nullptr,
                  d_it.p, d_rel.p, d_st.p, nullptr);
        }
        d2h(c, h_it.data(), d_it.p, B);
        d2h(c, h_rel.data(), d_rel.p, B);
        d2h(c, h_st.data(), d_st.p, B);
        CK(cudaStreamSynchronize(c->stream));
        for (int64_t i = 0; i < B; ++i) {
          iters[i * n_m + im] = h_it[i];
          final_rel[i * n_m + im] = h_rel[i];
          status[i * n_m + im] = h_st[i];
        }
      }
    } catch (...) {
      release(*c);
      swap_factors(saved);
      throw;
    }
    release(*c);
    swap_factors(saved);
  });
}

int vqpc_run_campaign(vqpc_ctx* c, const double* xi, int64_t B, int ld, double eps, int max_iter, int64_t chunk,
                      int32_t* labels, int32_t* iters, double* final_rel, uint8_t* status, int64_t* stats,
                      int64_t* summary) {
  return vqpc_run_campaign_ex(c, xi, B, ld, eps, max_iter, chunk, -1, labels, iters, final_rel, status, stats,
                              summary);
}

}  // extern "C"

// Diagnostics: per-phase cycles of the 2-D PCG (setup, sweeps, P1, P2), summed
// over CTAs by thread 0; nonzero only in a -DVQPC_PHASE_TIMING build.
extern "C" int vqpc_debug_pcg1d_phase_cycles(unsigned long long* out, int reset) {
  if (!out) return VQPC_INVALID_ARGUMENT;
#ifdef VQPC_PHASE_TIMING
  if (cudaMemcpyFromSymbol(out, vqpc::g_pcg1d_phase, 4 * sizeof(unsigned long long)) != cudaSuccess)
    return VQPC_CUDA_ERROR;
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    if (cudaMemcpyToSymbol(vqpc::g_pcg1d_phase, z, sizeof(z)) != cudaSuccess) return VQPC_CUDA_ERROR;
  }
#else
  (void)reset;
  for (int i = 0; i < 4; ++i) out[i] = 0;
#endif
  return VQPC_OK;
}

extern "C" int vqpc_debug_pcg2d_phase_cycles(unsigned long long* out, int reset) {
  if (!out) return VQPC_INVALID_ARGUMENT;
#ifdef VQPC_PHASE_TIMING
  if (cudaMemcpyFromSymbol(out, vqpc::g_pcg2d_phase, 4 * sizeof(unsigned long long)) != cudaSuccess)
    return VQPC_CUDA_ERROR;
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    if (cudaMemcpyToSymbol(vqpc::g_pcg2d_phase, z, sizeof(z)) != cudaSuccess) return VQPC_CUDA_ERROR;
  }
#else
  (void)reset;
  for (int i = 0; i < 4; ++i) out[i] = 0;
#endif
  return VQPC_OK;
}
