/*
 * vqpc.h — C-ABI boundary of the B200 Monte-Carlo sample-solve path.
 *
 * Replaces, for the hot path of the reference library `vqp`
 * (/root/reference/proj), the per-sample loop of
 *   run_campaign_with   proj/src/driver.cpp:193-281 (decl. driver.hpp:93-95)
 * and the functions it calls:
 *   assign              proj/src/quantizer.cpp:134-145 (decl. quantizer.hpp:92)
 *   lift / transport    proj/src/field.cpp:113-125, 138-145 (decl. field.hpp:67,76)
 *   assemble            proj/src/fem.cpp:213-256 (decl. fem.hpp:79), matrix-free here
 *   centroid_coefficient proj/src/quantizer.cpp:465-476 (decl. quantizer.hpp:141-142)
 *   build_cholesky      proj/src/solver.cpp:80-111,163-165 (decl. solver.hpp:26)
 *   Preconditioner      proj/include/vqp/solver.hpp:13-20 (apply/kind/built_from)
 *   pcg                 proj/src/solver.cpp:186-245 (decl. solver.hpp:75-76)
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *  - Every function returns an int status (0 = OK, see vqpc_code); no
 *    exception crosses the ABI. The codes map 1:1 onto the reference's
 *    vqp::Error strings (proj/include/vqp/error.hpp); vqpc_error_string()
 *    returns that string and vqpc_last_error() the context's last message.
 *  - Pointers are HOST memory unless the parameter name starts with d_
 *    (device memory on the context's device). Host arrays are borrowed for the
 *    duration of the call only; all device buffers created by a context are
 *    owned by it and released by vqpc_ctx_destroy().
 *  - Per-sample failures are status bytes (vqpc_sample_status), not call
 *    failures: the batch always completes (the reference aborts the process
 *    on pcg-breakdown inside a worker thread).
 *  - One context per CUDA stream; calls on one context are not re-entrant.
 *    Results are independent of chunk size, bucket order and grid size.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns VQPC_NO_DEVICE.
 */
#ifndef VQPC_H_
#define VQPC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (vqp::Error code strings) ------------------------------ */
enum vqpc_code {
  VQPC_OK = 0,
  VQPC_INVALID_LATENT = 1,          /* "invalid-latent"          quantizer.cpp:135-138 */
  VQPC_INVALID_COEFFICIENT = 2,     /* "invalid-coefficient"     fem.cpp:216-219 */
  VQPC_COEFFICIENT_OVERFLOW = 3,    /* "coefficient-overflow"    field.cpp:141-142 */
  VQPC_NOT_SPD = 4,                 /* "not-spd"                 solver.cpp:96 */
  VQPC_PCG_BREAKDOWN = 5,           /* "pcg-breakdown"           solver.cpp:207,214,238 */
  VQPC_INVALID_TOLERANCE = 6,       /* "invalid-tolerance"       solver.cpp:190 */
  VQPC_MODE_COUNT_OUT_OF_RANGE = 7, /* "mode-count-out-of-range" driver.cpp:179 */
  VQPC_INVALID_CODEBOOK = 8,        /* "invalid-codebook"        quantizer.cpp:95-109 */
  VQPC_INSUFFICIENT_SAMPLES = 9,    /* "insufficient-samples"    quantizer.cpp:200,351 */
  VQPC_INVALID_CONFIG = 10,         /* "invalid-config"          driver.cpp:36-41 */
  VQPC_INVALID_ARGUMENT = 11,
  VQPC_CUDA_ERROR = 20,
  VQPC_NO_DEVICE = 21,
  VQPC_OUT_OF_MEMORY = 22,
};

/* per-sample status (SURVEY Appendix B classes) */
enum vqpc_sample_status {
  VQPC_S_CONVERGED = 0,         /* rel < eps (solver.cpp:231-234) */
  VQPC_S_MAX_ITER = 1,          /* loop exhausted, converged=false */
  VQPC_S_BREAKDOWN = 2,         /* where the reference throws "pcg-breakdown" */
  VQPC_S_COEFF_OVERFLOW = 3,    /* transport produced a non-finite kappa */
  VQPC_S_INVALID_LATENT = 4,    /* non-finite xi */
  VQPC_S_INVALID_COEFF = 5,
  VQPC_S_NOT_SOLVED = 6,        /* realised + assigned only (beyond solve_limit) */
};

enum vqpc_method { VQPC_KMEANS = 0, VQPC_CLVQ = 1, VQPC_GRID = 2, VQPC_SIGN_GRID = 3 };
enum vqpc_map { VQPC_SCALE = 0, VQPC_CDF = 1 };
/* preconditioner kinds: the reference's PrecondKind (driver.hpp:13) numbering where
 * one exists (cholesky, amg); IC(0) is new. IDENTITY and block
 * Jacobi have no GPU implementation (invalid-config). */
enum vqpc_precond { VQPC_PC_IDENTITY = 0, VQPC_PC_CHOLESKY = 1, VQPC_PC_AMG = 3, VQPC_PC_IC0 = 4 };

/* Everything a campaign needs besides its xi draws (CampaignArtifacts,
 * driver.hpp:77-81, plus the CampaignConfig fields the solve uses). */
typedef struct vqpc_problem {
  int dim;                    /* 1: N-element 1-D model; 2: r x r structured mesh */
  int size;                   /* N (dim 1) or r (dim 2) */
  int n_kl;                   /* modes in the basis (KLBasis::n_kl) */
  int n_nodes;                /* field points: N (dim 1) or (r+1)^2 (dim 2) */
  const double* eigenvalues;  /* n_kl, nonincreasing                  (field.hpp:24) */
  const double* eigenvectors; /* n_kl x n_nodes, mode-major          (field.hpp:25) */
  int method;                 /* vqpc_method */
  int map;                    /* vqpc_map (T2Map::kind) */
  int P;                      /* centroids */
  int m;                      /* stochastic dimension d */
  const double* lambdas;      /* m: T2Map::lambdas                    (quantizer.hpp:33-35) */
  const double* centroids;    /* P x m, quantization space            (quantizer.hpp:74) */
  const double* latent;       /* P x m latent sites (grids), else NULL (quantizer.hpp:75) */
  int precond;                /* vqpc_precond */
  int device;                 /* CUDA ordinal */
} vqpc_problem;

typedef struct vqpc_ctx vqpc_ctx;

/* ---- context ------------------------------------------------------------- */
int vqpc_ctx_create(const vqpc_problem* problem, vqpc_ctx** out);
void vqpc_ctx_destroy(vqpc_ctx* ctx);
const char* vqpc_last_error(const vqpc_ctx* ctx);
const char* vqpc_error_string(int code);
/* Run all work of this context on an existing cudaStream_t (NULL: own stream). */
int vqpc_set_stream(vqpc_ctx* ctx, void* cuda_stream);
int vqpc_synchronize(vqpc_ctx* ctx);
/* Reference-order mode (parity instrument). enable != 0: every dot product is
 * summed serially in natural order (solver.cpp:176-180); in 1-D the solve also
 * runs Eigen's LL^T triangular solves on the reversed order (solver.cpp:98-110)
 * and the unfused vector updates (solver.cpp:224-241) on one thread per sample
 * (pcg1d_exact_kernel, ~0.5 ms per iteration at n = 4095). Either way the solve
 * is bit-identical to the reference arithmetic given the same coefficient bits.
 * Default 0 = the throughput kernels (block-tree reductions, chunked scans). */
int vqpc_set_exact_reductions(vqpc_ctx* ctx, int enable);
/* unknowns per sample system (n) and the number of device kernel launches
 * issued by this context so far (bench evidence). */
int vqpc_unknowns(const vqpc_ctx* ctx);
/* stored entries of one centroid's factor: 1-D tridiagonal 2n - 1, 2-D IC(0) 3n
 * (D, a_W, a_S), 2-D cholesky the RCM envelope of L (roofline accounting). */
int64_t vqpc_factor_entries(const vqpc_ctx* ctx);
int64_t vqpc_launch_count(const vqpc_ctx* ctx);

/* ---- (e) centroid factors: centroid_coefficient -> assemble -> build_cholesky
 * for every p (driver.cpp:212-219). Must precede any solve. --------------- */
int vqpc_factor_centroids(vqpc_ctx* ctx);
/* centroid coefficients kappa_p (P x n_nodes), for parity tests */
int vqpc_centroid_coefficients(vqpc_ctx* ctx, double* kappa_out);
/* Apply M_p^{-1} to r (n) -> z (n) for one centroid (Preconditioner::apply). */
int vqpc_precond_apply(vqpc_ctx* ctx, int p, const double* r, double* z);

/* ---- SA-AMG kind (VQPC_PC_AMG, 2-D): the hierarchy of centroid p built by
 * vqpc_factor_centroids (AmgPreconditioner ctor, amg.cpp:132-197). info[4l..4l+3]
 * = rows, nnz(A_l), nnz(P_l), columns of P_l; *dense_n = size of the coarsest
 * dense factor (0: smoother-only bottom). vqpc_amg_level copies level l's CSR
 * operator, its inverse diagonal, its prolongator (CSR, none on the coarsest) and,
 * on the coarsest level, the dense lower factor (row-major, nullable). */
int vqpc_amg_info(const vqpc_ctx* ctx, int p, int max_levels, int64_t* info, int* nlev, int* dense_n);
int vqpc_amg_level(const vqpc_ctx* ctx, int p, int l, int* a_rp, int* a_col, double* a_val, double* inv_diag,
                   int* p_rp, int* p_col, double* p_val, double* L);

/* ---- (b) assignment: labels[i] = assign(codebook, xi_i[0:m]) ------------- */
int vqpc_assign(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, int32_t* labels);
int vqpc_assign_d(vqpc_ctx* ctx, const double* d_xi, int64_t B, int ld, int32_t* d_labels);

/* ---- (c) bucketing: stable counting sort of sample ids by label; offsets
 * has P+1 entries (group p = perm[offsets[p] .. offsets[p+1])). ----------- */
int vqpc_bucket_d(vqpc_ctx* ctx, const int32_t* d_labels, int64_t B, int32_t* d_perm, int64_t* d_offsets);

/* ---- (a) realisation: kappa_i = transport(lift(basis, xi_i[0:m])) --------
 * status_out[i] (nullable): 0, VQPC_S_COEFF_OVERFLOW (a non-finite kappa:
 * transport's coefficient-overflow, field.cpp:141-142) or VQPC_S_INVALID_COEFF
 * (kappa == 0 after exp underflow: assembly's invalid-coefficient). */
int vqpc_realise(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, int m, double* kappa_out,
                 uint8_t* status_out);

/* ---- (d) batched PCG with labels given: per-sample J, final relative
 * residual and status; x_out (B x n, nullable). max_iter < 0 -> 10 n;
 * max_iter_arr (nullable) overrides it per sample (fixed-K parity runs). --- */
int vqpc_solve_batch(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, const int32_t* labels,
                     double eps, int max_iter, const int32_t* max_iter_arr, int32_t* iters,
                     double* final_rel, uint8_t* status, double* x_out);

/* ---- the whole hot path: run_campaign_with (driver.cpp:193-281) ----------
 * xi: B x ld rows (ld >= n_kl; all n_kl modes are lifted). Fills per-sample
 * labels / iters / final_rel / status, per-centroid stats (4P int64:
 * n_p | sum_j | conv_count | conv_sum) and summary (4 int64: total
 * iterations, unconverged, converged count, converged J sum).
 * chunk <= 0 -> one chunk. Host variant: xi and outputs in host memory,
 * copies included. Device variant: all pointers device-resident. -------- */
int vqpc_run_campaign(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, double eps, int max_iter,
                      int64_t chunk, int32_t* labels, int32_t* iters, double* final_rel, uint8_t* status,
                      int64_t* stats, int64_t* summary);
int vqpc_run_campaign_d(vqpc_ctx* ctx, const double* d_xi, int64_t B, int ld, double eps, int max_iter,
                        int64_t chunk, int32_t* d_labels, int32_t* d_iters, double* d_final_rel,
                        uint8_t* d_status, int64_t* d_stats, int64_t* d_summary);
/* Same, realising and assigning all B samples but solving only those with
 * index < solve_limit (BASELINE C5: 2^20 realised/assigned, 2^16 solved);
 * the others get status VQPC_S_NOT_SOLVED and are excluded from the stats. */
int vqpc_run_campaign_ex(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, double eps, int max_iter,
                         int64_t chunk, int64_t solve_limit, int32_t* labels, int32_t* iters,
                         double* final_rel, uint8_t* status, int64_t* stats, int64_t* summary);
int vqpc_run_campaign_ex_d(vqpc_ctx* ctx, const double* d_xi, int64_t B, int ld, double eps, int max_iter,
                           int64_t chunk, int64_t solve_limit, int32_t* d_labels, int32_t* d_iters,
                           double* d_final_rel, uint8_t* d_status, int64_t* d_stats, int64_t* d_summary);

/* Same as vqpc_run_campaign_ex without the final synchronisation: every copy and
 * kernel is enqueued on the context's stream and the call returns; the host
 * buffers (xi in, results out) must stay valid until vqpc_synchronize(ctx). With
 * pinned host buffers the copies overlap other work, so a caller alternating two
 * contexts pipelines consecutive batches (one batch's kernels start on the SMs the
 * previous batch's work-queue tail frees). Errors raised while enqueueing are
 * returned; asynchronous ones surface at vqpc_synchronize. */
int vqpc_run_campaign_async(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, double eps, int max_iter,
                            int64_t chunk, int64_t solve_limit, int32_t* labels, int32_t* iters,
                            double* final_rel, uint8_t* status, int64_t* stats, int64_t* summary);

/* Same as vqpc_run_campaign_ex, also returning the solutions the reference
 * computes and discards (driver.cpp:236-237, SURVEY §8b "run_campaign_with_
 * solutions"): x_out is B x n host memory; row i receives x of realisation i
 * (rows of samples that are not solved keep their input values). */
int vqpc_run_campaign_x(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, double eps, int max_iter,
                        int64_t chunk, int64_t solve_limit, int32_t* labels, int32_t* iters,
                        double* final_rel, uint8_t* status, int64_t* stats, int64_t* summary, double* x_out);

/* ---- ideal sweep (driver.cpp:290-340): for every realisation i (xi: B x ld host
 * rows, all n_kl modes lifted for the system) and every m of m_list, the
 * preconditioner of the context's kind built from the m-truncated coefficient
 * transport(lift(basis, xi_i[0:m])) and applied to the full-coefficient system.
 * Records are B x n_m row-major (record of (i, m_list[j]) at i * n_m + j); the
 * rows {m, relative energy, mean J over converged records} follow on the host.
 * The context's centroid factors are kept (set aside during the sweep). ----- */
int vqpc_ideal_sweep(vqpc_ctx* ctx, const double* xi, int64_t B, int ld, const int* m_list, int n_m, double eps,
                     int max_iter, int32_t* iters, double* final_rel, uint8_t* status);

/* ---- per-kernel device timing (CUDA events on the context's stream) ------
 * enable != 0 brackets every kernel launch with events; vqpc_profile_read
 * synchronises and returns, per kernel kind, the accumulated milliseconds and
 * launch counts (arrays of VQPC_NKINDS), optionally resetting them. */
enum vqpc_kernel_kind {
  VQPC_K_ASSIGN = 0, VQPC_K_BUCKET = 1, VQPC_K_REALISE = 2, VQPC_K_PCG = 3, VQPC_K_OTHER = 4, VQPC_NKINDS = 5
};
int vqpc_profile(vqpc_ctx* ctx, int enable);
int vqpc_profile_read(vqpc_ctx* ctx, double* ms, int64_t* counts, int reset);

/* fp64 roofline probe: a DFMA-throughput kernel on the given device; returns
 * the achieved fp64 TFLOP/s (2 flops per FMA) measured with CUDA events. */
int vqpc_fp64_peak(int device, double* tflops);

/* Diagnostics: cycles spent by the 2-D PCG in setup, IC(0) sweeps, P1 and P2,
 * summed over CTAs (all zero unless the library was built with
 * -DVQPC_PHASE_TIMING). */
int vqpc_debug_pcg2d_phase_cycles(unsigned long long* out4, int reset);
/* Same for the 1-D PCG: cycles between its four per-iteration barriers (CTA
 * thread 0 of every sample, summed). */
int vqpc_debug_pcg1d_phase_cycles(unsigned long long* out4, int reset);

/* ---- quantizer construction on the host with device assignment sweeps ----
 * kmeans = minmax seeding + Lloyd (quantizer.cpp:181-357), bit-identical to
 * the reference (labels and distances are exact; means are summed on the
 * host in sample order). samples: n x m latent draws. */
int vqpc_kmeans(int device, const double* samples, int n, int m, const double* lambdas, int map, int P,
                uint64_t init_seed, int max_iter, double rel_tol, double* centroids_out,
                double* history_out, int* n_history);

/* ---- KL basis on the device: build_kl_basis (field.cpp:22-82) by Lanczos with
 * full reorthogonalisation on the lumped-Galerkin operator W = M^1/2 C M^1/2,
 * applied matrix-free (1-D: element midpoints, weights h; 2-D: the structured
 * (size+1)^2 node grid with the Kronecker factorisation of the squared-exponential
 * kernel). Keeps the n_kl dominant modes above the reference's degeneracy cutoff
 * 1e-12 lambda_1 (cutoff != 0; else all positive ones), Phi = v / sqrt(mass),
 * first entry of largest magnitude positive. Outputs: eigenvalues (n_kl,
 * descending), eigenvectors (n_kl x n_nodes, mode-major), mass (n_nodes,
 * nullable); *kept = modes kept. */
int vqpc_kl_basis(int device, int dim, int size, double sigma2, double ell, int n_kl, int cutoff,
                  double* eigenvalues_out, double* eigenvectors_out, double* mass_out, int* kept);

/* ---- coefficient sampling (rng.hpp:14-31, rng.cpp:7-12) on the host -------
 * out[i*m+k] = gaussian_draw(seed, index0 + i, k). */
int vqpc_draw_standard_normal(int64_t n, int m, uint64_t seed, int64_t index0, double* out, int threads);
uint64_t vqpc_counter_hash(uint64_t seed, uint64_t index, uint64_t component);
double vqpc_normal_quantile(double p);

#ifdef __cplusplus
}
#endif

#endif /* VQPC_H_ */
