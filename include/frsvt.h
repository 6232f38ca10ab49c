/*
 * frsvt.h — C ABI of libfrsvt, the B200 (sm_100a) hot path of
 * "Fast Randomized Singular Value Thresholding for Low-rank Optimization"
 * (Oh, Matsushita, Tai, Kweon; arXiv 1509.00296). Citations "P:n" are lines of
 * the paper text; "S:n" lines of SPEC.md; readings Zn / Rn are
 * listed in DESIGN.md.
 *
 * Layout. Every matrix is COLUMN-MAJOR with an explicit leading dimension.
 * A matrix argument is a DEVICE pointer unless the comment says "host".
 * Element type is double (FRSVT_F64) or float (FRSVT_F32), fixed per handle.
 * A multi-GPU run row-shards every m-row operand: rank k owns rows
 * [row0, row0 + m_local) of the m_global x n matrix.
 *
 * Ownership. The caller owns A, X, D, E, the ALM operand and L and never
 * hands them over; the library never frees or reallocates them. The handle
 * owns Omega, every workspace, the carried basis Q~ and the NCCL communicator.
 * All handle memory is allocated in frsvt_create; no apply/step call
 * allocates, so one call is CUDA-graph capturable.
 *
 * Asynchrony. Work is enqueued on the handle's stream; calls return before it
 * completes unless a host output (info, rel_resid, get_* hooks) is requested,
 * which synchronises that stream. One handle per host thread.
 *
 * Errors. Arguments are validated before anything is enqueued; an invalid
 * call returns FRSVT_EINVAL and enqueues nothing. Numerical rank deficiency
 * is NOT an error: it is absorbed by truncation (info.s < l), the rank reveal
 * of QR-CP. A non-finite Gram diagonal sets FRSVT_FLAG_NONFINITE
 * (status FRSVT_ENONFINITE at the next synchronising call); a Jacobi solve that
 * hits its sweep cap sets FRSVT_FLAG_NOCONV (X is still written). CUDA / NCCL
 * failures map to FRSVT_ECUDA / FRSVT_ENCCL. No C++ exception crosses the ABI.
 */
#ifndef FRSVT_H
#define FRSVT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRSVT_LMAX 128  /* largest sketch width l supported */

typedef enum {
  FRSVT_OK = 0,
  FRSVT_EINVAL = 1,
  FRSVT_ENOCONV = 2,
  FRSVT_ECUDA = 3,
  FRSVT_ENCCL = 4,
  FRSVT_ENONFINITE = 5,
  FRSVT_ENOMEM = 6
} frsvt_status;

typedef enum { FRSVT_F32 = 0, FRSVT_F64 = 1 } frsvt_dtype;

#define FRSVT_LOOPBACK_MAX 8  /* ranks of a loopback group */

/* Loopback process group (see frsvt_loopback_create). */
typedef struct frsvt_group frsvt_group;

/* info.flags bits */
#define FRSVT_FLAG_NONFINITE 1
#define FRSVT_FLAG_NOCONV 2
#define FRSVT_FLAG_NONMONOTONE_W 4
#define FRSVT_FLAG_SINGLE_CTA 8   /* informational: frsvt_apply ran on the single-CTA path */

typedef struct {
  int32_t dtype;            /* frsvt_dtype */
  int64_t m_local;          /* rows held by this rank (>= 1) */
  int64_t n;                /* columns (>= 1) */
  int64_t m_global;         /* rows of the whole matrix (== m_local if nranks == 1) */
  int64_t row0;             /* first global row of this rank */
  int32_t l;                /* sketch width l = k + p (BASELINE "k", reading Z1), 1 <= l <= min(m_global, n, FRSVT_LMAX) */
  int32_t q;                /* power iterations eta >= 0 (reading Z2) */
  int32_t range_propagation;/* 1: carry Q~ between calls and draw only p = l - r fresh columns */
  uint64_t seed;            /* Omega of call c = Philox4x32-10(key = seed, stream 1000 + c) + Box-Muller */
  int32_t nranks;           /* 1 for a single GPU */
  int32_t rank;             /* 0 .. nranks-1 */
  const unsigned char* nccl_id; /* host, 128 bytes from frsvt_get_unique_id on rank 0; NULL if nranks == 1 */
  uint32_t options;         /* FRSVT_OPT_* bits (0 = defaults) */
  frsvt_group* group;       /* nranks > 1 without NCCL: the loopback group all ranks share (nccl_id ignored); NULL otherwise */
} frsvt_config;

/* frsvt_config.options bits */
#define FRSVT_OPT_FUSED_SKETCH 1u /* rpca_alm_step: form the next call's fresh sketch in the fused
                                     epilogue (see rpca_alm_step); fp32, range propagation, one rank */
#define FRSVT_OPT_TF32_OMEGA 2u   /* fp32 handles: every drawn Omega entry is rounded to tf32 (round to
                                     nearest, ties away: the fp32 draw with its low 13 mantissa bits
                                     cleared after adding 0x1000), so the tensor-core sketch multiplies
                                     A by Omega exactly. A
                                     different test matrix, not a different method: the oracle takes
                                     the same rounded Omega (synth.omega(..., tf32=True)). Omega set by
                                     frsvt_set_omega is used as given. EINVAL on fp64 handles. */

/* Host-side report of one call (filling it synchronises the stream). */
typedef struct {
  int32_t s;                /* basis width after rank reveal (s = min(l, rank)) */
  int32_t r;                /* kept rank #{d_i > 0} = width of the carried Q~ */
  int32_t flags;            /* FRSVT_FLAG_* */
  int32_t sweeps;           /* Jacobi sweeps of the small SVD */
  int64_t calls;            /* Omega call counter after this call */
  double sigma[FRSVT_LMAX]; /* singular values of B = Q^T A, descending (first s valid) */
  double d[FRSVT_LMAX];     /* shrunk values max(sigma_i - t_i, 0) */
  double mu;                /* rpca: mu used by the last step */
  int32_t l_next;           /* sketch width of the next call (adaptive rank prediction; l otherwise) */
  int32_t pad_;
  double varsigma;          /* Prop. 4 estimate of the sketch's residual sigma:
                               20 sqrt(2/pi) ||(I - QQ^T) y||, y the last fresh sample, Q the
                               basis before it; >= sigma_{k+1}(A) with probability >= 95%.
                               Reported by the tensor-core (fp32) path; 0 elsewhere. */
} frsvt_info;

typedef struct frsvt_handle frsvt_handle;

/* Batched FRSVT of `batch` independent small fp32 matrices (SURVEY.md §8(f)
 * NEXT-3; WNNM patch groups P:23/P:48, per-window problems P:643): one CTA per
 * matrix runs Algorithm 1 (no range propagation) in shared memory; one
 * launch, no handle. Matrix b is A + b strideA (m x n, column-major, leading
 * dim lda), its result X + b strideX (ldx); all device pointers. Omega: n x l
 * (ldo), shared by the batch. 1 <= l <= min(16, m, n), 0 <= q <= 16, and
 * 8 ((m + n) l + l^2 + 192) + 4 m n bytes of shared memory <= 227 KB.
 * wmode 0: t_i = tau, or tau_batch[b] (device, nullable); wmode 1: t_i = w[i]
 * (device, l values, by descending rank position). Outputs (device,
 * nullable): r_out[b] kept rank, sigma_out[b l + i] singular values of
 * B = Q^T A, descending. Enqueued on cuda_stream; returns before completion. */
frsvt_status frsvt_batched_apply(int32_t batch, int64_t m, int64_t n, int32_t l, int32_t q, const float* A,
                                 int64_t lda, int64_t strideA, const float* Omega, int64_t ldo, int32_t wmode,
                                 double tau, const double* tau_batch, const double* w, float* X, int64_t ldx,
                                 int64_t strideX, int32_t* r_out, double* sigma_out, void* cuda_stream);
/* The same for fp64 matrices (products, orthonormalisation and the small SVD
 * in fp64): 8 ((m + n) l + l^2 + 192) + 8 m n bytes of shared memory
 * <= 227 KB (e.g. BASELINE c1's 200 x 100, l = 10). */
frsvt_status frsvt_batched_apply_f64(int32_t batch, int64_t m, int64_t n, int32_t l, int32_t q, const double* A,
                                     int64_t lda, int64_t strideA, const double* Omega, int64_t ldo, int32_t wmode,
                                     double tau, const double* tau_batch, const double* w, double* X, int64_t ldx,
                                     int64_t strideX, int32_t* r_out, double* sigma_out, void* cuda_stream);

/* Loopback process group of `nranks` (2..FRSVT_LOOPBACK_MAX) virtual ranks:
 * the row-sharded path on ONE device and in ONE process,
 * each rank a handle created with cfg.group = this group, driven by its own
 * host thread and CUDA stream. Every all-reduce point of the path becomes a
 * host rendezvous: the last rank to arrive enqueues one kernel that sums (or
 * takes max/min over) all ranks' buffers in rank order and writes the result
 * into each of them; every rank's stream is ordered after it with events. No
 * kernel waits on another kernel. Collective calls (create, apply, step)
 * must be issued by all ranks in the same order. Not CUDA-graph capturable.
 * The caller destroys the group after every handle that uses it. */
frsvt_status frsvt_loopback_create(int32_t nranks, frsvt_group** out);
void frsvt_loopback_destroy(frsvt_group* g);

/* 128-byte NCCL unique id (rank 0 only); the caller broadcasts it, e.g. with
 * torch.distributed, and passes it to frsvt_create on every rank. */
frsvt_status frsvt_get_unique_id(unsigned char out[128]);

/* Validate cfg, allocate every workspace for width l on the current device,
 * bind the work to `cuda_stream` (a cudaStream_t, NULL = legacy default),
 * and initialise NCCL when nranks > 1 (collective over the ranks: the
 * m_local-dependent route of the orthonormalisation is agreed there, so every
 * rank takes the same one). *out is NULL on failure.
 * Multi-rank fp32 handles additionally require, on every call, a 16-byte
 * aligned operand with leading dimension % 4 == 0 (the tensor-core route must
 * be the same on all ranks); otherwise the call returns FRSVT_EINVAL. */
frsvt_status frsvt_create(const frsvt_config* cfg, void* cuda_stream, frsvt_handle** out);
void frsvt_destroy(frsvt_handle* h);
const char* frsvt_status_string(frsvt_status s);

/* X <- FRSVT_tau(A): Algorithm 1, Eq. (6), with the
 * singular value thresholding of Definition 1:
 *   sketch Y = A Omega (RP: Y = [Q~ | A Omega_p]), q power steps
 *   Q <- orth(A orth(A^T Q)), B = Q^T A, small SVD of B, shrink, compose.
 * A: m_local x n, leading dim lda >= m_local. X: m_local x n, ldx >= m_local,
 * may alias A (every read of A completes before X is written).
 * tau >= 0 finite. info: host, nullable (non-NULL synchronises).
 * A call small enough for one SM (no range propagation, one rank, l <= 16,
 * m, n <= 1024 and A plus the small blocks within 227 KB of shared memory,
 * e.g. BASELINE c1: 200 x 100 fp64) runs as ONE kernel launch (the
 * batched design below with batch 1; info.flags has FRSVT_FLAG_SINGLE_CTA);
 * explicit-weight calls of frsvt_apply_weighted take the same route. */
frsvt_status frsvt_apply(frsvt_handle* h, const void* A, int64_t lda, double tau,
                         void* X, int64_t ldx, frsvt_info* info);

/* Weighted SVT (WNNM's WSVT, footnote 1 P:48): per-index thresholds t_i on
 * sigma_i sorted descending.
 *   wmode 0 (explicit)     : t_i = w[i], w host array of l values >= 0
 *   wmode 1 (reciprocal)   : t_i = C / (sigma_i + eps) on this call's sigma
 *   wmode 2 (reweighted)   : t_i = C / (d_i^prev + eps), d^prev the shrunk
 *                            values of the handle's previous call (zeros past
 *                            its rank); the first call falls back to mode 1.
 * Non-monotone t is applied mechanically and flagged NONMONOTONE_W. */
frsvt_status frsvt_apply_weighted(frsvt_handle* h, const void* A, int64_t lda,
                                  int32_t wmode, const double* w, double C, double eps,
                                  void* X, int64_t ldx, frsvt_info* info);

/* Inexact-ALM Robust PCA step hosting FRSVT (order and constants of
 * S:449/S:471, reading Z9), with the stored operand A_k = D - E_{k+1} + Y_k/mu_k
 * so Y is never materialised (Y_{k+1} = mu_k (A_k - L_{k+1})):
 *   L_{k+1} = FRSVT_{1/mu_k}(A_k)             (no m x n write of L)
 *   resid_k = ||D - L_{k+1} - E_{k+1}||_F / ||D||_F
 *   mu_{k+1} = min(rho mu_k, mu_bar)
 *   E_{k+2} = S_{lambda/mu_{k+1}}(D - L_{k+1} + Y_{k+1}/mu_{k+1})
 *   A_{k+1} = D - E_{k+2} + Y_{k+1}/mu_{k+1}
 * all in ONE fused epilogue pass over D, A, E (reads D, A, E; writes A, E).
 * iter == 0 first runs the init: ||D||_2 (norm2_D, else a device block power
 * estimate), ||D||_inf, Y_0 = D / max(||D||_2, ||D||_inf / lambda),
 * mu_0 (mu0, else 1.25/||D||_2), E_1, A_1. finalize != 0 writes L_{k+1} into
 * st->L and leaves D, E, A, mu untouched (the textbook state after k+1 steps).
 * D, E, A, L: m_local x n, leading dim ld. rel_resid: host, nullable (syncs).
 * Fused next sketch (opt-in, FRSVT_OPT_FUSED_SKETCH; fp32 tensor path, range
 * propagation, one rank): when p = l - r <= 24 the epilogue also forms the next call's
 * fresh sketch A_{k+1} Omega_p and the next step skips that
 * pass. The contents of A (library-managed) must therefore not be changed by
 * the caller between consecutive steps unless a state setter runs in between
 * (frsvt_set_carry / _reset_carry / _set_omega / _set_call_index, rpca_set_mu,
 * any frsvt_apply*), each of which discards the fused sketch. */
typedef struct {
  const void* D;     /* observation */
  void* E;           /* sparse part; holds E_{k+1} on entry of step k */
  void* A;           /* ALM operand A_k (library-managed contents) */
  void* L;           /* low-rank output, written only when finalize != 0 */
  int64_t ld;
  double lambda;     /* <= 0 -> 1/sqrt(max(m_global, n)) */
  double rho;        /* mu growth factor (> 1) */
  double mu_max_factor; /* mu_bar = mu_max_factor * mu_0 (reading Z9: 1e7) */
  double norm2_D;    /* > 0 supplied ||D||_2; 0 -> estimated on device at iter 0 */
  double mu0;        /* > 0 supplied mu_0; 0 -> 1.25 / ||D||_2 */
  int32_t iter;      /* in/out: k; incremented by every non-finalize step */
  int32_t keep;      /* >= 0: partial SVT, the first `keep` singular values are not thresholded
                        (Type B truncated nuclear norm: argmin sum_{i>keep} sigma_i(L) + lambda ||S||_1);
                        0 = the nuclear norm (standard RPCA) */
  int32_t transfer;  /* 1: the init (iter == 0) keeps the handle's carried basis Q~ (range propagation
                        handles): the basis transfer between semi-online windows; 0: fresh */
} rpca_state;

frsvt_status rpca_alm_step(frsvt_handle* h, rpca_state* st, int32_t finalize, double* rel_resid);

/* ---- test / parity hooks (host outputs synchronise) ----------------------- */
/* Next call uses this n x l Omega (device, leading dim ldo) instead of Philox. */
frsvt_status frsvt_set_omega(frsvt_handle* h, const void* Omega, int64_t ldo);
/* Write the handle's Philox Omega of call `call` (n x l) to `out` (device). */
frsvt_status frsvt_draw_omega(frsvt_handle* h, int64_t call, void* out, int64_t ldo);
/* Carried basis Q~ (m_local x l, columns >= r zero) and its width r. */
frsvt_status frsvt_get_carry(frsvt_handle* h, void* Qt, int64_t ldq, int32_t* r);
frsvt_status frsvt_set_carry(frsvt_handle* h, const void* Qt, int64_t ldq, int32_t r);
frsvt_status frsvt_reset_carry(frsvt_handle* h);
/* Adaptive rank prediction (AP, §2.3, Eq. (7)): after a
 * call with sketch width l_i and kept rank r_i, the next call uses
 * l_{i+1} = min(r_i + p_{i+1}, b), p_{i+1} = a if r_i < l_i else p_jump
 * (= ceil(rho n)); with range propagation it draws l_{i+1} - r_i fresh columns
 * behind the r_i carried ones. Kept on the device (no host synchronisation;
 * the handle's buffers stay sized for l: the inactive columns are zero and
 * dropped by the rank reveal). l_0 = l0 after this call, after
 * frsvt_reset_carry and at the init of every rpca solve. 1 <= b <= l,
 * 1 <= l0 <= b, a, p_jump >= 1; a == 0 switches AP off. Synchronises. */
frsvt_status frsvt_set_adaptive_rank(frsvt_handle* h, int32_t a, int32_t p_jump, int32_t b, int32_t l0);
/* Set the Omega call counter (the next call draws Omega of call `call`). */
frsvt_status frsvt_set_call_index(frsvt_handle* h, int64_t call);
/* Last call's report (synchronises). */
frsvt_status frsvt_get_info(frsvt_handle* h, frsvt_info* info);
/* rpca: device mu (host copy) and set it (teacher forcing). */
frsvt_status rpca_get_mu(frsvt_handle* h, double* mu);
frsvt_status rpca_set_mu(frsvt_handle* h, double mu, double mu_bar);
/* Number of kernels this handle has launched since creation (host counter). */
int64_t frsvt_kernel_launches(const frsvt_handle* h);

/* Test hook: one streaming pass on a chosen route (synchronises).
 * kind 0: out (m_local x l, ld m_local) = A (m_local x n) * B (n x l, ld n)
 * kind 1: out (n x l, ld n) = A^T * B (m_local x l, ld m_local), summed over ranks
 * impl 0 = SIMT CUDA cores; 2 = the CTA-pair stream-K tcgen05 pass of the
 * product path, exact (fp32-level products); 3 = the same pass with the
 * tf32-rounded B, i.e. out = A * rna_tf32(B) (the span-only passes, DESIGN
 * reading R17). 2 and 3 need an fp32 handle, lda % 4 == 0 and a 16-byte
 * aligned A, else FRSVT_EINVAL. */
frsvt_status frsvt_debug_pass(frsvt_handle* h, int32_t kind, int32_t impl, const void* A, int64_t lda,
                              const void* B, void* out);
/* Same pass `reps` times back to back on the handle's stream (no host sync
 * in between), *ms = mean device time per pass (CUDA events). impl as above,
 * plus 8..263: impl 2 with parts of its pipeline switched off (bit field
 * impl - 8, see tc_pass3.cuh; outputs not meaningful). Synchronises. */
frsvt_status frsvt_debug_pass_timed(frsvt_handle* h, int32_t kind, int32_t impl, const void* A, int64_t lda,
                                    const void* B, void* out, int32_t reps, double* ms);

/* Test hook: the small SVD (Alg. 1 lines 16-18, reading Z8) alone, on an
 * l x l fp64 Gram G = B B^T (device, column-major, ld l; NULL = the Gram the
 * handle's last call decomposed). impl must be 0 (the production kernel:
 * one-sided Jacobi on G). Gcopy (device, nullable) receives the
 * Gram used. Outputs: sigma (device, l values, descending), UB (device, l x l,
 * ld l), *sweeps (host, nullable) and, when reps > 0, the mean device time of
 * `reps` back-to-back launches (*ms, host). Synchronises. */
frsvt_status frsvt_debug_small_svd(frsvt_handle* h, int32_t impl, const double* G, double* Gcopy, double* sigma,
                                   double* UB, int32_t* sweeps, int32_t reps, double* ms);

/* Test hook: the CholeskyQR factor kernel alone on an l x l fp64 Gram G
 * (device, column-major): T (device, l x l, handle dtype) with Y T an
 * orthonormal basis of range(Y) for Y^T Y = G, *s (host, nullable) = kept
 * rank; stamps (device, nullable, >= 8 x u64) = %globaltimer at phase
 * boundaries. Synchronises. */
frsvt_status frsvt_debug_chol(frsvt_handle* h, const double* G, void* T, int32_t* s, unsigned long long* stamps);

/* Test hook: the one-barrier-per-column factor kernel (chol_inv.cuh) alone,
 * fp32 handles. G: device, l x l fp64 Gram (column-major) of Y = [Q~ | Y_p]
 * whose first r columns (0 <= r <= l, host) are taken as orthonormal
 * (reading R11). T: device, l x l fp32
 * (column-major, ld l) receives, for r = 0, T with Y T orthonormal; for r > 0
 * the apply matrix Tp = [-G12 T22 ; T22] in its first p = l - r columns (the
 * rest zero), Y Tp spanning the part of range(Y) orthogonal to Q~. *s (host,
 * nullable) = r + kept fresh rank; stamps (device, nullable, >= 6 x u64) =
 * %globaltimer at the phase boundaries. EINVAL for a non-fp32 handle or r outside
 * [0, l]. Synchronises. */
frsvt_status frsvt_debug_chol_inv(frsvt_handle* h, const double* G, int32_t r, void* T, int32_t* s,
                                  unsigned long long* stamps);

/* Pass profiling: with enable != 0 every kernel that streams the m x n
 * operand is bracketed by CUDA events on the handle's stream (enabling resets
 * the totals). kind: 0 = A*X passes (sketch, power), 1 = A^T*Q passes (power,
 * B), 2 = composition / fused iALM epilogue, 3 = single-CTA calls (the whole
 * of Algorithm 1 in one kernel). Reading synchronises and returns the summed
 * event time (ms), the launch count and the algorithmic bytes of those
 * launches (m*n*elem per A pass; X write; 5 m*n*elem for the iALM epilogue:
 * D, A, E read, A, E written; 3 m*n*elem for a finalize step) -- for kind 3
 * the algorithmic FLOPs instead, 2 m n l (2q + 3) per call. */
frsvt_status frsvt_profile(frsvt_handle* h, int32_t enable);
frsvt_status frsvt_profile_read(frsvt_handle* h, int32_t kind, double* ms, int64_t* launches, double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* FRSVT_H */
