// libfrsvt: C ABI + orchestration of the FRSVT hot path on one B200 rank.
// Declarations, argument meaning and error behaviour: include/frsvt.h.
//
// One call of frsvt_apply* / rpca_alm_step enqueues, on the handle's stream
// (no host synchronisation, no allocation: a whole solve is graph-capturable):
//   omega -> Y = [Q~, A Omega_p]                              sketch   (Alg. 1 l.3-11)
//   orth(Y): fp64 Gram, Cholesky with column drop + explicit   rank reveal;
//     factor (chol_inv), applied on tensor cores; with a carry  RP: fresh block only (R13)
//   q x { Z = orth(A^T Q); Y = A Z; Q = orth2(Y) }              power iteration (l.13-15)
//   B^T = A^T Q; G = B B^T (fp64); Jacobi -> U_B, sigma         small SVD (l.16-18; R16)
//   shrink -> Mc, Mp; Q~ = Q Mc; Wt = B^T Mp                    Eq. (6) factors
//   X = Q~ Wt^T  (or the fused iALM epilogue, compose2)         composition (l.19)
// Row-sharded operands are reduced over ranks with NCCL where the contraction
// runs over rows (Grams of m-row matrices, A^T Q, residual, init norms).
#include "../../include/frsvt.h"
#include "common.cuh"
#include "gemm_simt.cuh"
#include "small.cuh"
#include "eig_jacobi.cuh"
#include "eig_warm.cuh"
#include "orth_chol.cuh"
#include "lowdin.cuh"
#include "chol_inv.cuh"
#include "gram_dmma.cuh"
#include "tc_pass.cuh"
#include "tc_compose.cuh"
#include "tc_util.cuh"
#include "tc_compose2.cuh"
#include "tc_pass3.cuh"
#include "batched.cuh"

#include <cudaTypedefs.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

using namespace frsvt;

namespace {

struct DevState {
  int s, r, flags, sweeps, have_prev, s2, fs_done, pad2;  // fs_done: next sketch formed by compose2
  double mu[2];        // mu_k, mu_bar
  double tau;
  double scal[4];      // 1/J, ||D||_2
  double dmax, dss;    // ||D||_inf, ||D||_F^2
  double resid[2];     // ||D-L-E||_F^2, relative residual
  double rep[2 * FRSVT_LMAX];
  int p_ap, l_act;     // adaptive rank prediction: fresh columns and width of the next call
  double varsig_raw;   // ||(I - QQ^T) y|| of the last sketch sample (Prop. 4 by-product)
};

struct Status {
  frsvt_status st = FRSVT_OK;
};

// Loopback reduction: out_r[i] = op over ranks k = 0..n-1 (in that order) of
// in_k[i], written back into every rank's buffer (in place: each element is
// read from all ranks before it is written).
struct LoopPtrs {
  void* p[FRSVT_LOOPBACK_MAX];
};
template <typename T>
__global__ void loopback_reduce_kernel(LoopPtrs b, int n, size_t count, int op) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T acc = reinterpret_cast<T*>(b.p[0])[i];
    for (int k = 1; k < n; ++k) {
      const T x = reinterpret_cast<T*>(b.p[k])[i];
      acc = op == 0 ? acc + x : (op == 1 ? (x > acc ? x : acc) : (x < acc ? x : acc));
    }
    for (int k = 0; k < n; ++k) reinterpret_cast<T*>(b.p[k])[i] = acc;
  }
}

}  // namespace

// Loopback process group (include/frsvt.h): n handles of one process on one
// device, each on its own host thread and stream. A reduction point is a host
// rendezvous: every rank records an event on its stream; the last to arrive
// makes its stream wait for all of them and enqueues one reduction kernel over
// all ranks' buffers; every rank's stream then waits for that kernel. No
// kernel waits on another kernel (stream-order dependencies only).
struct frsvt_group {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  void* bufs[FRSVT_LOOPBACK_MAX] = {};
  cudaEvent_t ready[FRSVT_LOOPBACK_MAX] = {};
  cudaEvent_t done = nullptr;
  size_t count = 0;
  int type = 0, op = 0;
  bool mismatch = false;
};

struct frsvt_handle {
  frsvt_config cfg;
  cudaStream_t st;
  int dev_id;
  int esz;  // element size
  int l, q, rp;
  int64_t m, n;
  // workspaces (element type = dtype)
  void *Om, *OmOv, *Y, *Q, *Qtmp, *Qt, *Z, *Zq, *Zt, *Wt;
  void *T1, *Mc, *Mp;
  double *wvec;
  // tcgen05 path (fp32): tf32 hi/lo splits of the small operands (ld padded to 4)
  float *Xh, *Xl, *Qh, *Ql;
  float *QtTh, *QtTl, *WtTh, *WtTl;  // K-major (Kp x rows) splits for the composition
  int Kp;
  int64_t ldxs, ldqs;
  int use_tc;        // fp32 handle with TMA available: tcgen05 passes (else SIMT, fp64 handles)
  int tc_m;          // tensor-core small-operand path for the m-row matrices (Y, Q); rank-uniform
  double* ewbuf;     // Gpad, Uf (32 x 32 each), sigma_f (32), G2 (l x l)
  int single_cta;    // the last frsvt_apply ran on the single-CTA path (FRSVT_FLAG_SINGLE_CTA)
  int fs;            // 1: fuse the next call's fresh sketch into the iALM composition (FRSVT_OPT_FUSED_SKETCH)
  int om_tf32;       // 1: drawn Omega entries rounded to tf32 (FRSVT_OPT_TF32_OMEGA)
  int ap_on, ap_a, ap_jump, ap_b, ap_l0;  // adaptive rank prediction (Eq. 7), frsvt_set_adaptive_rank
  int keep;          // partial SVT of the current rpca step (rpca_state.keep; 0 for frsvt_apply*)
  double* resid_out;  // where the next sketch orthonormalisation reports its last-sample residual
  bool fs_armed;     // the last composition may have formed Y_p for the next call (dev->fs_done)
  float* fspart;     // fused-sketch partial rows, one 24 x 128 block per composition CTA
  float* OmT;        // Omega^T, n x 24 (the fused sketch's TMA operand)
  size_t fspart_ctas;
  unsigned int* tilecnt;  // per-tile arrival counters (zero between passes)
  int ncnt;
  double* E2b;       // Loewdin workspace E^2 (l x l fp64)
  double* Rf;        // first-pass CholeskyQR factor R' (l x l row-major fp64)
  double *T2d, *Hd, *McD, *MpD;  // fp64 l x l: pending second CholeskyQR factor and fold scratch
  int t2_pending;    // 1: h->Q holds Q1 and the basis is Q1 T2d (T2d folded into G, Mc, Mp)
  int* lwd;          // device ints: [0] Loewdin ok, [2..3] max|E| (u64), [4] debug r, [6] create flag,
                     // [7] fresh-block sweeps, [8..9] sketch-width flags, [12..14] fresh-block width flags
  int nsm;           // SMs of the device (stream-K grid)
  float* skpart;     // stream-K partial-tile slots (nsm x 2 x 128 x 128 fp32)
  __nv_bfloat16 *Xb, *Qb;  // bf16 [b_l | b_h] operands of the stream-K passes (ld ldb16)
  int64_t ldb16;     // leading dimension of the bf16 low parts (multiple of 8)
  void* partq;       // split-K partials of A^T Q (dtype)
  size_t partq_elems;
  double* partd;     // Gram split-K partials (fp64)
  size_t partd_elems;
  double* redpart;   // per-block reduction partials
  size_t redpart_elems;
  double *G, *UB, *sigma, *dprev;
  double* redtmp;    // small fold outputs
  DevState* dev;
  int64_t call;
  int override_pending;
  ncclComm_t comm;
  frsvt_group* group;    // loopback process group (nranks > 1 without NCCL), not owned
  cudaEvent_t ev_ready;  // this rank's arrival at a loopback reduction
  int64_t launches;
  double last_mu_host;
  // pass profiling (frsvt_profile)
  int prof_on;
  std::vector<cudaEvent_t>* prof_ev;   // pool, pairs (start, end)
  std::vector<int>* prof_kind;         // kind per used pair
  size_t prof_used;
  double prof_ms[4], prof_bytes[4];
  int64_t prof_count[4];
};

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "libfrsvt: %s failed: %s (%s:%d)\n", #x, cudaGetErrorString(e_), \
              __FILE__, __LINE__);                                                 \
      return FRSVT_ECUDA;                                                          \
    }                                                                              \
  } while (0)

#define CKN(x)                                                                     \
  do {                                                                             \
    ncclResult_t r_ = (x);                                                         \
    if (r_ != ncclSuccess) {                                                       \
      fprintf(stderr, "libfrsvt: %s failed: %s\n", #x, ncclGetErrorString(r_));    \
      return FRSVT_ENCCL;                                                          \
    }                                                                              \
  } while (0)

#define TRY(x)                         \
  do {                                 \
    frsvt_status s_ = (x);             \
    if (s_ != FRSVT_OK) return s_;     \
  } while (0)

namespace {

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// NVTX range over one phase of the path (host-side markers for nsys/ncu
// timelines: range finder, small SVD, shrink/factors, composition/epilogue)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

frsvt_status post_launch(frsvt_handle* h) {
  h->launches++;
  CK(cudaGetLastError());
  return FRSVT_OK;
}

frsvt_status prof_flush(frsvt_handle* h) {
  if (!h->prof_used) return FRSVT_OK;
  CK(cudaEventSynchronize((*h->prof_ev)[2 * h->prof_used - 1]));
  for (size_t i = 0; i < h->prof_used; ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, (*h->prof_ev)[2 * i], (*h->prof_ev)[2 * i + 1]));
    h->prof_ms[(*h->prof_kind)[i]] += ms;
  }
  h->prof_used = 0;
  return FRSVT_OK;
}

// bracket one streaming pass with events (no-op unless profiling)
frsvt_status prof_begin(frsvt_handle* h) {
  if (!h->prof_on) return FRSVT_OK;
  if (2 * (h->prof_used + 1) > h->prof_ev->size()) {
    if (h->prof_ev->size() < 2 * 8192) {
      for (int i = 0; i < 256; ++i) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        h->prof_ev->push_back(e);
      }
      h->prof_kind->resize(h->prof_ev->size() / 2);
    } else {
      TRY(prof_flush(h));
    }
  }
  CK(cudaEventRecord((*h->prof_ev)[2 * h->prof_used], h->st));
  return FRSVT_OK;
}
frsvt_status prof_end(frsvt_handle* h, int kind, double bytes) {
  if (!h->prof_on) return FRSVT_OK;
  CK(cudaEventRecord((*h->prof_ev)[2 * h->prof_used + 1], h->st));
  (*h->prof_kind)[h->prof_used] = kind;
  h->prof_used++;
  h->prof_bytes[kind] += bytes;
  h->prof_count[kind]++;
  return FRSVT_OK;
}

int grid1d(int64_t total, int threads = 256) {
  int64_t b = cdiv(total, threads);
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

// ---------------------------------------------------------------- GEMM glue
template <typename Tin, typename Tacc, int BM, int BN, int BK, int TM, int TN, bool AMC, bool BKC,
          class Epi>
frsvt_status launch_tile(frsvt_handle* h, int M, int N, int K, int splits, const Tin* A,
                         int64_t lda, const Tin* B, int64_t ldb, const int* kdev, Epi epi) {
  if (M <= 0 || N <= 0) return FRSVT_OK;
  if (splits < 1) splits = 1;
  int kchunk = (int)cdiv(cdiv(K, splits), BK) * BK;
  if (kchunk < BK) kchunk = BK;
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, BN), (unsigned)splits);
  gemm_simt_kernel<Tin, Tacc, BM, BN, BK, TM, TN, AMC, BKC, Epi>
      <<<grid, 256, 0, h->st>>>(M, N, K, kchunk, A, lda, B, ldb, kdev, epi);
  return post_launch(h);
}

// skinny: N = l (<= 128)
template <typename Tin, typename Tacc, bool AMC, bool BKC, class Epi>
frsvt_status launch_skinny(frsvt_handle* h, int M, int N, int K, int splits, const Tin* A,
                           int64_t lda, const Tin* B, int64_t ldb, const int* kdev, Epi epi) {
  if (N <= 16)
    return launch_tile<Tin, Tacc, 256, 16, 16, 4, 4, AMC, BKC>(h, M, N, K, splits, A, lda, B, ldb, kdev, epi);
  if (N <= 32)
    return launch_tile<Tin, Tacc, 128, 32, 16, 4, 4, AMC, BKC>(h, M, N, K, splits, A, lda, B, ldb, kdev, epi);
  if (N <= 64)
    return launch_tile<Tin, Tacc, 128, 64, 16, 8, 4, AMC, BKC>(h, M, N, K, splits, A, lda, B, ldb, kdev, epi);
  return launch_tile<Tin, Tacc, 128, 128, 16, 8, 8, AMC, BKC>(h, M, N, K, splits, A, lda, B, ldb, kdev, epi);
}

// square l x l outputs (Gram)
template <typename Tin, class Epi>
frsvt_status launch_gram_tile(frsvt_handle* h, int l, int K, int splits, const Tin* Y, int64_t ld,
                              Epi epi) {
  if (l <= 16)
    return launch_tile<Tin, double, 16, 16, 32, 1, 1, false, true>(h, l, l, K, splits, Y, ld, Y, ld, nullptr, epi);
  if (l <= 32)
    return launch_tile<Tin, double, 32, 32, 16, 2, 2, false, true>(h, l, l, K, splits, Y, ld, Y, ld, nullptr, epi);
  if (l <= 64)
    return launch_tile<Tin, double, 64, 64, 16, 4, 4, false, true>(h, l, l, K, splits, Y, ld, Y, ld, nullptr, epi);
  return launch_tile<Tin, double, 128, 128, 16, 8, 8, false, true>(h, l, l, K, splits, Y, ld, Y, ld, nullptr, epi);
}

int gram_splits(int64_t rows) {
  int64_t s = cdiv(rows, 256);
  if (s > 148) s = 148;
  if (s < 1) s = 1;
  return (int)s;
}
int atq_splits(int64_t n, int64_t rows, int l) {
  const int bm = l <= 16 ? 256 : 128;
  int64_t tiles = cdiv(n, bm);
  int64_t s = cdiv(296, tiles);
  int64_t maxs = cdiv(rows, 128);
  if (s > maxs) s = maxs;
  if (s < 1) s = 1;
  return (int)s;
}

// ---------------------------------------------------------------- tcgen05 glue
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool tma_encode_available() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return true;
}

// 2-D fp32 tensor map over a column-major matrix (dim0 contiguous, ld elements)
bool make_map(CUtensorMap* map, const float* ptr, uint64_t dim0, uint64_t dim1, uint64_t ld, uint32_t box0,
              uint32_t box1, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {dim0, dim1};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tc_eligible(const frsvt_handle* h, const void* A, int64_t lda) {
  return h->use_tc && h->esz == 4 && (lda % 4) == 0 && ((uintptr_t)A % 16) == 0;
}

int tc_np(int l) { return l <= 32 ? 32 : (l <= 64 ? 64 : 128); }

template <int MODE, int NP>
frsvt_status launch_tc_np(frsvt_handle* h, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl,
                          int Mtot, int Ktot, int splits, float* out, int64_t ldo, int64_t zstride,
                          const float* add, int64_t ldadd) {
  const size_t smem = tc::PassSmem::total(NP);  // attribute set in frsvt_create
  const int nchunks = (int)cdiv(Ktot, tc::BK);
  const int cps = (int)cdiv(nchunks, splits);
  dim3 grid((unsigned)cdiv(Mtot, 128), (unsigned)splits);
  tc::tc_pass_kernel<MODE, NP><<<grid, tc::PASS_THREADS, smem, h->st>>>(mA, mBh, mBl, Mtot, Ktot, cps, h->l, out, ldo, zstride,
                                                           add, ldadd);
  return post_launch(h);
}

template <int MODE>
frsvt_status launch_tc(frsvt_handle* h, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl,
                       int Mtot, int Ktot, int splits, float* out, int64_t ldo, int64_t zstride, const float* add,
                       int64_t ldadd) {
  const int np = tc_np(h->l);
  if (np == 32) return launch_tc_np<MODE, 32>(h, mA, mBh, mBl, Mtot, Ktot, splits, out, ldo, zstride, add, ldadd);
  if (np == 64) return launch_tc_np<MODE, 64>(h, mA, mBh, mBl, Mtot, Ktot, splits, out, ldo, zstride, add, ldadd);
  return launch_tc_np<MODE, 128>(h, mA, mBh, mBl, Mtot, Ktot, splits, out, ldo, zstride, add, ldadd);
}

frsvt_status split_small(frsvt_handle* h, const float* X, int64_t rows, int64_t ldx, float* Hi, float* Lo,
                         int64_t ldo) {
  tc::split_tf32_kernel<<<grid1d(rows * h->l), 256, 0, h->st>>>(X, rows, h->l, ldx, Hi, Lo, ldo);
  return post_launch(h);
}

// partials (splits x Mcols x l) of A^T Q, A (rows x Mcols, lda), Q (rows x l, ldq), split-K over rows
frsvt_status tc_AtQ_gen(frsvt_handle* h, const float* A, int64_t lda, int64_t rows, int64_t Mcols, const float* Q,
                        int64_t ldq, float* part, int splits) {
  TRY(split_small(h, Q, rows, ldq, h->Qh, h->Ql, h->ldqs));
  const uint32_t np = (uint32_t)tc_np(h->l);
  CUtensorMap mA, mBh, mBl;
  if (!make_map(&mA, A, rows, Mcols, lda, tc::BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mBh, h->Qh, rows, h->l, h->ldqs, tc::BK, np, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mBl, h->Ql, rows, h->l, h->ldqs, tc::BK, np, CU_TENSOR_MAP_SWIZZLE_128B))
    return FRSVT_ECUDA;
  return launch_tc<tc::MODE_ATQ>(h, mA, mBh, mBl, (int)Mcols, (int)rows, splits, part, Mcols,
                                 (int64_t)Mcols * h->l, nullptr, 0);
}

// flags[0] = (p > thr), flags[1] = (p <= thr) for p = l - *r_dev, capped by
// *pmax_dev when adaptive rank prediction is on (the skip flags of the two
// sketch instances)
// adaptive rank prediction, Eq. (7): from this call's
// width l_i and kept rank r_i, p_{i+1} = a if r_i < l_i else ceil(rho n),
// l_{i+1} = min(r_i + p_{i+1}, b); the next call draws l_{i+1} - r_i fresh
// columns behind the r_i carried ones
__global__ void ap_update_kernel(DevState* __restrict__ d, int a, int jump, int b) {
  if (threadIdx.x == 0) {
    const int r = d->r, l = d->l_act;
    const int p = r < l ? a : jump;
    const int ln = min(r + p, b);
    d->l_act = ln;
    d->p_ap = ln - r;
  }
}
__global__ void ap_reset_kernel(DevState* __restrict__ d, int l0) {
  if (threadIdx.x == 0) {
    d->l_act = l0;
    d->p_ap = l0;
  }
}

__global__ void sketch_width_kernel(const int* __restrict__ r_dev, int l, int thr, int* __restrict__ flags,
                                    const int* __restrict__ pmax_dev) {
  if (threadIdx.x == 0) {
    int p = l - min(max(*r_dev, 0), l);
    if (pmax_dev) p = min(p, max(*pmax_dev, 0));
    flags[0] = p > thr ? 1 : 0;
    flags[1] = p > thr ? 0 : 1;
  }
}

// ---- CTA-pair (cta_group::2) stream-K passes (tc_pass3.cuh) -----------------
template <int MODE, int NP, int TERMS>
frsvt_status launch_p3(frsvt_handle* h, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBx,
                       int Mtot, int Ktot, float* out, int64_t ldo, const float* add, int64_t ldadd, int dbg,
                       const int* rp_dev, const int* skip_dev) {
  constexpr int CL = 2;
  const size_t smem = tc::Pass3Smem::total(NP, TERMS);  // attribute set in frsvt_create
  const int mtiles = (int)cdiv(Mtot, 128);
  const int64_t mgroups = cdiv(mtiles, CL);
  const int64_t total = mgroups * cdiv(Ktot, tc::BK);
  const int Gmax = h->nsm / CL;
  // small K (the l x l applies of the orthonormalisation): whole tiles per
  // cluster, no split tiles (dbg bit 8)
  const bool talign = Ktot <= 8 * tc::BK;
  if (talign) dbg |= 256;
  const int64_t units = talign ? mgroups : total;
  const int G = (int)(units < Gmax ? units : Gmax);
  if (mtiles > h->ncnt) return FRSVT_EINVAL;  // the tile counters cover every row tile (sized at create)
  // tiles shared by many clusters (few output tiles): the slots are summed by
  // a separate many-block kernel instead of the last covering CTA
  const bool sep_fix = !talign && (int64_t)G > 4 * mgroups;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(G * CL));
  lc.blockDim = dim3(tc::P3_THREADS);
  lc.dynamicSmemBytes = smem;
  lc.stream = h->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CK(cudaLaunchKernelEx(&lc, tc::tc_pass3_kernel<MODE, NP, TERMS>, mA, mBh, mBx, Mtot, Ktot, h->l, out, ldo, add,
                        ldadd, h->skpart, rp_dev, dbg, sep_fix ? nullptr : h->tilecnt, skip_dev));
  TRY(post_launch(h));
  if (!sep_fix) return FRSVT_OK;
  // columns per block: as many as keep ~2 waves of 4 blocks per SM (each
  // block first scans the covering clusters' ranges, once for all its columns)
  int fx_c = (int)((int64_t)mtiles * h->l / (8 * (int64_t)h->nsm));
  fx_c = fx_c < 1 ? 1 : (fx_c > tc::P3_FX_C ? tc::P3_FX_C : fx_c);
  tc::p3_fixup_kernel<NP><<<dim3((unsigned)mtiles, (unsigned)cdiv(h->l, fx_c)), 512, 0, h->st>>>(
      Mtot, Ktot, h->l, G, h->skpart, out, ldo, add, ldadd, rp_dev, skip_dev, fx_c);
  return post_launch(h);
}

// out (Mtot x l) = op(A) * B on CTA pairs, B (Ktot x l, ld ldb) the small
// operand: MODE_AX: A is Mtot x Ktot (lda); MODE_ATQ: A is Ktot x Mtot (lda),
// op = ^T. terms 3: fp32-level product; terms 2: product with the
// tf32-rounded B (span-only passes, reading R17).
template <int MODE>
frsvt_status tc_pass3(frsvt_handle* h, const float* A, int64_t lda, int64_t Mtot, int64_t Ktot, const float* B,
                      int64_t ldb, float* out, int64_t ldo, const float* add, int64_t ldadd, int terms, int dbg = 0,
                      const int* rp_dev = nullptr, const int* skip_dev = nullptr, int np_force = 0) {
  const int np = np_force ? np_force : tc_np(h->l);
  float* Bh = MODE == tc::MODE_AX ? h->Xh : h->Qh;
  __nv_bfloat16* Bx = MODE == tc::MODE_AX ? h->Xb : h->Qb;
  const int64_t ldh = MODE == tc::MODE_AX ? h->ldxs : h->ldqs;
  const int64_t kpad = cdiv(Ktot, tc::BK) * tc::BK;
  const uint32_t nb = (uint32_t)np / 2;  // each CTA of the pair holds an np/2-row half of a B stage
  CUtensorMap mA, mBh, mBx;
  bool ok = (MODE == tc::MODE_AX) ? make_map(&mA, A, Mtot, Ktot, lda, 128, tc::BK, CU_TENSOR_MAP_SWIZZLE_NONE)
                                  : make_map(&mA, A, Ktot, Mtot, lda, tc::BK, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok = ok && make_map(&mBh, Bh, Ktot, h->l, ldh, tc::BK, nb, CU_TENSOR_MAP_SWIZZLE_128B);
  if (terms == 3) {
    const int64_t kx = 2 * kpad;  // rows of the bf16 [b_l | b_h] operand
    tc::split_tf32_bf16x2_kernel<<<dim3((unsigned)cdiv(kx / 2, 512), (unsigned)h->l), 256, 0, h->st>>>(
        B, Ktot, h->l, ldb, Bh, ldh, Bx, h->ldb16);
    TRY(post_launch(h));
    cuuint64_t dims[2] = {(cuuint64_t)kx, (cuuint64_t)h->l};
    cuuint64_t strides[1] = {(cuuint64_t)h->ldb16 * 2};
    cuuint32_t box[2] = {(cuuint32_t)(2 * tc::BK), nb};
    cuuint32_t es[2] = {1, 1};
    ok = ok && g_encode(&mBx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)Bx, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  } else {
    tc::split_tf32_bf16_kernel<<<dim3((unsigned)cdiv(kpad / 2, 256), (unsigned)h->l), 256, 0, h->st>>>(
        B, Ktot, ldb, Bh, ldh, Bx, kpad);
    TRY(post_launch(h));
    cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)h->l};
    cuuint64_t strides[1] = {(cuuint64_t)kpad * 2};
    cuuint32_t box[2] = {(cuuint32_t)tc::BK, nb};
    cuuint32_t es[2] = {1, 1};
    ok = ok && g_encode(&mBx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)Bx, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (!ok) return FRSVT_ECUDA;
#define FRSVT_P3(NPV, TV) \
  launch_p3<MODE, NPV, TV>(h, mA, mBh, mBx, (int)Mtot, (int)Ktot, out, ldo, add, ldadd, dbg, rp_dev, skip_dev)
  if (terms == 3) {
    if (np == 32) return FRSVT_P3(32, 3);
    if (np == 64) return FRSVT_P3(64, 3);
    return FRSVT_P3(128, 3);
  }
  if (np == 32) return FRSVT_P3(32, 2);
  if (np == 64) return FRSVT_P3(64, 2);
  return FRSVT_P3(128, 2);
#undef FRSVT_P3
}

// tensor-core path for the small-operand GEMMs of a (rows x l, ld = rows)
// matrix. For the row-sharded m-row matrices (m_rows) the choice was made once
// in frsvt_create and agreed over the ranks (h->tc_m): every rank must take the
// same orthonormalisation route, or the replicated factors would differ.
bool tc_small_local(const frsvt_handle* h, int64_t rows) {
  return h->use_tc && h->esz == 4 && (rows % 4) == 0 && rows >= 128;
}
bool tc_small_ok(const frsvt_handle* h, int64_t rows, bool m_rows) {
  return m_rows ? h->tc_m != 0 : tc_small_local(h, rows);
}

// X = Q~ Wt^T fused with its consumer (tc::EPI_*) on tensor cores. Returns the
// number of residual partials written to h->redpart.
frsvt_status tc_compose(frsvt_handle* h, int epi, float* X, int64_t ldx, const float* D, float* A, float* E,
                        int64_t ld, double rho, double lambda, int* nparts, bool fs_next = false) {
  const int Kp = h->Kp;
  // compose2 (the iALM epilogue) splits Q~ itself while moving it to TMEM
  const bool tma_ok = epi == tc::EPI_STORE ? ((ldx % 4) == 0 && ((uintptr_t)X % 16) == 0)
                                           : ((ld % 4) == 0 && (((uintptr_t)D | (uintptr_t)A | (uintptr_t)E) % 16) == 0);
  const bool use2 = tma_ok && (h->m % 4) == 0;
  {
    if (!use2) {
      dim3 g1((unsigned)cdiv(h->m, 32), (unsigned)(Kp / 32));
      tc::split_transpose_kernel<<<g1, 256, 0, h->st>>>((const float*)h->Qt, h->m, h->l, h->m, Kp, h->QtTh,
                                                         h->QtTl);
      TRY(post_launch(h));
    }
    dim3 g2((unsigned)cdiv(h->n, 32), (unsigned)(Kp / 32));
    tc::split_transpose_kernel<<<g2, 256, 0, h->st>>>((const float*)h->Wt, h->n, h->l, h->n, Kp, h->WtTh, h->WtTl);
    TRY(post_launch(h));
  }
  CUtensorMap mQh, mQl, mWh, mWl;
  if (!make_map(&mQh, h->QtTh, Kp, h->m, Kp, tc::BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mQl, h->QtTl, Kp, h->m, Kp, tc::BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mWh, h->WtTh, Kp, h->n, Kp, tc::BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mWl, h->WtTl, Kp, h->n, Kp, tc::BK, 128, CU_TENSOR_MAP_SWIZZLE_128B))
    return FRSVT_ECUDA;
  const int rbs = (int)cdiv(h->m, 128), ntiles = (int)cdiv(h->n, 128);
  const int W = h->nsm;
  int nfull, rem, sp;
  if (rbs >= W) {
    nfull = (rbs / W) * W;
    rem = rbs - nfull;
    sp = rem ? (W / rem) : 1;
  } else {
    nfull = 0;
    rem = rbs;
    sp = (int)cdiv(2 * W, rbs);
  }
  if (sp > ntiles) sp = ntiles;
  if (sp < 1) sp = 1;
  dim3 grid((unsigned)(nfull + rem * sp));
  // compose2 streams D, A, E through TMA: 16-byte aligned columns required (use2)
  if (use2) {
    CUtensorMap mD, mA, mE, mQ;
    if (!make_map(&mQ, (const float*)h->Qt, h->m, h->l, h->m, 128, tc::BK, CU_TENSOR_MAP_SWIZZLE_NONE))
      return FRSVT_ECUDA;
    if (epi == tc::EPI_STORE) {  // no streamed operands: placeholder maps (never read)
      D = A = E = X;
      ld = ldx;
    }
    if (!make_map(&mD, D, h->m, h->n, ld, 128, 8, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !make_map(&mE, E, h->m, h->n, ld, 128, 8, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !make_map(&mA, epi == tc::EPI_ALM ? A : E, h->m, h->n, ld, 128, 8, CU_TENSOR_MAP_SWIZZLE_NONE))
      return FRSVT_ECUDA;
    // fused next sketch (fs): Omega of the next call (already drawn into h->Om)
    const bool fs = fs_next && epi == tc::EPI_ALM && grid.x <= h->fspart_ctas;
    CUtensorMap mOm = mD;
    if (fs) {
      tc::omega_t24_kernel<<<grid1d(h->n * tc::FS_PMAX), 256, 0, h->st>>>((const float*)h->Om, h->n, h->l, h->OmT);
      TRY(post_launch(h));
      if (!make_map(&mOm, h->OmT, tc::FS_PMAX, h->n, tc::FS_PMAX, tc::FS_PMAX, 8, CU_TENSOR_MAP_SWIZZLE_NONE))
        return FRSVT_ECUDA;
    }
    const size_t smem2 = tc::Compose2Smem::total();  // attributes set in frsvt_create
#define FRSVT_LAUNCH_CMP2(EPIV, FSV)                                                                            \
  do {                                                                                                          \
    tc::tc_compose2_kernel<EPIV, FSV><<<grid, tc::CMP_THREADS, smem2, h->st>>>(                                 \
        mQ, mWh, mWl, mD, mA, mE, mOm, (int)h->m, (int)h->n, h->l, &h->dev->r, nfull, sp, X, ldx, A, E, \
        ld, h->dev->mu, rho, lambda, h->redpart, h->fspart, &h->dev->fs_done);                                  \
  } while (0)
    if (epi == tc::EPI_ALM && fs) FRSVT_LAUNCH_CMP2(tc::EPI_ALM, true);
    else if (epi == tc::EPI_ALM) FRSVT_LAUNCH_CMP2(tc::EPI_ALM, false);
    else if (epi == tc::EPI_FINAL) FRSVT_LAUNCH_CMP2(tc::EPI_FINAL, false);
    else FRSVT_LAUNCH_CMP2(tc::EPI_STORE, false);
#undef FRSVT_LAUNCH_CMP2
    if (nparts) *nparts = (int)grid.x;
    TRY(post_launch(h));
    if (fs) {
      tc::fs_finish_kernel<<<(unsigned)rbs, 128, 0, h->st>>>(h->fspart, (int)h->m, h->l, &h->dev->r, nfull, sp,
                                                              (float*)h->Y, &h->dev->fs_done);
      TRY(post_launch(h));
      h->fs_armed = true;
    }
    return FRSVT_OK;
  }
  const size_t smem = tc::ComposeSmem::total();  // attributes set in frsvt_create
#define FRSVT_LAUNCH_CMP(EPIV)                                                                                  \
  do {                                                                                                          \
    tc::tc_compose_kernel<EPIV><<<grid, tc::CMP_THREADS, smem, h->st>>>(mQh, mQl, mWh, mWl, (int)h->m, (int)h->n, \
                                                                        &h->dev->r, nfull, sp, X, ldx, D, A, E, ld,    \
                                                                        h->dev->mu, rho, lambda, h->redpart);    \
  } while (0)
  if (epi == tc::EPI_STORE) FRSVT_LAUNCH_CMP(tc::EPI_STORE);
  else if (epi == tc::EPI_ALM) FRSVT_LAUNCH_CMP(tc::EPI_ALM);
  else FRSVT_LAUNCH_CMP(tc::EPI_FINAL);
#undef FRSVT_LAUNCH_CMP
  if (nparts) *nparts = (int)grid.x;
  return post_launch(h);
}

frsvt_status loopback_allreduce(frsvt_handle* h, void* buf, size_t count, ncclDataType_t t, ncclRedOp_t op) {
  frsvt_group* g = h->group;
  const int type = t == ncclFloat64 ? 0 : (t == ncclFloat32 ? 1 : 2);
  const int o = op == ncclSum ? 0 : (op == ncclMax ? 1 : 2);
  if ((t != ncclFloat64 && t != ncclFloat32 && t != ncclInt32) || (op != ncclSum && op != ncclMax && op != ncclMin))
    return FRSVT_EINVAL;
  std::unique_lock<std::mutex> lk(g->mu);
  const int me = h->cfg.rank;
  if (cudaEventRecord(h->ev_ready, h->st) != cudaSuccess) return FRSVT_ECUDA;
  g->bufs[me] = buf;
  g->ready[me] = h->ev_ready;
  if (g->arrived == 0) {
    g->count = count;
    g->type = type;
    g->op = o;
  } else if (g->count != count || g->type != type || g->op != o) {
    g->mismatch = true;  // ranks disagree on the reduction sequence
  }
  const uint64_t my_gen = g->gen;
  if (++g->arrived == g->n) {
    for (int r = 0; r < g->n; ++r)
      if (r != me) CK(cudaStreamWaitEvent(h->st, g->ready[r], 0));
    LoopPtrs ptrs{};
    for (int r = 0; r < g->n; ++r) ptrs.p[r] = g->bufs[r];
    const int blocks = (int)((count + 255) / 256 < 1024 ? (count + 255) / 256 : 1024);
    if (type == 0) loopback_reduce_kernel<double><<<blocks, 256, 0, h->st>>>(ptrs, g->n, count, o);
    else if (type == 1) loopback_reduce_kernel<float><<<blocks, 256, 0, h->st>>>(ptrs, g->n, count, o);
    else loopback_reduce_kernel<int><<<blocks, 256, 0, h->st>>>(ptrs, g->n, count, o);
    TRY(post_launch(h));
    CK(cudaEventRecord(g->done, h->st));
    g->arrived = 0;
    g->gen++;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->gen != my_gen; });
  }
  // inside the lock: the next reduction cannot re-record `done` before every
  // rank has ordered its stream after this one
  CK(cudaStreamWaitEvent(h->st, g->done, 0));
  return g->mismatch ? FRSVT_EINVAL : FRSVT_OK;
}

frsvt_status allreduce(frsvt_handle* h, void* buf, size_t count, ncclDataType_t t, ncclRedOp_t op) {
  if (h->cfg.nranks <= 1) return FRSVT_OK;
  if (h->group) return loopback_allreduce(h, buf, count, t, op);
  CKN(ncclAllReduce(buf, buf, count, t, op, h->comm, h->st));
  return FRSVT_OK;
}

template <typename T> ncclDataType_t nccl_type();
template <> ncclDataType_t nccl_type<float>() { return ncclFloat32; }
template <> ncclDataType_t nccl_type<double>() { return ncclFloat64; }

// G (l x l fp64) = Y^T Y over `rows` rows; summed over ranks if `sharded`.
template <typename T>
frsvt_status gram(frsvt_handle* h, const T* Y, int64_t rows, int64_t ld, bool sharded, const int* r_dev = nullptr) {
  const int l = h->l;
  // fp64 tensor cores (DMMA), upper 8x8 blocks only (gram_dmma.cuh); one wave
  // (1 CTA of 512 threads per SM at 128 registers), >= 32 rows each
  const bool narrow = l <= GS_LMAX && rows >= 32768;  // tall and narrow: entries per thread (gram_small_kernel)
  const int CR = narrow ? GS_ROWS : GD_ROWS;
  int S = (int)cdiv(rows, CR);
  const int Smax = (int)(h->partd_elems / ((size_t)l * l));
  if (S > h->nsm) S = h->nsm;
  if (S > Smax) S = Smax;
  if (S < 1) S = 1;
  const int64_t rpc = cdiv(cdiv(rows, S), CR) * CR;
  S = (int)cdiv(rows, rpc);
  if (narrow)  // (RP: all blocks are formed; chol_inv reads only the ones it needs)
    gram_small_kernel<T><<<S, GS_THREADS, 0, h->st>>>(Y, rows, ld, l, rpc, h->partd);
  else
    gram_dmma_kernel<T><<<S, GD_THREADS, 0, h->st>>>(Y, rows, ld, l, rpc, h->partd, r_dev);
  TRY(post_launch(h));
  splitk_reduce_wide_kernel<double, double><<<(unsigned)cdiv((int64_t)l * l, 32), 256, 0, h->st>>>(h->partd, S, l, l,
                                                                                                   h->G, l);
  TRY(post_launch(h));
  if (sharded) TRY(allreduce(h, h->G, (size_t)l * l, ncclFloat64, ncclSum));
  return FRSVT_OK;
}

template <typename T>
frsvt_status chol(frsvt_handle* h, T* Tout, const int* skip = nullptr) {
  const int l = h->l;
  const double tol = sizeof(T) == 4 ? 1e-12 : 1e-13;
  orth_chol_kernel<T><<<1, OC_THREADS, orth_chol_smem_bytes(l), h->st>>>(h->G, l, tol, Tout, &h->dev->s,
                                                                          &h->dev->flags, nullptr, skip);
  return post_launch(h);
}

// second-pass factor T2 of the nearly orthonormal Q1 (Gram in h->G): the
// Loewdin series when max|G - I| <= 0.05, else the Cholesky kernel (lowdin.cuh)
template <typename T>
frsvt_status chol2(frsvt_handle* h, T* Tout) {
  const int l = h->l;
  int* ok = h->lwd;
  unsigned long long* emax = (unsigned long long*)(h->lwd + 2);
  CK(cudaMemsetAsync(emax, 0, sizeof(unsigned long long), h->st));
  const dim3 g((unsigned)cdiv(l, LWD_T), (unsigned)cdiv(l, LWD_T));
  lowdin_sq_kernel<<<g, LWD_THREADS, lowdin_smem_bytes(l), h->st>>>(h->G, l, h->E2b, emax);
  TRY(post_launch(h));
  lowdin_series_kernel<T><<<g, LWD_THREADS, lowdin_smem_bytes(l), h->st>>>(h->G, h->E2b, l, emax, ok, Tout);
  TRY(post_launch(h));
  return chol<T>(h, Tout, ok);
}

// Out (rows x l) = In (rows x l) * M (l x l), fp32-accurate SIMT (used where
// the small factor is ill-conditioned: the first CholeskyQR pass)
template <typename T>
frsvt_status apply_small(frsvt_handle* h, const T* In, int64_t rows, int64_t ldin, const T* Msm,
                         T* Out, int64_t ldout) {
  EpiStore<T> epi{Out, ldout, 0};
  return launch_skinny<T, T, true, true>(h, (int)rows, h->l, h->l, 1, In, ldin, Msm, (int64_t)h->l,
                                          nullptr, epi);
}

// Out = In * M with a well-conditioned M (orthogonal-like): tensor cores when
// eligible (3xTF32, ~2e-6 relative), else SIMT
template <typename T>
frsvt_status apply_rows(frsvt_handle* h, const T* In, int64_t rows, const T* M, T* Out, const int* r_dev) {
  const int l = h->l;
  const unsigned g = (unsigned)cdiv(rows, 128);
  if (l <= 4) apply_rows_kernel<T, 4><<<g, 128, 0, h->st>>>(In, rows, rows, l, M, Out, rows, r_dev);
  else if (l <= 8) apply_rows_kernel<T, 8><<<g, 128, 0, h->st>>>(In, rows, rows, l, M, Out, rows, r_dev);
  else if (l <= 12) apply_rows_kernel<T, 12><<<g, 128, 0, h->st>>>(In, rows, rows, l, M, Out, rows, r_dev);
  else apply_rows_kernel<T, 16><<<g, 128, 0, h->st>>>(In, rows, rows, l, M, Out, rows, r_dev);
  return post_launch(h);
}

template <typename T>
frsvt_status apply_fast(frsvt_handle* h, const T* In, int64_t rows, bool m_rows, const T* Msm, T* Out) {
  if (h->l <= AR_LMAX) return apply_rows<T>(h, In, rows, Msm, Out, nullptr);  // narrow: one thread per row
  if constexpr (sizeof(T) == 4) {
    if (tc_small_ok(h, rows, m_rows))  // stream-K pass with K = l: whole tiles per CTA pair
      return tc_pass3<tc::MODE_AX>(h, (const float*)In, rows, rows, h->l, (const float*)Msm, h->l, (float*)Out, rows,
                                   nullptr, 0, 3);
  }
  return apply_small<T>(h, In, rows, rows, Msm, Out, rows);
}

// G = Y^T Y of a nearly orthonormal Y (second CholeskyQR pass): tensor cores
// when eligible (fp32 partials of 3xTF32 products, folded in fp64), else fp64 SIMT
template <typename T>
frsvt_status gram_fast(frsvt_handle* h, const T* Y, int64_t rows, bool m_rows) {
  const bool sharded = m_rows && h->cfg.nranks > 1;
  if constexpr (sizeof(T) == 4) {
    if (tc_small_ok(h, rows, m_rows)) {
      const int l = h->l;
      int S = (int)cdiv(rows, 256);
      if (S > 296) S = 296;
      TRY(tc_AtQ_gen(h, (const float*)Y, rows, rows, l, (const float*)Y, rows, (float*)h->partq, S));
      splitk_reduce_wide_kernel<float, double><<<(unsigned)cdiv((int64_t)l * l, 32), 256, 0, h->st>>>(
          (const float*)h->partq, S, l, l, h->G, l);
      TRY(post_launch(h));
      if (sharded) TRY(allreduce(h, h->G, (size_t)l * l, ncclFloat64, ncclSum));
      return FRSVT_OK;
    }
  }
  return gram<T>(h, Y, rows, rows, sharded);
}

// C (l x l) = op(A) op(B) in fp64 (small multi-CTA product)
template <typename Tout>
frsvt_status gemm_ll(frsvt_handle* h, const double* A, int ta, const double* B, int tb, Tout* C) {
  const int l = h->l;
  const dim3 g((unsigned)cdiv(l, LWD_T), (unsigned)cdiv(l, LWD_T));
  sgemm64_kernel<Tout><<<g, LWD_THREADS, (size_t)2 * LWD_T * l * sizeof(double), h->st>>>(l, l, l, A, l, ta, B, l, tb, C, l);
  return post_launch(h);
}

// the explicit CholeskyQR factor of h->G into T (l x l, ld l): 8 warps up to
// l = 64 (cheaper barriers), 32 warps above
void launch_chol_inv(frsvt_handle* h, const int* r_dev, float* T, unsigned long long* stamps, double* resid) {
  const int l = h->l;
  if (l <= FRSVT_LMAX / 2)
    chol_inv_kernel<float, 8><<<1, CI_THREADS_S, chol_inv_smem_bytes(), h->st>>>(
        h->G, l, r_dev, 1e-12, T, l, &h->dev->s, &h->dev->flags, nullptr, stamps, resid);
  else
    chol_inv_kernel<float, 16><<<1, 512, chol_inv_smem_bytes(), h->st>>>(
        h->G, l, r_dev, 1e-12, T, l, &h->dev->s, &h->dev->flags, nullptr, stamps, resid);
}

// CholeskyQR first pass with the explicit factor T of chol_inv_kernel (one
// barrier per column, no triangular solve) applied by the stream-K tensor-core
// pass. r_dev (range propagation, reading R11): In = [Q~ | Y_p]; only the
// fresh block is factored and, in place (Out == In), Y_p <- (Y_p - Q~ Q~^T Y_p) T22.
frsvt_status orth1_inv(frsvt_handle* h, const float* In, int64_t rows, float* Out, bool m_rows, const int* r_dev) {
  const int l = h->l;
  const bool sharded = m_rows && h->cfg.nranks > 1;
  TRY(gram<float>(h, In, rows, rows, sharded, r_dev));
  launch_chol_inv(h, r_dev, (float*)h->T1, nullptr, h->resid_out);
  h->resid_out = nullptr;  // only the sketch's orthonormalisation reports it
  TRY(post_launch(h));
  if (l <= AR_LMAX) return apply_rows<float>(h, In, rows, (const float*)h->T1, Out, r_dev);
  // r_dev: in place (Out == In): only the fresh columns are written; with
  // p <= 32 on the 32-column instance (the device-side choice of R11)
  if (r_dev && l > 32) {
    int* flags = h->lwd + 8;
    sketch_width_kernel<<<1, 32, 0, h->st>>>(r_dev, l, 32, flags, h->ap_on ? &h->dev->p_ap : nullptr);
    TRY(post_launch(h));
    TRY(tc_pass3<tc::MODE_AX>(h, In, rows, rows, l, (const float*)h->T1, l, Out, rows, nullptr, 0, 3, 0, r_dev,
                              flags + 1));
    return tc_pass3<tc::MODE_AX>(h, In, rows, rows, l, (const float*)h->T1, l, Out, rows, nullptr, 0, 3, 0, r_dev,
                                 flags, 32);
  }
  return tc_pass3<tc::MODE_AX>(h, In, rows, rows, l, (const float*)h->T1, l, Out, rows, nullptr, 0, 3, 0, r_dev);
}

// CholeskyQR, first pass (readings R2/R4/R14 in DESIGN.md): fp64 Gram,
// Cholesky with column drop and explicit factor, fp32-accurate apply. Out =
// Y T1 spans range(Y) and is orthonormal up to ~u kappa(Y): enough wherever
// only the span of the basis matters next (R9), so the second pass runs only
// on the final basis of the range finder (orth_final).
template <typename T>
frsvt_status orth1(frsvt_handle* h, const T* In, int64_t rows, T* Out, bool m_rows) {
  const bool sharded = m_rows && h->cfg.nranks > 1;
  if constexpr (sizeof(T) == 4) {
    if (tc_small_ok(h, rows, m_rows)) return orth1_inv(h, (const float*)In, rows, (float*)Out, m_rows, nullptr);
  }
  TRY(gram<T>(h, In, rows, rows, sharded));
  TRY(chol<T>(h, (T*)h->T1));
  return apply_small<T>(h, In, rows, rows, (const T*)h->T1, Out, rows);
}

// Final basis of the range finder: CholeskyQR2 = orth1 + a second factor T2 of
// the computed Q1 (Loewdin series or Cholesky, fp64). Q1 T2 is never formed:
// T2 is folded into the l x l factors downstream (t2_pending; small_svd,
// shrink_and_factors): B^T = (A^T Q1) T2, Q~ = Q1 (T2 Mc), Wt = (A^T Q1) (T2 Mp).
template <typename T>
frsvt_status orth_final(frsvt_handle* h, const T* In, int64_t rows, T* Out, bool m_rows) {
  TRY(orth1<T>(h, In, rows, Out, m_rows));
  TRY(gram_fast<T>(h, Out, rows, m_rows));
  TRY(chol2<double>(h, h->T2d));
  h->t2_pending = 1;
  return FRSVT_OK;
}

// Y (m x l) = A (m x n) * X (n x l)  [+ Add]. terms (tensor path): 3 exact,
// 2 with the tf32-rounded X (span-only passes, reading R17)
template <typename T>
frsvt_status gemm_AX(frsvt_handle* h, const T* A, int64_t lda, const T* X, T* Y, const T* Add, int terms) {
  if constexpr (sizeof(T) == 4) {
    if (tc_eligible(h, A, lda)) {
      TRY(prof_begin(h));
      TRY(tc_pass3<tc::MODE_AX>(h, (const float*)A, lda, h->m, h->n, (const float*)X, h->n, (float*)Y, h->m,
                                (const float*)Add, h->m, terms));
      return prof_end(h, 0, (double)h->m * h->n * sizeof(T));
    }
  }
  TRY(prof_begin(h));
  if (Add) {
    EpiStoreAdd<T> epi{Y, h->m, Add, h->m};
    TRY((launch_skinny<T, T, true, true>(h, (int)h->m, h->l, (int)h->n, 1, A, lda, X, h->n, nullptr, epi)));
  } else {
    EpiStore<T> epi{Y, h->m, 0};
    TRY((launch_skinny<T, T, true, true>(h, (int)h->m, h->l, (int)h->n, 1, A, lda, X, h->n, nullptr, epi)));
  }
  return prof_end(h, 0, (double)h->m * h->n * sizeof(T));
}

// Z (n x l) = A^T (n x m) * Q (m x l), split-K over rows, all-reduced over
// ranks. terms as in gemm_AX (3 for B^T = A^T Q, which enters X directly)
template <typename T>
frsvt_status gemm_AtQ(frsvt_handle* h, const T* A, int64_t lda, const T* Q, T* Z, int terms) {
  if constexpr (sizeof(T) == 4) {
    if (tc_eligible(h, A, lda)) {
      TRY(prof_begin(h));
      TRY(tc_pass3<tc::MODE_ATQ>(h, (const float*)A, lda, h->n, h->m, (const float*)Q, h->m, (float*)Z, h->n,
                                 nullptr, 0, terms));
      TRY(prof_end(h, 1, (double)h->m * h->n * sizeof(T)));
      TRY(allreduce(h, Z, (size_t)h->n * h->l, nccl_type<T>(), ncclSum));
      return FRSVT_OK;
    }
  }
  const int S = atq_splits(h->n, h->m, h->l);
  EpiStore<T> epi{(T*)h->partq, h->n, (int64_t)h->n * h->l};
  TRY(prof_begin(h));
  TRY((launch_skinny<T, T, false, true>(h, (int)h->n, h->l, (int)h->m, S, A, lda, Q, h->m, nullptr, epi)));
  TRY(prof_end(h, 1, (double)h->m * h->n * sizeof(T)));
  splitk_reduce_kernel<T, T><<<grid1d(h->n * h->l), 256, 0, h->st>>>((const T*)h->partq, S, (int)h->n, h->l, Z, h->n);
  TRY(post_launch(h));
  TRY(allreduce(h, Z, (size_t)h->n * h->l, nccl_type<T>(), ncclSum));
  return FRSVT_OK;
}

// range finder: Q (m x l) spanning (A A^T)^q A Omega' (+ Q~), Alg. 1 lines 3-15
template <typename T>
frsvt_status range_finder(frsvt_handle* h, const T* A, int64_t lda, int q, uint32_t stream,
                          bool use_carry, int64_t call, bool ap = true) {
  const int* pmax = (ap && h->ap_on) ? &h->dev->p_ap : nullptr;  // adaptive rank prediction (Eq. 7)
  const int l = h->l;
  const T* ov = h->override_pending ? (const T*)h->OmOv : nullptr;
  // RP on the stream-K path: multiply only the p fresh columns (Alg. 1 RP
  // branch) and place them behind the carried Q~
  bool rp_front = false;
  if constexpr (sizeof(T) == 4) rp_front = use_carry && tc_eligible(h, A, lda);
  omega_kernel<T><<<grid1d(h->n * l), 256, 0, h->st>>>((T*)h->Om, h->n, l, &h->dev->r, use_carry ? 1 : 0,
                                                       h->cfg.seed, stream + (uint32_t)call, ov, h->n,
                                                       rp_front ? 1 : 0, pmax, h->om_tf32);
  // the first orthonormalisation of the sketch reports the residual of its
  // last sample (tensor path), the Prop. 4 by-product
  CK(cudaMemsetAsync(&h->dev->varsig_raw, 0, sizeof(double), h->st));
  h->resid_out = &h->dev->varsig_raw;
  TRY(post_launch(h));
  h->override_pending = 0;
  if constexpr (sizeof(T) == 4) {
    if (rp_front) {
      // skipped on the device when the previous composition formed Y_p
      // (dev->fs_done); such a launch is not counted in the pass profile
      const int* skip = (h->fs_armed && ov == nullptr) ? &h->dev->fs_done : nullptr;
      if (!skip) TRY(prof_begin(h));
      if (h->l > 32 && !skip) {
        // p = l - r is known only on the device: both the full-width and the
        // 32-column instance are enqueued, each skips unless it is the one
        // for this p (flags[0]: p > 32, flags[1]: p <= 32); the carried
        // columns are copied first (the narrow instance writes the fresh ones)
        int* flags = h->lwd + 8;
        sketch_width_kernel<<<1, 32, 0, h->st>>>(&h->dev->r, h->l, 32, flags, pmax);
        TRY(post_launch(h));
        CK(cudaMemcpyAsync(h->Y, h->Qt, (size_t)h->m * h->l * sizeof(float), cudaMemcpyDeviceToDevice, h->st));
        TRY(tc_pass3<tc::MODE_AX>(h, (const float*)A, lda, h->m, h->n, (const float*)h->Om, h->n, (float*)h->Y,
                                  h->m, nullptr, 0, 2, 0, &h->dev->r, flags + 1));
        TRY(tc_pass3<tc::MODE_AX>(h, (const float*)A, lda, h->m, h->n, (const float*)h->Om, h->n, (float*)h->Y,
                                  h->m, nullptr, 0, 2, 0, &h->dev->r, flags, 32));
      } else {
        TRY(tc_pass3<tc::MODE_AX>(h, (const float*)A, lda, h->m, h->n, (const float*)h->Om, h->n, (float*)h->Y,
                                  h->m, (const float*)h->Qt, h->m, 2, 0, &h->dev->r, skip));
      }
      if (!skip) TRY(prof_end(h, 0, (double)h->m * h->n * sizeof(T)));
    }
  }
  h->fs_armed = false;
  if (!rp_front) TRY(gemm_AX<T>(h, A, lda, (const T*)h->Om, (T*)h->Y, use_carry ? (const T*)h->Qt : nullptr, 2));
  h->t2_pending = 0;
  if (q == 0) {
    TRY(orth_final<T>(h, (const T*)h->Y, h->m, (T*)h->Q, true));
    h->resid_out = nullptr;
    return FRSVT_OK;
  }
  // with range propagation on the tensor path the sketch basis is formed in
  // place in Y: [Q~ | orth(Y_p - Q~ Q~^T Y_p)] (reading R11)
  const T* Qcur = (const T*)h->Q;
  bool rp_orth = false;
  if constexpr (sizeof(T) == 4) rp_orth = rp_front && tc_small_ok(h, h->m, true);
  if (rp_orth) {
    if constexpr (sizeof(T) == 4) TRY(orth1_inv(h, (const float*)h->Y, h->m, (float*)h->Y, true, &h->dev->r));
    Qcur = (const T*)h->Y;
  } else {
    TRY(orth1<T>(h, (const T*)h->Y, h->m, (T*)h->Q, true));
  }
  h->resid_out = nullptr;
  for (int it = 0; it < q; ++it) {
    TRY(gemm_AtQ<T>(h, A, lda, it == 0 ? Qcur : (const T*)h->Q, (T*)h->Z, 2));
    TRY(orth1<T>(h, (const T*)h->Z, h->n, (T*)h->Zq, false));
    TRY(gemm_AX<T>(h, A, lda, (const T*)h->Zq, (T*)h->Y, nullptr, 2));
    if (it + 1 < q) TRY(orth1<T>(h, (const T*)h->Y, h->m, (T*)h->Q, true));
    else TRY(orth_final<T>(h, (const T*)h->Y, h->m, (T*)h->Q, true));
  }
  return FRSVT_OK;
}

// small SVD of the l x l fp64 Gram G (reading Z8): register-resident
// one-sided Jacobi on G (eig_jacobi.cuh); t_mode 0: no shortcut, 1: scalar
// threshold t_host, 2: scalar threshold *t_dev (exact Gershgorin early-out).
frsvt_status launch_eig_jacobi(frsvt_handle* h, const double* G, double* sigma, double* UB, int t_mode,
                               double t_host, const double* t_dev) {
  const int l = h->l;
  // fp64 handles: rotate down to 1e-15 relative, confirm with a clean sweep;
  // fp32 handles: rotate to 1e-9, stop after a sweep that measured <= 1e-4 (R3)
  const double tol_rot = h->esz == 8 ? 1e-15 : 1e-9;
  const double tol_stop = h->esz == 8 ? 0.0 : 1e-4;
  eig_jacobi_launch(h->st, G, l, t_dev, t_host, t_mode, tol_rot, tol_stop, 40, sigma, UB, &h->dev->sweeps,
                    &h->dev->flags);
  return post_launch(h);
}

// B^T = A^T Q, G = B B^T, Jacobi -> sigma, U_B   (Alg. 1 lines 16-18)
template <typename T>
frsvt_status small_svd(frsvt_handle* h, const T* A, int64_t lda, int t_mode = 0, double t_host = 0.0,
                       const double* t_dev = nullptr) {
  TRY(gemm_AtQ<T>(h, A, lda, (const T*)h->Q, (T*)h->Z, 3));
  TRY(gram<T>(h, (const T*)h->Z, h->n, h->n, false));
  if (h->t2_pending) {  // G = T2^T (Z'^T Z') T2 for B^T = Z' T2
    TRY(gemm_ll<double>(h, h->G, 0, h->T2d, 0, h->Hd));
    TRY(gemm_ll<double>(h, h->T2d, 1, h->Hd, 0, h->G));
  }
  if (h->rp != 0 && h->l > EW_P) {
    // warm start (R16): diagonalise the fresh block first, solve the rotated Gram
    // (only for l > EW_P: a cold solve of an l <= 32 Gram costs fewer rounds
    // than the 24- or 32-wide fresh-block solve it would save)
    int* flag = h->lwd + 12;  // [W, W == 24, W == 32] (lwd: [0..3] Loewdin, 4 debug, 7 sweeps scratch, 8..9 sketch)
    eig_fresh_pack_kernel<<<1, 256, 0, h->st>>>(h->G, h->l, &h->dev->r, h->ewbuf, flag);
    TRY(post_launch(h));
    double* Gpad = h->ewbuf;
    double* Uf = Gpad + EW_P * EW_P;
    double* sigf = Uf + EW_P * EW_P;
    double* G2 = sigf + EW_P;
    // fresh-block solve tolerances: those of the main solve (R3; the full
    // solve refines), fp64 handles to 1e-15
    const double ew_rot = h->esz == 4 ? 1e-9 : 1e-15, ew_stop = h->esz == 4 ? 1e-4 : 0.0;
    // the fresh-block solve at width 24 or 32 (whichever the device-side p selected)
    eig_jacobi_launch(h->st, Gpad, 24, nullptr, 0.0, 0, ew_rot, ew_stop, 40, sigf, Uf, h->lwd + 7, &h->dev->flags,
                      flag + 1);
    TRY(post_launch(h));
    eig_jacobi_launch(h->st, Gpad, EW_P, nullptr, 0.0, 0, ew_rot, ew_stop, 40, sigf, Uf, h->lwd + 7, &h->dev->flags,
                      flag + 2);
    TRY(post_launch(h));
    eig_fresh_rotate_kernel<<<(unsigned)cdiv((int64_t)h->l * h->l, 256), 256, 0, h->st>>>(h->G, h->l, &h->dev->r,
                                                                                          Uf, flag, G2);
    TRY(post_launch(h));
    TRY(launch_eig_jacobi(h, G2, h->sigma, h->UB, t_mode, t_host, t_dev));
    eig_fresh_back_kernel<<<(unsigned)cdiv(h->l, 128), 128, 0, h->st>>>(h->UB, h->l, &h->dev->r, Uf, flag);
    return post_launch(h);
  }
  return launch_eig_jacobi(h, h->G, h->sigma, h->UB, t_mode, t_host, t_dev);
}

// shrink + factors: Q~ = Q Mc, Wt = B^T Mp (Eq. 6 with the kept set)
template <typename T>
frsvt_status shrink_and_factors(frsvt_handle* h, int wmode, double tau, const double* tau_dev,
                                double C, double eps) {
  const int l = h->l;
  if (h->t2_pending) {  // Mc = T2 (U_B)_K, Mp = T2 (U_B)_K diag(d/sigma)
    shrink_kernel<double><<<1, 1024, 0, h->st>>>(h->sigma, h->UB, l, &h->dev->s, wmode, tau, tau_dev, h->wvec, C,
                                                eps, h->dprev, &h->dev->have_prev, h->McD, h->MpD, &h->dev->r,
                                                &h->dev->flags, h->dev->rep, h->keep);
    TRY(post_launch(h));
    TRY(gemm_ll<T>(h, h->T2d, 0, h->McD, 0, (T*)h->Mc));
    TRY(gemm_ll<T>(h, h->T2d, 0, h->MpD, 0, (T*)h->Mp));
  } else {
    shrink_kernel<T><<<1, 1024, 0, h->st>>>(h->sigma, h->UB, l, &h->dev->s, wmode, tau, tau_dev, h->wvec,
                                           C, eps, h->dprev, &h->dev->have_prev, (T*)h->Mc, (T*)h->Mp,
                                           &h->dev->r, &h->dev->flags, h->dev->rep, h->keep);
    TRY(post_launch(h));
  }
  TRY(apply_fast<T>(h, (const T*)h->Q, h->m, true, (const T*)h->Mc, (T*)h->Qt));
  TRY(apply_fast<T>(h, (const T*)h->Z, h->n, false, (const T*)h->Mp, (T*)h->Wt));
  return FRSVT_OK;
}

template <typename T>
frsvt_status frsvt_core(frsvt_handle* h, const T* A, int64_t lda, int wmode, double tau,
                        const double* tau_dev, double C, double eps) {
  {
    NvtxRange nv("frsvt.range_finder");
    TRY(range_finder<T>(h, A, lda, h->q, 1000u, h->rp != 0, h->call));
  }
  NvtxRange nv("frsvt.small_svd+shrink");
  // exact early-out of the small SVD when every sigma is certified <= the
  // smallest threshold (scalar tau, or the smallest explicit weight)
  // (partial SVT, keep > 0: t_min = 0, no shortcut and the standard Jacobi measure)
  if (wmode == 0 && h->keep > 0) TRY(small_svd<T>(h, A, lda));
  else if (wmode == 0) TRY(small_svd<T>(h, A, lda, tau_dev ? 2 : 1, tau, tau_dev));
  else if (wmode == 1) TRY(small_svd<T>(h, A, lda, 1, tau));
  else TRY(small_svd<T>(h, A, lda));
  TRY(shrink_and_factors<T>(h, wmode, tau, tau_dev, C, eps));
  if (h->ap_on) {
    ap_update_kernel<<<1, 32, 0, h->st>>>(h->dev, h->ap_a, h->ap_jump, h->ap_b);
    TRY(post_launch(h));
  }
  h->call++;
  return FRSVT_OK;
}

// X = Q~ Wt^T  (reconstruction, K = r)
template <typename T>
frsvt_status compose_X(frsvt_handle* h, T* X, int64_t ldx) {
  NvtxRange nv("frsvt.compose");
  if constexpr (sizeof(T) == 4) {
    if (h->use_tc) {
      TRY(prof_begin(h));
      TRY(tc_compose(h, tc::EPI_STORE, (float*)X, ldx, nullptr, nullptr, nullptr, 0, 0.0, 0.0, nullptr));
      return prof_end(h, 2, (double)h->m * h->n * sizeof(T));
    }
  }
  EpiStore<T> epi{X, ldx, 0};
  TRY(prof_begin(h));
  TRY((launch_tile<T, T, 128, 128, 16, 8, 8, true, false>(h, (int)h->m, (int)h->n, h->l, 1,
                                                         (const T*)h->Qt, h->m, (const T*)h->Wt,
                                                         h->n, &h->dev->r, epi)));
  return prof_end(h, 2, (double)h->m * h->n * sizeof(T));
}

frsvt_status fill_info(frsvt_handle* h, frsvt_info* info) {
  if (!info) return FRSVT_OK;
  CK(cudaStreamSynchronize(h->st));
  DevState ds;
  CK(cudaMemcpy(&ds, h->dev, sizeof(DevState), cudaMemcpyDeviceToHost));
  memset(info, 0, sizeof(*info));
  info->s = ds.s;
  info->r = ds.r;
  info->flags = ds.flags | (h->single_cta ? FRSVT_FLAG_SINGLE_CTA : 0);
  info->sweeps = ds.sweeps;
  info->calls = h->call;
  info->mu = ds.mu[0];
  info->l_next = h->ap_on ? ds.l_act : h->l;
  info->varsigma = 20.0 * sqrt(2.0 / M_PI) * ds.varsig_raw;
  for (int i = 0; i < FRSVT_LMAX; ++i) {
    info->sigma[i] = i < h->l ? ds.rep[i] : 0.0;
    info->d[i] = i < h->l ? ds.rep[FRSVT_LMAX + i] : 0.0;
  }
  if (ds.flags & FLAG_NONFINITE) return FRSVT_ENONFINITE;
  return FRSVT_OK;
}

// A call small enough for one SM (BASELINE c1: 200 x 100, l = 10) runs all of
// Algorithm 1 in one CTA's shared memory (batched.cuh with batch 1): no range
// propagation, one rank, plain or explicit-weight thresholds, l <= 16.
template <typename T>
bool single_cta_ok(const frsvt_handle* h, int wmode) {
  return !h->rp && h->cfg.nranks == 1 && h->group == nullptr && !h->ap_on && h->keep == 0 &&
         (wmode == 0 || wmode == 1) && bt_fits(h->m, h->n, h->l, (int)sizeof(T));
}

template <typename T>
frsvt_status single_cta_apply(frsvt_handle* h, const T* A, int64_t lda, int wmode, double tau, T* X,
                              int64_t ldx) {
  NvtxRange nv("frsvt.single_cta");
  // Omega: the override, else drawn inside the kernel (same generator and
  // stream as omega_kernel)
  const T* ov = h->override_pending ? (const T*)h->OmOv : nullptr;
  h->override_pending = 0;
  DevState* d = h->dev;
  BtArgs a{};
  a.m = (int)h->m;
  a.n = (int)h->n;
  a.l = h->l;
  a.q = h->q;
  a.A = A;
  a.lda = lda;
  a.Om = ov;
  a.ldo = h->n;
  a.om_seed = h->cfg.seed;
  a.om_stream = 1000u + (uint32_t)h->call;
  a.wmode = wmode;
  a.tau = tau;
  a.w = h->wvec;
  a.X = X;
  a.ldx = ldx;
  a.r_b = &d->r;
  a.sig_b = d->rep;
  a.d_b = d->rep + FRSVT_LMAX;
  a.s_b = &d->s;
  a.sweeps_b = &d->sweeps;
  a.vs_b = &d->varsig_raw;
  a.flags = &d->flags;
  a.flags_store = 1;
  TRY(prof_begin(h));
  CK(bt_launch<T>(a, 1, h->st));
  TRY(post_launch(h));
  TRY(prof_end(h, 3, 2.0 * (double)h->m * h->n * h->l * (2 * h->q + 3)));
  h->call++;
  return FRSVT_OK;
}

template <typename T>
frsvt_status apply_impl(frsvt_handle* h, const void* A, int64_t lda, int wmode, double tau,
                        const double* w_host, double C, double eps, void* X, int64_t ldx,
                        frsvt_info* info) {
  if (wmode == 1) {
    CK(cudaMemcpyAsync(h->wvec, w_host, sizeof(double) * h->l, cudaMemcpyHostToDevice, h->st));
    tau = w_host[0];  // smallest explicit threshold (the small SVD's exact early-out)
    for (int i = 1; i < h->l; ++i) tau = fmin(tau, w_host[i]);
  }
  h->keep = 0;  // partial SVT (keep) belongs to rpca_state only
  h->single_cta = single_cta_ok<T>(h, wmode) ? 1 : 0;
  if (!h->single_cta) CK(cudaMemsetAsync(&h->dev->flags, 0, sizeof(int), h->st));
  if (h->single_cta) {
    TRY(single_cta_apply<T>(h, (const T*)A, lda, wmode, tau, (T*)X, ldx));
    return fill_info(h, info);
  }
  TRY(frsvt_core<T>(h, (const T*)A, lda, wmode, tau, nullptr, C, eps));
  TRY(compose_X<T>(h, (T*)X, ldx));
  return fill_info(h, info);
}

// Power steps of the ||D||_2 estimate: c5's spectrum is flat at the top
// (sigma_1..4 = 447.8, 447.1, 446.9, 446.6), where 6 steps under-estimate by 3%;
// 24 steps are within 0.3% (446.7 vs 447.8, scripts/norm2_check.py).
#define FRSVT_NORM2_Q 24
// ||D||_2 estimate: block power (Rayleigh-Ritz on l columns), used only when
// the caller does not supply ||D||_2 (reading Z10). Writes sigma[0].
template <typename T>
frsvt_status estimate_norm2(frsvt_handle* h, const T* D, int64_t ld) {
  CK(cudaMemsetAsync(&h->dev->r, 0, sizeof(int), h->st));
  TRY(range_finder<T>(h, D, ld, FRSVT_NORM2_Q, 999u, false, 0, false));
  TRY(small_svd<T>(h, D, ld));
  return FRSVT_OK;
}

template <typename T>
frsvt_status rpca_impl(frsvt_handle* h, rpca_state* st, int finalize, double* rel_resid) {
  const double lambda = st->lambda > 0 ? st->lambda : 1.0 / sqrt((double)(h->cfg.m_global > h->n ? h->cfg.m_global : h->n));
  const T* D = (const T*)st->D;
  T* E = (T*)st->E;
  T* A = (T*)st->A;
  CK(cudaMemsetAsync(&h->dev->flags, 0, sizeof(int), h->st));
  h->keep = st->keep;
  h->single_cta = 0;
  if (st->iter == 0) {
    // ---- init: norms, mu_0, Y_0, E_1, A_1 ----
    const int nb = grid1d(h->m * h->n);
    absmax_sumsq_kernel<T><<<nb, 256, 0, h->st>>>(D, h->m, h->n, st->ld, h->redpart, h->redpart + nb);
    TRY(post_launch(h));
    fold_kernel<<<1, 256, 0, h->st>>>(h->redpart, h->redpart + nb, nb, &h->dev->dmax, &h->dev->dss);
    TRY(post_launch(h));
    TRY(allreduce(h, &h->dev->dmax, 1, ncclFloat64, ncclMax));
    TRY(allreduce(h, &h->dev->dss, 1, ncclFloat64, ncclSum));
    if (!(st->norm2_D > 0)) TRY(estimate_norm2<T>(h, D, st->ld));
    alm_scalars_kernel<<<1, 1, 0, h->st>>>(st->norm2_D, h->sigma, st->mu0, st->mu_max_factor, lambda,
                                           &h->dev->dmax, h->dev->mu, h->dev->scal);
    TRY(post_launch(h));
    alm_init_kernel<T><<<nb, 256, 0, h->st>>>(D, E, A, h->m, h->n, st->ld, h->dev->mu, h->dev->scal, lambda);
    TRY(post_launch(h));
    // fresh solve: empty carry (unless the basis is transferred from the
    // previous solve: the semi-online windows of P:645), Omega sequence
    // restarts at call 0
    if (!st->transfer) {
      CK(cudaMemsetAsync(&h->dev->r, 0, sizeof(int), h->st));
      CK(cudaMemsetAsync(h->Qt, 0, (size_t)h->m * h->l * h->esz, h->st));
    }
    CK(cudaMemsetAsync(&h->dev->have_prev, 0, sizeof(int), h->st));
    if (h->ap_on) {
      ap_reset_kernel<<<1, 32, 0, h->st>>>(h->dev, h->ap_l0);
      TRY(post_launch(h));
    }
    h->call = 0;
    h->fs_armed = false;
  }
  tau_from_mu_kernel<<<1, 1, 0, h->st>>>(h->dev->mu, &h->dev->tau);
  TRY(post_launch(h));
  TRY(frsvt_core<T>(h, A, st->ld, 0, 0.0, &h->dev->tau, 0.0, 0.0));
  // fused reconstruction + iALM epilogue (one pass over D, A, E)
  NvtxRange nv("rpca.epilogue");
  int nparts = (int)(cdiv(h->m, 128) * cdiv(h->n, 128));
  TRY(prof_begin(h));
  bool done = false;
  if constexpr (sizeof(T) == 4) {
    if (h->use_tc) {
      // fused next sketch: the next call's Omega and the carried columns of Y
      // are set up here; the composition forms Y_p when p = l - r <= FS_PMAX
      // (device-side decision) and the next sketch pass is then skipped
      const bool fs_next = !finalize && h->fs && h->rp != 0 && h->cfg.nranks == 1 &&
                           tc_eligible(h, A, st->ld) && !h->override_pending;
      if (fs_next) {
        omega_kernel<float><<<grid1d(h->n * h->l), 256, 0, h->st>>>((float*)h->Om, h->n, h->l, &h->dev->r, 1,
                                                                    h->cfg.seed, 1000u + (uint32_t)h->call, nullptr,
                                                                    h->n, 1, h->ap_on ? &h->dev->p_ap : nullptr,
                                                                    h->om_tf32);
        TRY(post_launch(h));
        CK(cudaMemcpyAsync(h->Y, h->Qt, (size_t)h->m * h->l * sizeof(float), cudaMemcpyDeviceToDevice, h->st));
      }
      TRY(tc_compose(h, finalize ? tc::EPI_FINAL : tc::EPI_ALM, (float*)st->L, st->ld, (const float*)D, (float*)A,
                     (float*)E, st->ld, st->rho, lambda, &nparts, fs_next));
      done = true;
    }
  }
  if (!done) {
    EpiAlm<T> epi{D, A, E, (T*)st->L, st->ld, h->dev->mu, st->rho, lambda, finalize, h->redpart};
    TRY((launch_tile<T, T, 128, 128, 16, 8, 8, true, false>(h, (int)h->m, (int)h->n, h->l, 1,
                                                           (const T*)h->Qt, h->m, (const T*)h->Wt, h->n,
                                                           &h->dev->r, epi)));
  }
  TRY(prof_end(h, 2, (double)h->m * h->n * sizeof(T) * (finalize ? 3.0 : 5.0)));
  fold_sum_kernel<<<1, 256, 0, h->st>>>(h->redpart, nparts, &h->dev->resid[0]);
  TRY(post_launch(h));
  TRY(allreduce(h, &h->dev->resid[0], 1, ncclFloat64, ncclSum));
  alm_mu_kernel<<<1, 1, 0, h->st>>>(st->rho, finalize, h->dev->mu, &h->dev->dss, h->dev->resid);
  TRY(post_launch(h));
  if (!finalize) st->iter++;
  if (rel_resid) {
    CK(cudaStreamSynchronize(h->st));
    CK(cudaMemcpy(rel_resid, &h->dev->resid[1], sizeof(double), cudaMemcpyDeviceToHost));
  }
  return FRSVT_OK;
}

// dynamic shared-memory limits of every kernel that needs more than 48 KB,
// set for the current device (attributes are per device; frsvt_create runs
// this on the handle's device)
frsvt_status set_smem_attrs() {
#define FRSVT_ATTR(K, BYTES) CK(cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(BYTES)))
  FRSVT_ATTR(orth_chol_kernel<float>, orth_chol_smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(orth_chol_kernel<double>, orth_chol_smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(sgemm64_kernel<float>, lowdin_smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(sgemm64_kernel<double>, lowdin_smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(lowdin_sq_kernel, lowdin_smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(lowdin_series_kernel<float>, lowdin_smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(lowdin_series_kernel<double>, lowdin_smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(eig_jacobi_kernel<8>, EigJacobi::smem_bytes(FRSVT_LMAX));
  FRSVT_ATTR(eig_jacobi_kernel<4>, EigJacobi::smem_bytes(40));
  FRSVT_ATTR((chol_inv_kernel<float, 16>), chol_inv_smem_bytes());
  FRSVT_ATTR((chol_inv_kernel<float, 8>), chol_inv_smem_bytes());
  CK(bt_set_attrs<float>());  // single-CTA path and frsvt_batched_apply
  CK(bt_set_attrs<double>());
  FRSVT_ATTR((tc::tc_pass_kernel<tc::MODE_ATQ, 32>), tc::PassSmem::total(32));
  FRSVT_ATTR((tc::tc_pass_kernel<tc::MODE_ATQ, 64>), tc::PassSmem::total(64));
  FRSVT_ATTR((tc::tc_pass_kernel<tc::MODE_ATQ, 128>), tc::PassSmem::total(128));
#define FRSVT_ATTR3(MODE, NPV, TV) FRSVT_ATTR((tc::tc_pass3_kernel<MODE, NPV, TV>), tc::Pass3Smem::total(NPV, TV))
  FRSVT_ATTR3(tc::MODE_AX, 32, 2);
  FRSVT_ATTR3(tc::MODE_AX, 64, 2);
  FRSVT_ATTR3(tc::MODE_AX, 128, 2);
  FRSVT_ATTR3(tc::MODE_AX, 32, 3);
  FRSVT_ATTR3(tc::MODE_AX, 64, 3);
  FRSVT_ATTR3(tc::MODE_AX, 128, 3);
  FRSVT_ATTR3(tc::MODE_ATQ, 32, 2);
  FRSVT_ATTR3(tc::MODE_ATQ, 64, 2);
  FRSVT_ATTR3(tc::MODE_ATQ, 128, 2);
  FRSVT_ATTR3(tc::MODE_ATQ, 32, 3);
  FRSVT_ATTR3(tc::MODE_ATQ, 64, 3);
  FRSVT_ATTR3(tc::MODE_ATQ, 128, 3);
#undef FRSVT_ATTR3
  FRSVT_ATTR((tc::tc_compose2_kernel<tc::EPI_ALM, false>), tc::Compose2Smem::total());
  FRSVT_ATTR((tc::tc_compose2_kernel<tc::EPI_ALM, true>), tc::Compose2Smem::total());
  FRSVT_ATTR((tc::tc_compose2_kernel<tc::EPI_FINAL, false>), tc::Compose2Smem::total());
  FRSVT_ATTR((tc::tc_compose2_kernel<tc::EPI_STORE, false>), tc::Compose2Smem::total());
  FRSVT_ATTR(tc::tc_compose_kernel<tc::EPI_STORE>, tc::ComposeSmem::total());
  FRSVT_ATTR(tc::tc_compose_kernel<tc::EPI_ALM>, tc::ComposeSmem::total());
  FRSVT_ATTR(tc::tc_compose_kernel<tc::EPI_FINAL>, tc::ComposeSmem::total());
#undef FRSVT_ATTR
  return FRSVT_OK;
}

}  // namespace

// Multi-rank handles: the pass route (tensor cores vs SIMT, and with it the
// range-propagation bookkeeping) depends on the operand's alignment, so every
// rank must see a TMA-compatible operand (16-byte aligned, ld % 4 == 0) on the
// tensor path; anything else would make ranks build different bases.
static bool rank_uniform_layout(const frsvt_handle* h, const void* A, int64_t lda) {
  return h->cfg.nranks <= 1 || !h->use_tc || tc_eligible(h, A, lda);
}

// ============================================================== C ABI
// frsvt_batched_apply / _f64: validation and one launch of the one-CTA kernel
template <typename T>
static frsvt_status batched_apply_t(int32_t batch, int64_t m, int64_t n, int32_t l, int32_t q, const T* A, int64_t lda,
                                    int64_t strideA, const T* Omega, int64_t ldo, int32_t wmode, double tau,
                                    const double* tau_batch, const double* w, T* X, int64_t ldx, int64_t strideX,
                                    int32_t* r_out, double* sigma_out, void* cuda_stream) {
  if (batch < 0 || m < 1 || n < 1 || l < 1 || l > BT_LMAX || l > m || l > n || q < 0 || q > 16) return FRSVT_EINVAL;
  if (lda < m || ldx < m || ldo < n || strideA < lda * n || strideX < ldx * n) return FRSVT_EINVAL;
  if (batch == 0) return FRSVT_OK;  // nothing to do (the pointers may be NULL)
  if (!A || !Omega || !X) return FRSVT_EINVAL;
  if (wmode == 0) {
    if (!tau_batch && (!(tau >= 0) || !std::isfinite(tau))) return FRSVT_EINVAL;
  } else if (wmode == 1) {
    if (!w) return FRSVT_EINVAL;
  } else {
    return FRSVT_EINVAL;
  }
  if (!bt_fits(m, n, l, (int)sizeof(T))) return FRSVT_EINVAL;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  CK(bt_set_attrs<T>());
  BtArgs a{};
  a.m = (int)m;
  a.n = (int)n;
  a.l = l;
  a.q = q;
  a.A = A;
  a.lda = lda;
  a.strideA = strideA;
  a.Om = Omega;
  a.ldo = ldo;
  a.wmode = wmode;
  a.tau = tau;
  a.tau_b = tau_batch;
  a.w = w;
  a.X = X;
  a.ldx = ldx;
  a.strideX = strideX;
  a.r_b = r_out;
  a.sig_b = sigma_out;
  CK(bt_launch<T>(a, batch, st));
  return FRSVT_OK;
}

extern "C" {

const char* frsvt_status_string(frsvt_status s) {
  switch (s) {
    case FRSVT_OK: return "ok";
    case FRSVT_EINVAL: return "invalid argument";
    case FRSVT_ENOCONV: return "Jacobi sweep cap reached";
    case FRSVT_ECUDA: return "CUDA error";
    case FRSVT_ENCCL: return "NCCL error";
    case FRSVT_ENONFINITE: return "non-finite value reached a Gram diagonal";
    case FRSVT_ENOMEM: return "out of device memory";
  }
  return "unknown status";
}

frsvt_status frsvt_batched_apply(int32_t batch, int64_t m, int64_t n, int32_t l, int32_t q, const float* A,
                                 int64_t lda, int64_t strideA, const float* Omega, int64_t ldo, int32_t wmode,
                                 double tau, const double* tau_batch, const double* w, float* X, int64_t ldx,
                                 int64_t strideX, int32_t* r_out, double* sigma_out, void* cuda_stream) {
  return batched_apply_t<float>(batch, m, n, l, q, A, lda, strideA, Omega, ldo, wmode, tau, tau_batch, w, X, ldx,
                                strideX, r_out, sigma_out, cuda_stream);
}

frsvt_status frsvt_batched_apply_f64(int32_t batch, int64_t m, int64_t n, int32_t l, int32_t q, const double* A,
                                     int64_t lda, int64_t strideA, const double* Omega, int64_t ldo, int32_t wmode,
                                     double tau, const double* tau_batch, const double* w, double* X, int64_t ldx,
                                     int64_t strideX, int32_t* r_out, double* sigma_out, void* cuda_stream) {
  return batched_apply_t<double>(batch, m, n, l, q, A, lda, strideA, Omega, ldo, wmode, tau, tau_batch, w, X, ldx,
                                 strideX, r_out, sigma_out, cuda_stream);
}

frsvt_status frsvt_loopback_create(int32_t nranks, frsvt_group** out) {
  if (!out) return FRSVT_EINVAL;
  *out = nullptr;
  if (nranks < 1 || nranks > FRSVT_LOOPBACK_MAX) return FRSVT_EINVAL;
  frsvt_group* g = new (std::nothrow) frsvt_group();
  if (!g) return FRSVT_ENOMEM;
  g->n = nranks;
  if (cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    delete g;
    return FRSVT_ECUDA;
  }
  *out = g;
  return FRSVT_OK;
}

void frsvt_loopback_destroy(frsvt_group* g) {
  if (!g) return;
  if (g->done) cudaEventDestroy(g->done);
  delete g;
}

frsvt_status frsvt_get_unique_id(unsigned char out[128]) {
  if (!out) return FRSVT_EINVAL;
  ncclUniqueId id;
  CKN(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(out, &id, 128);
  return FRSVT_OK;
}

static void free_handle(frsvt_handle* h) {
  if (!h) return;
  void* ptrs[] = {h->Om, h->OmOv, h->Y, h->Q, h->Qtmp, h->Qt, h->Z, h->Zq, h->Zt, h->Wt, h->T1, h->Mc,
                  h->Mp, h->wvec, h->Xh, h->Xl, h->Qh, h->Ql, h->QtTh, h->QtTl, h->WtTh, h->WtTl, h->partq, h->partd, h->redpart, h->skpart, h->Xb, h->Qb, h->tilecnt, h->fspart, h->OmT, h->ewbuf, h->E2b, h->Rf, h->T2d, h->Hd, h->McD, h->MpD, h->lwd, h->G, h->UB, h->sigma, h->dprev,
                  h->redtmp, h->dev};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->ev_ready) cudaEventDestroy(h->ev_ready);
  if (h->prof_ev) {
    for (cudaEvent_t e : *h->prof_ev) cudaEventDestroy(e);
    delete h->prof_ev;
  }
  delete h->prof_kind;
  delete h;
}

frsvt_status frsvt_create(const frsvt_config* cfg, void* cuda_stream, frsvt_handle** out) {
  if (!out) return FRSVT_EINVAL;
  *out = nullptr;
  if (!cfg) return FRSVT_EINVAL;
  const frsvt_config& c = *cfg;
  if (c.dtype != FRSVT_F32 && c.dtype != FRSVT_F64) return FRSVT_EINVAL;
  if ((c.options & FRSVT_OPT_TF32_OMEGA) && c.dtype != FRSVT_F32) return FRSVT_EINVAL;
  if (c.m_local < 1 || c.n < 1 || c.m_global < c.m_local || c.row0 < 0 || c.row0 + c.m_local > c.m_global)
    return FRSVT_EINVAL;
  if (c.l < 1 || c.l > FRSVT_LMAX || c.l > c.n || c.l > c.m_global || c.l > c.m_local) return FRSVT_EINVAL;
  if (c.q < 0 || c.q > 64) return FRSVT_EINVAL;
  if (c.nranks < 1 || c.rank < 0 || c.rank >= c.nranks) return FRSVT_EINVAL;
  if (c.nranks == 1 && c.m_local != c.m_global) return FRSVT_EINVAL;
  if (c.nranks > 1 && !c.nccl_id && !c.group) return FRSVT_EINVAL;
  if (c.group && (c.group->n != c.nranks || c.nranks > FRSVT_LOOPBACK_MAX)) return FRSVT_EINVAL;
  if (c.m_local > (int64_t)INT32_MAX || c.n > (int64_t)INT32_MAX) return FRSVT_EINVAL;

  frsvt_handle* h = new (std::nothrow) frsvt_handle();
  if (!h) return FRSVT_ENOMEM;
  memset(h, 0, sizeof(*h));
  h->cfg = c;
  h->cfg.nccl_id = nullptr;
  h->st = (cudaStream_t)cuda_stream;
  cudaGetDevice(&h->dev_id);
  h->esz = c.dtype == FRSVT_F32 ? 4 : 8;
  h->l = c.l;
  h->q = c.q;
  h->rp = c.range_propagation ? 1 : 0;
  h->m = c.m_local;
  h->n = c.n;
  h->prof_ev = new (std::nothrow) std::vector<cudaEvent_t>();
  h->prof_kind = new (std::nothrow) std::vector<int>();
  if (!h->prof_ev || !h->prof_kind) {
    free_handle(h);
    return FRSVT_ENOMEM;
  }
  const int l = c.l;
  const size_t ml = (size_t)h->m * l * h->esz, nl = (size_t)h->n * l * h->esz, ll = (size_t)l * l * h->esz;
  const int S_atq = atq_splits(h->n, h->m, l);
  h->partq_elems = (size_t)S_atq * h->n * l;
  if (h->partq_elems < (size_t)296 * l * l) h->partq_elems = (size_t)296 * l * l;
  const int64_t maxrows = h->m > h->n ? h->m : h->n;
  h->partd_elems = (size_t)(gram_splits(maxrows) > 2 * 148 ? gram_splits(maxrows) : 2 * 148) * l * l;
  const int64_t gx = cdiv(h->m, 128), gy = cdiv(h->n, 128);
  h->redpart_elems = (size_t)(gx * gy > 2 * 148 * 16 ? gx * gy : 2 * 148 * 16) + 64;
  struct {
    void** p;
    size_t bytes;
  } allocs[] = {{&h->Om, nl},          {&h->OmOv, nl},         {&h->Y, ml},
                {&h->Q, ml},           {&h->Qtmp, ml},         {&h->Qt, ml},
                {&h->Z, nl},           {&h->Zq, nl},           {&h->Zt, nl},
                {&h->Wt, nl},          {&h->T1, ll},           {&h->Mc, ll},
                {&h->Mp, ll},          {(void**)&h->wvec, sizeof(double) * FRSVT_LMAX},
                {&h->partq, h->partq_elems * h->esz},
                {(void**)&h->partd, h->partd_elems * sizeof(double)},
                {(void**)&h->redpart, h->redpart_elems * sizeof(double)},
                {(void**)&h->G, sizeof(double) * l * l},
                {(void**)&h->E2b, sizeof(double) * l * l},
                {(void**)&h->Rf, sizeof(double) * l * l},
                {(void**)&h->T2d, sizeof(double) * l * l},
                {(void**)&h->Hd, sizeof(double) * l * l},
                {(void**)&h->McD, sizeof(double) * l * l},
                {(void**)&h->MpD, sizeof(double) * l * l},
                {(void**)&h->lwd, sizeof(int) * (FRSVT_LMAX + 4)},
                {(void**)&h->UB, sizeof(double) * l * l},
                {(void**)&h->sigma, sizeof(double) * FRSVT_LMAX},
                {(void**)&h->dprev, sizeof(double) * FRSVT_LMAX},
                {(void**)&h->redtmp, sizeof(double) * 64},
                {(void**)&h->dev, sizeof(DevState)},
                {(void**)&h->Xh, c.dtype == FRSVT_F32 ? (size_t)cdiv(maxrows, 4) * 4 * l * 4 : 16},
                {(void**)&h->Xl, c.dtype == FRSVT_F32 ? (size_t)cdiv(maxrows, 4) * 4 * l * 4 : 16},
                {(void**)&h->Qh, c.dtype == FRSVT_F32 ? (size_t)cdiv(maxrows, 4) * 4 * l * 4 : 16},
                {(void**)&h->Ql, c.dtype == FRSVT_F32 ? (size_t)cdiv(maxrows, 4) * 4 * l * 4 : 16},
                {(void**)&h->QtTh, c.dtype == FRSVT_F32 ? (size_t)h->m * cdiv(l, 32) * 32 * 4 : 16},
                {(void**)&h->QtTl, c.dtype == FRSVT_F32 ? (size_t)h->m * cdiv(l, 32) * 32 * 4 : 16},
                {(void**)&h->WtTh, c.dtype == FRSVT_F32 ? (size_t)h->n * cdiv(l, 32) * 32 * 4 : 16},
                {(void**)&h->WtTl, c.dtype == FRSVT_F32 ? (size_t)h->n * cdiv(l, 32) * 32 * 4 : 16}};
  for (auto& a : allocs) {
    if (cudaMalloc(a.p, a.bytes) != cudaSuccess) {
      cudaGetLastError();
      free_handle(h);
      return FRSVT_ENOMEM;
    }
  }
  cudaMemset(h->Qt, 0, ml);
  h->ldxs = cdiv(maxrows, 4) * 4;
  h->Kp = (int)cdiv(l, 32) * 32;
  h->ldqs = cdiv(maxrows, 4) * 4;
  h->ldb16 = cdiv(maxrows, tc::BK) * 2 * tc::BK;
  {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm < 1) nsm = 148;
    if (nsm > 256) nsm = 256;  // stream-K fixup resolves <= 256 covering CTAs per tile
    h->nsm = nsm;
    if (cudaMalloc((void**)&h->ewbuf, sizeof(double) * (2 * EW_P * EW_P + EW_P + (size_t)l * l)) != cudaSuccess) {
      cudaGetLastError();
      free_handle(h);
      return FRSVT_ENOMEM;
    }
    h->fs = (c.options & FRSVT_OPT_FUSED_SKETCH) ? 1 : 0;
    h->om_tf32 = (c.options & FRSVT_OPT_TF32_OMEGA) ? 1 : 0;
    h->fs_armed = false;
    h->fspart_ctas = (size_t)cdiv(maxrows, 128) + 2 * (size_t)h->nsm + 8;
    if (cudaMalloc((void**)&h->fspart, sizeof(float) * tc::FS_PMAX * 128 * h->fspart_ctas) != cudaSuccess ||
        cudaMalloc((void**)&h->OmT, sizeof(float) * tc::FS_PMAX * (size_t)h->n) != cudaSuccess) {
      cudaGetLastError();
      free_handle(h);
      return FRSVT_ENOMEM;
    }
    h->ncnt = (int)cdiv(maxrows, 128) + 8;
    if (cudaMalloc((void**)&h->tilecnt, sizeof(unsigned int) * h->ncnt) != cudaSuccess ||
        cudaMemset(h->tilecnt, 0, sizeof(unsigned int) * h->ncnt) != cudaSuccess) {
      cudaGetLastError();
      free_handle(h);
      return FRSVT_ENOMEM;
    }
    if (c.dtype == FRSVT_F32 &&
        (cudaMalloc((void**)&h->skpart, (size_t)nsm * tc::P3_SLOTS * 128 * 128 * sizeof(float)) != cudaSuccess ||
         cudaMalloc((void**)&h->Xb, (size_t)h->ldb16 * l * 2) != cudaSuccess ||
         cudaMalloc((void**)&h->Qb, (size_t)h->ldb16 * l * 2) != cudaSuccess)) {
      cudaGetLastError();
      free_handle(h);
      return FRSVT_ENOMEM;
    }
  }
  h->use_tc = (c.dtype == FRSVT_F32) && tma_encode_available();
  h->tc_m = tc_small_local(h, h->m) ? 1 : 0;
  cudaMemset(h->dev, 0, sizeof(DevState));
  cudaMemset(h->sigma, 0, sizeof(double) * FRSVT_LMAX);
  cudaMemset(h->dprev, 0, sizeof(double) * FRSVT_LMAX);
  if (set_smem_attrs() != FRSVT_OK) {
    free_handle(h);
    return FRSVT_ECUDA;
  }
  if (c.nranks > 1) {
    if (c.group) {
      h->group = c.group;
      if (cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        free_handle(h);
        return FRSVT_ECUDA;
      }
    } else {
      ncclUniqueId id;
      memcpy(&id, c.nccl_id, 128);
      if (ncclCommInitRank(&h->comm, c.nranks, id, c.rank) != ncclSuccess) {
        free_handle(h);
        return FRSVT_ENCCL;
      }
    }
    // rank-uniform path choices (the tensor-core orthonormalisation of the
    // m-row matrices depends on m_local): agree on the minimum over ranks
    int* flag = h->lwd + 6;
    if (cudaMemcpyAsync(flag, &h->tc_m, sizeof(int), cudaMemcpyHostToDevice, h->st) != cudaSuccess ||
        allreduce(h, flag, 1, ncclInt32, ncclMin) != FRSVT_OK ||
        cudaMemcpyAsync(&h->tc_m, flag, sizeof(int), cudaMemcpyDeviceToHost, h->st) != cudaSuccess ||
        cudaStreamSynchronize(h->st) != cudaSuccess) {
      cudaGetLastError();
      free_handle(h);
      return FRSVT_ENCCL;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    free_handle(h);
    return FRSVT_ECUDA;
  }
  *out = h;
  return FRSVT_OK;
}

void frsvt_destroy(frsvt_handle* h) {
  if (!h) return;
  cudaStreamSynchronize(h->st);
  free_handle(h);
}

frsvt_status frsvt_apply(frsvt_handle* h, const void* A, int64_t lda, double tau, void* X, int64_t ldx,
                         frsvt_info* info) {
  if (h) h->fs_armed = false;  // a fused next sketch belongs to rpca_alm_step
  if (!h || !A || !X || lda < h->m || ldx < h->m || !(tau >= 0) || !std::isfinite(tau)) return FRSVT_EINVAL;
  h->keep = 0;
  if (!rank_uniform_layout(h, A, lda)) return FRSVT_EINVAL;
  if (h->cfg.dtype == FRSVT_F32) return apply_impl<float>(h, A, lda, 0, tau, nullptr, 0, 0, X, ldx, info);
  return apply_impl<double>(h, A, lda, 0, tau, nullptr, 0, 0, X, ldx, info);
}

frsvt_status frsvt_apply_weighted(frsvt_handle* h, const void* A, int64_t lda, int32_t wmode,
                                  const double* w, double C, double eps, void* X, int64_t ldx,
                                  frsvt_info* info) {
  if (h) h->fs_armed = false;
  if (!h || !A || !X || lda < h->m || ldx < h->m) return FRSVT_EINVAL;
  if (!rank_uniform_layout(h, A, lda)) return FRSVT_EINVAL;
  h->keep = 0;
  int km;
  if (wmode == 0) {
    if (!w) return FRSVT_EINVAL;
    for (int i = 0; i < h->l; ++i)
      if (!(w[i] >= 0) || !std::isfinite(w[i])) return FRSVT_EINVAL;
    km = 1;
  } else if (wmode == 1 || wmode == 2) {
    if (!(C >= 0) || !std::isfinite(C) || !(eps > 0) || !std::isfinite(eps)) return FRSVT_EINVAL;
    km = wmode == 1 ? 2 : 3;
  } else {
    return FRSVT_EINVAL;
  }
  if (h->cfg.dtype == FRSVT_F32) return apply_impl<float>(h, A, lda, km, 0.0, w, C, eps, X, ldx, info);
  return apply_impl<double>(h, A, lda, km, 0.0, w, C, eps, X, ldx, info);
}

frsvt_status rpca_alm_step(frsvt_handle* h, rpca_state* st, int32_t finalize, double* rel_resid) {
  if (!h || !st || !st->D || !st->E || !st->A || st->ld < h->m) return FRSVT_EINVAL;
  if (finalize && !st->L) return FRSVT_EINVAL;
  if (st->keep < 0 || st->keep > h->l || (st->transfer != 0 && st->transfer != 1) || (st->transfer && !h->rp))
    return FRSVT_EINVAL;
  if (!(st->rho > 1.0) || !std::isfinite(st->rho)) return FRSVT_EINVAL;
  if (st->iter < 0) return FRSVT_EINVAL;
  if (st->iter == 0 && !(st->mu_max_factor >= 1.0)) return FRSVT_EINVAL;
  if (st->norm2_D < 0 || st->mu0 < 0 || !std::isfinite(st->norm2_D) || !std::isfinite(st->mu0)) return FRSVT_EINVAL;
  if (!rank_uniform_layout(h, st->A, st->ld) || !rank_uniform_layout(h, st->D, st->ld)) return FRSVT_EINVAL;
  if (h->cfg.dtype == FRSVT_F32) return rpca_impl<float>(h, st, finalize, rel_resid);
  return rpca_impl<double>(h, st, finalize, rel_resid);
}

frsvt_status frsvt_set_omega(frsvt_handle* h, const void* Om, int64_t ldo) {
  if (!h || !Om || ldo < h->n) return FRSVT_EINVAL;
  h->fs_armed = false;  // a fused next sketch no longer matches
  CK(cudaMemcpy2DAsync(h->OmOv, h->n * h->esz, Om, ldo * h->esz, h->n * h->esz, h->l,
                       cudaMemcpyDeviceToDevice, h->st));
  h->override_pending = 1;
  return FRSVT_OK;
}

frsvt_status frsvt_draw_omega(frsvt_handle* h, int64_t call, void* out, int64_t ldo) {
  if (!h || !out || ldo < h->n || call < 0) return FRSVT_EINVAL;
  h->fs_armed = false;  // h->Om is overwritten
  if (h->cfg.dtype == FRSVT_F32)
    omega_kernel<float><<<grid1d(h->n * h->l), 256, 0, h->st>>>((float*)h->Om, h->n, h->l, &h->dev->r, 0,
                                                               h->cfg.seed, 1000u + (uint32_t)call, nullptr, h->n,
                                                               0, nullptr, h->om_tf32);
  else
    omega_kernel<double><<<grid1d(h->n * h->l), 256, 0, h->st>>>((double*)h->Om, h->n, h->l, &h->dev->r, 0,
                                                                h->cfg.seed, 1000u + (uint32_t)call, nullptr, h->n);
  TRY(post_launch(h));
  CK(cudaMemcpy2DAsync(out, ldo * h->esz, h->Om, h->n * h->esz, h->n * h->esz, h->l, cudaMemcpyDeviceToDevice,
                       h->st));
  CK(cudaStreamSynchronize(h->st));
  return FRSVT_OK;
}

frsvt_status frsvt_get_carry(frsvt_handle* h, void* Qt, int64_t ldq, int32_t* r) {
  if (!h || !Qt || ldq < h->m) return FRSVT_EINVAL;
  CK(cudaMemcpy2DAsync(Qt, ldq * h->esz, h->Qt, h->m * h->esz, h->m * h->esz, h->l, cudaMemcpyDeviceToDevice,
                       h->st));
  CK(cudaStreamSynchronize(h->st));
  if (r) {
    int rr = 0;
    CK(cudaMemcpy(&rr, &h->dev->r, sizeof(int), cudaMemcpyDeviceToHost));
    *r = rr;
  }
  return FRSVT_OK;
}

frsvt_status frsvt_set_carry(frsvt_handle* h, const void* Qt, int64_t ldq, int32_t r) {
  if (!h || r < 0 || r > h->l || (r > 0 && (!Qt || ldq < h->m))) return FRSVT_EINVAL;
  h->fs_armed = false;  // a fused next sketch no longer matches
  CK(cudaMemsetAsync(h->Qt, 0, (size_t)h->m * h->l * h->esz, h->st));
  if (r > 0)
    CK(cudaMemcpy2DAsync(h->Qt, h->m * h->esz, Qt, ldq * h->esz, h->m * h->esz, r, cudaMemcpyDeviceToDevice,
                         h->st));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(&h->dev->r, &r, sizeof(int), cudaMemcpyHostToDevice));
  return FRSVT_OK;
}

frsvt_status frsvt_reset_carry(frsvt_handle* h) {
  if (!h) return FRSVT_EINVAL;
  h->fs_armed = false;  // a fused next sketch no longer matches
  CK(cudaMemsetAsync(h->Qt, 0, (size_t)h->m * h->l * h->esz, h->st));
  CK(cudaMemsetAsync(&h->dev->r, 0, sizeof(int), h->st));
  CK(cudaMemsetAsync(&h->dev->have_prev, 0, sizeof(int), h->st));
  if (h->ap_on) {
    ap_reset_kernel<<<1, 32, 0, h->st>>>(h->dev, h->ap_l0);
    TRY(post_launch(h));
  }
  return FRSVT_OK;
}

frsvt_status frsvt_set_adaptive_rank(frsvt_handle* h, int32_t a, int32_t p_jump, int32_t b, int32_t l0) {
  if (!h) return FRSVT_EINVAL;
  if (a == 0) {
    h->ap_on = 0;
    return FRSVT_OK;
  }
  if (a < 1 || p_jump < 1 || b < 1 || b > h->l || l0 < 1 || l0 > b) return FRSVT_EINVAL;
  h->fs_armed = false;
  h->ap_on = 1;
  h->ap_a = a;
  h->ap_jump = p_jump;
  h->ap_b = b;
  h->ap_l0 = l0;
  ap_reset_kernel<<<1, 32, 0, h->st>>>(h->dev, l0);
  TRY(post_launch(h));
  CK(cudaStreamSynchronize(h->st));
  return FRSVT_OK;
}

frsvt_status frsvt_set_call_index(frsvt_handle* h, int64_t call) {
  if (!h || call < 0) return FRSVT_EINVAL;
  h->fs_armed = false;  // a fused next sketch no longer matches
  h->call = call;
  return FRSVT_OK;
}

frsvt_status frsvt_get_info(frsvt_handle* h, frsvt_info* info) {
  if (!h || !info) return FRSVT_EINVAL;
  return fill_info(h, info);
}

frsvt_status rpca_get_mu(frsvt_handle* h, double* mu) {
  if (!h || !mu) return FRSVT_EINVAL;
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(mu, h->dev->mu, sizeof(double), cudaMemcpyDeviceToHost));
  return FRSVT_OK;
}

frsvt_status rpca_set_mu(frsvt_handle* h, double mu, double mu_bar) {
  if (!h || !(mu > 0) || !(mu_bar >= mu)) return FRSVT_EINVAL;
  h->fs_armed = false;
  double v[2] = {mu, mu_bar};
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(h->dev->mu, v, sizeof(v), cudaMemcpyHostToDevice));
  return FRSVT_OK;
}

int64_t frsvt_kernel_launches(const frsvt_handle* h) { return h ? h->launches : -1; }

static frsvt_status debug_pass_nosync(frsvt_handle* h, int32_t kind, int32_t impl, const void* A, int64_t lda,
                                      const void* B, void* out) {
  // impl 0: SIMT passes; 2: the CTA-pair tcgen05 pass of the product path
  // (exact, 3 terms); 3: the same with the tf32-rounded small operand (2
  // terms, the span-only passes); 8..263: impl 2 with parts of its pipeline
  // switched off (dbg = impl - 8, outputs invalid)
  if (!h || !A || !B || !out || lda < h->m || kind < 0 || kind > 1 || impl < 0 || impl > 263 || impl == 1 ||
      (impl >= 4 && impl < 8))
    return FRSVT_EINVAL;
  if (impl >= 2 && !(h->esz == 4 && h->use_tc && tc_eligible(h, A, lda))) return FRSVT_EINVAL;
  if (impl >= 2) {
    const int terms = impl == 3 ? 2 : 3;
    const int dbg = impl >= 8 ? impl - 8 : 0;
    return kind == 0 ? tc_pass3<tc::MODE_AX>(h, (const float*)A, lda, h->m, h->n, (const float*)B, h->n, (float*)out,
                                             h->m, nullptr, 0, terms, dbg)
                     : tc_pass3<tc::MODE_ATQ>(h, (const float*)A, lda, h->n, h->m, (const float*)B, h->m,
                                              (float*)out, h->n, nullptr, 0, terms, dbg);
  }
  const int saved = h->use_tc;
  h->use_tc = 0;
  frsvt_status st;
  if (h->esz == 4) {
    st = kind == 0 ? gemm_AX<float>(h, (const float*)A, lda, (const float*)B, (float*)out, nullptr, 3)
                   : gemm_AtQ<float>(h, (const float*)A, lda, (const float*)B, (float*)out, 3);
  } else {
    st = kind == 0 ? gemm_AX<double>(h, (const double*)A, lda, (const double*)B, (double*)out, nullptr, 3)
                   : gemm_AtQ<double>(h, (const double*)A, lda, (const double*)B, (double*)out, 3);
  }
  h->use_tc = saved;
  return st;
}

frsvt_status frsvt_debug_small_svd(frsvt_handle* h, int32_t impl, const double* G, double* Gcopy, double* sigma,
                                   double* UB, int32_t* sweeps, int32_t reps, double* ms) {
  if (!h || !sigma || !UB || impl != 0 || reps < 0) return FRSVT_EINVAL;
  const size_t gb = sizeof(double) * h->l * h->l;
  if (G) CK(cudaMemcpyAsync(h->G, G, gb, cudaMemcpyDeviceToDevice, h->st));
  if (Gcopy) CK(cudaMemcpyAsync(Gcopy, h->G, gb, cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemsetAsync(&h->dev->flags, 0, sizeof(int), h->st));
  TRY(launch_eig_jacobi(h, h->G, sigma, UB, 0, 0.0, nullptr));
  if (reps > 0) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, h->st));
    for (int i = 0; i < reps; ++i) TRY(launch_eig_jacobi(h, h->G, sigma, UB, 0, 0.0, nullptr));
    CK(cudaEventRecord(e1, h->st));
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e0, e1));
    if (ms) *ms = t / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  CK(cudaStreamSynchronize(h->st));
  if (sweeps) CK(cudaMemcpy(sweeps, &h->dev->sweeps, sizeof(int), cudaMemcpyDeviceToHost));
  return FRSVT_OK;
}

frsvt_status frsvt_debug_pass(frsvt_handle* h, int32_t kind, int32_t impl, const void* A, int64_t lda,
                              const void* B, void* out) {
  TRY(debug_pass_nosync(h, kind, impl, A, lda, B, out));
  CK(cudaStreamSynchronize(h->st));
  return FRSVT_OK;
}

frsvt_status frsvt_debug_pass_timed(frsvt_handle* h, int32_t kind, int32_t impl, const void* A, int64_t lda,
                                    const void* B, void* out, int32_t reps, double* ms) {
  if (reps < 1 || !ms) return FRSVT_EINVAL;
  TRY(debug_pass_nosync(h, kind, impl, A, lda, B, out));  // warm-up (and argument check)
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, h->st));
  for (int i = 0; i < reps; ++i) TRY(debug_pass_nosync(h, kind, impl, A, lda, B, out));
  CK(cudaEventRecord(e1, h->st));
  CK(cudaEventSynchronize(e1));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, e0, e1));
  *ms = t / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return FRSVT_OK;
}

frsvt_status frsvt_debug_chol(frsvt_handle* h, const double* G, void* T, int32_t* s, unsigned long long* stamps) {
  if (!h || !G || !T) return FRSVT_EINVAL;
  CK(cudaMemcpyAsync(h->G, G, sizeof(double) * h->l * h->l, cudaMemcpyDeviceToDevice, h->st));
  const double tol = h->esz == 4 ? 1e-12 : 1e-13;
  if (h->esz == 4)
    orth_chol_kernel<float><<<1, OC_THREADS, orth_chol_smem_bytes(h->l), h->st>>>(h->G, h->l, tol, (float*)T,
                                                                                &h->dev->s, &h->dev->flags, stamps);
  else
    orth_chol_kernel<double><<<1, OC_THREADS, orth_chol_smem_bytes(h->l), h->st>>>(h->G, h->l, tol, (double*)T,
                                                                                 &h->dev->s, &h->dev->flags, stamps);
  TRY(post_launch(h));
  CK(cudaStreamSynchronize(h->st));
  if (s) CK(cudaMemcpy(s, &h->dev->s, sizeof(int), cudaMemcpyDeviceToHost));
  return FRSVT_OK;
}

frsvt_status frsvt_debug_chol_inv(frsvt_handle* h, const double* G, int32_t r, void* T, int32_t* s,
                                  unsigned long long* stamps) {
  if (!h || !G || !T || h->esz != 4 || r < 0 || r > h->l) return FRSVT_EINVAL;
  CK(cudaMemcpyAsync(h->G, G, sizeof(double) * h->l * h->l, cudaMemcpyDeviceToDevice, h->st));
  int* rd = h->lwd + 4;  // scratch int (lwd[0..3]: Loewdin flags)
  CK(cudaMemcpyAsync(rd, &r, sizeof(int), cudaMemcpyHostToDevice, h->st));
  launch_chol_inv(h, rd, (float*)T, stamps, nullptr);
  TRY(post_launch(h));
  CK(cudaStreamSynchronize(h->st));
  if (s) CK(cudaMemcpy(s, &h->dev->s, sizeof(int), cudaMemcpyDeviceToHost));
  return FRSVT_OK;
}

frsvt_status frsvt_profile(frsvt_handle* h, int32_t enable) {
  if (!h) return FRSVT_EINVAL;
  CK(cudaStreamSynchronize(h->st));
  h->prof_used = 0;
  for (int k = 0; k < 4; ++k) {
    h->prof_ms[k] = 0.0;
    h->prof_bytes[k] = 0.0;
    h->prof_count[k] = 0;
  }
  h->prof_on = enable ? 1 : 0;
  return FRSVT_OK;
}

frsvt_status frsvt_profile_read(frsvt_handle* h, int32_t kind, double* ms, int64_t* launches, double* bytes) {
  if (!h || kind < 0 || kind > 3) return FRSVT_EINVAL;
  TRY(prof_flush(h));
  if (ms) *ms = h->prof_ms[kind];
  if (launches) *launches = h->prof_count[kind];
  if (bytes) *bytes = h->prof_bytes[kind];
  return FRSVT_OK;
}

}  // extern "C"
