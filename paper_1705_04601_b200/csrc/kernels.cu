// sm_100a FP64 kernels of the H^2 sparsification hot path:
//   qr_kernel        step (i)   QR completion Q_t = [W_t, W_t^perp], R^_t
//   coupling_kernel             D~ = R^_t D R^_s^T
//   pair_kernel      (iv)+(ii)+(iii)  merge G_ts, H = Q_t^T G Q_s, freeze
//   strip_kernel     (ii)/(iii) strips W = Q_q^T Z, freeze                  (Eq. u1v1)
//   csr_cols_kernel  (iii)      CSR column indices of S
//   apply_*          U^T b, V y
// Dense contractions use FP64 DMMA (mma.sync m8n8k4 .f64, the native FP64
// tensor-core shape on sm_100a; tcgen05 has no f64 kind) with operands staged
// in shared memory; Q_t of the rotating cluster stays resident in shared
// memory across the run of items (a block row) of one CTA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "h2sp_internal.h"

namespace h2sp {

#define H2SP_CK(x)                                                                                       \
  do {                                                                                                   \
    cudaError_t e_ = (x);                                                                                \
    if (e_ != cudaSuccess) return fail(H2SP_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Dynamic shared-memory opt-in, per device and kernel (cudaFuncSetAttribute is a
// per-device setting): set on first use on each device, under a lock (builds on
// different devices may run on different host threads).
static h2sp_status ensure_smem(const void *fn, size_t bytes) {
  int dev = 0;
  H2SP_CK(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(dev, fn);
  const auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return H2SP_OK;
  H2SP_CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  done[key] = bytes;
  return H2SP_OK;
}

struct Clusters {  // device views of the per-cluster arrays in the meta region
  const int32_t *n_row, *k_row, *n_col, *k_col;
  const int64_t *q_off_row, *q_off_col, *rh_off_row, *rh_off_col;
  const int64_t *leaf_off_row, *leaf_off_col, *tr_off_row, *tr_off_col;
  const int64_t *s_off_row, *s_off_col, *zb_off_row, *zb_off_col;
  const int64_t *loc_off_row, *loc_off_col;
  const int8_t *need_row, *need_col;
};

static Clusters make_clusters(const h2sp_plan_s *p, const unsigned char *meta) {
  Clusters c;
  c.n_row = (const int32_t *)(meta + p->ca.n_row);
  c.k_row = (const int32_t *)(meta + p->ca.k_row);
  c.n_col = (const int32_t *)(meta + p->ca.n_col);
  c.k_col = (const int32_t *)(meta + p->ca.k_col);
  c.q_off_row = (const int64_t *)(meta + p->ca.q_off_row);
  c.q_off_col = (const int64_t *)(meta + p->ca.q_off_col);
  c.rh_off_row = (const int64_t *)(meta + p->ca.rh_off_row);
  c.rh_off_col = (const int64_t *)(meta + p->ca.rh_off_col);
  c.leaf_off_row = (const int64_t *)(meta + p->ca.leaf_off_row);
  c.leaf_off_col = (const int64_t *)(meta + p->ca.leaf_off_col);
  c.tr_off_row = (const int64_t *)(meta + p->ca.tr_off_row);
  c.tr_off_col = (const int64_t *)(meta + p->ca.tr_off_col);
  c.s_off_row = (const int64_t *)(meta + p->ca.s_off_row);
  c.s_off_col = (const int64_t *)(meta + p->ca.s_off_col);
  c.zb_off_row = (const int64_t *)(meta + p->ca.zb_off_row);
  c.zb_off_col = (const int64_t *)(meta + p->ca.zb_off_col);
  c.loc_off_row = (const int64_t *)(meta + p->ca.loc_off_row);
  c.loc_off_col = (const int64_t *)(meta + p->ca.loc_off_col);
  c.need_row = (const int8_t *)(meta + p->ca.need_row);
  c.need_col = (const int8_t *)(meta + p->ca.need_col);
  return c;
}

struct Side {  // one side (row or column) of the cluster arrays
  const int32_t *n, *k;
  const int64_t *q_off, *rh_off, *leaf_off, *tr_off, *s_off, *zb_off, *loc_off;
  const int8_t *need;
};

static Side side_of(const Clusters &c, bool col) {
  Side s;
  s.n = col ? c.n_col : c.n_row;
  s.k = col ? c.k_col : c.k_row;
  s.q_off = col ? c.q_off_col : c.q_off_row;
  s.rh_off = col ? c.rh_off_col : c.rh_off_row;
  s.leaf_off = col ? c.leaf_off_col : c.leaf_off_row;
  s.tr_off = col ? c.tr_off_col : c.tr_off_row;
  s.s_off = col ? c.s_off_col : c.s_off_row;
  s.zb_off = col ? c.zb_off_col : c.zb_off_row;
  s.loc_off = col ? c.loc_off_col : c.loc_off_row;
  s.need = col ? c.need_col : c.need_row;
  return s;
}

__host__ __device__ inline int64_t lvl_off_d(int L, int k) {
  return (int64_t(1) << (L + 1)) - (int64_t(1) << (L - k + 1));
}

// --------------------------------------------------------------------------
// DMMA helper: D(8x8) += A(8x4, row) * B(4x8, col), FP64.
// Fragments (PTX ISA, mma.m8n8k4 .f64): a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d = D[lane/4][2*(lane%4) + {0,1}].
// --------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Warp GEMM on shared-memory tiles with leading dimensions LDA / LDB:
//   acc[i][j] (8x8 tile at rows m0+8i, cols n0+8j) += sum_kk A(m, kk) B(kk, n)
//   A(m, kk) = AT ? sA[kk*LDA + m] : sA[m*LDA + kk];  B(kk, n) = sB[kk*LDB + n].
template <int LDA, int LDB, int TM, int TN, bool AT>
__device__ __forceinline__ void warp_gemm(const double *__restrict__ sA, const double *__restrict__ sB, int m0,
                                          int n0, int kmax, double (&acc)[TM][TN][2], int kmin = 0) {
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
#pragma unroll 4
  for (int k0 = kmin; k0 < kmax; k0 += 4) {
    double a[TM], b[TN];
#pragma unroll
    for (int i = 0; i < TM; i++) a[i] = AT ? sA[(k0 + q) * LDA + m0 + i * 8 + r] : sA[(m0 + i * 8 + r) * LDA + k0 + q];
#pragma unroll
    for (int j = 0; j < TN; j++) b[j] = sB[(k0 + q) * LDB + n0 + j * 8 + r];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++) dmma(acc[i][j], a[i], b[j]);
  }
}

template <int LD, int TM, int TN>
__device__ __forceinline__ void warp_store(double *sC, int m0, int n0, const double (&acc)[TM][TN][2]) {
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) {
      double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
      *reinterpret_cast<double2 *>(&sC[(m0 + i * 8 + r) * LD + n0 + j * 8 + 2 * q]) = v;
    }
}

template <int TM, int TN>
__device__ __forceinline__ void zero_acc(double (&acc)[TM][TN][2]) {
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// cp.async (LDGSTS) helpers: every global->shared tile load is issued as a batch
// of asynchronous 8-byte copies (zero-filled outside the valid region) and
// waited for once, so the loads of a tile overlap instead of serialising.
__device__ __forceinline__ void cp8(void *sdst, const void *gsrc, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void store2(double *d, double v0, double v1) {
  if ((reinterpret_cast<uintptr_t>(d) & 15) == 0) {
    *reinterpret_cast<double2 *>(d) = make_double2(v0, v1);
  } else {
    d[0] = v0;
    d[1] = v1;
  }
}
// Stores of final S values.  Compiling with -DH2SP_S_STREAM uses the
// evict-first (streaming) policy for them (they are never re-read by the
// build); measured 1 % slower on config 2, so plain stores are the default.
#ifdef H2SP_S_STREAM
__device__ __forceinline__ void st_s(double *d, double v) { __stcs(d, v); }
__device__ __forceinline__ void store2_s(double *d, double v0, double v1) {
  if ((reinterpret_cast<uintptr_t>(d) & 15) == 0) {
    __stcs(reinterpret_cast<double2 *>(d), make_double2(v0, v1));
  } else {
    __stcs(d, v0);
    __stcs(d + 1, v1);
  }
}
#else
__device__ __forceinline__ void st_s(double *d, double v) { *d = v; }
__device__ __forceinline__ void store2_s(double *d, double v0, double v1) { store2(d, v0, v1); }
#endif
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void cp16(void *sdst, const void *gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
// 16 zero bytes into shared memory through the async-copy path (src-size 0)
__device__ __forceinline__ void cp16_zero(void *sdst, const void *any) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;\n" ::"r"(s), "l"(any) : "memory");
}

// Asynchronously load an n x m row-major global block (leading dim ldg) into a
// padded NR x NC shared tile with leading dimension LD, zero fill.  Pairs of
// columns move as one 16-byte copy when the global block is 16-byte aligned.
// `any` is a valid global address used for the zero-filled (not read) copies.
template <int NR, int NC, int LD>
__device__ __forceinline__ void async_tile(double *s, const double *__restrict__ g, int n, int m, int64_t ldg,
                                           const void *any) {
  static_assert(NC % 2 == 0 && LD % 2 == 0, "paired columns");
  const bool al = ((reinterpret_cast<uintptr_t>(g) | uintptr_t(ldg * 8)) & 15) == 0;
  for (int idx = threadIdx.x; idx < NR * NC / 2; idx += blockDim.x) {
    const int i = idx / (NC / 2), j = 2 * (idx % (NC / 2));
    const bool v0 = i < n && j < m, v1 = i < n && j + 1 < m;
    const double *src = g + int64_t(i) * ldg + j;
    if (al && v0 && v1) {
      cp16(&s[i * LD + j], src);
    } else if (!v0 && ((LD & 1) == 0)) {  // both padding (v1 implies v0): one 16-byte zero fill
      cp16_zero(&s[i * LD + j], any);
    } else {
      cp8(&s[i * LD + j], v0 ? (const void *)src : any, v0);
      cp8(&s[i * LD + j + 1], v1 ? (const void *)(src + 1) : any, v1);
    }
  }
}

// --------------------------------------------------------------------------
// Step (i): QR completion (convention H, readings 1-2), one WARP per
// cluster (no block-level synchronisation):
//   X = R_leaf (level 0) or [R^_c1 T[:k1]; R^_c2 T[k1:]] (internal)
//   Householder on X (alpha = x_0, sigma = ||x_1:||; sigma == 0 -> tau = 0;
//   beta = -sgn(alpha) hypot(alpha, sigma), sgn(+-0) = +1), R^ = triu(X[:k]),
//   Q = H_0 ... H_{k-1} = I - V T V^T: the compact WY form of the same product
//   (T from the dlarft recurrence over V^T V), the three products V^T V, T V^T
//   and V (T V^T) on the DMMA pipe, Q written from the accumulators.
// Per-warp shared memory (doubles): X n x (k+1) | T K8 x LDT | G/M K4 x LDM | R^ staging
// --------------------------------------------------------------------------
__host__ __device__ inline int rup(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ inline int qr_ldt(int k) { return rup(rup(k, 4), 16) + 4; }
__host__ __device__ inline int qr_ldm(int n) { return rup(rup(n, 8), 16) + 4; }
__host__ __device__ inline int qr_warp_doubles(int n, int k, int rstage) {
  const int K4 = rup(k, 4), K8 = rup(k, 8);
  const int mm = K4 * qr_ldm(n) > K8 * K8 ? K4 * qr_ldm(n) : K8 * K8;
  const int stg = n * k > mm ? n * k : mm;   // transfer staging aliases G/M
  return n * (k + 1) + K8 * qr_ldt(k) + stg + rstage + 2;
}

__global__ void __launch_bounds__(128) qr_kernel(Side sd, int L, int level, int nclust, int per_warp,
                                                 const double *__restrict__ leaf, const double *__restrict__ transfer,
                                                 double *__restrict__ rh, double *__restrict__ qout,
                                                 const uint64_t *meta_magic, uint64_t magic, double *__restrict__ wy,
                                                 int wy_kp, int wy_n) {
  if (meta_magic && threadIdx.x == 0 && blockIdx.x == 0 && *meta_magic != magic) __trap();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * (blockDim.x >> 5) + warp;
  if (ci >= nclust) return;
  const int64_t base = lvl_off_d(L, level);
  const int64_t cl = base + ci;
  const int n = sd.n[cl], k = sd.k[cl];
  if (n == 0 || !sd.need[cl]) return;
  double *Qg = qout + sd.q_off[cl];
  // compact-WY copy (level 0 only), as qr_reg_kernel
  double *Wg = wy ? wy + int64_t(ci) * 2 * wy_n * wy_kp : nullptr;
  if (k == 0) {
    if (Wg) {
      for (int idx = lane; idx < 2 * wy_n * wy_kp; idx += 32) Wg[idx] = 0.0;
      return;
    }
    for (int idx = lane; idx < n * n; idx += 32) Qg[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
    return;
  }
  extern __shared__ __align__(16) double sm[];
  const int K4 = rup(k, 4), K8 = rup(k, 8), N4 = rup(n, 4), N8 = rup(n, 8);
  const int LDX = k + 1, LDT = qr_ldt(k), LDM = qr_ldm(n);
  double *X = sm + size_t(warp) * per_warp;
  double *Tw = X + n * LDX;                  // K8 x LDT
  double *Mm = Tw + K8 * LDT;                // G = V^T V (K8 x K8), then M = T V^T (K4 x LDM); T staging
  const int mm = K4 * LDM > K8 * K8 ? K4 * LDM : K8 * K8;
  double *RS = Mm + (n * k > mm ? n * k : mm);   // children R^ staging (level >= 1)
  for (int idx = lane; idx < K8 * LDT; idx += 32) Tw[idx] = 0.0;
  // ---- load X
  if (level == 0) {
    const double *R = leaf + sd.leaf_off[cl];
    for (int idx = lane; idx < n * k; idx += 32) cp8(&X[(idx / k) * LDX + idx % k], R + idx, true);
    cp_commit();
    cp_wait_all();
    __syncwarp();
  } else {
    const int64_t c1 = lvl_off_d(L, level - 1) + 2 * ci, c2 = c1 + 1;
    const int k1 = sd.k[c1], k2 = sd.k[c2];
    const double *T = transfer + sd.tr_off[cl];  // n x k
    double *sT = Mm, *sR1 = RS, *sR2 = RS + k1 * k1;
    const double *R1 = rh + sd.rh_off[c1];
    const double *R2 = rh + sd.rh_off[c2];
    for (int idx = lane; idx < n * k; idx += 32) cp8(&sT[idx], T + idx, true);
    for (int idx = lane; idx < k1 * k1; idx += 32) cp8(&sR1[idx], R1 + idx, true);
    for (int idx = lane; idx < k2 * k2; idx += 32) cp8(&sR2[idx], R2 + idx, true);
    cp_commit();
    cp_wait_all();
    __syncwarp();
    for (int idx = lane; idx < n * k; idx += 32) {
      const int i = idx / k, j = idx % k;
      double acc = 0.0;
      if (i < k1) {
        for (int l = i; l < k1; l++) acc = fma(sR1[i * k1 + l], sT[l * k + j], acc);
      } else {
        const int ii = i - k1;
        for (int l = ii; l < k2; l++) acc = fma(sR2[ii * k2 + l], sT[(k1 + l) * k + j], acc);
      }
      X[i * LDX + j] = acc;
    }
    __syncwarp();
  }
  // ---- Householder factorisation; tau_j kept on the diagonal of T
  for (int j = 0; j < k; j++) {
    double ss = 0.0;
    for (int i = j + 1 + lane; i < n; i += 32) ss = fma(X[i * LDX + j], X[i * LDX + j], ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double alpha = X[j * LDX + j];
    const double sigma = sqrt(ss);
    double beta, tau;
    if (sigma == 0.0) {
      tau = 0.0;
      beta = alpha;
    } else {
      const double sgn = alpha < 0.0 ? -1.0 : 1.0;
      beta = -sgn * hypot(alpha, sigma);
      tau = (beta - alpha) / beta;
    }
    __syncwarp();
    if (tau != 0.0) {
      const double div = alpha - beta;
      for (int i = j + 1 + lane; i < n; i += 32) X[i * LDX + j] = X[i * LDX + j] / div;
      __syncwarp();
      for (int c0 = j + 1; c0 < k; c0 += 4) {
        double w[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          w[u] = 0.0;
          if (c0 + u < k)
            for (int i = j + 1 + lane; i < n; i += 32) w[u] = fma(X[i * LDX + j], X[i * LDX + c0 + u], w[u]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < 4; u++) w[u] += __shfl_xor_sync(0xffffffffu, w[u], o);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          if (c0 + u >= k) continue;
          const double tw = tau * (w[u] + X[j * LDX + c0 + u]);
          for (int i = j + 1 + lane; i < n; i += 32) X[i * LDX + c0 + u] = fma(-tw, X[i * LDX + j], X[i * LDX + c0 + u]);
          __syncwarp();
          if (lane == 0) X[j * LDX + c0 + u] -= tw;
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      X[j * LDX + j] = beta;
      Tw[j * LDT + j] = tau;
    }
    __syncwarp();
  }
  // ---- R^ (k x k upper triangular)
  {
    double *R = rh + sd.rh_off[cl];
    for (int idx = lane; idx < k * k; idx += 32) {
      const int i = idx / k, j = idx % k;
      R[idx] = j >= i ? X[i * LDX + j] : 0.0;
    }
  }
  // V(i, l): unit lower trapezoidal reflector matrix (zero padding outside n x k)
  auto V = [&](int i, int l) -> double {
    if (i >= n || l >= k || i < l) return 0.0;
    return i == l ? 1.0 : X[i * LDX + l];
  };
  const int r = lane >> 2, q = lane & 3;
  // ---- G = V^T V (upper tiles) -> Mm (K8 x K8)
  for (int ta = 0; ta < K8 / 8; ta++)
    for (int tb = ta; tb < K8 / 8; tb++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < N4; k0 += 4) dmma(acc, V(k0 + q, ta * 8 + r), V(k0 + q, tb * 8 + r));
      Mm[(ta * 8 + r) * K8 + tb * 8 + 2 * q] = acc[0];
      Mm[(ta * 8 + r) * K8 + tb * 8 + 2 * q + 1] = acc[1];
    }
  __syncwarp();
  // ---- T recurrence (dlarft, forward, columnwise): T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]
  for (int j = 1; j < k; j++) {
    const double tj = Tw[j * LDT + j];
    double v[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int i = lane + 32 * u;
      if (i < j)
        for (int l = i; l < j; l++) v[u] = fma(Tw[i * LDT + l], Mm[l * K8 + j], v[u]);
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int i = lane + 32 * u;
      if (i < j) Tw[i * LDT + j] = -tj * v[u];
    }
    __syncwarp();
  }
  // ---- M = T V^T (K4 x N8) -> Mm (ld LDM); G is dead now
  for (int ta = 0; ta < K8 / 8; ta++)
    for (int tc = 0; tc < N8 / 8; tc++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < K4; k0 += 4) {
        const int a = ta * 8 + r;
        dmma(acc, Tw[a * LDT + k0 + q], V(tc * 8 + r, k0 + q));
      }
      __syncwarp();
      const int a = ta * 8 + r;
      if (a < K4) {
        Mm[a * LDM + tc * 8 + 2 * q] = acc[0];
        Mm[a * LDM + tc * 8 + 2 * q + 1] = acc[1];
      }
    }
  __syncwarp();
  if (Wg) {
    for (int idx = lane; idx < wy_n * wy_kp; idx += 32) {
      const int i = idx / wy_kp, c = idx - i * wy_kp;
      Wg[idx] = V(i, c);
    }
    for (int idx = lane; idx < wy_n * wy_kp; idx += 32) {
      const int a = idx / wy_n, c = idx - a * wy_n;
      Wg[wy_n * wy_kp + idx] = (a < k && c < n) ? Mm[a * LDM + c] : 0.0;
    }
    return;
  }
  // ---- Q = I - V M, straight to global
  for (int ti = 0; ti < N8 / 8; ti++)
    for (int tc = 0; tc < N8 / 8; tc++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < K4; k0 += 4) dmma(acc, V(ti * 8 + r, k0 + q), Mm[(k0 + q) * LDM + tc * 8 + r]);
      const int i = ti * 8 + r;
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int c = tc * 8 + 2 * q + e;
        if (i < n && c < n) Qg[i * n + c] = (i == c ? 1.0 : 0.0) - acc[e];
      }
    }
}

// Warp all-reduce of a P-vector (P a power of two, 8..32) by reduce-scatter +
// broadcast: log2(P) halving rounds (P-1 shuffles), the remaining rounds on a
// single value, then P broadcasts -- instead of 5 full butterfly rounds per entry.
template <int P>
__device__ __forceinline__ void warp_allreduce_vec(double (&w)[P], int lane) {
  int len = P;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const bool bit = (lane & o) != 0;
    if (len > 1) {
      const int half = len >> 1;
#pragma unroll
      for (int i = 0; i < P / 2; i++) {
        if (i < half) {
          const double send = bit ? w[i] : w[i + half];
          const double keep = bit ? w[i + half] : w[i];
          w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      len = half;
    } else {
      w[0] += __shfl_xor_sync(0xffffffffu, w[0], o);
    }
  }
  // lane holds the sum of component c(lane); component c lives in lane c * (32 / P)
  const double total = w[0];
#pragma unroll
  for (int c = 0; c < P; c++) w[c] = __shfl_sync(0xffffffffu, total, c * (32 / P));
}

// --------------------------------------------------------------------------
// Register-resident variant of the same QR completion for k <= KP <= 32 and
// n <= 32 * NR: lane l holds rows l, l+32 of X; the Householder loop is fully
// unrolled over the KP columns; every trailing-column dot product of one step
// is reduced in the same butterfly.  Same convention H, same compact-WY
// formation of Q (V staged once in shared memory with explicit unit diagonal).
// Per-warp shared memory (doubles): V N8 x LDV | T K8 x LDT | G/M max(K8*K8, K4*LDM)
// --------------------------------------------------------------------------
__host__ __device__ inline int qr_ldv(int k) { return rup(rup(k, 4), 16) + 4; }
__host__ __device__ inline int qr_reg_warp_doubles(int n, int k) {
  const int K4 = rup(k, 4), K8 = rup(k, 8), N8 = rup(n, 8);
  const int mm = K4 * qr_ldm(n) > K8 * K8 ? K4 * qr_ldm(n) : K8 * K8;
  return N8 * qr_ldv(k) + K8 * qr_ldt(k) + mm + 2;
}

template <int NR, int KP>
__global__ void __launch_bounds__(128) qr_reg_kernel(Side sd, int L, int level, int nclust, int per_warp,
                                                     const double *__restrict__ leaf,
                                                     const double *__restrict__ transfer, double *__restrict__ rh,
                                                     double *__restrict__ qout, const uint64_t *meta_magic,
                                                     uint64_t magic, double *__restrict__ wy, int wy_kp, int wy_n) {
  if (meta_magic && threadIdx.x == 0 && blockIdx.x == 0 && *meta_magic != magic) __trap();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * (blockDim.x >> 5) + warp;
  if (ci >= nclust) return;
  const int64_t base = lvl_off_d(L, level);
  const int64_t cl = base + ci;
  const int n = sd.n[cl], k = sd.k[cl];
  if (n == 0 || !sd.need[cl]) return;
  double *Qg = qout + sd.q_off[cl];
  // compact-WY copy (level 0 only): V (wy_n x wy_kp) then M = T V^T (wy_kp x wy_n), zero padded
  double *Wg = wy ? wy + int64_t(ci) * 2 * wy_n * wy_kp : nullptr;
  if (k == 0) {
    if (Wg) {  // V = M = 0: wy_form_q_kernel writes Q = I
      for (int idx = lane; idx < 2 * wy_n * wy_kp; idx += 32) Wg[idx] = 0.0;
      return;
    }
    for (int idx = lane; idx < n * n; idx += 32) Qg[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
    return;
  }
  double x[NR][KP];
  // ---- load X (rows lane + 32u)
  if (level == 0) {
    const double *R = leaf + sd.leaf_off[cl];
#pragma unroll
    for (int u = 0; u < NR; u++) {
      const int i = lane + 32 * u;
#pragma unroll
      for (int c = 0; c < KP; c++) x[u][c] = (i < n && c < k) ? __ldg(R + i * k + c) : 0.0;
    }
  } else {
    // X = [R^_c1 T[:k1]; R^_c2 T[k1:]]: stage T and both R^ with one batched copy
    extern __shared__ __align__(16) double smx[];
    const int64_t c1 = lvl_off_d(L, level - 1) + 2 * ci, c2 = c1 + 1;
    const int k1 = sd.k[c1], k2 = sd.k[c2];
    double *sT = smx + size_t(warp) * per_warp, *sR1 = sT + n * k, *sR2 = sR1 + k1 * k1;
    const double *T = transfer + sd.tr_off[cl];  // n x k
    const double *R1 = rh + sd.rh_off[c1];
    const double *R2 = rh + sd.rh_off[c2];
    for (int idx = lane; idx < n * k; idx += 32) cp8(&sT[idx], T + idx, true);
    for (int idx = lane; idx < k1 * k1; idx += 32) cp8(&sR1[idx], R1 + idx, true);
    for (int idx = lane; idx < k2 * k2; idx += 32) cp8(&sR2[idx], R2 + idx, true);
    cp_commit();
    cp_wait_all();
    __syncwarp();
#pragma unroll
    for (int u = 0; u < NR; u++) {
      const int i = lane + 32 * u;
#pragma unroll
      for (int c = 0; c < KP; c++) x[u][c] = 0.0;
      if (i < n) {
        const bool first = i < k1;
        const int ii = first ? i : i - k1, kk = first ? k1 : k2, roff = first ? 0 : k1;
        const double *Rr = first ? sR1 : sR2;
        for (int l = ii; l < kk; l++) {
          const double rv = Rr[ii * kk + l];
          const double *Trow = sT + (roff + l) * k;
#pragma unroll
          for (int c = 0; c < KP; c++)
            if (c < k) x[u][c] = fma(rv, Trow[c], x[u][c]);
        }
      }
    }
    __syncwarp();
  }
  // shared memory: V (unit lower trapezoidal, zero padded), T (tau on the diagonal), G/M
  extern __shared__ __align__(16) double sm[];
  const int K4 = rup(k, 4), K8 = rup(k, 8), N4 = rup(n, 4), N8 = rup(n, 8);
  const int LDV = qr_ldv(k), LDT = qr_ldt(k), LDM = qr_ldm(n);
  double *Vs = sm + size_t(warp) * per_warp;   // N8 x LDV
  double *Tw = Vs + N8 * LDV;                  // K8 x LDT
  double *Mm = Tw + K8 * LDT;                  // G (K8 x K8), then M (K4 x LDM)
  for (int idx = lane; idx < N8 * LDV; idx += 32) Vs[idx] = 0.0;
  for (int idx = lane; idx < K8 * LDT; idx += 32) Tw[idx] = 0.0;
  __syncwarp();
  double *Rg = rh + sd.rh_off[cl];
  for (int idx = lane; idx < k * k; idx += 32)  // strictly lower triangle of R^ (lane-parallel)
    if (idx % k < idx / k) Rg[idx] = 0.0;
  // ---- Householder factorisation.  Runtime loop over j with a shifting register
  //      window: x[u][0] is always the current column j, x[u][c] column j + c.
  for (int j = 0; j < k; j++) {
    const int w_left = k - j;   // columns j .. k-1 still in the window
    double ss = 0.0;
#pragma unroll
    for (int u = 0; u < NR; u++)
      if (lane + 32 * u > j && lane + 32 * u < n) ss = fma(x[u][0], x[u][0], ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double own0 = (NR == 1 || j < 32) ? x[0][0] : x[NR - 1][0];
    const double alpha = __shfl_sync(0xffffffffu, own0, j & 31);
    const double sigma = sqrt(ss);
    double beta, t;
    if (sigma == 0.0) {
      t = 0.0;
      beta = alpha;
    } else {
      const double sgn = alpha < 0.0 ? -1.0 : 1.0;
      beta = -sgn * hypot(alpha, sigma);
      t = (beta - alpha) / beta;
    }
    double v[NR];
    const double rdiv = 1.0 / (alpha - beta);
#pragma unroll
    for (int u = 0; u < NR; u++) {
      const int i = lane + 32 * u;
      v[u] = (i == j) ? 1.0 : ((t != 0.0 && i > j && i < n) ? x[u][0] * rdiv : 0.0);
    }
    if (t != 0.0) {
      constexpr int P2 = KP <= 8 ? 8 : KP <= 16 ? 16 : 32;
      double w[P2];
#pragma unroll
      for (int c = 0; c < P2; c++) {
        w[c] = 0.0;
        if (c >= 1 && c < KP && c < w_left)
#pragma unroll
          for (int u = 0; u < NR; u++) w[c] = fma(v[u], x[u][c < KP ? c : 0], w[c]);
      }
      warp_allreduce_vec<P2>(w, lane);
#pragma unroll
      for (int c = 1; c < KP; c++)
        if (c < w_left) {
          const double tw = t * w[c];
#pragma unroll
          for (int u = 0; u < NR; u++) x[u][c] = fma(-tw, v[u], x[u][c]);
        }
    }
    // reflector j -> V (rows > j; unit diagonal), tau_j -> T diagonal, row j of R^
#pragma unroll
    for (int u = 0; u < NR; u++) {
      const int i = lane + 32 * u;
      if (i >= j && i < n) Vs[i * LDV + j] = v[u];
      if (i == j) {
        Rg[j * k + j] = beta;
#pragma unroll
        for (int c = 1; c < KP; c++)
          if (c < w_left) Rg[j * k + j + c] = x[u][c];
      }
    }
    if (lane == 0) Tw[j * LDT + j] = t;
    // shift the window
#pragma unroll
    for (int u = 0; u < NR; u++) {
#pragma unroll
      for (int c = 0; c < KP - 1; c++) x[u][c] = x[u][c + 1];
      x[u][KP - 1] = 0.0;
    }
  }
  __syncwarp();
  const int r = lane >> 2, q = lane & 3;
  // ---- G = V^T V (upper tiles)
  for (int ta = 0; ta < K8 / 8; ta++)
    for (int tb = ta; tb < K8 / 8; tb++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < N4; k0 += 4)
        dmma(acc, Vs[(k0 + q) * LDV + ta * 8 + r], Vs[(k0 + q) * LDV + tb * 8 + r]);
      Mm[(ta * 8 + r) * K8 + tb * 8 + 2 * q] = acc[0];
      Mm[(ta * 8 + r) * K8 + tb * 8 + 2 * q + 1] = acc[1];
    }
  __syncwarp();
  // ---- T recurrence (dlarft, forward, columnwise): T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]
  for (int j = 1; j < k; j++) {
    const double tj = Tw[j * LDT + j];
    double v = 0.0;
    if (lane < j)
      for (int l = lane; l < j; l++) v = fma(Tw[lane * LDT + l], Mm[l * K8 + j], v);
    __syncwarp();
    if (lane < j) Tw[lane * LDT + j] = -tj * v;
    __syncwarp();
  }
  // ---- M = T V^T
  for (int ta = 0; ta < K8 / 8; ta++)
    for (int tc = 0; tc < N8 / 8; tc++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < K4; k0 += 4)
        dmma(acc, Tw[(ta * 8 + r) * LDT + k0 + q], Vs[(tc * 8 + r) * LDV + k0 + q]);
      __syncwarp();
      const int a = ta * 8 + r;
      if (a < K4) {
        Mm[a * LDM + tc * 8 + 2 * q] = acc[0];
        Mm[a * LDM + tc * 8 + 2 * q + 1] = acc[1];
      }
    }
  __syncwarp();
  if (Wg) {
    // V and M for the compact-WY congruence; Q itself is formed later off the
    // critical path (wy_form_q_kernel)
    {  // V: row-major wy_n x wy_kp (row / column advanced incrementally, no division)
      int i = lane / wy_kp, c = lane % wy_kp;
      for (int idx = lane; idx < wy_n * wy_kp; idx += 32) {
        Wg[idx] = (i < n && c < k) ? Vs[i * LDV + c] : 0.0;
        for (c += 32; c >= wy_kp; c -= wy_kp) i++;
      }
    }
    {  // M: row-major wy_kp x wy_n
      int a = lane / wy_n, c = lane % wy_n;
      for (int idx = lane; idx < wy_n * wy_kp; idx += 32) {
        Wg[wy_n * wy_kp + idx] = (a < k && c < n) ? Mm[a * LDM + c] : 0.0;
        for (c += 32; c >= wy_n; c -= wy_n) a++;
      }
    }
    return;
  }
  // ---- Q = I - V M, straight to global
  for (int ti = 0; ti < N8 / 8; ti++)
    for (int tc = 0; tc < N8 / 8; tc++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < K4; k0 += 4)
        dmma(acc, Vs[(ti * 8 + r) * LDV + k0 + q], Mm[(k0 + q) * LDM + tc * 8 + r]);
      const int i = ti * 8 + r;
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int c = tc * 8 + 2 * q + e;
        if (i < n && c < n) Qg[i * n + c] = (i == c ? 1.0 : 0.0) - acc[e];
      }
    }
}

// --------------------------------------------------------------------------
// Level-0 QR completion for leaves with 64 < n <= 128 (config 5: B = 128, k <= 32):
// one CTA of 128 threads per leaf, thread i owns row i of X in registers
// (shifting column window as qr_reg_kernel); the per-column reductions are a
// warp butterfly plus a 4-way cross-warp sum through shared memory.  Same
// convention H; emits R^ and the compact-WY factors V, M = T V^T only (leaves
// this large always take the compact-WY congruence; wy_form_q_kernel forms Q).
// --------------------------------------------------------------------------
// Also at levels >= 1 (X = [R^_c1 T[:k1]; R^_c2 T[k1:]], the children's R^ and
// T staged in the V / T / M region first) and with the explicit Q = I - V M
// written to `qout` when wy == nullptr: the k = n / 2 clusters of configs 4 and
// 5 (n = 64, k = 32) run here at 5 CTAs (10 warps) per SM instead of the
// warp-per-cluster kernel's 45 KB of shared memory per warp (4 warps per SM).
template <int KP, int NW>
__global__ void __launch_bounds__(32 * NW) qr_cta_kernel(Side sd, int nclust, const double *__restrict__ leaf,
                                                     double *__restrict__ rh, double *__restrict__ wy, int wy_kp,
                                                     int wy_n, const uint64_t *meta_magic, uint64_t magic, int L = 0,
                                                     int level = 0, const double *__restrict__ transfer = nullptr,
                                                     double *__restrict__ qout = nullptr) {
  if (meta_magic && threadIdx.x == 0 && blockIdx.x == 0 && *meta_magic != magic) __trap();
  constexpr int NROW = 32 * NW;  // rows (one per thread)
  constexpr int LDV = KP + 4, LDT = KP + 4, LDM = NROW + 4;
  extern __shared__ __align__(16) double smc[];
  double *Vs = smc;               // NROW x LDV (unit lower trapezoidal, zero padded)
  double *Tw = Vs + NROW * LDV;   // KP x LDT
  double *Mm = Tw + KP * LDT;    // G = V^T V (KP x KP, ld LDT), then M = T V^T (KP x LDM)
  __shared__ double red_ss[2][NW], red_w[2][NW][KP], wsum[KP];
  __shared__ double s_alpha[2];
  const int ci = blockIdx.x;
  if (ci >= nclust) return;
  const int64_t cl = lvl_off_d(L, level) + ci;
  const int n = sd.n[cl], k = sd.k[cl];
  if (n == 0 || !sd.need[cl]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *Wg = wy ? wy + int64_t(ci) * 2 * wy_n * wy_kp : nullptr;
  double *Qg = wy ? nullptr : qout + sd.q_off[cl];
  if (k == 0) {
    if (Wg)
      for (int idx = tid; idx < 2 * wy_n * wy_kp; idx += blockDim.x) Wg[idx] = 0.0;
    else
      for (int idx = tid; idx < n * n; idx += blockDim.x) Qg[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
    return;
  }
  double x[KP];
  if (level == 0) {
    const double *R = leaf + sd.leaf_off[cl];
#pragma unroll
    for (int c = 0; c < KP; c++) x[c] = (tid < n && c < k) ? __ldg(R + int64_t(tid) * k + c) : 0.0;
  } else {  // X = [R^_c1 T[:k1]; R^_c2 T[k1:]]
    const int64_t c1 = lvl_off_d(L, level - 1) + 2 * int64_t(ci), c2 = c1 + 1;
    const int k1 = sd.k[c1], k2 = sd.k[c2];
    double *sT = smc, *sR1 = sT + n * k, *sR2 = sR1 + k1 * k1;
    const double *T = transfer + sd.tr_off[cl];
    for (int idx = tid; idx < n * k; idx += blockDim.x) cp8(&sT[idx], T + idx, true);
    for (int idx = tid; idx < k1 * k1; idx += blockDim.x) cp8(&sR1[idx], rh + sd.rh_off[c1] + idx, true);
    for (int idx = tid; idx < k2 * k2; idx += blockDim.x) cp8(&sR2[idx], rh + sd.rh_off[c2] + idx, true);
    cp_commit();
    cp_wait_all();
    __syncthreads();
#pragma unroll
    for (int c = 0; c < KP; c++) x[c] = 0.0;
    if (tid < n) {
      const bool first = tid < k1;
      const int ii = first ? tid : tid - k1, kk = first ? k1 : k2, roff = first ? 0 : k1;
      const double *Rr = first ? sR1 : sR2;
      for (int l = ii; l < kk; l++) {
        const double rv = Rr[ii * kk + l];
        const double *Trow = sT + (roff + l) * k;
#pragma unroll
        for (int c = 0; c < KP; c++)
          if (c < k) x[c] = fma(rv, Trow[c], x[c]);
      }
    }
    __syncthreads();  // the staging region becomes V / T / M
  }
  for (int idx = tid; idx < NROW * LDV; idx += blockDim.x) Vs[idx] = 0.0;
  for (int idx = tid; idx < KP * LDT; idx += blockDim.x) Tw[idx] = 0.0;
  double *Rg = rh + sd.rh_off[cl];
  for (int j = 0; j < k; j++) {
    const int b = j & 1, w_left = k - j;
    double ss = (tid > j && tid < n) ? x[0] * x[0] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red_ss[b][warp] = ss;
    if (tid == j) s_alpha[b] = x[0];
    __syncthreads();
    ss = 0.0;
#pragma unroll
    for (int w_ = 0; w_ < NW; w_++) ss += red_ss[b][w_];
    const double alpha = s_alpha[b];
    const double sigma = sqrt(ss);
    double beta, t;
    if (sigma == 0.0) {
      t = 0.0;
      beta = alpha;
    } else {
      const double sgn = alpha < 0.0 ? -1.0 : 1.0;
      beta = -sgn * hypot(alpha, sigma);
      t = (beta - alpha) / beta;
    }
    const double rdiv = 1.0 / (alpha - beta);
    const double v = (tid == j) ? 1.0 : ((t != 0.0 && tid > j && tid < n) ? x[0] * rdiv : 0.0);
    if (t != 0.0) {  // uniform over the CTA
      double w[KP];
#pragma unroll
      for (int c = 0; c < KP; c++) w[c] = (c >= 1 && c < w_left) ? v * x[c] : 0.0;
      warp_allreduce_vec<KP>(w, lane);
      if (lane < KP) {
        double mine = w[0];
#pragma unroll
        for (int c = 1; c < KP; c++)
          if (lane == c) mine = w[c];
        red_w[b][warp][lane] = mine;
      }
      __syncthreads();
      if (tid < KP) {
        double acc_ = 0.0;
#pragma unroll
        for (int w_ = 0; w_ < NW; w_++) acc_ += red_w[b][w_][tid];
        wsum[tid] = acc_;
      }
      __syncthreads();
#pragma unroll
      for (int c = 1; c < KP; c++)
        if (c < w_left) x[c] = fma(-(t * wsum[c]), v, x[c]);
    }
    if (tid >= j && tid < n) Vs[tid * LDV + j] = v;
    if (tid == j) {
      for (int c = 0; c < j; c++) Rg[j * k + c] = 0.0;
      Rg[j * k + j] = beta;
#pragma unroll
      for (int c = 1; c < KP; c++)
        if (c < w_left) Rg[j * k + j + c] = x[c];
    }
    if (tid == 0) Tw[j * LDT + j] = t;
#pragma unroll
    for (int c = 0; c < KP - 1; c++) x[c] = x[c + 1];
    x[KP - 1] = 0.0;
  }
  __syncthreads();
  const int r = lane >> 2, q = lane & 3;
  constexpr int KT = KP / 8;
  // ---- G = V^T V (KP x KP, all tiles; warps take tiles round robin)
  for (int tile = warp; tile < KT * KT; tile += NW) {
    const int ta = tile / KT, tb = tile % KT;
    double acc[2] = {0.0, 0.0};
    for (int k0 = 0; k0 < NROW; k0 += 4) dmma(acc, Vs[(k0 + q) * LDV + ta * 8 + r], Vs[(k0 + q) * LDV + tb * 8 + r]);
    Mm[(ta * 8 + r) * LDT + tb * 8 + 2 * q] = acc[0];
    Mm[(ta * 8 + r) * LDT + tb * 8 + 2 * q + 1] = acc[1];
  }
  __syncthreads();
  // ---- T recurrence (dlarft, forward, columnwise), warp 0
  if (warp == 0) {
    for (int j = 1; j < k; j++) {
      const double tj = Tw[j * LDT + j];
      double vv = 0.0;
      if (lane < j)
        for (int l = lane; l < j; l++) vv = fma(Tw[lane * LDT + l], Mm[l * LDT + j], vv);
      __syncwarp();
      if (lane < j) Tw[lane * LDT + j] = -tj * vv;
      __syncwarp();
    }
  }
  __syncthreads();
  // ---- M = T V^T (KP x 128); G is dead.  Compact-WY output with the leaf's
  // padded layout (wy_kp == KP, wy_n == NROW): straight from the accumulators to
  // global (rows a >= k and columns c >= n come out zero: T and V are zero
  // there), so the launch needs no M staging (4 instead of 2 CTAs per SM);
  // otherwise -> Mm (ld LDM) for the explicit Q below / the padded copy.
  const bool m_direct = Wg && wy_kp == KP && wy_n == NROW;
  for (int tile = warp; tile < KT * (NROW / 8); tile += NW) {
    const int ta = tile / (NROW / 8), tc = tile % (NROW / 8);
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 4) dmma(acc, Tw[(ta * 8 + r) * LDT + k0 + q], Vs[(tc * 8 + r) * LDV + k0 + q]);
    __syncwarp();
    if (m_direct) {
      double *Mg = Wg + wy_n * wy_kp + (ta * 8 + r) * wy_n + tc * 8 + 2 * q;
      Mg[0] = acc[0];
      Mg[1] = acc[1];
    } else {
      Mm[(ta * 8 + r) * LDM + tc * 8 + 2 * q] = acc[0];
      Mm[(ta * 8 + r) * LDM + tc * 8 + 2 * q + 1] = acc[1];
    }
  }
  __syncthreads();
  if (!Wg) {  // Q = I - V M (n x n) from 8 x 8 DMMA tiles, straight to global
    const int N8 = (n + 7) / 8;
    for (int tile = warp; tile < N8 * N8; tile += NW) {
      const int ti = tile / N8, tc = tile % N8;
      double acc[2] = {0.0, 0.0};
#pragma unroll
      for (int k0 = 0; k0 < KP; k0 += 4) dmma(acc, Vs[(ti * 8 + r) * LDV + k0 + q], Mm[(k0 + q) * LDM + tc * 8 + r]);
      const int i = ti * 8 + r;
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int c = tc * 8 + 2 * q + e;
        if (i < n && c < n) Qg[i * n + c] = (i == c ? 1.0 : 0.0) - acc[e];
      }
    }
    return;
  }
  for (int idx = tid; idx < wy_n * wy_kp; idx += blockDim.x) {
    const int i = idx / wy_kp, c = idx - i * wy_kp;
    Wg[idx] = (i < n && c < k) ? Vs[i * LDV + c] : 0.0;
  }
  if (!m_direct)
    for (int idx = tid; idx < wy_n * wy_kp; idx += blockDim.x) {
      const int a = idx / wy_n, c = idx - a * wy_n;
      Wg[wy_n * wy_kp + idx] = (a < k && c < n) ? Mm[a * LDM + c] : 0.0;
    }
}

// --------------------------------------------------------------------------
// Level-0 Q from its compact-WY form, Q = I - V M (the same product qr_reg_kernel
// forms at the other levels), when the level-0 congruence runs on V / M: it is
// only an output (and input of the applies), so it is formed off the critical
// path.  One CTA (4 warps) per leaf; warp w computes rows 16w..16w+15.
// --------------------------------------------------------------------------
template <int KP, int NW>
__global__ void __launch_bounds__(NW * 2) wy_form_q_kernel(Side sr, Side sc, const double *__restrict__ wy_r,
                                                           const double *__restrict__ wy_c, double *__restrict__ q_r,
                                                           double *__restrict__ q_c, int64_t nclust) {
  constexpr int LDV = KP + 4, LDM = NW + 4;
  extern __shared__ __align__(16) double smw[];
  double *sV = smw, *sM = smw + NW * LDV;
  const bool col = blockIdx.x >= nclust;  // second half of the grid: column side (general mode)
  const int64_t cl = col ? blockIdx.x - nclust : blockIdx.x;
  const Side &sd = col ? sc : sr;
  const double *wy = col ? wy_c : wy_r;
  double *qout = col ? q_c : q_r;
  const int n = sd.n[cl];
  if (n == 0 || !sd.need[cl]) return;
  const double *g = wy + cl * (2 * NW * KP);
  async_tile<NW, KP, LDV>(sV, g, NW, KP, KP, g);
  async_tile<KP, NW, LDM>(sM, g + NW * KP, KP, NW, NW, g);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int m0 = warp * 16;
  double *Q = qout + sd.q_off[cl];
  for (int n0 = 0; n0 < NW; n0 += 64) {  // 16 x 64 output tiles per warp
    double acc[2][8][2];
    zero_acc(acc);
    warp_gemm<LDV, LDM, 2, 8, false>(sV, sM, m0, n0, KP, acc);
#pragma unroll
    for (int i = 0; i < 2; i++) {
      const int row = m0 + i * 8 + r;
      if (row >= n) continue;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int c = n0 + j * 8 + 2 * q;
        const double v0 = (row == c ? 1.0 : 0.0) - acc[i][j][0];
        const double v1 = (row == c + 1 ? 1.0 : 0.0) - acc[i][j][1];
        if (c + 1 < n)
          store2(Q + int64_t(row) * n + c, v0, v1);
        else if (c < n)
          Q[int64_t(row) * n + c] = v0;
      }
    }
  }
}

template <int KP, int NW>
static h2sp_status launch_wy_form_q(unsigned grid, cudaStream_t st, const Side &rs, const Side &cs, const double *wr,
                             const double *wc, double *qr, double *qc, int64_t nleaf) {
  constexpr size_t smem = size_t(NW * (KP + 4) + KP * (NW + 4)) * sizeof(double);
  if (h2sp_status e = ensure_smem((const void *)wy_form_q_kernel<KP, NW>, smem)) return e;
  wy_form_q_kernel<KP, NW><<<grid, NW * 2, smem, st>>>(rs, cs, wr, wc, qr, qc, nleaf);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}

// --------------------------------------------------------------------------
// Couplings in orthogonalised coordinates: D~ = R^R_t D R^C_s^T.
// One warp per admissible pair, `ipc` pairs per CTA.  Operands staged with
// cp.async into the warp's slice of shared memory (zero padded), then the two
// small products on the DMMA pipe: W = D R^_s^T, D~ = R^_t W.
// Per-warp shared memory (doubles): D A8 x LDB | Rs B8 x LDB | Rt A8 x LDA | W A8 x LDB
// --------------------------------------------------------------------------
// Kernel function of h2sp_close_gen for two distinct points x, y (dim coordinates):
// r^2 summed without FMA contraction in coordinate order (K(x, y) == K(y, x)
// bitwise), rsqrt and multiplications by precomputed constants instead of sqrt
// and divisions.  Shared by h2sp_eval_kernel_blocks and the matrix-free couplings.
struct CloseGen {
  const double *pts;
  int dim, kind;
  double p0, p1;
  double q0;                         // exp: -1 / p0; Laplace: 1 / (4 pi)
  const double *nodes_row, *nodes_col;  // matrix-free couplings (nullptr: read D)
};

__device__ __forceinline__ double kernel_eval(const CloseGen &g, const double *x, const double *y) {
  const double d0 = __dsub_rn(__ldg(x), __ldg(y));
  double r2 = __dmul_rn(d0, d0);
  if (g.dim > 1) {
    const double d1 = __dsub_rn(__ldg(x + 1), __ldg(y + 1));
    r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
  }
  if (g.dim > 2) {
    const double d2 = __dsub_rn(__ldg(x + 2), __ldg(y + 2));
    r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
  }
  const double ir = rsqrt(r2);
  if (g.kind == H2SP_KERNEL_LAPLACE) return g.q0 * ir;
  const double r = r2 > 0.0 ? r2 * ir : 0.0;
  return g.kind == H2SP_KERNEL_EXP ? exp(r * g.q0) : 1.0 / (r + g.p0);
}

__host__ __device__ inline int coup_ld(int k) { return rup(rup(k, 8), 16) + 4; }
__host__ __device__ inline int coup_warp_doubles(int kt, int ks) {
  const int A8 = rup(kt, 8), B8 = rup(ks, 8);
  return A8 * coup_ld(ks) * 2 + B8 * coup_ld(ks) + A8 * coup_ld(kt) + 2;
}

// Register variant for ranks <= KP <= 32 (every BASELINE config): one warp per
// pair, no shared memory -- X = R^_t D with both operands' DMMA fragments read
// straight from L1/L2 (R^ blocks are shared by many pairs), then
// D~ = X R^_s^T with X's A fragments taken from the accumulators by quad
// shuffles.  Zero-padded to KP; ragged ranks take the predicated loads.
// GEN: D evaluated from the cluster nodes (h2sp_close_gen.nodes_*): B fragment
// (kk, n) = K(node kk of t, node n of s), each entry of D exactly once per warp.
template <int KP, bool GEN>
__global__ void __launch_bounds__(128, KP == 32 ? 3 : 4) coupling_reg_kernel(const CouplingItem *__restrict__ items, int64_t n_items,
                                                           Side rs, Side cs, const double *__restrict__ rh_row,
                                                           const double *__restrict__ rh_col,
                                                           const double *__restrict__ D, double *__restrict__ dt,
                                                           CloseGen g) {
  constexpr int T = KP / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (item >= n_items) return;
  const CouplingItem it = items[item];
  const int kt = rs.k[it.t], ks = cs.k[it.s];
  const double *Rt = rh_row + rs.rh_off[it.t];   // kt x kt, row-major
  const double *Rs = rh_col + cs.rh_off[it.s];   // ks x ks
  const double *Dg = GEN ? nullptr : D + it.d_src;  // kt x ks
  const double *xt = GEN ? g.nodes_row + rs.zb_off[it.t] * g.dim : nullptr;  // nodes of t, s
  const double *xs = GEN ? g.nodes_col + cs.zb_off[it.s] * g.dim : nullptr;
  const int r = lane >> 2, q = lane & 3;
  // ---- X = R^_t D: A(m, kk) = R^_t[m][kk], B(kk, n) = D[kk][n]
  double X[T][T][2];
#pragma unroll
  for (int i = 0; i < T; i++)
#pragma unroll
    for (int j = 0; j < T; j++) X[i][j][0] = X[i][j][1] = 0.0;
#pragma unroll 2
  for (int k0 = 0; k0 < KP; k0 += 4) {
    const int kk = k0 + q;
    double a[T], b[T];
#pragma unroll
    for (int i = 0; i < T; i++) {
      const int m = i * 8 + r;
      a[i] = (m < kt && kk < kt) ? __ldg(Rt + m * kt + kk) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < T; j++) {
      const int n = j * 8 + r;
      if constexpr (GEN)
        b[j] = (kk < kt && n < ks) ? kernel_eval(g, xt + kk * g.dim, xs + n * g.dim) : 0.0;
      else
        b[j] = (kk < kt && n < ks) ? __ldg(Dg + kk * ks + n) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < T; i++)
#pragma unroll
      for (int j = 0; j < T; j++) dmma(X[i][j], a[i], b[j]);
  }
  // ---- D~ = X R^_s^T: A(m, kk) = X[m][kk] (lane (r, (k0 % 8 + q) / 2), element q % 2),
  //      B(kk, n) = R^_s[n][kk]
  //      in passes of JH column tiles (KP = 32: two passes, to stay within 128 registers)
  constexpr int JH = KP == 32 ? T / 2 : T;
  const int src_lo = r * 4 + (q >> 1), src_hi = src_lo + 2;
  double *out = dt + it.dt_dst;
#pragma unroll
  for (int j0 = 0; j0 < T; j0 += JH) {
    double Y[T][JH][2];
#pragma unroll
    for (int i = 0; i < T; i++)
#pragma unroll
      for (int j = 0; j < JH; j++) Y[i][j][0] = Y[i][j][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const int kk = k0 + q;
      double a[T], b[JH];
#pragma unroll
      for (int i = 0; i < T; i++) {
        const double e0 = __shfl_sync(0xffffffffu, X[i][jt][0], srcl);
        const double e1 = __shfl_sync(0xffffffffu, X[i][jt][1], srcl);
        a[i] = (q & 1) ? e1 : e0;
      }
#pragma unroll
      for (int j = 0; j < JH; j++) {
        const int n = (j0 + j) * 8 + r;
        b[j] = (n < ks && kk < ks) ? __ldg(Rs + n * ks + kk) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < T; i++)
#pragma unroll
        for (int j = 0; j < JH; j++) dmma(Y[i][j], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < T; i++) {
      const int m = i * 8 + r;
      if (m >= kt) continue;
#pragma unroll
      for (int j = 0; j < JH; j++) {
        const int n = (j0 + j) * 8 + 2 * q;
        if (n < ks) out[m * ks + n] = Y[i][j][0];
        if (n + 1 < ks) out[m * ks + n + 1] = Y[i][j][1];
      }
    }
  }
}

__global__ void __launch_bounds__(128) coupling_kernel(const CouplingItem *__restrict__ items, int64_t n_items,
                                                       int per_warp, Side rs, Side cs,
                                                       const double *__restrict__ rh_row,
                                                       const double *__restrict__ rh_col,
                                                       const double *__restrict__ D, double *__restrict__ dt) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (item >= n_items) return;
  const CouplingItem it = items[item];
  const int kt = rs.k[it.t], ks = cs.k[it.s];
  const int A8 = rup(kt, 8), B8 = rup(ks, 8), A4 = rup(kt, 4), B4 = rup(ks, 4);
  const int LDA = coup_ld(kt), LDB = coup_ld(ks);
  extern __shared__ __align__(16) double sm[];
  double *sD = sm + size_t(warp) * per_warp;   // A8 x LDB
  double *sRs = sD + A8 * LDB;                 // B8 x LDB
  double *sRt = sRs + B8 * LDB;                // A8 x LDA
  double *sW = sRt + A8 * LDA;                 // A8 x LDB
  const double *Rt = rh_row + rs.rh_off[it.t];
  const double *Rs = rh_col + cs.rh_off[it.s];
  const double *Dg = D + it.d_src;
  for (int idx = lane; idx < A8 * B8; idx += 32) {
    const int i = idx / B8, j = idx % B8;
    const bool v = i < kt && j < ks;
    cp8(&sD[i * LDB + j], v ? (const void *)(Dg + i * ks + j) : (const void *)Dg, v);
  }
  for (int idx = lane; idx < B8 * B8; idx += 32) {
    const int i = idx / B8, j = idx % B8;
    const bool v = i < ks && j < ks;
    cp8(&sRs[i * LDB + j], v ? (const void *)(Rs + i * ks + j) : (const void *)Rs, v);
  }
  for (int idx = lane; idx < A8 * A8; idx += 32) {
    const int i = idx / A8, j = idx % A8;
    const bool v = i < kt && j < kt;
    cp8(&sRt[i * LDA + j], v ? (const void *)(Rt + i * kt + j) : (const void *)Rt, v);
  }
  cp_commit();
  cp_wait_all();
  __syncwarp();
  const int r = lane >> 2, q = lane & 3;
  // W = D R^_s^T : A(m, kk) = D[m][kk], B(kk, n) = R^_s[n][kk]
  for (int ti = 0; ti < A8 / 8; ti++)
    for (int tj = 0; tj < B8 / 8; tj++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < B4; k0 += 4)
        dmma(acc, sD[(ti * 8 + r) * LDB + k0 + q], sRs[(tj * 8 + r) * LDB + k0 + q]);
      sW[(ti * 8 + r) * LDB + tj * 8 + 2 * q] = acc[0];
      sW[(ti * 8 + r) * LDB + tj * 8 + 2 * q + 1] = acc[1];
    }
  __syncwarp();
  // D~ = R^_t W : A(m, kk) = R^_t[m][kk], B(kk, n) = W[kk][n]
  double *out = dt + it.dt_dst;
  for (int ti = 0; ti < A8 / 8; ti++)
    for (int tj = 0; tj < B8 / 8; tj++) {
      double acc[2] = {0.0, 0.0};
      for (int k0 = 0; k0 < A4; k0 += 4)
        dmma(acc, sRt[(ti * 8 + r) * LDA + k0 + q], sW[(k0 + q) * LDB + tj * 8 + r]);
      const int i = ti * 8 + r;
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int j = tj * 8 + 2 * q + e;
        if (i < kt && j < ks) out[i * ks + j] = acc[e];
      }
    }
}

// --------------------------------------------------------------------------
// Steps (iv)+(ii)+(iii): one CTA per chunk of pairs (t, s_1..s_c) of one block
// row t.  Q_t resident in shared memory; per pair: gather G (level 0: C_ts;
// else the 2x2 children arrangement of bb parts / D~) and Q_s with cp.async,
// T = Q_t^T G, H = T Q_s on the FP64 tensor pipe (DMMA), then scatter H's
// four parts (nn -> S, bb -> next level, bn / nb -> strips).
// --------------------------------------------------------------------------
template <int NP>
struct PairCfg {
  static constexpr int LD = NP + 4;       // conflict-free DMMA fragment loads
  static constexpr int TM = 1;                    // 8-row tiles per warp
  static constexpr int WARPS = NP / (8 * TM);     // warp w owns rows [8*TM*w, 8*TM*(w+1)) of T and H
  static constexpr int THREADS = WARPS * 32;
  static constexpr int TN = NP / 8;
  static constexpr size_t SMEM = size_t(3) * NP * LD * sizeof(double);
  static constexpr int MIN_BLOCKS = (NP == 64) ? 2 : (NP == 48) ? 3 : 6;  // smem-bound anyway at 48, 64
};


struct PairArgs {
  const PairItem *items;
  const Chunk *chunks;
  Side rs, cs;
  int L, level, B;
  int sym;
  const double *close;
  CloseGen gen;
  const double *bb_in, *dt_in;        // level k-1 results
  const double *q_row, *q_col;
  double *s_val, *bb_out, *yr, *yc;   // yc: transposed column strips (general) / yr (symmetric)
  const double *bw;                   // bench mode: w (S column order)
  double2 *part;                      // bench mode: partial slots {S w, |S|^2}
  int debug;                          // -DH2SP_TIMING_KNOBS builds only (attribution): 1 = skip scatter, 2 = skip loads
};

// close_gen mode: C_ts[i][j] = K(x_{tB+i}, x_{sB+j}) (include/h2sp.h).  A thread
// owns column j of the tile (point y_j of s, kept in registers) and evaluates
// rows i on request.  r^2 is summed without FMA contraction in coordinate
// order, so r(i, j) == r(j, i) bitwise and diagonal blocks come out symmetric.
// rsqrt / multiplications by precomputed constants replace sqrt and the
// divisions (a few ulp from the numpy generator; parity tolerance 1e-13).
struct GenCol {
  const double *xt;  // points of t
  double y0, y1, y2;
  int j, nt;
  bool jok, tss;     // column inside the tile; t == s
};

__device__ __forceinline__ GenCol gen_col(const CloseGen &g, int t, int s, int nt, int ns, int B, int j) {
  GenCol c;
  c.j = j;
  c.nt = nt;
  c.jok = j < ns;
  c.tss = t == s;
  c.xt = g.pts + int64_t(t) * B * g.dim;
  c.y0 = c.y1 = c.y2 = 0.0;
  if (c.jok) {
    const double *ys = g.pts + (int64_t(s) * B + j) * g.dim;
    c.y0 = __ldg(ys);
    if (g.dim > 1) c.y1 = __ldg(ys + 1);
    if (g.dim > 2) c.y2 = __ldg(ys + 2);
  }
  return c;
}

__device__ __forceinline__ double gen_entry(const CloseGen &g, const GenCol &c, int i) {
  if (!c.jok || i >= c.nt) return 0.0;
  const double *x = c.xt + i * g.dim;
  const double d0 = __dsub_rn(__ldg(x), c.y0);
  double r2 = __dmul_rn(d0, d0);
  if (g.dim > 1) {
    const double d1 = __dsub_rn(__ldg(x + 1), c.y1);
    r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
  }
  if (g.dim > 2) {
    const double d2 = __dsub_rn(__ldg(x + 2), c.y2);
    r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
  }
  const bool same = c.tss && i == c.j;
  const double ir = rsqrt(r2);                 // +inf at r = 0
  if (g.kind == H2SP_KERNEL_LAPLACE) return same ? g.p1 : g.q0 * ir;   // q0 = 1 / (4 pi)
  const double r = r2 > 0.0 ? r2 * ir : 0.0;
  double v = g.kind == H2SP_KERNEL_EXP ? exp(r * g.q0)                  // q0 = -1 / p0
                                       : 1.0 / (r + g.p0);
  return same ? v + g.p1 : v;
}

// exp(x) for x <= 0 with a 64-entry table of 2^(j/64) (in shared memory): x =
// (k/64) ln 2 + f, |f| <= ln2/128, exp(f) by its degree-6 Taylor polynomial
// (truncation < 3e-20), result 2^(k>>6) * tab[k & 63] * exp(f): ~10 FP64
// operations instead of the library exp's ~25, within a few ulp of it -- the
// FP64 datapath is shared with the DMMA (DMMA = DFMA rate on sm_100a).
__device__ const double g_exp2_64[64] = {1.0,1.0108892860517005,1.0218971486541166,1.0330248790212284,1.0442737824274138,1.0556451783605572,1.0671404006768237,1.0787607977571199,1.0905077326652577,1.102382583307841,1.1143867425958924,1.1265216186082418,1.1387886347566916,1.1511892299529827,1.1637248587775775,1.1763969916502812,1.189207115002721,1.202156731452703,1.215247359980469,1.22848053610687,1.241857812073484,1.255380757024691,1.2690509571917332,1.2828700160787783,1.2968395546510096,1.3109612115247644,1.3252366431597413,1.339667524053303,1.3542555469368927,1.3690024229745905,1.383909881963832,1.3989796725383112,1.4142135623730951,1.42961333839197,1.4451808069770467,1.460917794180647,1.4768261459394993,1.4929077282912648,1.5091644275934228,1.5255981507445384,1.5422108254079407,1.559004400237837,1.5759808451078865,1.593142151342267,1.6104903319492543,1.6280274218573478,1.645755478153965,1.6636765803267364,1.681792830507429,1.7001063537185235,1.718619298122478,1.7373338352737062,1.7562521603732995,1.7753764925265212,1.7947090750031072,1.8142521755003989,1.8340080864093424,1.8539791250833855,1.8741676341103,1.8945759815869656,1.9152065613971474,1.9360617934922943,1.9571441241754002,1.978456026387951};

__device__ __forceinline__ double exp_neg_tab(double x, const double *tab) {
  if (x < -700.0) return 0.0;
  const double kd = rint(x * 92.33248261689366);                         // 64 / ln 2
  const double f = fma(kd, -2.9815858269852933e-12, fma(kd, -0.01083042469326756, x));  // x - kd ln2/64
  double pz = fma(f, 1.0 / 720.0, 1.0 / 120.0);
  pz = fma(pz, f, 1.0 / 24.0);
  pz = fma(pz, f, 1.0 / 6.0);
  pz = fma(pz, f, 0.5);
  pz = fma(pz, f, 1.0);
  pz = fma(pz, f, 1.0);
  const int k = int(kd);
  return __hiloint2double((1023 + (k >> 6)) << 20, 0) * (tab[k & 63] * pz);
}

// gen_entry with t's points staged in shared memory (xs: nt x dim) and the exp table
__device__ __forceinline__ double gen_entry_s(const CloseGen &g, const GenCol &c, int i, const double *xs,
                                              const double *tab) {
  if (!c.jok || i >= c.nt) return 0.0;
  const double *x = xs + i * g.dim;
  const double d0 = __dsub_rn(x[0], c.y0);
  double r2 = __dmul_rn(d0, d0);
  if (g.dim > 1) {
    const double d1 = __dsub_rn(x[1], c.y1);
    r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
  }
  if (g.dim > 2) {
    const double d2 = __dsub_rn(x[2], c.y2);
    r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
  }
  const bool same = c.tss && i == c.j;
  const double ir = rsqrt(r2);
  if (g.kind == H2SP_KERNEL_LAPLACE) return same ? g.p1 : g.q0 * ir;
  const double r = r2 > 0.0 ? r2 * ir : 0.0;
  const double v = g.kind == H2SP_KERNEL_EXP ? exp_neg_tab(r * g.q0, tab) : 1.0 / (r + g.p0);
  return same ? v + g.p1 : v;
}

template <int NP, int LD>
__device__ __forceinline__ void gen_close_tile(double *sG, const CloseGen &g, int t, int s, int nt, int ns, int B) {
  const GenCol c = gen_col(g, t, s, nt, ns, B, threadIdx.x % NP);
  for (int i = threadIdx.x / NP; i < NP; i += blockDim.x / NP) sG[i * LD + c.j] = gen_entry(g, c, i);
}

// h2sp_eval_kernel_blocks: one CTA per block, threads over its entries (same
// distance arithmetic as gen_entry, so K(x, y) == K(y, x) bitwise).
__global__ void __launch_bounds__(128) kernel_blocks_kernel(CloseGen g, const double *__restrict__ xn,
                                                            const double *__restrict__ yn,
                                                            const h2sp_block_desc *__restrict__ blocks,
                                                            double *__restrict__ out) {
  const h2sp_block_desc bd = blocks[blockIdx.x];
  const int ne = bd.nx * bd.ny;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const int i = e / bd.ny, j = e - i * bd.ny;
    const double *x = xn + (bd.x_off + i) * g.dim, *y = yn + (bd.y_off + j) * g.dim;
    out[bd.out_off + e] = kernel_eval(g, x, y);
  }
}

h2sp_status launch_kernel_blocks(const h2sp_close_gen *k, const double *xn, const double *yn,
                                 const h2sp_block_desc *blocks, int64_t n_blocks, double *out, void *stream) {
  if (n_blocks == 0) return H2SP_OK;
  CloseGen g{};
  g.pts = nullptr;
  g.dim = k->dim;
  g.kind = k->kernel;
  g.p0 = k->p0;
  g.p1 = k->p1;
  g.q0 = g.kind == H2SP_KERNEL_EXP ? -1.0 / g.p0 : 1.0 / (4.0 * 3.141592653589793);
  for (int64_t b0 = 0; b0 < n_blocks; b0 += (int64_t(1) << 30)) {
    const int64_t nb = std::min<int64_t>(n_blocks - b0, int64_t(1) << 30);
    kernel_blocks_kernel<<<unsigned(nb), 128, 0, (cudaStream_t)stream>>>(g, xn, yn, blocks + b0, out);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return fail(H2SP_ECUDA, std::string("kernel blocks: ") + cudaGetErrorString(err));
  }
  return H2SP_OK;
}

// Level-0 G = C_ts: cp.async copy of the stored block, or evaluated (close_gen).
template <int NP, int LD, bool GEN>
__device__ __forceinline__ void load_close(const PairArgs &A, const PairItem &it, double *sG) {
  if constexpr (GEN)
    gen_close_tile<NP, LD>(sG, A.gen, it.t, it.s, it.nt, it.ns, A.B);
  else
    async_tile<NP, NP, LD>(sG, A.close + it.g_src[0], it.nt, it.ns, A.B, A.chunks);
}

// Issue the cp.async copies of G_ts (level 0: C_ts; else the 2x2 arrangement of
// the children's bb parts / D~) into sG.
template <int NP, bool GEN>
__device__ __forceinline__ void pair_load_G(const PairArgs &A, const PairItem &it, double *sG) {
  constexpr int LD = PairCfg<NP>::LD;
  const int nt = it.nt, ns = it.ns;
  const void *any = A.chunks;
  if (A.level == 0) {
    load_close<NP, LD, GEN>(A, it, sG);
  } else {
    const int kr0 = it.kr0, kr1 = it.kr1;
    const int kc0 = it.kc0, kc1 = it.kc1;
    // blockDim.x is a multiple of NP: each thread keeps one column j and walks
    // rows i = tid/NP, +R, ...; the two quadrant sources of that column (a = 0, 1)
    // are resolved once into a base pointer and a row stride.
    const int j = threadIdx.x % NP;
    const int R = blockDim.x / NP;
    const int b = j >= kc0;
    const int jj = b ? j - kc0 : j, kb = b ? kc1 : kc0;
    const bool jok = j < ns;
    const double *base[2];
    int64_t st[2];
#pragma unroll
    for (int a = 0; a < 2; a++) {
      const int ka = a ? kr1 : kr0;
      const int q = a * 2 + b;
      const int kind = (it.gkind >> (4 * q)) & 15;
      const int64_t off = it.g_src[q];
      base[a] = nullptr;
      st[a] = 0;
      switch (kind) {
        case G_BB: base[a] = A.bb_in + off + jj; st[a] = kb; break;
        case G_BB_T: base[a] = A.bb_in + off + int64_t(jj) * ka; st[a] = 1; break;
        case G_DT: base[a] = A.dt_in + off + jj; st[a] = kb; break;
        case G_DT_T: base[a] = A.dt_in + off + int64_t(jj) * ka; st[a] = 1; break;
        default: break;
      }
    }
    for (int i = threadIdx.x / NP; i < NP; i += R) {
      const int a = i >= kr0;
      const int ii = a ? i - kr0 : i;
      const double *bp = a ? base[1] : base[0];
      const bool ok = jok && i < nt && bp != nullptr;
      const double *src = ok ? bp + ii * (a ? st[1] : st[0]) : reinterpret_cast<const double *>(any);
      cp8(&sG[i * LD + j], src, ok);
    }
  }
}

// Scatter of one lane's two horizontally adjacent H entries (row, col), (row, col+1)
// of an 8x8 tile to the four parts of step (iii): nn -> S (+ mirror), bb -> next
// level, bn -> row-strip panel, nb^T -> column-strip panel.  Whole tiles inside
// one region (the common case) take the short branch; tiles that straddle
// k_t / k_s or the matrix edge, and diagonal blocks in symmetric mode
// (H_sym[i][j] = H[min][max], each upper entry written twice) go per element.
struct PairDst {          // the destinations of one pair, kept in registers
  int64_t s_dst, s_dst_m, bb_dst, yr_dst, yc_dst;
  int32_t s_ld, s_ld_m, yr_ld, yc_ld;
  int32_t nt, ns, kt, ks;
  bool dsym;
};

// BENCH (bench mode): the nn part is not stored here (bench_pair reduces it).
template <bool BENCH = false>
__device__ __forceinline__ void scatter_pair2(const PairArgs &A, const PairDst &D, int row0, int col0, int row,
                                              int col, double v0, double v1) {
  const bool r_nn = row0 >= D.kt, r_bb = row0 + 8 <= D.kt;
  const bool c_nn = col0 >= D.ks, c_bb = col0 + 8 <= D.ks;
  if (row0 + 8 <= D.nt && col0 + 8 <= D.ns && !D.dsym && (r_nn || r_bb) && (c_nn || c_bb)) {
    if (r_nn && c_nn) {
      if (BENCH) return;
      const int a = row - D.kt, b = col - D.ks;
      if (D.s_dst >= 0) store2_s(A.s_val + D.s_dst + int64_t(a) * D.s_ld + b, v0, v1);
      if (D.s_dst_m >= 0 && !(A.debug & 4)) {
        double *d = A.s_val + D.s_dst_m + int64_t(b) * D.s_ld_m + a;
        st_s(d, v0);
        st_s(d + D.s_ld_m, v1);
      }
    } else if (r_nn) {
      if (D.yc_dst >= 0) {
        double *d = A.yc + D.yc_dst + int64_t(col) * D.yc_ld + (row - D.kt);
        d[0] = v0;
        d[D.yc_ld] = v1;
      }
    } else if (c_bb) {
      if (D.bb_dst >= 0) store2(A.bb_out + D.bb_dst + row * D.ks + col, v0, v1);
    } else if (D.yr_dst >= 0) {
      store2(A.yr + D.yr_dst + int64_t(row) * D.yr_ld + (col - D.ks), v0, v1);
    }
    return;
  }
  if (row >= D.nt) return;
#pragma unroll 1
  for (int e = 0; e < 2; e++) {
    const int c = col + e;
    if (c >= D.ns) continue;
    const double v = e ? v1 : v0;
    if (row >= D.kt) {
      const int a = row - D.kt;
      if (c >= D.ks) {
        if (BENCH) continue;
        const int b = c - D.ks;
        if (D.dsym) {
          if (a <= b) {
            st_s(A.s_val + D.s_dst + int64_t(a) * D.s_ld + b, v);
            st_s(A.s_val + D.s_dst + int64_t(b) * D.s_ld + a, v);
          }
        } else {
          if (D.s_dst >= 0) st_s(A.s_val + D.s_dst + int64_t(a) * D.s_ld + b, v);
          if (D.s_dst_m >= 0) st_s(A.s_val + D.s_dst_m + int64_t(b) * D.s_ld_m + a, v);
        }
      } else if (D.yc_dst >= 0) {
        A.yc[D.yc_dst + int64_t(c) * D.yc_ld + a] = v;
      }
    } else if (c < D.ks) {
      if (D.bb_dst >= 0) {
        if (D.dsym) {
          if (row <= c) {
            A.bb_out[D.bb_dst + row * D.ks + c] = v;
            A.bb_out[D.bb_dst + c * D.ks + row] = v;
          }
        } else {
          A.bb_out[D.bb_dst + row * D.ks + c] = v;
        }
      }
    } else if (D.yr_dst >= 0) {
      A.yr[D.yr_dst + int64_t(row) * D.yr_ld + (c - D.ks)] = v;
    }
  }
}

// Sums over the 8 lane rows r = lane >> 2 of a DMMA accumulator layout (lane
// bits 4, 3, 2) of NV (8 or 4) per-lane values by recursive halving: lanes 16,
// 8, 4 apart exchange the half they do not keep (7 shuffles for 8 values instead
// of 24; 4 values: two halvings and one butterfly step).  Afterwards v[0] of lane
// (r, q) is the total of value index r (NV = 8) or r >> 1 (NV = 4, both lanes of
// a pair) over the 8 lanes with the same q.  Fixed order.
template <int NV>
__device__ __forceinline__ void lane_rows_reduce(double (&v)[NV], int lane) {
  static_assert(NV == 8 || NV == 4, "8 or 4 values per lane");
  int cnt = NV;
#pragma unroll
  for (int o = 16; o >= 4; o >>= 1) {
    if (cnt > 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < cnt / 2; i++) {
        const double send = up ? v[i] : v[i + cnt / 2];
        const double keep = up ? v[i + cnt / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
      cnt >>= 1;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}

// Bench mode (H2SP_PLAN_BENCH, include/h2sp.h h2sp_outputs): the nn part of H --
// S block (t@k, s@k) and, symmetric, its mirror (s@k, t@k) = H_nn^T -- reduced
// to per-row partials {sum_j S[i][j] w[j], sum_j S[i][j]^2} in a fixed order:
// a row's entries are summed by its lane quad (shuffles), a mirror row's
// (= H column's) by the 8 lanes of a tile column (shuffles) and then over the
// warps in warp order through `scratch` (WARPS * NP + NP double2; all threads
// of the CTA must call this).  Diagonal blocks of symmetric mode (H_sym[a][b] =
// H[min(a,b)][max(a,b)]): entries with a <= b come from row a, a > b from
// column a.  Lane (r, q) of warp w holds H[m0 + r][8j + 2q + e].
template <int NP, int TN, int WARPS>
__device__ __forceinline__ void bench_pair(const PairArgs &A, const PairDst &D, int t, int s, const double (&H)[TN][2],
                                           int m0, double2 *scratch, double2 *rowp_ = nullptr,
                                           const double *ws_sm = nullptr, const double *wt_sm = nullptr) {
  static_assert(WARPS * 8 == NP && TN * 8 == NP, "warp w owns rows 8w..8w+7 of the NP x NP tile");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r = lane >> 2, q = lane & 3;
  double2 *colp = scratch, *rowp = rowp_ ? rowp_ : scratch + WARPS * NP;
  const int row = m0 + r, a = row - D.kt;
  const bool vrow = row >= D.kt && row < D.nt;
  const bool cols = D.dsym || D.s_dst_m >= 0;   // CTA-uniform
  const double *w_s = A.bw + A.cs.s_off[s];      // weights of block (t, s)'s columns
  // ws_sm / wt_sm: the weights staged in shared memory by the caller, indexed by tile column / row
  // (zero outside the frozen range) instead of read through L1 per element
  const double wa = (vrow && cols) ? (wt_sm ? wt_sm[row] : __ldg(A.bw + A.cs.s_off[t] + a)) : 0.0;  // weight of mirror column a
  double ry = 0.0, rr = 0.0;
  constexpr int GS = 2;   // accumulator tiles per group of column sums (4 values per lane: 8 shuffles per group
                          // and quantity pair instead of 24; groups of 4 tiles save one more but cost 8 registers)
  static_assert(TN % GS == 0, "whole groups");
#pragma unroll
  for (int j0 = 0; j0 < TN; j0 += GS) {
    // this warp's 8 rows summed per column, one quantity at a time (registers): lane (r, q) ends
    // with value ix of its 2 GS
    const int ix = GS == 4 ? r : r >> 1;
    double2 cres = make_double2(0.0, 0.0);
    {
      double cy[2 * GS];
#pragma unroll
      for (int jj = 0; jj < GS; jj++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int j = j0 + jj;
          const int col = j * 8 + 2 * q + e, b = col - D.ks;
          const bool v = vrow && col >= D.ks && col < D.ns;
          const double h = H[j][e];
          if (v && D.s_dst >= 0 && (!D.dsym || a <= b)) {
            ry = fma(h, ws_sm ? ws_sm[col] : __ldg(w_s + b), ry);
            rr = fma(h, h, rr);
          }
          cy[jj * 2 + e] = (v && (D.dsym ? a < b : true)) ? h * wa : 0.0;
        }
      if (cols) {
        lane_rows_reduce(cy, lane);
        cres.x = cy[0];
      }
    }
    if (cols) {
      double cr[2 * GS];
#pragma unroll
      for (int jj = 0; jj < GS; jj++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int j = j0 + jj;
          const int col = j * 8 + 2 * q + e, b = col - D.ks;
          const bool v = vrow && col >= D.ks && col < D.ns;
          const double h = H[j][e];
          cr[jj * 2 + e] = (v && (D.dsym ? a < b : true)) ? h * h : 0.0;
        }
      lane_rows_reduce(cr, lane);
      cres.y = cr[0];
      if (GS == 4 || (r & 1) == 0) colp[warp * NP + (j0 + (ix >> 1)) * 8 + 2 * q + (ix & 1)] = cres;
    }
  }
  ry += __shfl_xor_sync(0xffffffffu, ry, 1);
  rr += __shfl_xor_sync(0xffffffffu, rr, 1);
  ry += __shfl_xor_sync(0xffffffffu, ry, 2);
  rr += __shfl_xor_sync(0xffffffffu, rr, 2);
  if (q == 0) rowp[row] = make_double2(ry, rr);
  __syncthreads();
  for (int i = threadIdx.x; i < NP; i += blockDim.x) {
    if (D.s_dst >= 0 && i >= D.kt && i < D.nt) {  // row i - kt of block (t, s)
      double2 v = rowp[i];
      if (D.dsym)
#pragma unroll
        for (int w_ = 0; w_ < WARPS; w_++) {
          v.x += colp[w_ * NP + i].x;
          v.y += colp[w_ * NP + i].y;
        }
      A.part[D.s_dst + int64_t(i - D.kt) * D.s_ld] = v;
    }
    if (!D.dsym && D.s_dst_m >= 0 && i >= D.ks && i < D.ns) {  // row i - ks of the mirror block (s, t)
      double2 v = make_double2(0.0, 0.0);
#pragma unroll
      for (int w_ = 0; w_ < WARPS; w_++) {
        v.x += colp[w_ * NP + i].x;
        v.y += colp[w_ * NP + i].y;
      }
      A.part[D.s_dst_m + int64_t(i - D.ks) * D.s_ld_m] = v;
    }
  }
  __syncthreads();
}

// Stage the chunk's work items (<= PAIR_CHUNK_MAX, 144 B each, everything a
// pair needs precomputed by the plan) into shared memory with one batch of
// 16-byte async copies: one global round trip per CTA instead of a chain of
// dependent descriptor loads per pair.
__device__ __forceinline__ int stage_items(const PairItem *items, const Chunk &ch, PairItem *s_it) {
  const int nit = ch.end - ch.begin;
  const char *src = reinterpret_cast<const char *>(items + ch.begin);
  for (int c = threadIdx.x; c < nit * int(sizeof(PairItem) / 16); c += blockDim.x)
    cp16(reinterpret_cast<char *>(s_it) + 16 * c, src + 16 * c);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  return nit;
}

// Steps (iv)+(ii)+(iii) for one chunk of pairs (t, s_1..s_c) of block row t.
// Shared memory: Q_t (resident), G, Q_s; G and Q_s of pair p+1 are fetched
// (cp.async) while pair p computes.  Warp w computes rows [8w, 8w+8) of
// T = Q_t^T G and keeps them in registers; H = T Q_s takes its A fragments
// from T by quad shuffles.  The scatter of pair p's H is software-pipelined
// into the T-GEMM of pair p+1 (8x8 tiles spread over the k-steps), so the
// stores fill issue slots between DMMAs instead of forming an idle phase.
template <int NP, bool GEN, bool BENCH>
__global__ void __launch_bounds__(PairCfg<NP>::THREADS, PairCfg<NP>::MIN_BLOCKS) pair_kernel(PairArgs A) {
  using C = PairCfg<NP>;
  constexpr int LD = C::LD;
  constexpr int TN = C::TN;
  constexpr int TM = C::TM;
  extern __shared__ __align__(16) double sm[];
  double *sQt = sm;
  double *sG = sm + NP * LD;
  double *sQs = sm + 2 * NP * LD;
  __shared__ __align__(16) PairItem s_it[PAIR_CHUNK_MAX];
  const Chunk ch = A.chunks[blockIdx.x];
  stage_items(A.items, ch, s_it);
  int t = s_it[0].t;   // current block row (the chunk may cross rows)
  int nt = s_it[0].nt, ktt = s_it[0].kt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int m0 = warp * 8 * TM;
  // prologue: Q_t, G_0, Q_s0
  async_tile<NP, NP, LD>(sQt, A.q_row + s_it[0].q_off_t, nt, nt, nt, A.chunks);
  pair_load_G<NP, GEN>(A, s_it[0], sG);
  async_tile<NP, NP, LD>(sQs, A.q_col + s_it[0].q_off_s, s_it[0].ns, s_it[0].ns, s_it[0].ns, A.chunks);
  cp_commit();
  double H[TM][TN][2];  // result of the previous pair, scattered during the next T-GEMM
  PairDst prev;
  bool have_prev = false;
  for (int p = ch.begin; p <= ch.end; p++) {
    if (p == ch.end) {  // drain: scatter the last pair
      if (have_prev && !(A.debug & 1)) {
#pragma unroll
        for (int i = 0; i < TM; i++)
#pragma unroll
          for (int j = 0; j < TN; j++)
            scatter_pair2<BENCH>(A, prev, m0 + i * 8, j * 8, m0 + i * 8 + r, j * 8 + 2 * q, H[i][j][0], H[i][j][1]);
      }
      break;
    }
    const PairItem &it = s_it[p - ch.begin];
    const int s = it.s;
    cp_wait_all();
    __syncthreads();
    if (it.t != t) {  // new block row: reload the resident Q_t (G and Q_s of this pair are in flight/landed)
      t = it.t;
      nt = it.nt;
      ktt = it.kt;
      async_tile<NP, NP, LD>(sQt, A.q_row + it.q_off_t, nt, nt, nt, A.chunks);
      cp_commit();
      cp_wait_all();
      __syncthreads();
    }
    // ---- T = Q_t^T G (rows m0..m0+15), interleaved with the scatter of the previous H
    double T[TM][TN][2];
    zero_acc(T);
    const bool scat = have_prev && !(A.debug & 1);
#pragma unroll
    for (int k0 = 0; k0 < NP; k0 += 4) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i++) a[i] = sQt[(k0 + q) * LD + m0 + i * 8 + r];
#pragma unroll
      for (int j = 0; j < TN; j++) b[j] = sG[(k0 + q) * LD + j * 8 + r];
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) dmma(T[i][j], a[i], b[j]);
      // tiles of the previous H spread over the NP/4 k-steps
      constexpr int TPK = (TM * TN + NP / 4 - 1) / (NP / 4);
#pragma unroll
      for (int u = 0; u < TPK; u++) {
        const int tile = (k0 / 4) * TPK + u;
        if (tile < TM * TN && scat) {
          const int i = tile / TN, j = tile % TN;
          scatter_pair2<BENCH>(A, prev, m0 + i * 8, j * 8, m0 + i * 8 + r, j * 8 + 2 * q, H[i][j][0], H[i][j][1]);
        }
      }
    }
    __syncthreads();  // every warp is done with G
    const bool more = p + 1 < ch.end && !(A.debug & 2);
    if (more) {
      pair_load_G<NP, GEN>(A, s_it[p + 1 - ch.begin], sG);
      cp_commit();
    }
    // ---- H = T Q_s; A fragment (row m0+8i+r, col k0+q) lives in lane (r, (k0%8+q)/2), element q%2
    zero_acc(H);
    const int src_lo = r * 4 + (q >> 1), src_hi = src_lo + 2;
#pragma unroll
    for (int k0 = 0; k0 < NP; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i++) {
        const double e0 = __shfl_sync(0xffffffffu, T[i][jt][0], srcl);
        const double e1 = __shfl_sync(0xffffffffu, T[i][jt][1], srcl);
        a[i] = (q & 1) ? e1 : e0;
      }
#pragma unroll
      for (int j = 0; j < TN; j++) b[j] = sQs[(k0 + q) * LD + j * 8 + r];
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) dmma(H[i][j], a[i], b[j]);
    }
    __syncthreads();  // every warp is done with Q_s
    prev.s_dst = it.s_dst;
    prev.s_dst_m = it.s_dst_m;
    prev.bb_dst = it.bb_dst;
    prev.yr_dst = it.yr_dst;
    prev.yc_dst = it.yc_dst;
    prev.s_ld = it.s_ld;
    prev.s_ld_m = it.s_ld_m;
    prev.yr_ld = it.yr_ld;
    prev.yc_ld = it.yc_ld;
    prev.nt = nt;
    prev.ns = it.ns;
    prev.kt = ktt;
    prev.ks = it.ks;
    prev.dsym = A.sym && s == t;
    have_prev = true;
    // bench mode: the S part reduced now (Q_s's buffer is the scratch), the
    // other parts scattered during the next pair's T-GEMM as usual
    if constexpr (BENCH) bench_pair<NP, TN, C::WARPS>(A, prev, t, s, H[0], m0, reinterpret_cast<double2 *>(sQs));
    if (more) {
      const PairItem &nx = s_it[p + 1 - ch.begin];
      async_tile<NP, NP, LD>(sQs, A.q_col + nx.q_off_s, nx.ns, nx.ns, nx.ns, A.chunks);
      cp_commit();
    }
  }
}

// --------------------------------------------------------------------------
// Level-0 congruence with Q in compact-WY form (H2SP_PLAN_EXPLICIT_Q unset):
// Q = I - V M, M = T V^T (V: the n x k Householder vectors of step (i)), so
//   H = Q_t^T G Q_s = T1 - (T1 V_s) M_s,   T1 = G - M_t^T (V_t^T G),
// four skinny products costing 4 n_t n_s (k_t + k_s) flops instead of the
// 2 n_t n_s (n_t + n_s) of the explicit product (1.78x fewer at n = 64, k = 16).
// Same result up to rounding; when every reflector has tau = 0 (M = 0) it is
// G itself, bit for bit.  Block layout as pair_kernel<64>: 8 warps, warp w owns
// rows 8w..8w+7 of T1 and H (registers), V_t / M_t resident per block row,
// G and V_s / M_s reloaded per pair, the previous H scattered during step 1.
// --------------------------------------------------------------------------
#ifndef WY_SPLIT
#define WY_SPLIT 2  // partial sums per tile in the skinny products of pair_wy_kernel
#endif
template <int KP>
struct PairWyCfg {
  static constexpr int NP = 64;
  static constexpr int LD = NP + 4;       // G, P, M (rows of 64)
  static constexpr int LDV = KP + 4;      // V (rows of KP): LDV = 4 (mod 8) -> conflict-free fragments
  static constexpr int WARPS = 8;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int V_D = NP * LDV, M_D = KP * LD, G_D = NP * LD, P_D = KP * LD;
  // V_s / M_s double-buffered (loaded a whole pair ahead) when two CTAs still fit an SM
  static constexpr bool DB = size_t(3 * V_D + 3 * M_D + G_D + P_D) * sizeof(double) + 2048 <= 113 * 1024;
  static constexpr size_t SMEM = size_t((DB ? 3 : 2) * (V_D + M_D) + G_D + P_D) * sizeof(double);
};

template <int KP>
__device__ __forceinline__ void wy_load(double *sV, double *sM, const double *wy, int64_t c) {
  using C = PairWyCfg<KP>;
  const double *g = wy + c * (2 * 64 * KP);
  async_tile<64, KP, C::LDV>(sV, g, 64, KP, KP, g);
  async_tile<KP, 64, C::LD>(sM, g + 64 * KP, KP, 64, 64, g);
}

template <int KP, bool GEN, bool BENCH>
__global__ void __launch_bounds__(PairWyCfg<KP>::THREADS, 2) pair_wy_kernel(PairArgs A, const double *wy_row,
                                                                              const double *wy_col) {
  using C = PairWyCfg<KP>;
  constexpr int LD = C::LD, LDV = C::LDV, TN = 8;
  extern __shared__ __align__(16) double sm[];
  double *sVt = sm, *sMt = sVt + C::V_D;
  double *sG = sMt + C::M_D, *sP = sG + C::G_D;
  double *sVM = sP + C::P_D;  // V_s / M_s stage(s), each V_D + M_D
  __shared__ __align__(16) PairItem s_it[PAIR_CHUNK_MAX];
  const Chunk ch = A.chunks[blockIdx.x];
  stage_items(A.items, ch, s_it);
  int t = s_it[0].t;
  int nt = s_it[0].nt, ktt = s_it[0].kt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int m0 = warp * 8;
  wy_load<KP>(sVt, sMt, wy_row, t);
  load_close<64, LD, GEN>(A, s_it[0], sG);
  wy_load<KP>(sVM, sVM + C::V_D, wy_col, s_it[0].s);
  cp_commit();
  double H[TN][2];
  PairDst prev;
  bool have_prev = false;
  const int src_lo = r * 4 + (q >> 1), src_hi = src_lo + 2;
  for (int p = ch.begin;; p++) {
    if (p == ch.end) {
      if (have_prev && !(A.debug & 1)) {
#pragma unroll
        for (int j = 0; j < TN; j++) scatter_pair2<BENCH>(A, prev, m0, j * 8, m0 + r, j * 8 + 2 * q, H[j][0], H[j][1]);
      }
      break;
    }
    const PairItem &it = s_it[p - ch.begin];
    const int s = it.s;
    const int stg = C::DB ? ((p - ch.begin) & 1) : 0;
    double *sVs = sVM + stg * (C::V_D + C::M_D), *sMs = sVs + C::V_D;
    cp_wait_all();
    __syncthreads();
    if (it.t != t) {
      t = it.t;
      nt = it.nt;
      ktt = it.kt;
      wy_load<KP>(sVt, sMt, wy_row, t);
      cp_commit();
      cp_wait_all();
      __syncthreads();
    }
    const bool more = p + 1 < ch.end && !(A.debug & 2);
    if (C::DB && more) {  // V_s / M_s of pair p+1 into the other stage (free since the barrier above)
      double *nV = sVM + (stg ^ 1) * (C::V_D + C::M_D);
      wy_load<KP>(nV, nV + C::V_D, wy_col, s_it[p + 1 - ch.begin].s);
      cp_commit();
    }
    const bool scat = have_prev && !(A.debug & 1);
    // ---- step 1: P = V_t^T G (KP x 64); warp w computes columns 8w..8w+7,
    //      interleaved with the scatter of the previous H (one tile per k-step)
    {
      // two partial sums per tile (even / odd k-steps): twice the independent
      // DMMA chains of this skinny product
      constexpr int NS = WY_SPLIT;  // partial sums per tile (k-steps round robin): independent DMMA chains
      double pacc[NS][KP / 8][2];
#pragma unroll
      for (int u = 0; u < NS; u++)
#pragma unroll
        for (int i = 0; i < KP / 8; i++) pacc[u][i][0] = pacc[u][i][1] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < 64; k0 += 4) {
        const double b = sG[(k0 + q) * LD + m0 + r];
#pragma unroll
        for (int i = 0; i < KP / 8; i++) dmma(pacc[(k0 >> 2) % NS][i], sVt[(k0 + q) * LDV + i * 8 + r], b);
        // one tile of the previous H every (64/4)/TN k-steps: the stores are spread
        // over the whole product instead of bunched at its start
        constexpr int EVERY = (64 / 4) / TN;
        if ((k0 / 4) % EVERY == 0 && scat) {
          const int j = (k0 / 4) / EVERY;
          scatter_pair2<BENCH>(A, prev, m0, j * 8, m0 + r, j * 8 + 2 * q, H[j][0], H[j][1]);
        }
      }
#pragma unroll
      for (int i = 0; i < KP / 8; i++) {
#pragma unroll
        for (int u = 1; u < NS; u++) {
          pacc[0][i][0] += pacc[u][i][0];
          pacc[0][i][1] += pacc[u][i][1];
        }
        sP[(i * 8 + r) * LD + m0 + 2 * q] = pacc[0][i][0];
        sP[(i * 8 + r) * LD + m0 + 2 * q + 1] = pacc[0][i][1];
      }
    }
    __syncthreads();
    // ---- step 2: T1 = G - M_t^T P (rows m0..m0+7 of T1 in H's registers)
#pragma unroll
    for (int j = 0; j < TN; j++) {
      H[j][0] = sG[(m0 + r) * LD + j * 8 + 2 * q];
      H[j][1] = sG[(m0 + r) * LD + j * 8 + 2 * q + 1];
    }
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const double a = -sMt[(k0 + q) * LD + m0 + r];
#pragma unroll
      for (int j = 0; j < TN; j++) dmma(H[j], a, sP[(k0 + q) * LD + j * 8 + r]);
    }
    __syncthreads();  // every warp is done with G and P
    // close_gen: G of pair p+1 is evaluated during step 3 (one row per k-step)
    const bool gnext = GEN && more;
    GenCol gc;
    if (more) {
      const PairItem &nx = s_it[p + 1 - ch.begin];
      if (gnext) {
        gc = gen_col(A.gen, nx.t, nx.s, nx.nt, nx.ns, A.B, threadIdx.x & 63);
      } else {
        async_tile<64, 64, LD>(sG, A.close + nx.g_src[0], nx.nt, nx.ns, A.B, A.chunks);
        cp_commit();
      }
    }
    // ---- step 3: R = T1 V_s (8 x KP per warp), A fragments from the T1 accumulators
    constexpr int NS3 = WY_SPLIT;
    double Rp[NS3][KP / 8][2];
#pragma unroll
    for (int u = 0; u < NS3; u++)
#pragma unroll
      for (int i = 0; i < KP / 8; i++) Rp[u][i][0] = Rp[u][i][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 64; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const double e0 = __shfl_sync(0xffffffffu, H[jt][0], srcl);
      const double e1 = __shfl_sync(0xffffffffu, H[jt][1], srcl);
      const double a = (q & 1) ? e1 : e0;
#pragma unroll
      for (int i = 0; i < KP / 8; i++) dmma(Rp[(k0 >> 2) % NS3][i], a, sVs[(k0 + q) * LDV + i * 8 + r]);
      if (gnext) {  // 256 threads x 16 k-steps = the 64 x 64 entries
        const int gi = (threadIdx.x >> 6) + 4 * (k0 >> 2);
        sG[gi * LD + gc.j] = gen_entry(A.gen, gc, gi);
      }
    }
    double R[KP / 8][2];
#pragma unroll
    for (int i = 0; i < KP / 8; i++) {
      R[i][0] = Rp[0][i][0];
      R[i][1] = Rp[0][i][1];
#pragma unroll
      for (int u = 1; u < NS3; u++) {
        R[i][0] += Rp[u][i][0];
        R[i][1] += Rp[u][i][1];
      }
    }
    // ---- step 4: H = T1 - R M_s
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const double e0 = __shfl_sync(0xffffffffu, R[jt][0], srcl);
      const double e1 = __shfl_sync(0xffffffffu, R[jt][1], srcl);
      const double a = -((q & 1) ? e1 : e0);
#pragma unroll
      for (int j = 0; j < TN; j++) dmma(H[j], a, sMs[(k0 + q) * LD + j * 8 + r]);
    }
    if constexpr (BENCH) {
      // the S part of H reduced now; this pair's V_s / M_s stage is the scratch
      // (with DB it is next written at the top of pair p + 1, after a barrier)
      PairDst cur;
      cur.s_dst = it.s_dst;
      cur.s_dst_m = it.s_dst_m;
      cur.s_ld = it.s_ld;
      cur.s_ld_m = it.s_ld_m;
      cur.nt = nt;
      cur.ns = it.ns;
      cur.kt = ktt;
      cur.ks = it.ks;
      cur.dsym = A.sym && s == t;
      __syncthreads();  // every warp is done with V_s / M_s
      bench_pair<64, TN, C::WARPS>(A, cur, t, s, H, m0, reinterpret_cast<double2 *>(sVs));
    }
    if (!C::DB) {
      __syncthreads();  // every warp is done with V_s / M_s
      if (more) {
        wy_load<KP>(sVs, sMs, wy_col, s_it[p + 1 - ch.begin].s);
        cp_commit();
      }
    }
    prev.s_dst = it.s_dst;
    prev.s_dst_m = it.s_dst_m;
    prev.bb_dst = it.bb_dst;
    prev.yr_dst = it.yr_dst;
    prev.yc_dst = it.yc_dst;
    prev.s_ld = it.s_ld;
    prev.s_ld_m = it.s_ld_m;
    prev.yr_ld = it.yr_ld;
    prev.yc_ld = it.yc_ld;
    prev.nt = nt;
    prev.ns = it.ns;
    prev.kt = ktt;
    prev.ks = it.ks;
    prev.dsym = A.sym && s == t;
    have_prev = true;
  }
}

// --------------------------------------------------------------------------
// Level-0 compact-WY congruence for 128-point leaves (config 5: B = 128, r = 32).
// Same four products as pair_wy_kernel; a 128 x 128 G plus one V / M pair fill
// 206 KB of shared memory, so one CTA (16 warps) per SM and the two sides' V / M
// share one buffer: V_t, M_t for steps 1-2 (P = V_t^T G lands in the V buffer),
// then V_s, M_s for steps 3-4 (their load is the one exposed latency per pair;
// the next G streams in behind steps 3-4).  Warp w owns rows 8w..8w+7.
// --------------------------------------------------------------------------
template <int KP>
struct PairWy128Cfg {
  static constexpr int NP = 128;
  static constexpr int LD = NP + 4;    // G, M, P rows
  static constexpr int LDV = KP + 4;   // V rows
  static constexpr int WARPS = 16;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int G_D = NP * LD, V_D = NP * LDV, M_D = KP * LD;
  static_assert(KP * LD <= NP * LDV, "P aliases the V buffer");
  static constexpr size_t SMEM = size_t(G_D + V_D + M_D) * sizeof(double);
};

template <int KP>
__device__ __forceinline__ void wy128_load(double *sV, double *sM, const double *wy, int64_t c) {
  using C = PairWy128Cfg<KP>;
  const double *g = wy + c * (2 * 128 * KP);
  async_tile<128, KP, C::LDV>(sV, g, 128, KP, KP, g);
  async_tile<KP, 128, C::LD>(sM, g + 128 * KP, KP, 128, 128, g);
}

template <int KP, bool GEN, bool BENCH>
__global__ void __launch_bounds__(PairWy128Cfg<KP>::THREADS, 1) pair_wy128_kernel(PairArgs A, const double *wy_row,
                                                                                   const double *wy_col) {
  using C = PairWy128Cfg<KP>;
  constexpr int LD = C::LD, LDV = C::LDV, TN = 16;
  extern __shared__ __align__(16) double sm[];
  double *sG = sm, *sV = sG + C::G_D, *sM = sV + C::V_D;
  double *sP = sV;  // KP x LD, after step 1
  __shared__ __align__(16) PairItem s_it[PAIR_CHUNK_MAX];
  // close_gen: points of the next pair's row cluster t (staged once per t) and the exp table
  __shared__ __align__(16) double s_xt[GEN ? 128 * 3 : 2];
  __shared__ double s_tab[GEN ? 64 : 1];
  __shared__ double s_wst[BENCH ? 256 : 1];   // bench mode: w of the pair's S columns (by tile column) | S rows' mirror (by tile row)
  if (GEN && threadIdx.x < 64) s_tab[threadIdx.x] = g_exp2_64[threadIdx.x];
  const Chunk ch = A.chunks[blockIdx.x];
  stage_items(A.items, ch, s_it);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int m0 = warp * 8;
  const int src_lo = r * 4 + (q >> 1), src_hi = src_lo + 2;
  int xt_staged = -1;   // cluster whose points are in s_xt
  if constexpr (GEN) {  // the first G with the same evaluation as the rest (bitwise independent of chunking)
    xt_staged = s_it[0].t;
    const double *src = A.gen.pts + int64_t(xt_staged) * A.B * A.gen.dim;
    for (int c = threadIdx.x; c < A.B * A.gen.dim; c += blockDim.x) cp8(s_xt + c, src + c, true);
    cp_commit();
    cp_wait_all();
    __syncthreads();
    const GenCol c0 = gen_col(A.gen, s_it[0].t, s_it[0].s, s_it[0].nt, s_it[0].ns, A.B, threadIdx.x & 127);
    for (int i = threadIdx.x >> 7; i < 128; i += blockDim.x >> 7) sG[i * LD + c0.j] = gen_entry_s(A.gen, c0, i, s_xt, s_tab);
  } else {
    load_close<128, LD, GEN>(A, s_it[0], sG);
  }
  wy128_load<KP>(sV, sM, wy_row, s_it[0].t);
  cp_commit();
  for (int p = ch.begin; p < ch.end; p++) {
    const PairItem &it = s_it[p - ch.begin];
    cp_wait_all();
    __syncthreads();
    // ---- step 1: P = V_t^T G (KP x 128); warp w: columns 8w..8w+7
    {
      double pacc[2][KP / 8][2];
#pragma unroll
      for (int i = 0; i < KP / 8; i++) pacc[0][i][0] = pacc[0][i][1] = pacc[1][i][0] = pacc[1][i][1] = 0.0;
#pragma unroll 8
      for (int k0 = 0; k0 < 128; k0 += 4) {
        const double b = sG[(k0 + q) * LD + m0 + r];
#pragma unroll
        for (int i = 0; i < KP / 8; i++) dmma(pacc[(k0 >> 2) & 1][i], sV[(k0 + q) * LDV + i * 8 + r], b);
      }
      __syncthreads();  // every warp is done with V_t: P overwrites it
#pragma unroll
      for (int i = 0; i < KP / 8; i++) {
        sP[(i * 8 + r) * LD + m0 + 2 * q] = pacc[0][i][0] + pacc[1][i][0];
        sP[(i * 8 + r) * LD + m0 + 2 * q + 1] = pacc[0][i][1] + pacc[1][i][1];
      }
    }
    __syncthreads();
    // ---- step 2: T1 = G - M_t^T P (rows m0..m0+7 in registers)
    double H[TN][2];
#pragma unroll
    for (int j = 0; j < TN; j++) {
      H[j][0] = sG[(m0 + r) * LD + j * 8 + 2 * q];
      H[j][1] = sG[(m0 + r) * LD + j * 8 + 2 * q + 1];
    }
#pragma unroll 2
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const double a = -sM[(k0 + q) * LD + m0 + r];
#pragma unroll
      for (int j = 0; j < TN; j++) dmma(H[j], a, sP[(k0 + q) * LD + j * 8 + r]);
    }
    __syncthreads();  // G, P, M_t are dead
    const bool more = p + 1 < ch.end && !(A.debug & 2);
    // close_gen: G of pair p+1 is evaluated during step 3 (one row per k-step)
    const bool gnext = GEN && more;
    wy128_load<KP>(sV, sM, wy_col, it.s);
    if constexpr (BENCH) {  // this pair's weights for the epilogue (land with V_s / M_s)
      if (threadIdx.x < 256) {
        const bool colside = threadIdx.x < 128;
        const int i = threadIdx.x & 127;
        const int lo = colside ? it.ks : it.kt, hi = colside ? it.ns : it.nt;
        const bool ok = i >= lo && i < hi;
        const double *src = A.bw + A.cs.s_off[colside ? it.s : it.t] + (i - lo);
        cp8(s_wst + threadIdx.x, ok ? (const void *)src : (const void *)A.chunks, ok);
      }
    }
    if (gnext && s_it[p + 1 - ch.begin].t != xt_staged) {  // points of the next row cluster
      xt_staged = s_it[p + 1 - ch.begin].t;
      const double *src = A.gen.pts + int64_t(xt_staged) * A.B * A.gen.dim;
      for (int c = threadIdx.x; c < A.B * A.gen.dim; c += blockDim.x) cp8(s_xt + c, src + c, true);
    }
    cp_commit();
    if (more && !gnext) {  // G of pair p+1 streams in behind steps 3-4
      const PairItem &nx = s_it[p + 1 - ch.begin];
      async_tile<128, 128, LD>(sG, A.close + nx.g_src[0], nx.nt, nx.ns, A.B, A.chunks);
      cp_commit();
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // V_s / M_s landed
    } else {
      cp_wait_all();
    }
    __syncthreads();
    // ---- step 3: R = T1 V_s (8 x KP per warp)
    double R[2][KP / 8][2];
#pragma unroll
    for (int i = 0; i < KP / 8; i++) R[0][i][0] = R[0][i][1] = R[1][i][0] = R[1][i][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 128; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const double e0 = __shfl_sync(0xffffffffu, H[jt][0], srcl);
      const double e1 = __shfl_sync(0xffffffffu, H[jt][1], srcl);
      const double a = (q & 1) ? e1 : e0;
#pragma unroll
      for (int i = 0; i < KP / 8; i++) dmma(R[(k0 >> 2) & 1][i], a, sV[(k0 + q) * LDV + i * 8 + r]);
    }
#pragma unroll
    for (int i = 0; i < KP / 8; i++) {
      R[0][i][0] += R[1][i][0];
      R[0][i][1] += R[1][i][1];
    }
    // ---- step 4: H = T1 - R M_s
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const double e0 = __shfl_sync(0xffffffffu, R[0][jt][0], srcl);
      const double e1 = __shfl_sync(0xffffffffu, R[0][jt][1], srcl);
      const double a = -((q & 1) ? e1 : e0);
#pragma unroll
      for (int j = 0; j < TN; j++) dmma(H[j], a, sM[(k0 + q) * LD + j * 8 + r]);
    }
    // G of pair p+1 (512 threads x 32 rows = the 128 x 128 entries) in a rolled loop
    // after step 4, where R is dead (after step 3, with R and H live, the kernel
    // spilled at 128 registers); the evaluations share the FP64 datapath with the
    // DMMA anyway, and inlining one per unrolled k-step made the kernel 188 KB of
    // code (i-cache misses)
    if (gnext) {
      const PairItem &nx = s_it[p + 1 - ch.begin];
      const GenCol gc = gen_col(A.gen, nx.t, nx.s, nx.nt, nx.ns, A.B, threadIdx.x & 127);
#pragma unroll 2
      for (int gi = threadIdx.x >> 7; gi < 128; gi += 4) sG[gi * LD + gc.j] = gen_entry_s(A.gen, gc, gi, s_xt, s_tab);
    }
    __syncthreads();  // every warp is done with V_s / M_s
    PairDst D;
    D.s_dst = it.s_dst;
    D.s_dst_m = it.s_dst_m;
    D.bb_dst = it.bb_dst;
    D.yr_dst = it.yr_dst;
    D.yc_dst = it.yc_dst;
    D.s_ld = it.s_ld;
    D.s_ld_m = it.s_ld_m;
    D.yr_ld = it.yr_ld;
    D.yc_ld = it.yc_ld;
    D.nt = it.nt;
    D.ns = it.ns;
    D.kt = it.kt;
    D.ks = it.ks;
    D.dsym = A.sym && it.s == it.t;
    // bench mode: the S part reduced with the (free) V / M buffer as scratch
    if constexpr (BENCH)
      bench_pair<128, TN, C::WARPS>(A, D, it.t, it.s, H, m0, reinterpret_cast<double2 *>(sV), nullptr, s_wst, s_wst + 128);
    if (more) {  // V_t / M_t of the next pair, in flight during the scatter
      wy128_load<KP>(sV, sM, wy_row, s_it[p + 1 - ch.begin].t);
      cp_commit();
    }
    if (!(A.debug & 1)) {
#pragma unroll
      for (int j = 0; j < TN; j++) scatter_pair2<BENCH>(A, D, m0, j * 8, m0 + r, j * 8 + 2 * q, H[j][0], H[j][1]);
    }
  }
}


// --------------------------------------------------------------------------
// Level-0 compact-WY congruence for 128-point leaves with matrix-free close
// blocks (close_gen; config 5).  G_ts = C_ts is never stored: its entries are
// evaluated where the products consume them -- as the B operand of
// P = V_t^T G (warp w: column 8w+r, rows k) and as the initial accumulator of
// T1 = G - M_t^T P (warp w: rows 8w..8w+7) -- 64 evaluations per thread per
// pair instead of 32, and no 135 KB G buffer.  That leaves room for V_t, M_t
// resident over the chunk (one block row t) and for V_s, M_s of pair p+1
// loading during the epilogue of pair p and steps 1-2 of pair p+1: no load is
// exposed in the pair loop (the FP64 datapath -- DMMA and the kernel
// evaluations -- is the bottleneck resource).
// --------------------------------------------------------------------------
template <int KP>
struct PairWy128gCfg {
  static constexpr int NP = 128;
  static constexpr int LD = NP + 4;    // M, P rows
  static constexpr int LDV = KP + 4;   // V rows
  static constexpr int WARPS = 16;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int V_D = NP * LDV, M_D = KP * LD, P_D = KP * LD, X_D = NP * 3;
  static constexpr size_t SMEM = size_t(2 * V_D + 3 * M_D + 2 * X_D) * sizeof(double);
  static_assert(P_D * 2 >= WARPS * NP * 2, "the bench column partials fit the P buffer");
};

// K(x, y) of h2sp_close_gen for row point x and column point y (the same
// arithmetic as gen_entry_s); `same`: the same point (diagonal of t == s)
__device__ __forceinline__ double gen_eval(const CloseGen &g, const double *x, const double *y, bool same,
                                           const double *tab) {
  const double d0 = __dsub_rn(x[0], y[0]);
  double r2 = __dmul_rn(d0, d0);
  if (g.dim > 1) {
    const double d1 = __dsub_rn(x[1], y[1]);
    r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
  }
  if (g.dim > 2) {
    const double d2 = __dsub_rn(x[2], y[2]);
    r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
  }
  const double ir = rsqrt(r2);
  if (g.kind == H2SP_KERNEL_LAPLACE) return same ? g.p1 : g.q0 * ir;
  const double r = r2 > 0.0 ? r2 * ir : 0.0;
  const double v = g.kind == H2SP_KERNEL_EXP ? exp_neg_tab(r * g.q0, tab) : 1.0 / (r + g.p0);
  return same ? v + g.p1 : v;
}

template <int KP, bool BENCH>
__global__ void __launch_bounds__(PairWy128gCfg<KP>::THREADS, 1) pair_wy128g_kernel(PairArgs A, const double *wy_row,
                                                                                     const double *wy_col) {
  using C = PairWy128gCfg<KP>;
  constexpr int LD = C::LD, LDV = C::LDV, TN = 16;
  extern __shared__ __align__(16) double sm[];
  double *sVt = sm, *sMt = sVt + C::V_D, *sP = sMt + C::M_D, *sVs = sP + C::P_D, *sMs = sVs + C::V_D;
  double *sXt = sMs + C::M_D, *sYs = sXt + C::X_D;   // points of t (rows), of s (columns): 128 x dim
  __shared__ __align__(16) PairItem s_it[PAIR_CHUNK_MAX];
  __shared__ double s_tab[64];
  __shared__ double2 s_rowp[BENCH ? 128 : 1];
  if (threadIdx.x < 64) s_tab[threadIdx.x] = g_exp2_64[threadIdx.x];
  const Chunk ch = A.chunks[blockIdx.x];
  stage_items(A.items, ch, s_it);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int m0 = warp * 8;
  const int src_lo = r * 4 + (q >> 1), src_hi = src_lo + 2;
  const int dim = A.gen.dim;
  auto load_pts = [&](double *dst, int c) {   // the B points of leaf c
    const double *src = A.gen.pts + int64_t(c) * A.B * dim;
    for (int e = threadIdx.x; e < A.B * dim; e += blockDim.x) cp8(dst + e, src + e, true);
  };
  int t = s_it[0].t;
  wy128_load<KP>(sVt, sMt, wy_row, t);
  load_pts(sXt, t);
  wy128_load<KP>(sVs, sMs, wy_col, s_it[0].s);
  load_pts(sYs, s_it[0].s);
  cp_commit();
  for (int p = ch.begin; p < ch.end; p++) {
    const PairItem &it = s_it[p - ch.begin];
    cp_wait_all();
    __syncthreads();
    if (it.t != t) {  // new block row (chunks are one row each; kept for generality)
      t = it.t;
      wy128_load<KP>(sVt, sMt, wy_row, t);
      load_pts(sXt, t);
      cp_commit();
      cp_wait_all();
      __syncthreads();
    }
    const int nt = it.nt, ns = it.ns;
    const bool tss = it.t == it.s;
    // ---- step 1: P = V_t^T G (KP x 128); warp w: columns 8w..8w+7, B operand
    //      G[k0 + q][8w + r] evaluated in place
    {
      const int c1 = m0 + r;
      double yc[3] = {0.0, 0.0, 0.0};
      for (int a = 0; a < dim; a++) yc[a] = sYs[c1 * dim + a];
      double pacc[2][KP / 8][2];
#pragma unroll
      for (int i = 0; i < KP / 8; i++) pacc[0][i][0] = pacc[0][i][1] = pacc[1][i][0] = pacc[1][i][1] = 0.0;
#pragma unroll 4
      for (int k0 = 0; k0 < 128; k0 += 4) {
        const int i = k0 + q;
        const double b = (i < nt && c1 < ns) ? gen_eval(A.gen, sXt + i * dim, yc, tss && i == c1, s_tab) : 0.0;
#pragma unroll
        for (int ii = 0; ii < KP / 8; ii++) dmma(pacc[(k0 >> 2) & 1][ii], sVt[(k0 + q) * LDV + ii * 8 + r], b);
      }
#pragma unroll
      for (int ii = 0; ii < KP / 8; ii++) {
        sP[(ii * 8 + r) * LD + m0 + 2 * q] = pacc[0][ii][0] + pacc[1][ii][0];
        sP[(ii * 8 + r) * LD + m0 + 2 * q + 1] = pacc[0][ii][1] + pacc[1][ii][1];
      }
    }
    __syncthreads();
    // ---- step 2: T1 = G - M_t^T P (rows m0..m0+7 in registers), G evaluated as the accumulator
    double H[TN][2];
    {
      const int row = m0 + r;
      double xr[3] = {0.0, 0.0, 0.0};
      for (int a = 0; a < dim; a++) xr[a] = sXt[row * dim + a];
#pragma unroll
      for (int j = 0; j < TN; j++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = j * 8 + 2 * q + e;
          H[j][e] = (row < nt && c < ns) ? gen_eval(A.gen, xr, sYs + c * dim, tss && row == c, s_tab) : 0.0;
        }
    }
#pragma unroll 2
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const double a = -sMt[(k0 + q) * LD + m0 + r];
#pragma unroll
      for (int j = 0; j < TN; j++) dmma(H[j], a, sP[(k0 + q) * LD + j * 8 + r]);
    }
    // ---- step 3: R = T1 V_s (8 x KP per warp), A fragments from the T1 accumulators
    double R[2][KP / 8][2];
#pragma unroll
    for (int i = 0; i < KP / 8; i++) R[0][i][0] = R[0][i][1] = R[1][i][0] = R[1][i][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 128; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const double e0 = __shfl_sync(0xffffffffu, H[jt][0], srcl);
      const double e1 = __shfl_sync(0xffffffffu, H[jt][1], srcl);
      const double a = (q & 1) ? e1 : e0;
#pragma unroll
      for (int i = 0; i < KP / 8; i++) dmma(R[(k0 >> 2) & 1][i], a, sVs[(k0 + q) * LDV + i * 8 + r]);
    }
#pragma unroll
    for (int i = 0; i < KP / 8; i++) {
      R[0][i][0] += R[1][i][0];
      R[0][i][1] += R[1][i][1];
    }
    // ---- step 4: H = T1 - R M_s
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const double e0 = __shfl_sync(0xffffffffu, R[0][jt][0], srcl);
      const double e1 = __shfl_sync(0xffffffffu, R[0][jt][1], srcl);
      const double a = -((q & 1) ? e1 : e0);
#pragma unroll
      for (int j = 0; j < TN; j++) dmma(H[j], a, sMs[(k0 + q) * LD + j * 8 + r]);
    }
    __syncthreads();  // every warp is done with V_s, M_s, the points of s and P
    if (p + 1 < ch.end) {  // V_s, M_s, points of the next pair: in flight until its step 3
      const PairItem &nx = s_it[p + 1 - ch.begin];
      wy128_load<KP>(sVs, sMs, wy_col, nx.s);
      load_pts(sYs, nx.s);
      cp_commit();
    }
    PairDst D;
    D.s_dst = it.s_dst;
    D.s_dst_m = it.s_dst_m;
    D.bb_dst = it.bb_dst;
    D.yr_dst = it.yr_dst;
    D.yc_dst = it.yc_dst;
    D.s_ld = it.s_ld;
    D.s_ld_m = it.s_ld_m;
    D.yr_ld = it.yr_ld;
    D.yc_ld = it.yc_ld;
    D.nt = nt;
    D.ns = ns;
    D.kt = it.kt;
    D.ks = it.ks;
    D.dsym = A.sym && tss;
    // bench mode: the S part reduced with the (free) P buffer as scratch
    if constexpr (BENCH)
      bench_pair<128, TN, C::WARPS>(A, D, it.t, it.s, H, m0, reinterpret_cast<double2 *>(sP), s_rowp);
#pragma unroll
    for (int j = 0; j < TN; j++) scatter_pair2<BENCH>(A, D, m0, j * 8, m0 + r, j * 8 + 2 * q, H[j][0], H[j][1]);
  }
}

// --------------------------------------------------------------------------
// Strips (Eq. u1v1): one CTA per column tile (TN columns) of one
// rotating cluster's panel.  Z = [Y_c1; Y_c2] is gathered from the children's
// panels (union of their frozen groups), W = Q_q^T Z on the DMMA pipe, then
// rows [k_q, n_q) -> S (contiguous row segments, and/or the transposed blocks),
// rows [0, k_q) -> q's panel for the next level.
// --------------------------------------------------------------------------
template <int NP, int TN>
struct StripCfg {
  static constexpr int LDQ = NP + 4;
  static constexpr int LDZ = TN + 4;
  static constexpr int WN = 32;                    // warp tile 16 x 32
  static constexpr int NWM = NP / 16, NWN = TN / WN;
  static constexpr int WARPS = NWM * NWN;
  static constexpr int THREADS = WARPS * 32;
#ifndef STRIP_MINB
#define STRIP_MINB 5
#endif
  // NP == 32: 5 CTAs per SM (46 KB of shared memory -- the tile's groups,
  // staged before the gather, alias the Z buffer -- and <= 48 registers).
  // Other widths keep the separate group array and no minimum-blocks hint
  // (__launch_bounds__(512, 1) let NP = 48 / 64 grow to 76 registers = one CTA
  // per SM: 1.35x slower strips on the config-5 recipe).
  static constexpr bool SMALL = NP == 32 && TN == 128;
  // NP == 48: aliasing the group array alone (no hint, 54 registers) fits 3 CTAs
  // per SM instead of 2 (74 KB of shared memory each)
  static constexpr bool ALIAS = SMALL || (NP == 48 && TN == 128);
  // (NP == 48: the minimum-blocks hint 3 pins the register budget at <= 56 so the
  // 3 CTAs per SM cannot silently drop to 2 after a code change)
  static constexpr int MIN_BLOCKS = SMALL ? STRIP_MINB : (NP == 48 && TN == 128) ? 3 : 0;
  static constexpr size_t SMEM = (size_t(NP) * LDQ + size_t(NP) * LDZ) * sizeof(double) + TN * 16 + (ALIAS ? 0 : 64);
  static_assert(size_t(NP) * LDZ * sizeof(double) >= (TN + 1) * sizeof(StripGroup), "groups alias sZ");
};

struct StripArgs {
  const StripTileX *tiles;
  const StripGroup *groups;
  int L, level;
  const double *q;
  const double *y_in;
  double *y_out;
  double *s_val;
  const double *bw;   // bench mode: w (S column order)
  double2 *part;      // bench mode: partial slots
  int aligned;        // bench mode: every frozen group width is a multiple of 32 (plan-wide)
};

// BENCH (bench mode, include/h2sp.h): rows [k_q, n_q) of W are reduced instead
// of stored -- per (row, frozen group) of the direct block {sum W w, sum W^2}
// and per column of the transposed blocks, the weights w staged per tile.
// Aligned plans (every group 32k wide, so each warp's 32 columns lie in one
// group): straight from the accumulators -- a row's 8 values per lane, the
// lane quad (shuffles), then the group's warp slabs in order; a column's rows
// over the 8 lane rows (shuffles), then the row warps in order.  Otherwise W is
// staged in the Z buffer: 8 lanes per (row, group), TPC lanes per column.
// Fixed orders either way (the choice is plan-wide, so shards agree).  Tiles
// hold whole groups (plan.cpp).
#ifdef H2SP_STRIP_CLOCKS
// Attribution build only (tools/strip_clocks.py): thread 0 of a sample of CTAs stamps clock64() at the
// phase boundaries of strip_kernel into a global table read back by h2sp_debug_strip_clocks.
struct StripClk {
  unsigned grid, smid;
  unsigned long long gt0;
  long long c[10];
};
__device__ StripClk g_strip_clk[16384];
__device__ unsigned g_strip_clk_n;
#define STRIP_CLK(i)                                        \
  do {                                                      \
    if (clk_slot >= 0 && threadIdx.x == 0) g_strip_clk[clk_slot].c[i] = clock64(); \
  } while (0)
#else
#define STRIP_CLK(i) do { } while (0)
#endif
template <int NP, int TN, bool BENCH>
__global__ void __launch_bounds__(StripCfg<NP, TN>::THREADS, StripCfg<NP, TN>::MIN_BLOCKS) strip_kernel(StripArgs A) {
  using C = StripCfg<NP, TN>;
  extern __shared__ __align__(16) double sm[];
  double *sQ = sm;                           // NP x LDQ
  double *sZ = sm + NP * C::LDQ;             // NP x LDZ
  int64_t *tdst = reinterpret_cast<int64_t *>(sZ + NP * C::LDZ);  // per column: transposed S dst (b*ld folded in)
  int32_t *src1 = reinterpret_cast<int32_t *>(tdst + TN);          // per column: column in child-1 panel or -1
  int32_t *src2 = src1 + TN;
  double *s_wc = reinterpret_cast<double *>(src2 + TN);   // bench: w of every tile column (TN)
  double *s_wq = s_wc + TN;                               // bench: w of q's frozen rows (NP)
  __shared__ StripGroup sg_own[C::ALIAS ? 1 : TN + 1];
  __shared__ int4 s_gtab[BENCH ? TN + 1 : 1];   // bench: the tile's groups {first column, width, w index}
  __shared__ int s_ngt;
  // groups overlapping this tile (<= TN + 1); when aliased, dead before the gather
  StripGroup *sg = C::ALIAS ? reinterpret_cast<StripGroup *>(sZ) : sg_own;
  __shared__ __align__(16) StripTileX s_tile;
#ifdef H2SP_STRIP_CLOCKS
  int clk_slot = -1;
  if (threadIdx.x == 0 && (blockIdx.x & 63) == 0) {
    const unsigned sl = atomicAdd(&g_strip_clk_n, 1u);
    if (sl < 16384u) {
      clk_slot = int(sl);
      unsigned smid;
      unsigned long long gt;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      g_strip_clk[sl].grid = gridDim.x;
      g_strip_clk[sl].smid = smid;
      g_strip_clk[sl].gt0 = gt;
    }
  }
#endif
  STRIP_CLK(0);
  // round trip 1: the self-contained tile descriptor
  if (threadIdx.x < sizeof(StripTileX) / 16)
    cp16(reinterpret_cast<char *>(&s_tile) + 16 * threadIdx.x,
         reinterpret_cast<const char *>(A.tiles + blockIdx.x) + 16 * threadIdx.x);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  STRIP_CLK(1);
  const StripTileX &T = s_tile;
  const int n = T.n, kq = T.kq, k1 = T.k1, k2 = T.k2;
  const int ncol = T.ncol;
  // round trip 2: Q_q and the (at most TN + 1) groups overlapping the tile
  async_tile<NP, NP, C::LDQ>(sQ, A.q + T.q_off, n, n, n, A.tiles);
  const int ng = min(T.gend - T.g0, TN + 1);
  for (int g = threadIdx.x; g < ng * 2; g += blockDim.x)
    cp16(reinterpret_cast<char *>(&sg[g >> 1]) + 16 * (g & 1),
         reinterpret_cast<const char *>(&A.groups[T.g0 + (g >> 1)]) + 16 * (g & 1));
  cp_commit();
  cp_wait_all();
  __syncthreads();
  STRIP_CLK(2);
  // per-column source / destination maps
  for (int cc = threadIdx.x; cc < TN; cc += blockDim.x) {
    int32_t a1 = -1, a2 = -1;
    int64_t td = -1;
    if (cc < ncol) {
      const int c = T.c0 + cc;
      int g = 0;
      while (g + 1 < ng && sg[g + 1].col0 <= c) g++;
      const StripGroup gr = sg[g];
      const int b = c - gr.col0;
      if (gr.pos_c1 >= 0) a1 = gr.pos_c1 + b;
      if (gr.pos_c2 >= 0) a2 = gr.pos_c2 + b;
      if (gr.s_dst_t >= 0) td = gr.s_dst_t + int64_t(b) * gr.s_ld_t;
      // (bench weights: asynchronous copies that land with the gather -- a plain load here put a
      // global round trip into this phase: 2.3 of the tile's 20.9 kcycles, tools/strip_clocks.py)
      if (BENCH) cp8(&s_wc[cc], T.s_dst >= 0 ? (const void *)(A.bw + gr.wc0 + b) : (const void *)A.tiles, T.s_dst >= 0);
    } else if (BENCH) {
      s_wc[cc] = 0.0;
    }
    src1[cc] = a1;
    src2[cc] = a2;
    tdst[cc] = td;
  }
  if constexpr (BENCH) {  // the tile's whole groups (tile starts at group g0's first column)
    for (int a = threadIdx.x; a < NP; a += blockDim.x)
      cp8(&s_wq[a], a < n - kq ? (const void *)(A.bw + T.wq0 + a) : (const void *)A.tiles, a < n - kq);
    for (int g = threadIdx.x; g < ng; g += blockDim.x)
      if (sg[g].col0 < T.c0 + ncol) s_gtab[g] = make_int4(sg[g].col0 - T.c0, sg[g].m, sg[g].wc0, 0);
    if (threadIdx.x == 0) {
      int c = 0;
      while (c < ng && sg[c].col0 < T.c0 + ncol) c++;
      s_ngt = c;
    }
  }
  __syncthreads();
  STRIP_CLK(3);
  // gather Z: each thread keeps one column pair (cc, cc + 1) and walks its rows
  // (blockDim.x is a multiple of TN / 2); a pair contiguous and 16-byte aligned
  // in a child's panel (the common case: even group widths) is one 16-byte copy.
  // Rows of an absent child and rows [n, n4) are zero-filled.
  const int n4 = rup(n, 4);
  {
    const int cc = 2 * (threadIdx.x % (TN / 2)), R = blockDim.x / (TN / 2);
    const double *b1 = src1[cc] >= 0 ? A.y_in + T.src_c1 + src1[cc] : nullptr;
    const double *b2 = src2[cc] >= 0 ? A.y_in + T.src_c2 + src2[cc] : nullptr;
    const double *b1n = src1[cc + 1] >= 0 ? A.y_in + T.src_c1 + src1[cc + 1] : nullptr;
    const double *b2n = src2[cc + 1] >= 0 ? A.y_in + T.src_c2 + src2[cc + 1] : nullptr;
    // 16-byte copies need: second column right after the first in the same child
    // panel, and every row start 16-byte aligned (even ld, even first offset)
    const bool v1 = b1 && b1n == b1 + 1 && ((reinterpret_cast<uintptr_t>(b1) | (uintptr_t(T.ld_c1) * 8)) & 15) == 0;
    const bool v2 = b2 && b2n == b2 + 1 && ((reinterpret_cast<uintptr_t>(b2) | (uintptr_t(T.ld_c2) * 8)) & 15) == 0;
    const void *any = A.tiles;
    // aligned bench plans: the product skips the k range of an absent child for this column's
    // 32-wide slab (below), so those rows of Z need not even be zero-filled
    const bool skip = BENCH && A.aligned && (k1 & 3) == 0;
    for (int i = threadIdx.x / (TN / 2); i < n4; i += R) {
      const bool first = i < k1, second = !first && i < k1 + k2;
      if (skip && ((first && !b1) || (second && !b2))) continue;
      const int64_t off = int64_t(first ? i : i - k1) * (first ? T.ld_c1 : T.ld_c2);
      const double *p0 = first ? b1 : (second ? b2 : nullptr);
      const double *p1 = first ? b1n : (second ? b2n : nullptr);
      double *d = &sZ[i * C::LDZ + cc];
      if ((first && v1) || (second && v2)) {
        cp16(d, p0 + off);
      } else if (!p0 && !p1) {
        cp16_zero(d, any);
      } else {
        cp8(d, p0 ? (const void *)(p0 + off) : any, p0 != nullptr);
        cp8(d + 1, p1 ? (const void *)(p1 + off) : any, p1 != nullptr);
      }
    }
  }
  cp_commit();
  cp_wait_all();
  __syncthreads();
  STRIP_CLK(4);
  const int warp = threadIdx.x >> 5;
  const int m0 = (warp / C::NWN) * 16, n0 = (warp % C::NWN) * C::WN;
  if (!BENCH && m0 >= n) return;  // no rows of W for this warp (nothing after this needs the CTA barrier)
  double acc[2][C::WN / 8][2];
  zero_acc(acc);
  // aligned bench plans: a warp's 32 columns are one frozen group, present in one
  // or both children -- the k range of an absent child's rows (zero in Z) is
  // skipped (the algorithmic count 2 n_p (sum of present k_c) m, bitwise equal)
  int kb = 0, ke = n4;
  if (BENCH && A.aligned && (k1 & 3) == 0) {
    const bool p1 = src1[n0] >= 0, p2 = src2[n0] >= 0;
    if (!p1 && !p2) ke = 0;
    else if (p1 && !p2) ke = k1;
    else if (!p1 && p2) kb = k1;
  }
  if (m0 < n) warp_gemm<C::LDQ, C::LDZ, 2, C::WN / 8, true>(sQ, sZ, m0, n0, ke, acc, kb);
  STRIP_CLK(5);
  // epilogue straight from the accumulators: lane (r, q) holds W[row][col], W[row][col + 1]
  // rows [0, k_q) -> q's panel; rows [k_q, n_q) -> S row segment and the transposed block
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q4 = lane & 3;
  if (BENCH && A.aligned) {
    // rows [0, k_q) -> q's panel first: the stores leave while the slower warps finish their product
    if (m0 < kq && T.y_dst >= 0) {
#pragma unroll
      for (int i = 0; i < 2; i++) {
        const int row = m0 + i * 8 + r;
        if (row >= kq) continue;
#pragma unroll
        for (int j = 0; j < C::WN / 8; j++) {
          const int col = n0 + j * 8 + 2 * q4;
          if (col >= ncol) continue;
          double *d = A.y_out + T.y_dst + int64_t(row) * T.y_ld + T.c0 + col;
          if (col + 1 < ncol)
            store2(d, acc[i][j][0], acc[i][j][1]);
          else
            d[0] = acc[i][j][0];
        }
      }
    }
    STRIP_CLK(6);
    __syncthreads();  // every warp is done reading Z: its space holds the slab partials
    STRIP_CLK(7);
    double2 *dslab = reinterpret_cast<double2 *>(sZ);   // [NWN][NP]: (row, warp column slab)
    double2 *tslab = dslab + C::NWN * NP;               // [NWM][TN]: (column, warp row slab)
    const int wn = warp % C::NWN, wm = warp / C::NWN;
    if (m0 < n) {
#pragma unroll
      for (int i = 0; i < 2; i++) {  // direct: a row's values of this warp's 32 columns
        const int row = m0 + i * 8 + r;
        double y = 0.0, y2 = 0.0;
#pragma unroll
        for (int j = 0; j < C::WN / 8; j++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const double v = acc[i][j][e];
            y = fma(v, s_wc[n0 + j * 8 + 2 * q4 + e], y);
            y2 = fma(v, v, y2);
          }
        y += __shfl_xor_sync(0xffffffffu, y, 1);
        y2 += __shfl_xor_sync(0xffffffffu, y2, 1);
        y += __shfl_xor_sync(0xffffffffu, y, 2);
        y2 += __shfl_xor_sync(0xffffffffu, y2, 2);
        if (q4 == 0) dslab[wn * NP + row] = make_double2(y, y2);
      }
      {  // transposed: a column's values of this warp's 16 rows; lane (r, q4) ends with column r of its 8
        static_assert(C::WN == 32, "8 columns per lane");
        double2 cres;
        {
          double cy[8];
#pragma unroll
          for (int j = 0; j < C::WN / 8; j++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
              double y = 0.0;
#pragma unroll
              for (int i = 0; i < 2; i++) {
                const int row = m0 + i * 8 + r;
                y = fma(row >= kq ? acc[i][j][e] : 0.0, s_wq[row >= kq ? row - kq : 0], y);
              }
              cy[j * 2 + e] = y;
            }
          lane_rows_reduce(cy, lane);
          cres.x = cy[0];
        }
        {
          double cr[8];
#pragma unroll
          for (int j = 0; j < C::WN / 8; j++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
              double y2 = 0.0;
#pragma unroll
              for (int i = 0; i < 2; i++) {
                const double v = m0 + i * 8 + r >= kq ? acc[i][j][e] : 0.0;
                y2 = fma(v, v, y2);
              }
              cr[j * 2 + e] = y2;
            }
          lane_rows_reduce(cr, lane);
          cres.y = cr[0];
        }
        tslab[wm * TN + n0 + (r >> 1) * 8 + 2 * q4 + (r & 1)] = cres;
      }
    }
    __syncthreads();
    STRIP_CLK(8);
    const int nfz = n - kq;
    const int nwm = (n + 15) / 16;   // row warps that computed
    if (T.s_dst >= 0) {              // (row a, group g): the group's column slabs in order
      const int ngt = s_ngt;
      for (int it = threadIdx.x; it < nfz * ngt; it += blockDim.x) {
        const int a = it / ngt, g = it - a * ngt;
        const int4 gt = s_gtab[g];
        double2 v = make_double2(0.0, 0.0);
        for (int sl = gt.x / C::WN; sl < (gt.x + gt.y) / C::WN; sl++) {
          v.x += dslab[sl * NP + kq + a].x;
          v.y += dslab[sl * NP + kq + a].y;
        }
        A.part[T.s_dst + g + int64_t(a) * T.s_ld] = v;
      }
    }
    for (int cc = threadIdx.x; cc < ncol; cc += blockDim.x) {   // transposed: row slabs in order
      const int64_t td = tdst[cc];
      if (td < 0) continue;
      double2 v = make_double2(0.0, 0.0);
      for (int sl = kq / 16; sl < nwm; sl++) {
        v.x += tslab[sl * TN + cc].x;
        v.y += tslab[sl * TN + cc].y;
      }
      A.part[td] = v;
    }
    STRIP_CLK(9);
    return;   // (the panel rows were stored before the slab reduction)
  } else if constexpr (BENCH) {
    __syncthreads();  // every warp is done reading Z: stage W there
    if (m0 < n) {
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < C::WN / 8; j++) {
          const int row = m0 + i * 8 + r, col = n0 + j * 8 + 2 * q4;
          sZ[row * C::LDZ + col] = acc[i][j][0];
          sZ[row * C::LDZ + col + 1] = acc[i][j][1];
        }
    }
    __syncthreads();
    const int nfz = n - kq;  // frozen rows of W
    if (T.s_dst >= 0) {      // direct block(s): item (row a, group g) on 8 lanes
      const int ngt = s_ngt;
      const int items = nfz * ngt;
      const int sub = threadIdx.x & 7;
      for (int it0 = threadIdx.x >> 3; it0 < rup(items, int(blockDim.x) >> 3); it0 += blockDim.x >> 3) {
        double y = 0.0, r2 = 0.0;
        int a = 0, g = 0;
        if (it0 < items) {
          a = it0 / ngt;
          g = it0 - a * ngt;
          const int4 gt = s_gtab[g];
          const double *wr = sZ + (kq + a) * C::LDZ + gt.x;
          const double *ww = s_wc + gt.x;
          for (int c = sub; c < gt.y; c += 8) {
            const double v = wr[c];
            y = fma(v, ww[c], y);
            r2 = fma(v, v, r2);
          }
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          y += __shfl_xor_sync(0xffffffffu, y, o);
          r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        }
        if (sub == 0 && it0 < items) A.part[T.s_dst + g + int64_t(a) * T.s_ld] = make_double2(y, r2);
      }
    }
    {  // transposed blocks: column cc on TPC lanes
      constexpr int TPC = C::THREADS / TN >= 4 ? 4 : C::THREADS / TN >= 2 ? 2 : 1;  // power of two
      static_assert(C::THREADS >= TN, "one lane per column at least");
      const int cc = threadIdx.x / TPC, sub = threadIdx.x % TPC;
      const int64_t td = cc < ncol ? tdst[cc] : -1;
      double y = 0.0, r2 = 0.0;
      if (td >= 0) {
        for (int a = sub; a < nfz; a += TPC) {
          const double v = sZ[(kq + a) * C::LDZ + cc];
          y = fma(v, s_wq[a], y);
          r2 = fma(v, v, r2);
        }
      }
#pragma unroll
      for (int o = 1; o < TPC; o <<= 1) {
        y += __shfl_xor_sync(0xffffffffu, y, o);
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
      }
      if (sub == 0 && td >= 0) A.part[td] = make_double2(y, r2);
    }
    if (m0 >= n) return;
  }
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const int row = m0 + i * 8 + r;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < C::WN / 8; j++) {
      const int col = n0 + j * 8 + 2 * q4;
      if (col >= ncol) continue;
      const bool two = col + 1 < ncol;
      const double v0 = acc[i][j][0], v1 = acc[i][j][1];
      double *d = nullptr;
      if (row < kq) {
        if (T.y_dst >= 0) d = A.y_out + T.y_dst + int64_t(row) * T.y_ld + T.c0 + col;
      } else if (!BENCH) {
        const int a = row - kq;
        if (T.s_dst >= 0) {
          double *ds = A.s_val + T.s_dst + int64_t(a) * T.s_ld + T.c0 + col;
          if (two)
            store2_s(ds, v0, v1);
          else
            st_s(ds, v0);
        }
        const int64_t t0 = tdst[col];
        if (t0 >= 0) st_s(A.s_val + t0 + a, v0);
        if (two) {
          const int64_t t1 = tdst[col + 1];
          if (t1 >= 0) st_s(A.s_val + t1 + a, v1);
        }
      }
      if (d) {
        if (two)
          store2(d, v0, v1);
        else
          d[0] = v0;
      }
    }
  }
}

// --------------------------------------------------------------------------
// Strips, bench mode on aligned plans (config 5): a persistent, software-
// pipelined version of strip_kernel.  One CTA per SM walks a contiguous range
// of tiles (consecutive tiles share a panel, so Q_q stays loaded); while the
// DMMA of tile i runs, Z of tile i+1 is in flight (double-buffered), the groups
// of tile i+2 and the descriptor of tile i+3 too (4 metadata stages).  Per
// tile the same arithmetic as strip_kernel's aligned path (same GEMM order,
// same slab reductions), so results are bitwise equal to it.  The one-tile-
// per-CTA kernel spends most of its time in dependent round trips (descriptor
// -> Q / groups -> Z) that only 2 co-resident CTAs can overlap.
// --------------------------------------------------------------------------
template <int NP, int TN>
struct PipeMeta {
  StripTileX tile;
  StripGroup grp[TN + 1];
};
template <int NP, int TN>
struct PipeMaps {
  int64_t tdst[TN];
  int32_t src1[TN], src2[TN];
  double wc[TN];
  double wq[NP];
  int4 gtab[TN + 1];
  int ngt, pad_[3];
};
template <int NP, int TN>
struct StripPipeCfg {
  using C = StripCfg<NP, TN>;
  static constexpr size_t Q_B = size_t(NP) * C::LDQ * sizeof(double);
  static constexpr size_t Z_B = size_t(NP) * C::LDZ * sizeof(double);
  static constexpr size_t SMEM = Q_B + 2 * Z_B + 4 * sizeof(PipeMeta<NP, TN>) + 2 * sizeof(PipeMaps<NP, TN>);
};

template <int NP, int TN>
__global__ void __launch_bounds__(StripCfg<NP, TN>::THREADS, 1) strip_pipe_kernel(StripArgs A, int64_t ntiles) {
  using C = StripCfg<NP, TN>;
  using PC = StripPipeCfg<NP, TN>;
  extern __shared__ __align__(16) double sm[];
  unsigned char *base = reinterpret_cast<unsigned char *>(sm);
  double *sQ = sm;
  double *sZ0 = reinterpret_cast<double *>(base + PC::Q_B);
  PipeMeta<NP, TN> *meta = reinterpret_cast<PipeMeta<NP, TN> *>(base + PC::Q_B + 2 * PC::Z_B);
  PipeMaps<NP, TN> *maps = reinterpret_cast<PipeMaps<NP, TN> *>(meta + 4);
  const int64_t tb = ntiles * blockIdx.x / gridDim.x, te = ntiles * (blockIdx.x + 1) / gridDim.x;
  if (tb >= te) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q4 = lane & 3;
  const int m0 = (warp / C::NWN) * 16, n0 = (warp % C::NWN) * C::WN;
  auto zbuf = [&](int64_t i) { return sZ0 + ((i - tb) & 1) * (size_t(NP) * C::LDZ); };
  auto load_desc = [&](int64_t i) {
    if (i < te && threadIdx.x < int(sizeof(StripTileX) / 16))
      cp16(reinterpret_cast<char *>(&meta[(i - tb) & 3].tile) + 16 * threadIdx.x,
           reinterpret_cast<const char *>(A.tiles + i) + 16 * threadIdx.x);
  };
  auto load_groups = [&](int64_t i) {   // needs the descriptor of tile i in shared memory
    if (i >= te) return;
    PipeMeta<NP, TN> &M = meta[(i - tb) & 3];
    const int ng = min(M.tile.gend - M.tile.g0, TN + 1);
    for (int g = threadIdx.x; g < ng * 2; g += blockDim.x)
      cp16(reinterpret_cast<char *>(&M.grp[g >> 1]) + 16 * (g & 1),
           reinterpret_cast<const char *>(&A.groups[M.tile.g0 + (g >> 1)]) + 16 * (g & 1));
  };
  // per-column maps, weights and the group table of tile i (its descriptor and groups landed)
  auto make_maps = [&](int64_t i) {
    const PipeMeta<NP, TN> &M = meta[(i - tb) & 3];
    PipeMaps<NP, TN> &X = maps[(i - tb) & 1];
    const StripTileX &T = M.tile;
    const int ng = min(T.gend - T.g0, TN + 1);
    for (int cc = threadIdx.x; cc < TN; cc += blockDim.x) {
      int32_t a1 = -1, a2 = -1;
      int64_t td = -1;
      double wc = 0.0;
      if (cc < T.ncol) {
        const int c = T.c0 + cc;
        int g = 0;
        while (g + 1 < ng && M.grp[g + 1].col0 <= c) g++;
        const StripGroup gr = M.grp[g];
        const int b = c - gr.col0;
        if (gr.pos_c1 >= 0) a1 = gr.pos_c1 + b;
        if (gr.pos_c2 >= 0) a2 = gr.pos_c2 + b;
        if (gr.s_dst_t >= 0) td = gr.s_dst_t + int64_t(b) * gr.s_ld_t;
        if (T.s_dst >= 0) wc = __ldg(A.bw + gr.wc0 + b);
      }
      X.src1[cc] = a1;
      X.src2[cc] = a2;
      X.tdst[cc] = td;
      X.wc[cc] = wc;
    }
    for (int a = threadIdx.x; a < NP; a += blockDim.x) X.wq[a] = a < T.n - T.kq ? __ldg(A.bw + T.wq0 + a) : 0.0;
    for (int g = threadIdx.x; g < ng; g += blockDim.x)
      if (M.grp[g].col0 < T.c0 + T.ncol) X.gtab[g] = make_int4(M.grp[g].col0 - T.c0, M.grp[g].m, M.grp[g].wc0, 0);
    if (threadIdx.x == 0) {
      int c = 0;
      while (c < ng && M.grp[c].col0 < T.c0 + T.ncol) c++;
      X.ngt = c;
    }
  };
  // asynchronous gather of Z of tile i (maps of tile i complete, CTA barrier passed)
  auto gather = [&](int64_t i) {
    const StripTileX &T = meta[(i - tb) & 3].tile;
    const PipeMaps<NP, TN> &X = maps[(i - tb) & 1];
    double *sZ = zbuf(i);
    const int n4 = rup(int(T.n), 4), k1 = T.k1, k2 = T.k2;
    const int cc = 2 * (threadIdx.x % (TN / 2)), R = blockDim.x / (TN / 2);
    const double *b1 = X.src1[cc] >= 0 ? A.y_in + T.src_c1 + X.src1[cc] : nullptr;
    const double *b2 = X.src2[cc] >= 0 ? A.y_in + T.src_c2 + X.src2[cc] : nullptr;
    const double *b1n = X.src1[cc + 1] >= 0 ? A.y_in + T.src_c1 + X.src1[cc + 1] : nullptr;
    const double *b2n = X.src2[cc + 1] >= 0 ? A.y_in + T.src_c2 + X.src2[cc + 1] : nullptr;
    const bool v1 = b1 && b1n == b1 + 1 && ((reinterpret_cast<uintptr_t>(b1) | (uintptr_t(T.ld_c1) * 8)) & 15) == 0;
    const bool v2 = b2 && b2n == b2 + 1 && ((reinterpret_cast<uintptr_t>(b2) | (uintptr_t(T.ld_c2) * 8)) & 15) == 0;
    const void *any = A.tiles;
    for (int i_ = threadIdx.x / (TN / 2); i_ < n4; i_ += R) {
      const bool first = i_ < k1, second = !first && i_ < k1 + k2;
      const int64_t off = int64_t(first ? i_ : i_ - k1) * (first ? T.ld_c1 : T.ld_c2);
      const double *p0 = first ? b1 : (second ? b2 : nullptr);
      const double *p1 = first ? b1n : (second ? b2n : nullptr);
      double *d = &sZ[i_ * C::LDZ + cc];
      if ((first && v1) || (second && v2)) {
        cp16(d, p0 + off);
      } else if (!p0 && !p1) {
        cp16_zero(d, any);
      } else {
        cp8(d, p0 ? (const void *)(p0 + off) : any, p0 != nullptr);
        cp8(d + 1, p1 ? (const void *)(p1 + off) : any, p1 != nullptr);
      }
    }
  };
  // ---- prologue: tile tb ready to compute, tb+1 groups landed, tb+2 descriptor landed
  load_desc(tb);
  load_desc(tb + 1);
  load_desc(tb + 2);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  load_groups(tb);
  load_groups(tb + 1);
  async_tile<NP, NP, C::LDQ>(sQ, A.q + meta[0].tile.q_off, meta[0].tile.n, meta[0].tile.n, meta[0].tile.n, A.tiles);
  int64_t q_loaded = meta[0].tile.q_off;
  cp_commit();
  cp_wait_all();
  __syncthreads();
  make_maps(tb);
  __syncthreads();
  gather(tb);
  load_desc(tb + 3);
  cp_commit();
  for (int64_t i = tb; i < te; i++) {
    cp_wait_all();
    __syncthreads();  // Z_i, groups(i+1), descriptors(i+2, i+3) landed; tile i-1 fully done
    const StripTileX &T = meta[(i - tb) & 3].tile;
    const PipeMaps<NP, TN> &X = maps[(i - tb) & 1];
    if (T.q_off != q_loaded) {  // panel change: Q_q (exposed, rare)
      async_tile<NP, NP, C::LDQ>(sQ, A.q + T.q_off, T.n, T.n, T.n, A.tiles);
      cp_commit();
      cp_wait_all();
      __syncthreads();
      q_loaded = T.q_off;
    }
    // ---- prepare tile i+1 (maps, then Z in flight), groups of i+2
    if (i + 1 < te) {
      make_maps(i + 1);
      __syncthreads();
      gather(i + 1);
    }
    load_groups(i + 2);
    cp_commit();
    // ---- W = Q_q^T Z_i
    const int n = T.n, kq = T.kq, ncol = T.ncol;
    double *sZ = zbuf(i);
    double acc[2][C::WN / 8][2];
    zero_acc(acc);
    if (m0 < n) warp_gemm<C::LDQ, C::LDZ, 2, C::WN / 8, true>(sQ, sZ, m0, n0, rup(n, 4), acc);
    // ---- epilogue: carry rows [0, kq) -> q's panel; rows [kq, n) reduced (aligned slabs)
#pragma unroll
    for (int i2 = 0; i2 < 2; i2++) {
      const int row = m0 + i2 * 8 + r;
      if (row >= kq || row >= n || T.y_dst < 0) continue;
#pragma unroll
      for (int j = 0; j < C::WN / 8; j++) {
        const int col = n0 + j * 8 + 2 * q4;
        if (col >= ncol) continue;
        double *d = A.y_out + T.y_dst + int64_t(row) * T.y_ld + T.c0 + col;
        if (col + 1 < ncol)
          store2(d, acc[i2][j][0], acc[i2][j][1]);
        else
          d[0] = acc[i2][j][0];
      }
    }
    __syncthreads();  // every warp is done reading Z_i: its space holds the slab partials
    double2 *dslab = reinterpret_cast<double2 *>(sZ);
    double2 *tslab = dslab + C::NWN * NP;
    const int wn = warp % C::NWN, wm = warp / C::NWN;
    if (m0 < n) {
#pragma unroll
      for (int i2 = 0; i2 < 2; i2++) {
        const int row = m0 + i2 * 8 + r;
        double y = 0.0, y2 = 0.0;
#pragma unroll
        for (int j = 0; j < C::WN / 8; j++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const double v = acc[i2][j][e];
            y = fma(v, X.wc[n0 + j * 8 + 2 * q4 + e], y);
            y2 = fma(v, v, y2);
          }
        y += __shfl_xor_sync(0xffffffffu, y, 1);
        y2 += __shfl_xor_sync(0xffffffffu, y2, 1);
        y += __shfl_xor_sync(0xffffffffu, y, 2);
        y2 += __shfl_xor_sync(0xffffffffu, y2, 2);
        if (q4 == 0) dslab[wn * NP + row] = make_double2(y, y2);
      }
#pragma unroll
      for (int j = 0; j < C::WN / 8; j++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          double y = 0.0, y2 = 0.0;
#pragma unroll
          for (int i2 = 0; i2 < 2; i2++) {
            const int row = m0 + i2 * 8 + r;
            const double v = row >= kq ? acc[i2][j][e] : 0.0;
            y = fma(v, X.wq[row >= kq ? row - kq : 0], y);
            y2 = fma(v, v, y2);
          }
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) {
            y += __shfl_xor_sync(0xffffffffu, y, o);
            y2 += __shfl_xor_sync(0xffffffffu, y2, o);
          }
          if (r == 0) tslab[wm * TN + n0 + j * 8 + 2 * q4 + e] = make_double2(y, y2);
        }
    }
    __syncthreads();
    const int nfz = n - kq;
    const int nwm = (n + 15) / 16;
    if (T.s_dst >= 0) {
      const int ngt = X.ngt;
      for (int it = threadIdx.x; it < nfz * ngt; it += blockDim.x) {
        const int a = it / ngt, g = it - a * ngt;
        const int4 gt = X.gtab[g];
        double2 v = make_double2(0.0, 0.0);
        for (int sl = gt.x / C::WN; sl < (gt.x + gt.y) / C::WN; sl++) {
          v.x += dslab[sl * NP + kq + a].x;
          v.y += dslab[sl * NP + kq + a].y;
        }
        A.part[T.s_dst + g + int64_t(a) * T.s_ld] = v;
      }
    }
    for (int cc = threadIdx.x; cc < ncol; cc += blockDim.x) {
      const int64_t td = X.tdst[cc];
      if (td < 0) continue;
      double2 v = make_double2(0.0, 0.0);
      for (int sl = kq / 16; sl < nwm; sl++) {
        v.x += tslab[sl * TN + cc].x;
        v.y += tslab[sl * TN + cc].y;
      }
      A.part[td] = v;
    }
    __syncthreads();  // tile i's metadata stage is free again
    load_desc(i + 4);
    cp_commit();
  }
}

// Bench mode: y[i] = sum of row i's partial slots, in block order (one warp per
// S row, lanes round robin over the blocks, fixed shuffle tree), and the row
// norms likewise.  One CTA per S block row.
__global__ void __launch_bounds__(256) bench_reduce_kernel(const CsrBlockRow *__restrict__ rows,
                                                           const double2 *__restrict__ part, double *__restrict__ y,
                                                           double *__restrict__ r2) {
  const CsrBlockRow br = rows[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int a = warp; a < br.m_r; a += blockDim.x >> 5) {
    const double2 *p = part + br.part_base + int64_t(a) * br.nblk;
    double sy = 0.0, sr = 0.0;
    for (int j = lane; j < br.nblk; j += 32) {
      const double2 v = __ldcs(p + j);
      sy += v.x;
      sr += v.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
      sr += __shfl_xor_sync(0xffffffffu, sr, o);
    }
    if (lane == 0) {
      y[br.grow0 + a] = sy;
      if (r2) r2[br.grow0 + a] = sr;
    }
  }
}

// --------------------------------------------------------------------------
// CSR column indices.  A block row (rows [row0, row0 + m_r)) is one contiguous
// panel of m_r x rowlen entries in s_col, every row carrying the same column
// pattern: expand the pattern once into shared memory, then stream the panel
// out with coalesced stores.  Long panels are split over several CTAs.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) csr_cols_kernel(const CsrBlockRow *__restrict__ rows,
                                                       const int32_t *__restrict__ pat, int32_t *__restrict__ col,
                                                       int splits, int64_t nwork) {
  // grid-stride over the (block row, part) work items: a capped grid
  // (H2SP_CSR_GRID) keeps this bandwidth filler from crowding the latency-bound
  // kernels it overlaps
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
  const CsrBlockRow br = rows[w / splits];
  const int part = int(w % splits);
  const int rowlen = br.rowlen;
  // this CTA writes whole rows [a0, a1) of the panel: a broadcast copy of the
  // block row's precomputed column pattern
  const int a0 = int((int64_t(br.m_r) * part) / splits), a1 = int((int64_t(br.m_r) * (part + 1)) / splits);
  const int32_t *src = pat + br.pat_off;
  int32_t *dst = col + br.p_base + int64_t(a0) * rowlen;
  constexpr int PER = 12;  // pattern entries held in registers per thread (chunk of 256 * PER columns)
  for (int c0 = 0; c0 < rowlen; c0 += 256 * PER) {
    int32_t v[PER];
#pragma unroll
    for (int i = 0; i < PER; i++) {
      const int p = c0 + threadIdx.x + 256 * i;
      v[i] = p < rowlen ? __ldg(src + p) : 0;
    }
    for (int a = 0; a < a1 - a0; a++) {
      int32_t *d = dst + int64_t(a) * rowlen + c0;
#pragma unroll
      for (int i = 0; i < PER; i++) {
        const int p = threadIdx.x + 256 * i;
        if (c0 + p < rowlen) d[p] = v[i];
      }
    }
  }
  }
}

// --------------------------------------------------------------------------
// Apply, one launch per direction.
// y = U^T b, leaves -> root: one CTA per leaf; after a cluster is done, the
// CTA that completes the second child of a parent (atomic arrival counter)
// continues with the parent, so the whole upward pass is one kernel.
// x = V y, root -> leaves: one CTA per leaf walks its root-to-leaf path,
// recomputing the (few, small) ancestor products it needs.
// Vectors column-major (ld) with nrhs columns; zb = basis coefficients.
// --------------------------------------------------------------------------
// APPLY_RC: right-hand sides per pass over Q (each Q element read once per pass):
// 1 for a single vector, 8 otherwise
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sum NV per-lane values over the 32 lanes of a warp: recursive halving (lanes
// o apart exchange the half they do not keep: NV - 1 shuffles instead of
// 5 NV), then a butterfly over the remaining lane bits.  Afterwards v[0] is the
// warp total of value `slot` (returned); the 32 / NV lanes sharing a slot hold
// the same total.  Fixed order.
template <int NV>
__device__ __forceinline__ int warp_reduce_many(double (&v)[NV], int lane) {
  static_assert(NV >= 1 && NV <= 32 && (NV & (NV - 1)) == 0, "power of two");
  int slot = 0, o = 16;
#pragma unroll
  for (int cnt = NV; cnt > 1; cnt >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < cnt / 2; i++) {
      const double send = up ? v[i] : v[i + cnt / 2];
      const double keep = up ? v[i + cnt / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    slot = 2 * slot + (up ? 1 : 0);
    o >>= 1;
  }
#pragma unroll
  for (int o2 = 16 / NV; o2 > 0; o2 >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o2);
  return slot;
}

// predicated 16-byte read-only load (zeros when !ok); one LDG.128 whatever the predicate's shape
__device__ __forceinline__ double2 ldg2(const double *p, bool ok) {
  double2 v = make_double2(0.0, 0.0);
  asm volatile("{ .reg .pred pp; setp.ne.b32 pp, %3, 0; @pp ld.global.nc.v2.f64 {%0, %1}, [%2]; }"
               : "+d"(v.x), "+d"(v.y)
               : "l"(p), "r"(int(ok)));
  return v;
}

// z[j] = sum_i Q[i n + j] x[i] (j in [0, n), n <= 128; x = sx[i * APPLY_RC + rr]),
// per-warp partial sums into red[(rr * 4 + warp) * 128 + j] (4 warps).  The warps split
// the rows (UR consecutive rows each per round), the lanes the columns in
// 16-byte pairs (2 lane, 2 lane + 1 and + 64): every load of a round is issued
// before the first FMA, so a lane keeps 2 UR 16-byte loads in flight.
template <int APPLY_RC>
__device__ __forceinline__ void apply_cols(const double *__restrict__ Q, int n, const double *sx, int rc, double *red) {
  constexpr int UR = APPLY_RC == 1 ? 8 : 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool vec = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(Q) & 15) == 0;
  double acc[4][APPLY_RC];
#pragma unroll
  for (int c = 0; c < 4; c++)
#pragma unroll
    for (int rr = 0; rr < APPLY_RC; rr++) acc[c][rr] = 0.0;
  if (vec) {
    const int ja = 2 * lane, jb = 2 * lane + 64;
    for (int base = 0; base < n; base += nw * UR) {
      double2 qa[UR], qb[UR];
#pragma unroll
      for (int u = 0; u < UR; u++) {
        const int i = base + warp * UR + u;
        const double *row = Q + int64_t(i) * n;
        qa[u] = ldg2(row + ja, i < n && ja < n);
        qb[u] = ldg2(row + jb, i < n && jb < n);
      }
#pragma unroll
      for (int u = 0; u < UR; u++) {
        const int i = min(base + warp * UR + u, n - 1);   // rows past n carry zeros in qa / qb
#pragma unroll
        for (int rr = 0; rr < APPLY_RC; rr++) {
          if (rr >= rc) continue;
          const double xv = sx[i * APPLY_RC + rr];
          acc[0][rr] = fma(qa[u].x, xv, acc[0][rr]);
          acc[1][rr] = fma(qa[u].y, xv, acc[1][rr]);
          acc[2][rr] = fma(qb[u].x, xv, acc[2][rr]);
          acc[3][rr] = fma(qb[u].y, xv, acc[3][rr]);
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < APPLY_RC; rr++) {   // [rhs][warp][column]: conflict-free 16-byte stores
      double *rw = red + (rr * 4 + warp) * 128;
      if (ja < n) *reinterpret_cast<double2 *>(rw + ja) = make_double2(acc[0][rr], acc[1][rr]);
      if (jb < n) *reinterpret_cast<double2 *>(rw + jb) = make_double2(acc[2][rr], acc[3][rr]);
    }
  } else {
    for (int base = 0; base < n; base += nw * UR) {
      double qv[UR][4];
#pragma unroll
      for (int u = 0; u < UR; u++) {
        const int i = base + warp * UR + u;
#pragma unroll
        for (int c = 0; c < 4; c++) qv[u][c] = (i < n && lane + 32 * c < n) ? __ldg(Q + int64_t(i) * n + lane + 32 * c) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UR; u++) {
        const int i = min(base + warp * UR + u, n - 1);
#pragma unroll
        for (int rr = 0; rr < APPLY_RC; rr++) {
          if (rr >= rc) continue;
          const double xv = sx[i * APPLY_RC + rr];
#pragma unroll
          for (int c = 0; c < 4; c++) acc[c][rr] = fma(qv[u][c], xv, acc[c][rr]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 4; c++)
      if (lane + 32 * c < n)
#pragma unroll
        for (int rr = 0; rr < APPLY_RC; rr++) red[(rr * 4 + warp) * 128 + lane + 32 * c] = acc[c][rr];
  }
}

// --------------------------------------------------------------------------
// y = U^T b, leaves -> root, one launch: one CTA (4 warps) per leaf computes
// z = Q_t^T x_t with Q read straight from global memory (apply_cols); the CTA
// that completes the second child of a parent (atomic arrival counter)
// continues with the parent, so the whole upward pass is one kernel.
// --------------------------------------------------------------------------
template <int APPLY_RC>
__global__ void __launch_bounds__(128) apply_ut_kernel(Side sd, int L, const double *__restrict__ q,
                                                       const double *__restrict__ b, int64_t ldb, double *__restrict__ y,
                                                       int64_t ldy, double *__restrict__ zb, int64_t zbl, int nrhs, int B,
                                                       int *__restrict__ arrive, int64_t leaf0) {
  __shared__ double sx[128 * APPLY_RC];
  __shared__ __align__(16) double red[4 * 128 * APPLY_RC];   // [rhs][warp][column]
  __shared__ int s_go;
  // metadata of every cluster this CTA may climb through (the leaf's ancestors)
  // and of their children, in one round trip (level l in slot l)
  __shared__ int m_n[64], m_k[64], m_k1[64];
  __shared__ int64_t m_q[64], m_zb[64], m_loc[64], m_zb1[64], m_zb2[64];
  int level = 0;
  int64_t idx = leaf0 + blockIdx.x;  // in-level index (global)
  for (int lv = threadIdx.x; lv <= L; lv += blockDim.x) {
    const int64_t a = idx >> lv, cl = lvl_off_d(L, lv) + a;
    m_n[lv] = sd.n[cl];
    m_k[lv] = sd.k[cl];
    m_q[lv] = sd.q_off[cl];
    m_zb[lv] = sd.zb_off[cl];
    m_loc[lv] = sd.loc_off[cl];
    if (lv > 0) {
      const int64_t c1 = lvl_off_d(L, lv - 1) + 2 * a;
      m_k1[lv] = sd.k[c1];
      m_zb1[lv] = sd.zb_off[c1];
      m_zb2[lv] = sd.zb_off[c1 + 1];
    }
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  while (true) {
    const int n = m_n[level], k = m_k[level];
    if (level < L) {  // the parent's Q into L2 now: the CTA that climbs reads it after the arrival
      const int np = m_n[level + 1];
      const double *Qp = q + m_q[level + 1];
      for (int e = threadIdx.x * 16; e < np * np; e += blockDim.x * 16)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(Qp + e));
    }
    if (n > 0) {
      const double *Q = q + m_q[level];
      const int k1 = level > 0 ? m_k1[level] : 0;
      for (int r0 = 0; r0 < nrhs; r0 += APPLY_RC) {
        const int rc = min(APPLY_RC, nrhs - r0);
        __syncthreads();
        for (int e = threadIdx.x; e < n * rc; e += blockDim.x) {
          const int i = e % n, rr = e / n, r = r0 + rr;
          double v;
          if (level == 0) v = b[((idx - leaf0) * B + i) + r * ldb];
          else if (i < k1) v = __ldcg(zb + m_zb1[level] + i + r * zbl);
          else v = __ldcg(zb + m_zb2[level] + (i - k1) + r * zbl);
          sx[i * APPLY_RC + rr] = v;
        }
        __syncthreads();
        apply_cols<APPLY_RC>(Q, n, sx, rc, red);
        __syncthreads();
        for (int e = threadIdx.x; e < n * rc; e += blockDim.x) {
          const int tj = e % n, rr = e / n, r = r0 + rr;
          double acc = red[rr * 4 * 128 + tj];
          for (int u = 1; u < nw; u++) acc += red[(rr * 4 + u) * 128 + tj];
          if (tj < k) zb[m_zb[level] + tj + r * zbl] = acc;
          else y[m_loc[level] + (tj - k) + r * ldy] = acc;
        }
      }
    }
    if (level == L) break;
    // arrival at the parent: the second child's CTA continues upward
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t parent = lvl_off_d(L, level + 1) + idx / 2;
      s_go = atomicAdd(&arrive[parent], 1) == 1;
    }
    __syncthreads();
    if (!s_go) break;
    __threadfence();
    level++;
    idx >>= 1;
  }
}

// out[i] = sum_j Q[i n + j] v[j] for i in [0, n), n <= 128, APPLY_RC right-hand
// sides at once (sv[rr * 128 + j]: conflict-free 16-byte reads).  Per round warp w takes rows
// base + UR w .. + UR - 1; the lanes stride one row's columns in 16-byte pairs
// (2 lane and 2 lane + 64), every load of a round issued before the first FMA;
// the UR x APPLY_RC partial sums of a lane meet by recursive halving
// (warp_reduce_many).  ready() is called by every thread once, after the first
// round's loads are issued and before sv is read: it completes sv and ends with
// a CTA barrier (the loads stay in flight across it).  emit(i, rr, value): one
// lane per result.
template <int APPLY_RC, class R, class F>
__device__ __forceinline__ void apply_rows(const double *__restrict__ Q, int n, const double *sv, int rc, R &&ready,
                                           F &&emit) {
  constexpr int UR = APPLY_RC == 1 ? 8 : 2, NV = UR * APPLY_RC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool vec = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(Q) & 15) == 0;
  const int ja = 2 * lane, jb = 2 * lane + 64;
  for (int base = 0; base < n; base += nw * UR) {
    const int i0 = base + warp * UR;
    double acc[NV];
#pragma unroll
    for (int e = 0; e < NV; e++) acc[e] = 0.0;
    if (vec) {
      double2 qa[UR], qb[UR];
#pragma unroll
      for (int u = 0; u < UR; u++) {
        const double *row = Q + int64_t(i0 + u) * n;
        qa[u] = ldg2(row + ja, i0 + u < n && ja < n);
        qb[u] = ldg2(row + jb, i0 + u < n && jb < n);
      }
      if (base == 0) ready();
      const int jas = min(ja, n - 2), jbs = min(jb, n - 2);   // lanes past n carry zeros in qa / qb
#pragma unroll
      for (int rr = 0; rr < APPLY_RC; rr++) {
        if (rr >= rc) continue;
        const double2 va = *reinterpret_cast<const double2 *>(sv + rr * 128 + jas);
        const double2 vb = *reinterpret_cast<const double2 *>(sv + rr * 128 + jbs);
#pragma unroll
        for (int u = 0; u < UR; u++)
          acc[u * APPLY_RC + rr] = fma(qb[u].y, vb.y, fma(qb[u].x, vb.x, fma(qa[u].y, va.y, fma(qa[u].x, va.x, 0.0))));
      }
    } else {
      if (base == 0) ready();
      for (int j = lane; j < n; j += 32) {
        double qv[UR];
#pragma unroll
        for (int u = 0; u < UR; u++) qv[u] = i0 + u < n ? __ldg(Q + int64_t(i0 + u) * n + j) : 0.0;
#pragma unroll
        for (int rr = 0; rr < APPLY_RC; rr++) {
          if (rr >= rc) continue;
          const double v0 = sv[rr * 128 + j];
#pragma unroll
          for (int u = 0; u < UR; u++) acc[u * APPLY_RC + rr] = fma(qv[u], v0, acc[u * APPLY_RC + rr]);
        }
      }
    }
    const int slot = warp_reduce_many<NV>(acc, lane);
    const int u = slot / APPLY_RC, rr = slot % APPLY_RC;
    if ((lane & (32 / NV - 1)) == 0 && i0 + u < n && rr < rc) emit(i0 + u, rr, acc[0]);
  }
}

// --------------------------------------------------------------------------
// x = V y, root -> leaves, one launch: one CTA (8 warps) per cluster of the
// shard's tree (its subtree and the path above it).  CTAs take their cluster
// from a ticket counter in start order, the tickets numbering the clusters
// level by level from the root down (the leaves last): cluster t's product
// [c_1; c_2] = Q_t [c_t; y_t] is computed once -- its Q rows and y_t are
// requested first, then the CTA waits for the parent's flag (acquire), reads
// c_t from zb, multiplies, writes the children's coefficients to zb and
// publishes its own flag (release).  A cluster's parent has a smaller ticket,
// i.e. belongs to a CTA that is already running, so the waits cannot deadlock
// whatever the hardware's block scheduling order; the upper levels are done
// while the first wide levels stream, and the leaves (most of the bytes) find
// their parents finished.  flags: [ncl] cluster flags + the ticket, zeroed
// before the launch.
// --------------------------------------------------------------------------
template <int APPLY_RC>
__global__ void __launch_bounds__(256) apply_v_kernel(Side sd, int L, const double *__restrict__ q,
                                                      const double *__restrict__ y, int64_t ldy, double *__restrict__ x,
                                                      int64_t ldx, double *zb, int64_t zbl, int nrhs, int B, int *flags,
                                                      int64_t ncl, int64_t leaf0, int64_t nleaves) {
  __shared__ __align__(16) double sv[128 * APPLY_RC];   // [rhs][column]
  __shared__ int s_ticket;
  if (threadIdx.x == 0) s_ticket = atomicAdd(flags + ncl, 1);
  __syncthreads();
  // ticket -> (level, in-level index): levels L .. 0, max(1, nleaves >> level) clusters each
  int64_t t = s_ticket;
  int lv = L;
  for (; lv > 0; lv--) {
    const int64_t cnt = max(int64_t(1), nleaves >> lv);
    if (t < cnt) break;
    t -= cnt;
  }
  const int64_t a = (leaf0 >> lv) + t, cl = lvl_off_d(L, lv) + a;
  const int n = sd.n[cl], k = sd.k[cl];
  int *flag = flags + cl;
  if (n == 0) {  // nothing to multiply (levels without admissible blocks): the children carry no coefficients
    if (lv > 0 && threadIdx.x == 0) st_release_gpu(flag, 1);
    return;
  }
  const double *Q = q + sd.q_off[cl];
  const int64_t loc = sd.loc_off[cl], zin = sd.zb_off[cl];
  int k1 = 0;
  int64_t zo1 = 0, zo2 = 0;
  if (lv > 0) {
    const int64_t c1 = lvl_off_d(L, lv - 1) + 2 * a;
    k1 = sd.k[c1];
    zo1 = sd.zb_off[c1];
    zo2 = sd.zb_off[c1 + 1];
  }
  const int *pflag = (lv < L && k > 0) ? flags + lvl_off_d(L, lv + 1) + (a >> 1) : nullptr;
  for (int r0 = 0; r0 < nrhs; r0 += APPLY_RC) {
    const int rc = min(APPLY_RC, nrhs - r0);
    auto ready = [&]() {  // (called with the Q loads in flight)
      for (int e = threadIdx.x; e < (n - k) * rc; e += blockDim.x) {  // the cluster's own part of the vector
        const int jj = e % (n - k), rr = e / (n - k);
        sv[rr * 128 + k + jj] = y[loc + jj + (r0 + rr) * ldy];
      }
      if (r0 == 0 && pflag) {  // the parent's part, once its product is published
        if (threadIdx.x == 0)
          while (ld_acquire_gpu(pflag) == 0) __nanosleep(20);
        __syncthreads();
      }
      for (int e = threadIdx.x; e < k * rc; e += blockDim.x) {
        const int jj = e % k, rr = e / k;
        sv[rr * 128 + jj] = __ldcg(zb + zin + jj + (r0 + rr) * zbl);
      }
      __syncthreads();
    };
    if (lv == 0) {
      double *xo = x + (a - leaf0) * B + r0 * ldx;
      apply_rows<APPLY_RC>(Q, n, sv, rc, ready, [&](int i, int rr, double v) { xo[i + rr * ldx] = v; });
    } else {
      double *z1 = zb + zo1 + r0 * zbl, *z2 = zb + zo2 + r0 * zbl - k1;
      apply_rows<APPLY_RC>(Q, n, sv, rc, ready, [&](int i, int rr, double v) { (i < k1 ? z1 : z2)[i + rr * zbl] = v; });
    }
    __syncthreads();   // sv free for the next pass; every thread's zb stores ordered before the release
  }
  if (lv > 0 && threadIdx.x == 0) st_release_gpu(flag, 1);
}

// --------------------------------------------------------------------------
// Host orchestration
// --------------------------------------------------------------------------
template <int KP, bool GEN, bool BENCH>
static h2sp_status launch_pairs_wy128_t(const PairArgs &a, const double *wy_row, const double *wy_col, int64_t nchunks,
                                        cudaStream_t st) {
  using C = PairWy128Cfg<KP>;
  if (h2sp_status e = ensure_smem((const void *)pair_wy128_kernel<KP, GEN, BENCH>, C::SMEM)) return e;
  pair_wy128_kernel<KP, GEN, BENCH><<<unsigned(nchunks), C::THREADS, C::SMEM, st>>>(a, wy_row, wy_col);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}
template <int KP, bool BENCH>
static h2sp_status launch_pairs_wy128g_t(const PairArgs &a, const double *wy_row, const double *wy_col,
                                         int64_t nchunks, cudaStream_t st) {
  using C = PairWy128gCfg<KP>;
  if (h2sp_status e = ensure_smem((const void *)pair_wy128g_kernel<KP, BENCH>, C::SMEM)) return e;
  pair_wy128g_kernel<KP, BENCH><<<unsigned(nchunks), C::THREADS, C::SMEM, st>>>(a, wy_row, wy_col);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}
template <int KP>
static h2sp_status launch_pairs_wy128(const PairArgs &a, const double *wy_row, const double *wy_col, int64_t nchunks,
                                      cudaStream_t st, bool bench) {
  const bool gen = a.gen.pts != nullptr;
  // matrix-free close blocks, H2SP_WY128_GEVAL=1: G evaluated inside the products
  // (pair_wy128g_kernel, no G buffer, no exposed load) -- measured 8 % slower
  // than evaluating every entry once into the G buffer (config 5: 2996 vs
  // 2795 ms per step; the FP64 datapath, shared by DMMA and the evaluations,
  // is the bottleneck, so the second evaluation costs more than the loads it hides)
  static const bool geval = getenv("H2SP_WY128_GEVAL") && atoi(getenv("H2SP_WY128_GEVAL")) != 0;
  if (gen && geval)
    return bench ? launch_pairs_wy128g_t<KP, true>(a, wy_row, wy_col, nchunks, st)
                 : launch_pairs_wy128g_t<KP, false>(a, wy_row, wy_col, nchunks, st);
  if (bench)
    return gen ? launch_pairs_wy128_t<KP, true, true>(a, wy_row, wy_col, nchunks, st)
               : launch_pairs_wy128_t<KP, false, true>(a, wy_row, wy_col, nchunks, st);
  return gen ? launch_pairs_wy128_t<KP, true, false>(a, wy_row, wy_col, nchunks, st)
             : launch_pairs_wy128_t<KP, false, false>(a, wy_row, wy_col, nchunks, st);
}

template <int NP, bool GEN, bool BENCH>
static h2sp_status launch_pairs_t(const PairArgs &a, int64_t nchunks, cudaStream_t st) {
  using C = PairCfg<NP>;
  if (h2sp_status e = ensure_smem((const void *)pair_kernel<NP, GEN, BENCH>, C::SMEM)) return e;
  pair_kernel<NP, GEN, BENCH><<<unsigned(nchunks), C::THREADS, C::SMEM, st>>>(a);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}
template <int NP>
static h2sp_status launch_pairs(const PairArgs &a, int64_t nchunks, cudaStream_t st, bool bench) {
  static_assert(PairCfg<NP>::WARPS >= 1, "");
  const bool gen = a.level == 0 && a.gen.pts != nullptr;
  if (bench)
    return gen ? launch_pairs_t<NP, true, true>(a, nchunks, st) : launch_pairs_t<NP, false, true>(a, nchunks, st);
  return gen ? launch_pairs_t<NP, true, false>(a, nchunks, st) : launch_pairs_t<NP, false, false>(a, nchunks, st);
}

template <int KP, bool GEN, bool BENCH>
static h2sp_status launch_pairs_wy_t(const PairArgs &a, const double *wy_row, const double *wy_col, int64_t nchunks,
                                     cudaStream_t st) {
  using C = PairWyCfg<KP>;
  if (h2sp_status e = ensure_smem((const void *)pair_wy_kernel<KP, GEN, BENCH>, C::SMEM)) return e;
  pair_wy_kernel<KP, GEN, BENCH><<<unsigned(nchunks), C::THREADS, C::SMEM, st>>>(a, wy_row, wy_col);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}
template <int KP>
static h2sp_status launch_pairs_wy(const PairArgs &a, const double *wy_row, const double *wy_col, int64_t nchunks,
                                   cudaStream_t st, bool bench) {
  const bool gen = a.gen.pts != nullptr;
  if (bench)
    return gen ? launch_pairs_wy_t<KP, true, true>(a, wy_row, wy_col, nchunks, st)
               : launch_pairs_wy_t<KP, false, true>(a, wy_row, wy_col, nchunks, st);
  return gen ? launch_pairs_wy_t<KP, true, false>(a, wy_row, wy_col, nchunks, st)
             : launch_pairs_wy_t<KP, false, false>(a, wy_row, wy_col, nchunks, st);
}

template <int NP, int TN, bool BENCH>
static h2sp_status launch_strips1(const StripArgs &a, int64_t ntiles, cudaStream_t st) {
  using C = StripCfg<NP, TN>;
  // bench mode, aligned plans: the pipelined persistent kernel (H2SP_STRIP_PIPE=0: one tile per CTA)
  // (measured slower: config 5 serial strips 1.11 vs 0.96 s -- one CTA of 16 warps
  // per SM hides the DMMA / shared-memory latencies worse than two one-tile CTAs)
  static const bool pipe = getenv("H2SP_STRIP_PIPE") && atoi(getenv("H2SP_STRIP_PIPE")) != 0;
  if constexpr (BENCH && NP >= 32) {
    if (pipe && a.aligned) {
      using PC = StripPipeCfg<NP, TN>;
      if (h2sp_status e = ensure_smem((const void *)strip_pipe_kernel<NP, TN>, PC::SMEM)) return e;
      int dev = 0, nsm = 148;
      H2SP_CK(cudaGetDevice(&dev));
      H2SP_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      const int64_t grid = std::min<int64_t>(ntiles, nsm);
      if (grid > 0) strip_pipe_kernel<NP, TN><<<unsigned(grid), C::THREADS, PC::SMEM, st>>>(a, ntiles);
      H2SP_CK(cudaGetLastError());
      return H2SP_OK;
    }
  }
  constexpr size_t smem = C::SMEM + (BENCH ? size_t(TN + NP) * sizeof(double) : 0);  // + staged weights
  static_assert(!BENCH || size_t(NP) * C::LDZ * sizeof(double) >= (C::NWN * NP + (NP / 16) * TN) * 16,
                "slab partials fit the Z buffer");
  if (h2sp_status e = ensure_smem((const void *)strip_kernel<NP, TN, BENCH>, smem)) return e;
  strip_kernel<NP, TN, BENCH><<<unsigned(ntiles), C::THREADS, smem, st>>>(a);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}

static int pad16(int x) { return x <= 16 ? 16 : x <= 32 ? 32 : x <= 48 ? 48 : 64; }

template <int TN, bool BENCH>
static h2sp_status launch_strips_tn(const StripArgs &a, int np, int64_t ntiles, cudaStream_t st) {
  switch (pad16(np)) {
    case 16: return launch_strips1<16, TN, BENCH>(a, ntiles, st);
    case 32: return launch_strips1<32, TN, BENCH>(a, ntiles, st);
    case 48: return launch_strips1<48, TN, BENCH>(a, ntiles, st);
    default: return launch_strips1<64, TN, BENCH>(a, ntiles, st);
  }
}

// tn: the tile width the plan cut this level's panels into (strip_tn_of_level)
static h2sp_status launch_strips(const StripArgs &a, int np, int tn, int64_t ntiles, cudaStream_t st, bool bench) {
  if (bench)
    return tn == STRIP_TN_SMALL ? launch_strips_tn<STRIP_TN_SMALL, true>(a, np, ntiles, st)
                                : launch_strips_tn<STRIP_TN, true>(a, np, ntiles, st);
  return tn == STRIP_TN_SMALL ? launch_strips_tn<STRIP_TN_SMALL, false>(a, np, ntiles, st)
                              : launch_strips_tn<STRIP_TN, false>(a, np, ntiles, st);
}

// Side streams and events used to overlap the independent chains of one build
// (QR + couplings of all levels, CSR index expansion) with the congruence
// chain.  Created once per device; fork/join through events on the caller's
// stream, so a build stays stream-ordered (and CUDA-graph capturable).
struct DeviceAux {
  bool init = false;
  cudaStream_t side[8];    // QR/coupling chain, CSR, strips (set 0 / first half), main chain, strips (set 1),
                           // strips (set 0, second half), h2sp_build_host's early CSR + D2H, level-0 Q from V / M
  cudaEvent_t host_fork = nullptr, host_join = nullptr;
  std::vector<cudaEvent_t> ev;
};
static DeviceAux g_aux[64];

static h2sp_status get_aux(int L, DeviceAux **out) {
  int dev = 0;
  H2SP_CK(cudaGetDevice(&dev));
  DeviceAux &a = g_aux[dev & 63];
  if (!a.init) {
    // s1 (QR / coupling chain, latency-bound, on the critical path of level 1)
    // gets the highest priority so its CTAs take SM slots as soon as they free
    // up; s2 (CSR index expansion, bandwidth filler) the lowest.
    int lo = 0, hi = 0;
    H2SP_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    int qr_off = 0;  // H2SP_PRIO_QR: levels below the highest for the QR / coupling chain
    if (const char *e = getenv("H2SP_PRIO_QR")) qr_off = atoi(e);
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[0], cudaStreamNonBlocking, hi < lo ? std::min(lo, hi + qr_off) : hi));
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[1], cudaStreamNonBlocking, lo));
    // priorities: QR/coupling chain (feeds every level) > main chain = strips > CSR.
    // H2SP_PRIO="a,b,c" (scheduling experiments): levels below the highest for
    // strips set 0, main chain, strips set 1 (clamped to the device range)
    int off[3] = {2, 1, 2};  // main chain above the strips (measured: 1.30 vs 1.31 ms)
    if (const char *e = getenv("H2SP_PRIO")) sscanf(e, "%d,%d,%d", &off[0], &off[1], &off[2]);
    auto pr = [&](int o) { return hi < lo ? std::min(lo, hi + o) : hi; };
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[2], cudaStreamNonBlocking, pr(off[0])));  // strips, set 0
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[3], cudaStreamNonBlocking, pr(off[1])));  // main chain
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[4], cudaStreamNonBlocking, pr(off[2])));  // strips, set 1
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[5], cudaStreamNonBlocking, pr(off[0])));  // strips, set 0 B
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[6], cudaStreamNonBlocking, lo));  // build_host: early CSR + D2H
    H2SP_CK(cudaStreamCreateWithPriority(&a.side[7], cudaStreamNonBlocking, hi < lo ? std::min(lo, hi + qr_off) : hi));
    H2SP_CK(cudaEventCreateWithFlags(&a.host_fork, cudaEventDisableTiming));
    H2SP_CK(cudaEventCreateWithFlags(&a.host_join, cudaEventDisableTiming));
    a.init = true;
  }
  while (int(a.ev.size()) < 3 * L + 16) {
    cudaEvent_t e;
    H2SP_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    a.ev.push_back(e);
  }
  *out = &a;
  return H2SP_OK;
}

h2sp_status launch_build(const h2sp_plan_s *P, const h2sp_inputs *in, const h2sp_outputs *out,
                         const unsigned char *meta, unsigned char *scratch, void *stream, int64_t *launches,
                         void *const *events, int64_t n_events, const h2sp_apply_args *ap, unsigned char *ap_scratch) {
  cudaStream_t st = (cudaStream_t)stream;
  // workspace regions: plan offsets count from the start of a combined
  // meta | scratch workspace; the two parts may live in separate buffers
  auto reg = [&](size_t off) { return scratch + (off - P->meta_bytes); };
  const Clusters cl = make_clusters(P, meta);
  const Side rs = side_of(cl, false), cs = side_of(cl, true);
  // h2sp_plan_set_qr_mode: H2SP_QR_ALL -- the QR kernels (and the level-0 Q
  // formation) take every cluster of the tree, not just this shard's need set;
  // H2SP_QR_REUSE -- they are not launched: R^ / V, M (the head of scratch, at
  // plan-independent offsets) and Q still hold an H2SP_QR_ALL build's results
  Side rs_qr = rs, cs_qr = cs;
  if (P->qr_mode == H2SP_QR_ALL) rs_qr.need = cs_qr.need = (const int8_t *)(meta + P->ca.need_all);
  const bool qr_reuse = P->qr_mode == H2SP_QR_REUSE;
  const bool sym = P->sym != 0;
  double *rh_row = (double *)reg(P->ws_rh_row);
  double *rh_col = sym ? rh_row : (double *)reg(P->ws_rh_col);
  double *dt = (double *)reg(P->ws_dt);
  double *bb = (double *)reg(P->ws_bb);
  double *yr = (double *)reg(P->ws_yr);
  double *yc = sym ? yr : (double *)reg(P->ws_yc);
  const double *leaf_col = sym ? in->leaf_basis_row : in->leaf_basis_col;
  const double *tr_col = sym ? in->transfer_row : in->transfer_col;
  double *q_col = sym ? out->q_row : out->q_col;
  double *wy_row = P->wy_kp ? (double *)reg(P->ws_wy_row) : nullptr;
  double *wy_col = P->wy_kp ? (double *)reg(P->ws_wy_col) : nullptr;
  const int L = P->L;
  DeviceAux *aux = nullptr;
  if (h2sp_status e = get_aux(L, &aux)) return e;
  cudaStream_t s1 = aux->side[0], s2 = aux->side[1], s3 = aux->side[2], s4 = aux->side[4], s5 = aux->side[5];
  cudaStream_t s7 = aux->side[7];
  const cudaStream_t user_st = st;
  cudaEvent_t ev_begin = aux->ev[6 + 2 * L], ev_end = aux->ev[7 + 2 * L];
  static const bool serial = [] {
    const char *e = getenv("H2SP_SERIAL");  // debugging / attribution: run every launch on `stream`
    return e && e[0] == '1';
  }();
  if (serial) {
    s1 = s2 = s3 = s4 = s5 = s7 = st;
  } else {
    // the main chain runs on an internal high-priority stream forked from the
    // caller's stream (the CSR stream has the lowest priority and fills gaps)
    H2SP_CK(cudaEventRecord(ev_begin, user_st));
    st = aux->side[3];
    H2SP_CK(cudaStreamWaitEvent(st, ev_begin, 0));
  }
  cudaEvent_t ev_fork = aux->ev[0], ev_qr0 = aux->ev[1], ev_csr = aux->ev[2];
  auto ev_ready = [&](int k) { return aux->ev[3 + k]; };   // QR_k and couplings_{k-1} done
  auto ev_pairs = [&](int k) { return aux->ev[4 + L + k]; };  // congruence of level k done (main stream)
  cudaEvent_t ev_strips_done = aux->ev[5 + 2 * L];
  cudaEvent_t ev_pairs_a = aux->ev[10 + 3 * L], ev_a_last = aux->ev[11 + 3 * L], ev_s5_done = aux->ev[12 + 3 * L];
  bool a_recorded = false;  // ev_a_last recorded in this build (never wait on a stale record: graph capture)
  // The launch order (and so the index of h2sp_plan_launches / profiling
  // events) is: per level QR row, QR col, couplings, pairs, row strips,
  // column strips; then the CSR expansion.  Events 2i / 2i+1 bracket launch i
  // on the stream it runs on.
  int64_t nl = 0;
  auto pre = [&](cudaStream_t s, int64_t i) -> h2sp_status {
    if (events && 2 * i < n_events) H2SP_CK(cudaEventRecord((cudaEvent_t)events[2 * i], s));
    return H2SP_OK;
  };
  auto post = [&](cudaStream_t s, int64_t i) -> h2sp_status {
    if (events && 2 * i + 1 < n_events) H2SP_CK(cudaEventRecord((cudaEvent_t)events[2 * i + 1], s));
    return H2SP_OK;
  };
  if (h2sp_status e = ensure_smem((const void *)qr_kernel, 200 * 1024)) return e;
  if (h2sp_status e = ensure_smem((const void *)coupling_kernel, 200 * 1024)) return e;
  // Launch indices are assigned in the plan's canonical order; precompute them.
  struct LvlIdx {
    int64_t qr_row = -1, qr_col = -1, coup = -1, pairs = -1, rstr[2] = {-1, -1}, cstr[2] = {-1, -1}, rstr_b = -1;
  };
  std::vector<LvlIdx> li(L + 1);
  int64_t csr_idx = -1, qform_idx = -1;
  {
    int64_t c = 0;
    for (int k = 0; k <= L; k++) {
      const LevelPlan &lp = P->levels[k];
      if (lp.np_row > 0) li[k].qr_row = c++;
      if (!sym && lp.np_col > 0) li[k].qr_col = c++;
      if (lp.n_coup) li[k].coup = c++;
      if (lp.n_pairs) li[k].pairs = c++;
      for (int set = 0; set < 2; set++) {
        if (lp.sp[set].n_rtiles) li[k].rstr[set] = c++;
        if (lp.sp[set].n_rtiles_a) li[k].rstr_b = c++;
        if (lp.sp[set].n_ctiles) li[k].cstr[set] = c++;
      }
    }
    if (P->n_csr_rows) csr_idx = c++;
    if (P->wy_kp) qform_idx = c++;
    nl = c;
  }
  auto qr = [&](int k, cudaStream_t s) -> h2sp_status {
    const LevelPlan &lp = P->levels[k];
    const int M = int(int64_t(1) << (L - k));
    auto launch = [&](const Side &sd, const std::vector<int32_t> &nn, const std::vector<int32_t> &kk, const double *leaf,
                      const double *tr, double *rh, double *qo, const uint64_t *magic_ptr,
                      double *wyo) -> h2sp_status {
      int per_warp = 2, nmax = 0, kmax = 0, per_warp_reg = 2;
      for (int i = 0; i < M; i++) {
        const int64_t c = lvl_off_d(L, k) + i;
        int rs_ = 0;
        if (k > 0) {
          const int64_t c1 = lvl_off_d(L, k - 1) + 2 * i;
          rs_ = kk[c1] * kk[c1] + kk[c1 + 1] * kk[c1 + 1];
        }
        per_warp = std::max(per_warp, qr_warp_doubles(nn[c], kk[c], rs_));
        per_warp_reg = std::max(per_warp_reg, std::max(qr_reg_warp_doubles(nn[c], kk[c]), nn[c] * kk[c] + rs_ + 2));
        nmax = std::max(nmax, int(nn[c]));
        kmax = std::max(kmax, int(kk[c]));
      }
      // level 0 on the compact-WY path: one CTA per leaf, one row per thread --
      // 128-point leaves always; <= 64-point leaves only with H2SP_QR_CTA=1 (measured
      // slower there than the warp-per-leaf register kernel: 62 vs 52 us alone)
      static const bool qr_cta64 = getenv("H2SP_QR_CTA") && atoi(getenv("H2SP_QR_CTA")) != 0;
      if (k == 0 && wyo && kmax <= 32 && (nmax > 64 || qr_cta64)) {
        const int kp = kmax <= 16 ? 16 : 32;
        const int nw = nmax > 64 ? 4 : 2;
        // M goes straight to global when the compact-WY layout is unpadded
        // (wy_kp == kp, wy_n == 32 nw): the M staging shrinks to the K x K Gram
        const bool m_direct = P->wy_kp == kp && P->wy_n == 32 * nw;
        const size_t smem = size_t(32 * nw * (kp + 4) + kp * (kp + 4) +
                                   (m_direct ? kp * (kp + 4) : kp * (32 * nw + 4))) * sizeof(double);
#define H2SP_QR_CTA(KP_, NW_)                                                                              \
  do {                                                                                                     \
    if (h2sp_status e_ = ensure_smem((const void *)qr_cta_kernel<KP_, NW_>, smem)) return e_;            \
    qr_cta_kernel<KP_, NW_><<<unsigned(M), 32 * NW_, smem, s>>>(sd, M, leaf, rh, wyo, P->wy_kp, P->wy_n,   \
                                                               magic_ptr, P->magic);                      \
  } while (0)
        if (nw == 4) {
          if (kp == 16) H2SP_QR_CTA(16, 4); else H2SP_QR_CTA(32, 4);
        } else {
          if (kp == 16) H2SP_QR_CTA(16, 2); else H2SP_QR_CTA(32, 2);
        }
#undef H2SP_QR_CTA
        H2SP_CK(cudaGetLastError());
        return H2SP_OK;
      }
      // k = n / 2 = 32 (configs 4 and 5 above the leaves, config 4's leaves): one
      // 64-thread CTA per cluster, explicit Q (H2SP_QR_WARP32=1: the warp kernel)
      static const bool qr_warp32 = getenv("H2SP_QR_WARP32") && atoi(getenv("H2SP_QR_WARP32")) != 0;
      if (!wyo && kmax > 24 && kmax <= 32 && nmax > 32 && nmax <= 64 && !qr_warp32) {
        constexpr size_t smem = size_t(64 * (32 + 4) + 32 * (32 + 4) + 32 * (64 + 4)) * sizeof(double);
        if (h2sp_status e_ = ensure_smem((const void *)qr_cta_kernel<32, 2>, smem)) return e_;
        qr_cta_kernel<32, 2><<<unsigned(M), 64, smem, s>>>(sd, M, leaf, rh, nullptr, 0, 0, magic_ptr, P->magic, L, k,
                                                            tr, qo);
        H2SP_CK(cudaGetLastError());
        return H2SP_OK;
      }
      if (kmax <= 32 && nmax <= 64) {
        // 4 independent warps (clusters) per CTA: same per-cluster latency, a quarter of
        // the SM slots taken from the concurrent congruence
        const int wpb = std::max(1, std::min(4, int((96 * 1024) / (size_t(per_warp_reg) * 8))));
        const unsigned grid = unsigned((M + wpb - 1) / wpb);
        const size_t smem = size_t(per_warp_reg) * 8 * wpb;
        const int kp = kmax <= 8 ? 8 : kmax <= 16 ? 16 : kmax <= 24 ? 24 : 32;
#define H2SP_QR_REG(NR_, KP_)                                                                              \
  do {                                                                                                     \
    if (h2sp_status e_ = ensure_smem((const void *)qr_reg_kernel<NR_, KP_>, 100 * 1024)) return e_;      \
    qr_reg_kernel<NR_, KP_><<<grid, 32 * wpb, smem, s>>>(sd, L, k, M, per_warp_reg, leaf, tr, rh, qo,        \
                                                        magic_ptr, P->magic, wyo, P->wy_kp, P->wy_n);      \
  } while (0)
        if (nmax <= 32) {
          switch (kp) {
            case 8: H2SP_QR_REG(1, 8); break;
            case 16: H2SP_QR_REG(1, 16); break;
            case 24: H2SP_QR_REG(1, 24); break;
            default: H2SP_QR_REG(1, 32); break;
          }
        } else {
          switch (kp) {
            case 8: H2SP_QR_REG(2, 8); break;
            case 16: H2SP_QR_REG(2, 16); break;
            case 24: H2SP_QR_REG(2, 24); break;
            default: H2SP_QR_REG(2, 32); break;
          }
        }
#undef H2SP_QR_REG
        H2SP_CK(cudaGetLastError());
        return H2SP_OK;
      }
      const int wpb = std::max(1, std::min(4, int((96 * 1024) / (size_t(per_warp) * 8))));
      qr_kernel<<<unsigned((M + wpb - 1) / wpb), 32 * wpb, size_t(per_warp) * 8 * wpb, s>>>(
          sd, L, k, M, per_warp, leaf, tr, rh, qo, magic_ptr, P->magic, wyo, P->wy_kp, P->wy_n);
      H2SP_CK(cudaGetLastError());
      return H2SP_OK;
    };
    if (lp.np_row > 0) {
      if (h2sp_status e = pre(s, li[k].qr_row)) return e;
      if (!qr_reuse)
        if (h2sp_status e = launch(rs_qr, P->n_row, P->k_row, in->leaf_basis_row, in->transfer_row, rh_row, out->q_row,
                                   k == 0 ? (const uint64_t *)meta : nullptr, k == 0 ? wy_row : nullptr))
          return e;
      if (h2sp_status e = post(s, li[k].qr_row)) return e;
    }
    if (!sym && lp.np_col > 0) {
      if (h2sp_status e = pre(s, li[k].qr_col)) return e;
      if (!qr_reuse)
        if (h2sp_status e = launch(cs_qr, P->n_col, P->k_col, leaf_col, tr_col, rh_col, q_col, nullptr,
                                   k == 0 ? wy_col : nullptr))
          return e;
      if (h2sp_status e = post(s, li[k].qr_col)) return e;
    }
    return H2SP_OK;
  };
  // matrix-free close blocks / couplings (h2sp_close_gen)
  CloseGen cgen{};
  if (in->close_gen) {
    cgen.pts = in->close_gen->points;
    cgen.dim = in->close_gen->dim;
    cgen.kind = in->close_gen->kernel;
    cgen.p0 = in->close_gen->p0;
    cgen.p1 = in->close_gen->p1;
    cgen.q0 = cgen.kind == H2SP_KERNEL_EXP ? -1.0 / cgen.p0 : 1.0 / (4.0 * 3.141592653589793);
    if (!in->coupling) {
      cgen.nodes_row = in->close_gen->nodes_row;
      cgen.nodes_col = sym ? in->close_gen->nodes_row : in->close_gen->nodes_col;
    }
  }
  const bool coup_gen = cgen.nodes_row != nullptr;
  auto coupling = [&](int k, cudaStream_t s) -> h2sp_status {
    const LevelPlan &lp = P->levels[k];
    if (!lp.n_coup) return H2SP_OK;
    int kmax = 0;
    for (int64_t i = 0; i < (int64_t(1) << (L - k)); i++)
      kmax = std::max(kmax, std::max(P->k_row[lvl_off_d(L, k) + i], P->k_col[lvl_off_d(L, k) + i]));
    if (h2sp_status e = pre(s, li[k].coup)) return e;
    const CouplingItem *items = (const CouplingItem *)(meta + lp.coup_off);
    static const bool coup_smem = [] {  // H2SP_COUPLING_SMEM=1: the shared-memory kernel at every rank
      const char *e = getenv("H2SP_COUPLING_SMEM");
      return e && e[0] == '1';
    }();
    if (coup_gen && !(kmax <= 32 && !coup_smem))
      return fail(H2SP_EUNSUPPORTED, "matrix-free couplings need ranks <= 32");
    if (kmax <= 32 && !coup_smem) {
      const unsigned grid = unsigned((lp.n_coup + 3) / 4);
      switch ((kmax + 7) / 8) {
        case 0:
        case 1:
          if (coup_gen) coupling_reg_kernel<8, true><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, nullptr, dt, cgen);
          else coupling_reg_kernel<8, false><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, in->coupling, dt, cgen);
          break;
        case 2:
          if (coup_gen) coupling_reg_kernel<16, true><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, nullptr, dt, cgen);
          else coupling_reg_kernel<16, false><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, in->coupling, dt, cgen);
          break;
        case 3:
          if (coup_gen) coupling_reg_kernel<24, true><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, nullptr, dt, cgen);
          else coupling_reg_kernel<24, false><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, in->coupling, dt, cgen);
          break;
        default:
          if (coup_gen) coupling_reg_kernel<32, true><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, nullptr, dt, cgen);
          else coupling_reg_kernel<32, false><<<grid, 128, 0, s>>>(items, lp.n_coup, rs, cs, rh_row, rh_col, in->coupling, dt, cgen);
          break;
      }
    } else {
      const int per_warp = coup_warp_doubles(kmax, kmax);
      const int ipc = std::max(1, std::min(4, int((96 * 1024) / (size_t(per_warp) * 8))));
      coupling_kernel<<<unsigned((lp.n_coup + ipc - 1) / ipc), 32 * ipc, size_t(per_warp) * 8 * ipc, s>>>(
          items, lp.n_coup, per_warp, rs, cs, rh_row, rh_col, in->coupling, dt);
    }
    H2SP_CK(cudaGetLastError());
    return post(s, li[k].coup);
  };

  // ---- CSR index expansion on s2 (independent of all values): a pure HBM write
  //      stream at the lowest priority, started with the build by default
  //      (H2SP_CSR_AT below).
#ifdef H2SP_TIMING_KNOBS
  // attribution builds only (-DH2SP_TIMING_KNOBS): skip the index expansion
  static const bool no_csr = [] {
    const char *e = getenv("H2SP_NO_CSR");
    return e && e[0] == '1';
  }();
#else
  constexpr bool no_csr = false;
#endif
  const bool bench = P->bench != 0;
  auto csr = [&]() -> h2sp_status {
    if (csr_idx >= 0 && !no_csr && !bench) {
      if (h2sp_status e = pre(s2, csr_idx)) return e;
      if (out->s_rowptr)
        H2SP_CK(cudaMemcpyAsync(out->s_rowptr, meta + P->rowptr_off, size_t(P->n_rows_local + 1) * sizeof(int64_t),
                                cudaMemcpyDeviceToDevice, s2));
      if (out->s_col) {
        const int splits = 4;
        static const int64_t grid_cap = getenv("H2SP_CSR_GRID") ? atoll(getenv("H2SP_CSR_GRID")) : 0;
        const int64_t nwork = P->n_csr_rows * splits;
        const int64_t grid = grid_cap > 0 ? std::min(grid_cap, nwork) : nwork;
        csr_cols_kernel<<<unsigned(grid), 256, 0, s2>>>((const CsrBlockRow *)(meta + P->csr_rows_off),
                                                        (const int32_t *)(meta + P->csr_pat_off), out->s_col, splits,
                                                        nwork);
        H2SP_CK(cudaGetLastError());
      }
      if (h2sp_status e = post(s2, csr_idx)) return e;
    } else if (out->s_rowptr) {
      H2SP_CK(cudaMemcpyAsync(out->s_rowptr, meta + P->rowptr_off, size_t(P->n_rows_local + 1) * sizeof(int64_t),
                              cudaMemcpyDeviceToDevice, s2));
    }
    H2SP_CK(cudaEventRecord(ev_csr, s2));
    return H2SP_OK;
  };
  // CSR expansion start (H2SP_CSR_AT, scheduling experiments): 0 (default) at the
  // start of the build, overlapping the latency-bound QR0 and the level-0
  // congruence; 1 after QR0; 2 after the level-0 congruence (upper-level gaps)
  static const int csr_at = [] {
    const char *e = getenv("H2SP_CSR_AT");
    return e ? atoi(e) : 0;
  }();
  static const int csr_level = [] {  // H2SP_CSR_AT=2: after the congruence of this level
    const char *e = getenv("H2SP_CSR_LEVEL");
    return e ? atoi(e) : 0;
  }();
  if (csr_at == 0) {
    if (!serial) H2SP_CK(cudaStreamWaitEvent(s2, ev_begin, 0));
    if (h2sp_status e = csr()) return e;
  }
  // ---- step (i) at level 0 on the main stream; the rest of the QR chain and
  //      all couplings on s1, overlapping the level-0 congruence
  if (h2sp_status e = qr(0, st)) return e;
  H2SP_CK(cudaEventRecord(ev_qr0, st));
  if (csr_at == 1) {
    H2SP_CK(cudaStreamWaitEvent(s2, ev_qr0, 0));
    if (h2sp_status e = csr()) return e;
  }
  (void)ev_fork;
  H2SP_CK(cudaStreamWaitEvent(s1, ev_qr0, 0));
  for (int k = 0; k <= L; k++) {
    if (k < L) {
      if (h2sp_status e = coupling(k, s1)) return e;
      if (h2sp_status e = qr(k + 1, s1)) return e;
      H2SP_CK(cudaEventRecord(ev_ready(k + 1), s1));
    }
  }
  // ---- level-0 Q from V / M (compact-WY path): only an output and an input of
  //      the applies.  It needs only QR0, so it runs on its own stream (s7, the
  //      QR chain's priority) right after QR0; the applies on s1 wait for it.
  //      (Trailing the chain on s1 it delayed the applies -- on the step's
  //      critical path -- by its own duration; first on s1 it delayed the chain.)
  if (P->wy_kp) {
    cudaEvent_t ev_qform = aux->ev[13 + 3 * L];
    H2SP_CK(cudaStreamWaitEvent(s7, ev_qr0, 0));
    if (h2sp_status e = pre(s7, qform_idx)) return e;
    const int64_t nleaf = int64_t(1) << L;
    const unsigned grid = unsigned(nleaf * (sym ? 1 : 2));
    if (qr_reuse) {
      // Q is already there
    } else if (P->wy_n == 128) {
      if (P->wy_kp == 16)
        { if (h2sp_status e = launch_wy_form_q<16, 128>(grid, s7, rs_qr, cs_qr, wy_row, wy_col, out->q_row, q_col, nleaf)) return e; }
      else
        { if (h2sp_status e = launch_wy_form_q<32, 128>(grid, s7, rs_qr, cs_qr, wy_row, wy_col, out->q_row, q_col, nleaf)) return e; }
    } else if (P->wy_kp == 16) {
      { if (h2sp_status e = launch_wy_form_q<16, 64>(grid, s7, rs_qr, cs_qr, wy_row, wy_col, out->q_row, q_col, nleaf)) return e; }
    } else {
      { if (h2sp_status e = launch_wy_form_q<24, 64>(grid, s7, rs_qr, cs_qr, wy_row, wy_col, out->q_row, q_col, nleaf)) return e; }
    }
    H2SP_CK(cudaGetLastError());
    if (h2sp_status e = post(s7, qform_idx)) return e;
    H2SP_CK(cudaEventRecord(ev_qform, s7));
    H2SP_CK(cudaStreamWaitEvent(s1, ev_qform, 0));
  }
  // ---- the applies of the same pass (need Q only): on s1 after the QR chain
  cudaEvent_t ev_apply = aux->ev[8 + 2 * L];
  if (ap) {
    unsigned char *aws = ap_scratch;  // the applies' own scratch; the work lists are the build's
    // V w with w independent of U^T b's output: on s7 beside U^T b (both need
    // only Q; V w uses neither the coefficient buffer nor the arrival counters)
    // ... only when the four vectors' byte ranges are pairwise disjoint (x may
    // alias b, w may be y: then V w runs after U^T b on s1, in order)
    auto range = [&](const void *p, int64_t ld, int64_t rows) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(p);
      return std::make_pair(a, a + uintptr_t((ld * (ap->nrhs - 1) + rows) * 8));
    };
    const int64_t ntree = P->n_leaves_local * P->B;
    bool disjoint = ap->w && ap->b && ap->x && ap->y;
    if (disjoint) {
      const std::pair<uintptr_t, uintptr_t> r[4] = {range(ap->b, ap->ldb, ntree), range(ap->y, ap->ldy, P->n_rows_local),
                                                    range(ap->w, ap->ldw, P->n_cols_local), range(ap->x, ap->ldx, ntree)};
      for (int i = 0; i < 4; i++)
        for (int j = i + 1; j < 4; j++)
          if (r[i].first < r[j].second && r[j].first < r[i].second) disjoint = false;
    }
    const bool v_beside = disjoint && s7 != s1;
    cudaEvent_t ev_chain = aux->ev[14 + 3 * L], ev_v = aux->ev[15 + 3 * L];
    if (v_beside) {
      H2SP_CK(cudaEventRecord(ev_chain, s1));
      H2SP_CK(cudaStreamWaitEvent(s7, ev_chain, 0));
      if (h2sp_status e = launch_apply_V(P, sym ? out->q_row : q_col, ap->w, ap->ldw, ap->x, ap->ldx, ap->nrhs, meta,
                                         aws, s7, !sym))
        return e;
      H2SP_CK(cudaEventRecord(ev_v, s7));
    }
    if (ap->b) {
      if (h2sp_status e = launch_apply_Ut(P, out->q_row, ap->b, ap->ldb, ap->y, ap->ldy, ap->nrhs, meta, aws, s1, false))
        return e;
    }
    if (v_beside) {
      H2SP_CK(cudaStreamWaitEvent(s1, ev_v, 0));
    } else if (ap->w) {
      if (h2sp_status e = launch_apply_V(P, sym ? out->q_row : q_col, ap->w, ap->ldw, ap->x, ap->ldx, ap->nrhs, meta,
                                         aws, s1, !sym))
        return e;
    }
  }
  // everything on s1 (QR chain, level-0 Q formation, applies) joins through ev_apply
  H2SP_CK(cudaEventRecord(ev_apply, s1));
  for (int k = 0; k <= L; k++) {
    const LevelPlan &lp = P->levels[k];
    if (k > 0) H2SP_CK(cudaStreamWaitEvent(st, ev_ready(k), 0));
    // ---- merge + congruence + freeze
    if (lp.n_pairs) {
      PairArgs a;
      a.items = (const PairItem *)(meta + lp.pairs_off);
      a.chunks = (const Chunk *)(meta + lp.pair_chunks_off);
      a.rs = rs;
      a.cs = cs;
      a.L = L;
      a.level = k;
      a.B = P->B;
      a.sym = P->sym;
      a.close = in->close;
      a.gen = cgen;
      a.bb_in = bb;
      a.dt_in = dt;
      a.q_row = out->q_row;
      a.q_col = q_col;
      a.s_val = out->s_val;
      a.bb_out = bb;
      a.yr = yr;
      a.yc = yc;
#ifdef H2SP_TIMING_KNOBS
      // attribution builds only (-DH2SP_TIMING_KNOBS): 1 = skip the scatter, 2 = skip the loads
      static const int pair_debug = [] {
        const char *e = getenv("H2SP_PAIR_DEBUG");
        return e ? atoi(e) : 0;
      }();
      a.debug = pair_debug;
#else
      a.debug = 0;
#endif
      a.bw = out->bench_w;
      a.part = bench ? (double2 *)reg(P->ws_part) : nullptr;
      if (h2sp_status e = pre(st, li[k].pairs)) return e;
      // level 0 may run as two launches (first / second half of the leaves), with
      // ev_pairs_a recorded in between for the first half's strips
      const int64_t split = k == 0 ? lp.pair_split : 0;
      for (int part = 0; part < (split ? 2 : 1); part++) {
        PairArgs ap_ = a;
        int64_t nch = lp.n_pair_chunks;
        if (split) {
          ap_.chunks = a.chunks + (part ? split : 0);
          nch = part ? lp.n_pair_chunks - split : split;
        }
        h2sp_status s;
        if (k == 0 && P->wy_kp && P->wy_n == 128) {
          s = P->wy_kp == 16 ? launch_pairs_wy128<16>(ap_, wy_row, wy_col, nch, st, bench)
                             : launch_pairs_wy128<32>(ap_, wy_row, wy_col, nch, st, bench);
        } else if (k == 0 && P->wy_kp) {
          s = P->wy_kp == 16 ? launch_pairs_wy<16>(ap_, wy_row, wy_col, nch, st, bench)
                             : launch_pairs_wy<24>(ap_, wy_row, wy_col, nch, st, bench);
        } else switch (pad16(lp.np_pair)) {
          case 16: s = launch_pairs<16>(ap_, nch, st, bench); break;
          case 32: s = launch_pairs<32>(ap_, nch, st, bench); break;
          case 48: s = launch_pairs<48>(ap_, nch, st, bench); break;
          default: s = launch_pairs<64>(ap_, nch, st, bench); break;
        }
        if (s != H2SP_OK) return s;
        if (split && part == 0) H2SP_CK(cudaEventRecord(ev_pairs_a, st));
      }
      if (h2sp_status e = post(st, li[k].pairs)) return e;
    }
    // ---- strips arriving from level k-1.  Set 0 (groups born at level 0) on s3:
    //      it needs only the level-0 congruence and Q_k, so it runs concurrently
    //      with the whole upper-level congruence chain.  Set 1 (born at a level
    //      >= 1) on s4: it needs the level-(k-1) congruence (its new strips).
    H2SP_CK(cudaEventRecord(ev_pairs(k), st));
    if (k == std::min(csr_level, L) && csr_at == 2) {
      H2SP_CK(cudaStreamWaitEvent(s2, ev_pairs(k), 0));
      if (h2sp_status e = csr()) return e;
    }
    for (int set = 0; set < 2; set++) {
      const LevelPlan::StripSet &sp = lp.sp[set];
      // set 0 with a split: first half on s3 (needs only the first half of the
      // level-0 pairs), second half + column strips on s5; unsplit set 0 on s5
      // too when level 0 was split (its panels may mix both halves)
      const bool split0 = set == 0 && P->levels[0].pair_split > 0;
      cudaStream_t ss = set == 0 ? (split0 ? s5 : s3) : s4;
      if (sp.n_rtiles || sp.n_ctiles) {
        H2SP_CK(cudaStreamWaitEvent(ss, ev_pairs(set == 0 ? 0 : k - 1), 0));
        H2SP_CK(cudaStreamWaitEvent(ss, ev_ready(k), 0));
        if (split0 && a_recorded) H2SP_CK(cudaStreamWaitEvent(ss, ev_a_last, 0));  // children in the first half
      }
      if (sp.n_rtiles) {
        StripArgs a;
        a.tiles = (const StripTileX *)(meta + sp.rtiles_off);
        a.groups = (const StripGroup *)(meta + sp.rgroups_off);
        a.L = L;
        a.level = k;
        a.q = out->q_row;
        a.y_in = yr;
        a.y_out = yr;
        a.s_val = out->s_val;
        a.bw = out->bench_w;
        a.part = bench ? (double2 *)reg(P->ws_part) : nullptr;
        a.aligned = P->strip_aligned;
        const int64_t na = sp.n_rtiles_a;
        if (na > 0) {
          H2SP_CK(cudaStreamWaitEvent(s3, ev_pairs_a, 0));
          H2SP_CK(cudaStreamWaitEvent(s3, ev_ready(k), 0));
          if (h2sp_status e = pre(s3, li[k].rstr[set])) return e;
          if (h2sp_status e = launch_strips(a, lp.np_rstrip, lp.mp, na, s3, bench)) return e;
          if (h2sp_status e = post(s3, li[k].rstr[set])) return e;
          H2SP_CK(cudaEventRecord(ev_a_last, s3));
          a_recorded = true;
          StripArgs b = a;
          b.tiles = a.tiles + na;
          if (h2sp_status e = pre(ss, li[k].rstr_b)) return e;
          if (h2sp_status e = launch_strips(b, lp.np_rstrip, lp.mp, sp.n_rtiles - na, ss, bench)) return e;
          if (h2sp_status e = post(ss, li[k].rstr_b)) return e;
        } else {
          if (h2sp_status e = pre(ss, li[k].rstr[set])) return e;
          h2sp_status s = launch_strips(a, lp.np_rstrip, lp.mp, sp.n_rtiles, ss, bench);
          if (s != H2SP_OK) return s;
          if (h2sp_status e = post(ss, li[k].rstr[set])) return e;
        }
      }
      if (sp.n_ctiles) {
        StripArgs a;
        a.tiles = (const StripTileX *)(meta + sp.ctiles_off);
        a.groups = (const StripGroup *)(meta + sp.cgroups_off);
        a.L = L;
        a.level = k;
        a.q = q_col;
        a.y_in = yc;
        a.y_out = yc;
        a.s_val = out->s_val;
        a.bw = out->bench_w;
        a.part = bench ? (double2 *)reg(P->ws_part) : nullptr;
        a.aligned = P->strip_aligned;
        if (h2sp_status e = pre(ss, li[k].cstr[set])) return e;
        h2sp_status s = launch_strips(a, lp.np_cstrip, lp.mp, sp.n_ctiles, ss, bench);
        if (s != H2SP_OK) return s;
        if (h2sp_status e = post(ss, li[k].cstr[set])) return e;
      }
    }
  }
  H2SP_CK(cudaEventRecord(ev_strips_done, s3));
  H2SP_CK(cudaEventRecord(ev_s5_done, s5));
  cudaEvent_t ev_strips1_done = aux->ev[9 + 2 * L];
  H2SP_CK(cudaEventRecord(ev_strips1_done, s4));
  // ---- join
  if (L > 0) H2SP_CK(cudaStreamWaitEvent(st, ev_ready(L), 0));
  H2SP_CK(cudaStreamWaitEvent(st, ev_apply, 0));
  H2SP_CK(cudaStreamWaitEvent(st, ev_csr, 0));
  H2SP_CK(cudaStreamWaitEvent(st, ev_strips_done, 0));
  H2SP_CK(cudaStreamWaitEvent(st, ev_s5_done, 0));
  H2SP_CK(cudaStreamWaitEvent(st, ev_strips1_done, 0));
  // ---- bench mode: every S block has left its partials; sum them per row
  if (bench && P->n_csr_rows) {
    if (h2sp_status e = pre(st, csr_idx)) return e;
    bench_reduce_kernel<<<unsigned(P->n_csr_rows), 256, 0, st>>>((const CsrBlockRow *)(meta + P->csr_rows_off),
                                                                 (const double2 *)reg(P->ws_part), out->bench_y,
                                                                 out->bench_r2);
    H2SP_CK(cudaGetLastError());
    if (h2sp_status e = post(st, csr_idx)) return e;
  }
  if (st != user_st) {
    H2SP_CK(cudaEventRecord(ev_end, st));
    H2SP_CK(cudaStreamWaitEvent(user_st, ev_end, 0));
  }
  if (launches) *launches = nl;
  return H2SP_OK;
}

// h2sp_build_host: the CSR index arrays depend on the plan only, so they are
// expanded and read back to the host on a side stream that starts with the call,
// overlapping the host-to-device copies of the inputs and the build; the caller
// joins through launch_csr_early_join after its own work.
h2sp_status launch_csr_early(const h2sp_plan_s *P, unsigned char *ws, int64_t *d_rowptr, int32_t *d_col,
                             int64_t *h_rowptr, int32_t *h_col, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  DeviceAux *aux = nullptr;
  if (h2sp_status e = get_aux(P->L, &aux)) return e;
  cudaStream_t s = aux->side[6];
  const unsigned char *meta = ws;
  H2SP_CK(cudaEventRecord(aux->host_fork, st));
  H2SP_CK(cudaStreamWaitEvent(s, aux->host_fork, 0));
  const size_t rp_bytes = size_t(P->n_rows_local + 1) * sizeof(int64_t);
  if (d_rowptr) H2SP_CK(cudaMemcpyAsync(d_rowptr, meta + P->rowptr_off, rp_bytes, cudaMemcpyDeviceToDevice, s));
  if (d_col && P->n_csr_rows) {
    const int splits = 4;
    const int64_t nwork = P->n_csr_rows * splits;
    csr_cols_kernel<<<unsigned(nwork), 256, 0, s>>>((const CsrBlockRow *)(meta + P->csr_rows_off),
                                                    (const int32_t *)(meta + P->csr_pat_off), d_col, splits, nwork);
    H2SP_CK(cudaGetLastError());
  }
  if (h_col && d_col) H2SP_CK(cudaMemcpyAsync(h_col, d_col, size_t(P->s_nnz) * 4, cudaMemcpyDeviceToHost, s));
  if (h_rowptr && d_rowptr) H2SP_CK(cudaMemcpyAsync(h_rowptr, d_rowptr, rp_bytes, cudaMemcpyDeviceToHost, s));
  H2SP_CK(cudaEventRecord(aux->host_join, s));
  return H2SP_OK;
}

h2sp_status launch_csr_early_join(const h2sp_plan_s *P, void *stream) {
  DeviceAux *aux = nullptr;
  if (h2sp_status e = get_aux(P->L, &aux)) return e;
  H2SP_CK(cudaStreamWaitEvent((cudaStream_t)stream, aux->host_join, 0));
  return H2SP_OK;
}

h2sp_status launch_apply_Ut(const h2sp_plan_s *P, const double *q, const double *b, int64_t ldb, double *y,
                            int64_t ldy, int nrhs, const unsigned char *meta, unsigned char *scratch, void *stream,
                            bool col_side) {
  cudaStream_t st = (cudaStream_t)stream;
  const Clusters cl = make_clusters(P, meta);
  const Side sd = side_of(cl, col_side);
  double *zb = (double *)scratch;
  const int64_t zbl = col_side ? P->zb_col_len : P->zb_row_len;
  int *arrive = (int *)(scratch + ((size_t(std::max(P->zb_row_len, P->zb_col_len)) * nrhs * 8 + 255) / 256) * 256);
  H2SP_CK(cudaMemsetAsync(arrive, 0, size_t(P->ncl) * sizeof(int), st));
  if (nrhs == 1)
    apply_ut_kernel<1><<<unsigned(P->n_leaves_local), 128, 0, st>>>(sd, P->L, q, b, ldb, y, ldy, zb, zbl, nrhs, P->B,
                                                                    arrive, P->first_leaf);
  else
    apply_ut_kernel<8><<<unsigned(P->n_leaves_local), 128, 0, st>>>(sd, P->L, q, b, ldb, y, ldy, zb, zbl, nrhs, P->B,
                                                                    arrive, P->first_leaf);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}

h2sp_status launch_apply_V(const h2sp_plan_s *P, const double *q, const double *y, int64_t ldy, double *x,
                           int64_t ldx, int nrhs, const unsigned char *meta, unsigned char *scratch, void *stream,
                           bool col_side) {
  cudaStream_t st = (cudaStream_t)stream;
  const Clusters cl = make_clusters(P, meta);
  const Side sd = side_of(cl, col_side);
  // the downward pass's own half of the apply scratch (U^T b may run beside it):
  // basis coefficients | cluster flags + ticket
  const size_t zbytes = (size_t(std::max(P->zb_row_len, P->zb_col_len)) * nrhs * 8 + 255) / 256 * 256;
  const size_t abytes = (size_t(P->ncl) * 4 + 255) / 256 * 256;
  double *zb = (double *)(scratch + zbytes + abytes);
  const int64_t zbl = col_side ? P->zb_col_len : P->zb_row_len;
  int *flags = (int *)(scratch + zbytes + abytes + zbytes);
  H2SP_CK(cudaMemsetAsync(flags, 0, (size_t(P->ncl) + 1) * sizeof(int), st));
  // one CTA per cluster of the shard's tree: levels L .. 0, max(1, n_leaves_local >> level) each
  int64_t nunits = 0;
  for (int lv = 0; lv <= P->L; lv++) nunits += std::max<int64_t>(1, P->n_leaves_local >> lv);
  if (nrhs == 1)
    apply_v_kernel<1><<<unsigned(nunits), 256, 0, st>>>(sd, P->L, q, y, ldy, x, ldx, zb, zbl, nrhs, P->B, flags, P->ncl,
                                                        P->first_leaf, P->n_leaves_local);
  else
    apply_v_kernel<8><<<unsigned(nunits), 256, 0, st>>>(sd, P->L, q, y, ldy, x, ldx, zb, zbl, nrhs, P->B, flags, P->ncl,
                                                        P->first_leaf, P->n_leaves_local);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}



// --------------------------------------------------------------------------
// GPU H^2 construction (the input side of the path):
// nested bases by tensor Chebyshev interpolation on each cluster's box -- the
// recipe of the synthetic inputs evaluated where the build
// consumes it.  Per cluster of rank k = prod(p_a) > 0:
//   box padded by max(1e-9 ext, 1e-12) per axis; orders p_a = the base orders
//   assigned to the axes by decreasing extent (stable);
//   axis nodes  mid + half * c_j (c_j = the host's cosine table; p = 1: mid);
//   nodes       tensor grid, axis 0 slowest;
//   basis(x)[j] = prod_a l_{j_a}(x_a), l_j(x) = prod_{m != j} (x - n_m) / (n_j - n_m)
//               multiplied in the order m = 0.., axes 0..d-1;
//   leaf R_t = basis_t(points of t), transfer rows of child c = basis_p(nodes_c).
// Every operation is an explicitly rounded IEEE op (no contraction), so the
// arrays equal the numpy generator's bit for bit.
// --------------------------------------------------------------------------
struct ChebArgs {
  int dim, ords[3];
  double cosv[9][8];            // cosv[p][j], p = 1..8
  const double *lo, *hi;        // tight cluster boxes, n_clusters x dim
};

struct ChebBox {
  int p[3];
  double nodes[3][8];
};

__device__ __forceinline__ ChebBox cheb_box(const ChebArgs &A, int64_t c) {
  ChebBox b;
  double lo[3], hi[3], ext[3];
  for (int a = 0; a < 3; a++) {
    lo[a] = hi[a] = ext[a] = 0.0;
    b.p[a] = 1;
  }
  for (int a = 0; a < A.dim; a++) {
    const double l = A.lo[c * A.dim + a], h = A.hi[c * A.dim + a];
    ext[a] = __dsub_rn(h, l);
    const double pad = fmax(__dmul_rn(ext[a], 1e-9), 1e-12);
    lo[a] = __dsub_rn(l, pad);
    hi[a] = __dadd_rn(h, pad);
  }
  // axes by decreasing extent, stable (argsort of -ext)
  int order[3] = {0, 1, 2};
  for (int i = 1; i < A.dim; i++)
    for (int j = i; j > 0 && ext[order[j]] > ext[order[j - 1]]; j--) {
      const int t = order[j];
      order[j] = order[j - 1];
      order[j - 1] = t;
    }
  for (int i = 0; i < A.dim; i++) b.p[order[i]] = A.ords[i];
  for (int a = 0; a < A.dim; a++) {
    const int p = b.p[a];
    const double mid = __ddiv_rn(__dadd_rn(lo[a], hi[a]), 2.0);
    const double half = __ddiv_rn(__dsub_rn(hi[a], lo[a]), 2.0);
    for (int j = 0; j < 8; j++) b.nodes[a][j] = (j < p) ? (p == 1 ? mid : __dadd_rn(mid, __dmul_rn(half, A.cosv[p][j]))) : 0.0;
  }
  return b;
}

// Lagrange polynomial j of the p nodes of axis a at x: prod_{m != j} (x - n_m) / (n_j - n_m),
// multiplied in the order m = 0, 1, ... (the generator's order)
__device__ __forceinline__ double cheb_lagrange(const ChebBox &b, int a, int j, double x) {
  double v = 1.0;
#pragma unroll
  for (int m = 0; m < 8; m++)
    if (m < b.p[a] && m != j) v = __dmul_rn(v, __ddiv_rn(__dsub_rn(x, b.nodes[a][m]), __dsub_rn(b.nodes[a][j], b.nodes[a][m])));
  return v;
}

// basis function jj (axis-0-slowest multi-index) of box b at the point (x0, x1, x2):
// ((l_0 * l_1) * l_2) as the generator's reshaped outer products
__device__ __forceinline__ double cheb_basis_fn(const ChebBox &b, int dim, int jj, double x0, double x1, double x2) {
  const int p1 = dim > 1 ? b.p[1] : 1, p2 = dim > 2 ? b.p[2] : 1;
  const int j0 = jj / (p1 * p2), j1 = (jj / p2) % p1, j2 = jj % p2;
  double v = cheb_lagrange(b, 0, j0, x0);
  if (dim > 1) v = __dmul_rn(v, cheb_lagrange(b, 1, j1, x1));
  if (dim > 2) v = __dmul_rn(v, cheb_lagrange(b, 2, j2, x2));
  return v;
}

// one thread per (cluster, node): the node coordinates
__global__ void __launch_bounds__(256) cheb_nodes_kernel(ChebArgs A, Side sd, int64_t ncl, int r, double *__restrict__ nodes) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= ncl * r) return;
  const int64_t c = t / r;
  const int j = int(t - c * r);
  if (sd.k[c] == 0) return;
  const ChebBox b = cheb_box(A, c);
  const int p1 = A.dim > 1 ? b.p[1] : 1, p2 = A.dim > 2 ? b.p[2] : 1;
  const int j0 = j / (p1 * p2), j1 = (j / p2) % p1, j2 = j % p2;
  double *o = nodes + (sd.zb_off[c] + j) * A.dim;
  o[0] = b.nodes[0][j0];
  if (A.dim > 1) o[1] = b.nodes[1][j1];
  if (A.dim > 2) o[2] = b.nodes[2][j2];
}

// one thread per (leaf, point): row i of R_t
__global__ void __launch_bounds__(128) cheb_leaf_kernel(ChebArgs A, Side sd, int64_t nleaf, int B,
                                                        const double *__restrict__ pts, double *__restrict__ leaf) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nleaf * B) return;
  const int64_t c = t / B;
  const int i = int(t - c * B);
  const int k = sd.k[c];
  if (k == 0) return;
  const ChebBox b = cheb_box(A, c);
  const double *xp = pts + t * A.dim;
  const double x0 = xp[0], x1 = A.dim > 1 ? xp[1] : 0.0, x2 = A.dim > 2 ? xp[2] : 0.0;
  double *o = leaf + sd.leaf_off[c] + int64_t(i) * k;
  for (int j = 0; j < k; j++) o[j] = cheb_basis_fn(b, A.dim, j, x0, x1, x2);
}

// one thread per (internal cluster p, row of T_p): row i is child c's node
// i (child 1 first) under p's basis; zero rows when p has rank 0 handled by
// the k == 0 exit (T_p has no columns then)
__global__ void __launch_bounds__(128) cheb_transfer_kernel(ChebArgs A, Side sd, int L, int64_t nint, int rmax,
                                                            const double *__restrict__ nodes, double *__restrict__ tr) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nint * 2 * rmax) return;
  const int64_t pi = t / (2 * rmax);           // internal cluster index (level-major, after the leaves)
  const int i = int(t - pi * 2 * rmax);        // row of T_p (< k_c1 + k_c2)
  const int64_t p = (int64_t(1) << L) + pi;
  const int kp = sd.k[p], n = sd.n[p];
  if (kp == 0 || i >= n) return;
  int k_ = 0;  // level of p
  while (p >= lvl_off_d(L, k_ + 1)) k_++;
  const int64_t c1 = lvl_off_d(L, k_ - 1) + 2 * (p - lvl_off_d(L, k_));
  const int k1 = sd.k[c1];
  const int64_t c = i < k1 ? c1 : c1 + 1;
  const int ii = i < k1 ? i : i - k1;
  const ChebBox b = cheb_box(A, p);
  const double *xp = nodes + (sd.zb_off[c] + ii) * A.dim;
  const double x0 = xp[0], x1 = A.dim > 1 ? xp[1] : 0.0, x2 = A.dim > 2 ? xp[2] : 0.0;
  double *o = tr + sd.tr_off[p] + int64_t(i) * kp;
  for (int j = 0; j < kp; j++) o[j] = cheb_basis_fn(b, A.dim, j, x0, x1, x2);
}

h2sp_status launch_cheb_construct(const h2sp_plan_s *P, const unsigned char *meta, int side, const h2sp_cheb_spec *s,
                                  const double *points, const double *box_lo, const double *box_hi, double *leaf,
                                  double *transfer, double *nodes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const Clusters cl = make_clusters(P, meta);
  const Side sd = side_of(cl, side != 0);
  ChebArgs A{};
  A.dim = s->dim;
  for (int a = 0; a < 3; a++) A.ords[a] = a < s->dim ? s->orders[a] : 1;
  for (int p = 0; p <= 8; p++)
    for (int j = 0; j < 8; j++) A.cosv[p][j] = (p >= 1 && j < p) ? s->cheb_cos[(p - 1) * 8 + j] : 0.0;
  A.lo = box_lo;
  A.hi = box_hi;
  int r = 1;
  for (int a = 0; a < s->dim; a++) r *= s->orders[a];
  const int64_t ncl = P->ncl, nleaf = int64_t(1) << P->L;
  cheb_nodes_kernel<<<unsigned((ncl * r + 255) / 256), 256, 0, st>>>(A, sd, ncl, r, nodes);
  H2SP_CK(cudaGetLastError());
  cheb_leaf_kernel<<<unsigned((nleaf * P->B + 127) / 128), 128, 0, st>>>(A, sd, nleaf, P->B, points, leaf);
  H2SP_CK(cudaGetLastError());
  const int64_t nint = ncl - nleaf;
  if (nint > 0) {
    cheb_transfer_kernel<<<unsigned((nint * 2 * r + 127) / 128), 128, 0, st>>>(A, sd, P->L, nint, r, nodes, transfer);
    H2SP_CK(cudaGetLastError());
  }
  return H2SP_OK;
}
}  // namespace h2sp

#ifdef H2SP_STRIP_CLOCKS
// attribution build: copy the strip phase stamps out (count returned; table reset)
extern "C" int64_t h2sp_debug_strip_clocks(void *out, int64_t max_entries) {
  unsigned n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, h2sp::g_strip_clk_n, sizeof(n));
  int64_t m = n < 16384u ? n : 16384;
  if (m > max_entries) m = max_entries;
  cudaMemcpyFromSymbol(out, h2sp::g_strip_clk, size_t(m) * sizeof(h2sp::StripClk));
  unsigned z = 0;
  cudaMemcpyToSymbol(h2sp::g_strip_clk_n, &z, sizeof(z));
  return m;
}
#endif
