// The paper's preconditioning workload on the device (SURVEY §8(f) #3,
// "Sparsification method as a preconditioner") and the direct
// solve it shares its factorisation with (§8(f) #1, x = V S^-1 U^T b):
//
//   * ilut_kernel   -- ILUT(tau, p) of S (reading 24: Saad's
//                      Algorithm 10.6 with the dual dropping rule); tau = 0,
//                      p < 0 is the complete LU (the direct solve).
//   * trsv kernels  -- (L U)^-1 b by forward / backward substitution.
//   * csr_spmv      -- S x (the H^2 matvec A x = U S U^T x of GMRES).
//   * GMRES(m)      -- right-preconditioned restarted GMRES (Saad Alg. 9.5),
//                      Arnoldi by classical Gram-Schmidt with one
//                      re-orthogonalisation (CGS2: two batched dot-product
//                      launches per step instead of j + 1 dependent ones).
//
// ILUT on a GPU.  Row i of the factor needs the U rows of every k < i its work
// row touches, so rows form a dependency DAG that follows the (evolving) fill.
// One warp factorises one row at a time; rows are handed out in increasing
// order by an atomic ticket, a row waits (acquire) on the completion flag of
// each U row it uses and publishes its own U row (release) BEFORE it selects
// and writes its L part -- the L part is off every other row's critical path.
// Tickets are taken only by running warps and a row waits only on smaller
// rows, so there is no deadlock whatever the grid size.  The work row w is a
// dense per-warp vector in HBM (touched entries only: O(row) per row) with a
// presence bitmap in shared memory, scanned with warp ballots for "the next
// k with w_k present" (new fill from U row k lands right of k, so one forward
// cursor visits every k in increasing order, as the algorithm does).
//
// Arithmetic order: every update is w_j - (w_k * u_kj) with two roundings
// (__dmul_rn / __dsub_rn: no contraction), in increasing k; the row norm is a
// sequential sum of squares in column order; the p-largest selection is exact
// (radix select on |w| bits, ties to the smaller column).  So the factors are
// bitwise those of the plain-C oracle (oracle/ilut.c) on the same input.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "h2sp_internal.h"

using namespace h2sp;

#define KCK(x)                                                                                           \
  do {                                                                                                   \
    cudaError_t e_ = (x);                                                                                \
    if (e_ != cudaSuccess) return fail(H2SP_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int32_t *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flag(const int32_t *p, int want) {
  if (ld_acquire(p) >= want) return;
  while (ld_acquire(p) < want) __nanosleep(32);
}

__device__ __forceinline__ unsigned long long dkey(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(fabs(v)));
}

// ---------------------------------------------------------------------------
// ILUT
// ---------------------------------------------------------------------------

struct IlutArgs {
  int64_t n;
  const int64_t *rp;
  const int32_t *ci;
  const double *av;
  double tau;
  int32_t p;
  int32_t nwords;  // bitmap words per warp = ceil(n / 32)
  int64_t *l_start, *u_start;
  int32_t *l_len, *u_len;
  double *diag;
  int32_t *pool_col;
  double *pool_val;
  int64_t cap;
  unsigned long long *cursor;  // pool entries reserved so far
  unsigned long long *ticket;  // next row
  int32_t *done;               // [n] 1 once U row i and u_ii are published
  int32_t *status;             // [0] bit 1 = pool overflow, bit 2 = zero pivot; [1] first zero-pivot row
  double *w;                   // [slots][n] work rows (zero between rows)
  int32_t *ccol;               // [slots][n] candidate columns
  double *cval;                // [slots][n] candidate values
};

// Next set bit in [from, lim) of the warp's bitmap, or lim.
__device__ __forceinline__ int64_t next_bit(const uint32_t *bits, int64_t from, int64_t lim, int lane) {
  if (from >= lim) return lim;
  const int64_t w0 = from >> 5, wl = (lim + 31) >> 5;
  for (int64_t base = w0; base < wl; base += 32) {
    const int64_t wi = base + lane;
    uint32_t v = 0;
    if (wi < wl) {
      v = bits[wi];
      const int64_t lo = from - (wi << 5);
      if (lo > 0) v &= ~0u << lo;
      const int64_t hi = lim - (wi << 5);
      if (hi < 32) v &= (1u << hi) - 1u;
    }
    const unsigned m = __ballot_sync(FULL, v != 0);
    if (m) {
      const int src = __ffs(m) - 1;
      const uint32_t vv = __shfl_sync(FULL, v, src);
      return ((base + src) << 5) + __ffs(vv) - 1;
    }
  }
  return lim;
}

// Compact the present entries of w in [lo, hi] (bitmap order = ascending
// column) into (ccol, cval); U part (upper = true): only entries surviving the
// tau rule; L part: every present entry (rule 1 already dropped the rest).
__device__ int64_t gather(const uint32_t *bits, const double *w, int64_t lo, int64_t hi, bool upper, double taui,
                          int32_t *ccol, double *cval, int lane) {
  int64_t cnt = 0;
  if (lo > hi) return 0;
  const int64_t w0 = lo >> 5, w1 = hi >> 5;
  for (int64_t base = w0; base <= w1; base += 32) {
    const int64_t wi = base + lane;
    uint32_t v = 0;
    if (wi <= w1) {
      v = bits[wi];
      const int64_t l = lo - (wi << 5);
      if (l > 0) v &= ~0u << l;
      const int64_t h = hi - (wi << 5);
      if (h < 31) v &= (2u << h) - 1u;
    }
    uint32_t keep = v;
    if (upper) {
      keep = 0;
      for (uint32_t t = v; t; t &= t - 1) {
        const int b = __ffs(t) - 1;
        const double x = w[(wi << 5) + b];
        if (!(fabs(x) < taui || x == 0.0)) keep |= 1u << b;
      }
    }
    const int c = __popc(keep);
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    int64_t pos = cnt + incl - c;
    for (uint32_t t = keep; t; t &= t - 1) {
      const int b = __ffs(t) - 1;
      const int64_t j = (wi << 5) + b;
      ccol[pos] = int32_t(j);
      cval[pos] = w[j];
      pos++;
    }
    cnt += __shfl_sync(FULL, incl, 31);
  }
  __syncwarp();
  return cnt;
}

// Keep the p largest |cval| of c candidates (ties: smaller column, i.e.
// earlier position), in place, column order preserved.  Returns the count.
__device__ int64_t keep_largest(int32_t *ccol, double *cval, int64_t c, int p, int *hist, int lane) {
  if (p < 0 || c <= p) return c;
  if (p == 0) return 0;
  unsigned long long prefix = 0, mask = 0;
  int64_t rem = p;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int64_t a = lane; a < c; a += 32) {
      const unsigned long long k = dkey(cval[a]);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
    }
    __syncwarp();
    // lane l owns bins 255-8l .. 248-8l (descending)
    int s = 0;
    for (int q = 0; q < 8; q++) s += hist[255 - 8 * lane - q];
    int incl = s;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned m = __ballot_sync(FULL, incl >= rem);
    const int src = __ffs(m) - 1;
    int digit = 0;
    int64_t above = 0;
    if (lane == src) {
      int64_t run = incl - s;
      for (int q = 0; q < 8; q++) {
        const int b = 255 - 8 * lane - q;
        if (run + hist[b] >= rem) {
          digit = b;
          above = run;
          break;
        }
        run += hist[b];
      }
    }
    digit = __shfl_sync(FULL, digit, src);
    above = __shfl_sync(FULL, above, src);
    rem -= above;
    prefix |= static_cast<unsigned long long>(digit) << shift;
    mask |= 255ull << shift;
    __syncwarp();
  }
  // keys > T kept; of the keys == T, the first `rem` in column order
  const unsigned long long T = prefix;
  int64_t out = 0, eq_seen = 0;
  for (int64_t base = 0; base < c; base += 32) {
    const int64_t a = base + lane;
    int32_t cc = 0;
    double vv = 0.0;
    unsigned long long k = 0;
    if (a < c) {
      cc = ccol[a];
      vv = cval[a];
      k = dkey(vv);
    }
    const unsigned lt = (1u << lane) - 1u;
    const unsigned eq = __ballot_sync(FULL, a < c && k == T);
    const bool keep = a < c && (k > T || (k == T && eq_seen + __popc(eq & lt) < rem));
    const unsigned km = __ballot_sync(FULL, keep);
    __syncwarp();
    if (keep) {
      ccol[out + __popc(km & lt)] = cc;
      cval[out + __popc(km & lt)] = vv;
    }
    out += __popc(km);
    eq_seen += __popc(eq);
    __syncwarp();
  }
  return out;
}

__device__ int64_t reserve(const IlutArgs &A, int64_t cnt, int lane) {
  unsigned long long st = 0;
  if (lane == 0 && cnt > 0) {
    st = atomicAdd(A.cursor, static_cast<unsigned long long>(cnt));
    if (int64_t(st) + cnt > A.cap) atomicOr(&A.status[0], 1);
  }
  st = __shfl_sync(FULL, st, 0);
  return int64_t(st);
}

__global__ void __launch_bounds__(256) ilut_kernel(IlutArgs A, int warps_per_cta) {
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= warps_per_cta) return;
  uint32_t *bits = smem + size_t(wid) * A.nwords;
  int *hist = reinterpret_cast<int *>(smem + size_t(warps_per_cta) * A.nwords) + 256 * wid;
  const int64_t slot = int64_t(blockIdx.x) * warps_per_cta + wid;
  double *w = A.w + slot * A.n;
  int32_t *ccol = A.ccol + slot * A.n;
  double *cval = A.cval + slot * A.n;
  for (int i = lane; i < A.nwords; i += 32) bits[i] = 0;
  __syncwarp();
  for (;;) {
    unsigned long long row = 0;
    if (lane == 0) row = atomicAdd(A.ticket, 1ull);
    const int64_t i = int64_t(__shfl_sync(FULL, row, 0));
    if (i >= A.n) break;
    const int64_t e0 = A.rp[i], e1 = A.rp[i + 1];
    // tau_i = tau * ||a_i||_2, the sum of squares in column order
    double taui = 0.0;
    if (lane == 0) {
      double s = 0.0;
      for (int64_t e = e0; e < e1; e++) s = __dadd_rn(s, __dmul_rn(A.av[e], A.av[e]));
      taui = __dmul_rn(A.tau, sqrt(s));
    }
    taui = __shfl_sync(FULL, taui, 0);
    int64_t lo = i, hi = i;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int32_t j = A.ci[e];
      w[j] = A.av[e];
      atomicOr(&bits[j >> 5], 1u << (j & 31));
      lo = min(lo, int64_t(j));
      hi = max(hi, int64_t(j));
    }
    for (int o = 16; o; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(FULL, lo, o));
      hi = max(hi, __shfl_xor_sync(FULL, hi, o));
    }
    __syncwarp();
    // for k < i with w_k present, in increasing k
    for (int64_t k = next_bit(bits, lo, i, lane); k < i; k = next_bit(bits, k + 1, i, lane)) {
      if (lane == 0) wait_flag(A.done + k, 1);
      __syncwarp();
      const double wk = __ddiv_rn(w[k], __ldcg(A.diag + k));
      if (fabs(wk) < taui || wk == 0.0) {  // rule 1
        __syncwarp();
        if (lane == 0) {
          w[k] = 0.0;
          bits[k >> 5] &= ~(1u << (k & 31));
        }
        __syncwarp();
        continue;
      }
      __syncwarp();
      if (lane == 0) w[k] = wk;
      const int64_t us = __ldcg(A.u_start + k);
      const int32_t ul = __ldcg(A.u_len + k);
      for (int32_t e = lane; e < ul; e += 32) {
        const int32_t j = __ldcg(A.pool_col + us + e);
        const double u = __ldcg(A.pool_val + us + e);
        w[j] = __dsub_rn(w[j], __dmul_rn(wk, u));
        atomicOr(&bits[j >> 5], 1u << (j & 31));
        hi = max(hi, int64_t(j));
      }
      __syncwarp();
    }
    for (int o = 16; o; o >>= 1) hi = max(hi, __shfl_xor_sync(FULL, hi, o));
    // rule 2, U part; publish U row i and u_ii first
    int64_t cu = gather(bits, w, i + 1, hi, true, taui, ccol, cval, lane);
    cu = keep_largest(ccol, cval, cu, A.p, hist, lane);
    int64_t st = reserve(A, cu, lane);
    const bool fits = st + cu <= A.cap;
    if (fits)
      for (int64_t a = lane; a < cu; a += 32) {
        A.pool_col[st + a] = ccol[a];
        A.pool_val[st + a] = cval[a];
      }
    const double uii = w[i];
    __syncwarp();
    if (lane == 0) {
      A.u_start[i] = st;
      A.u_len[i] = fits ? int32_t(cu) : 0;
      A.diag[i] = uii;
      if (uii == 0.0) {
        atomicOr(&A.status[0], 2);
        atomicMin(&A.status[1], int32_t(i));
      }
      __threadfence();
      st_release(A.done + i, 1);
    }
    // L part (kept entries of rule 1)
    int64_t cl = gather(bits, w, lo, i - 1, false, taui, ccol, cval, lane);
    cl = keep_largest(ccol, cval, cl, A.p, hist, lane);
    st = reserve(A, cl, lane);
    const bool lfits = st + cl <= A.cap;
    if (lfits)
      for (int64_t a = lane; a < cl; a += 32) {
        A.pool_col[st + a] = ccol[a];
        A.pool_val[st + a] = cval[a];
      }
    if (lane == 0) {
      A.l_start[i] = st;
      A.l_len[i] = lfits ? int32_t(cl) : 0;
    }
    // clear the touched range of w and the bitmap
    __syncwarp();
    for (int64_t wi = (lo >> 5) + lane; wi <= (hi >> 5); wi += 32) {
      for (uint32_t t = bits[wi]; t; t &= t - 1) w[(wi << 5) + __ffs(t) - 1] = 0.0;
      bits[wi] = 0;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Triangular solves: x = U^-1 L^-1 b (L unit lower), one warp per row.
// ---------------------------------------------------------------------------

struct TrsvArgs {
  int64_t n;
  const int64_t *l_start, *u_start;
  const int32_t *l_len, *u_len;
  const double *diag;
  const int32_t *pool_col;
  const double *pool_val;
  const double *b;
  double *x;
  int32_t *flag;
  unsigned long long *ticket;  // [0] forward, [1] backward
};

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__global__ void __launch_bounds__(256) trsv_lower_kernel(TrsvArgs A) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(A.ticket, 1ull);
    const int64_t i = int64_t(__shfl_sync(FULL, t, 0));
    if (i >= A.n) return;
    const int64_t s0 = A.l_start[i];
    const int32_t len = A.l_len[i];
    double acc = 0.0;
    for (int32_t e = lane; e < len; e += 32) {
      const int32_t j = A.pool_col[s0 + e];
      wait_flag(A.flag + j, 1);
      acc += A.pool_val[s0 + e] * __ldcg(A.x + j);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      A.x[i] = A.b[i] - acc;
      __threadfence();
      st_release(A.flag + i, 1);
    }
  }
}

__global__ void __launch_bounds__(256) trsv_upper_kernel(TrsvArgs A) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(A.ticket + 1, 1ull);
    const int64_t tt = int64_t(__shfl_sync(FULL, t, 0));
    if (tt >= A.n) return;
    const int64_t i = A.n - 1 - tt;
    const int64_t s0 = A.u_start[i];
    const int32_t len = A.u_len[i];
    double acc = 0.0;
    for (int32_t e = lane; e < len; e += 32) {
      const int32_t j = A.pool_col[s0 + e];
      wait_flag(A.flag + j, 2);
      acc += A.pool_val[s0 + e] * __ldcg(A.x + j);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      A.x[i] = (__ldcg(A.x + i) - acc) / A.diag[i];
      __threadfence();
      st_release(A.flag + i, 2);
    }
  }
}

// ---------------------------------------------------------------------------
// CSR SpMV and the GMRES vector kernels (fixed grids: deterministic)
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) spmv_kernel(int64_t n, const int64_t *rp, const int32_t *ci, const double *av,
                                                   const double *x, double *y) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
    double acc = 0.0;
    for (int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) acc += av[e] * __ldg(x + ci[e]);
    acc = warp_sum(acc);
    if (lane == 0) y[i] = acc;
  }
}

constexpr int DOT_BLOCKS = 296, DOT_THREADS = 256, DOT_MAXV = 8;

// part[blk * nv + v] = sum over the block's slice of V[v] . w  (nv <= DOT_MAXV per launch)
__global__ void __launch_bounds__(DOT_THREADS) dots_kernel(const double *V, int64_t ldv, int nv, const double *w,
                                                           int64_t n, double *part) {
  __shared__ double red[DOT_MAXV][DOT_THREADS / 32];
  double acc[DOT_MAXV];
#pragma unroll
  for (int v = 0; v < DOT_MAXV; v++) acc[v] = 0.0;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const double we = w[e];
#pragma unroll
    for (int v = 0; v < DOT_MAXV; v++)
      if (v < nv) acc[v] += V[v * ldv + e] * we;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < DOT_MAXV; v++) {
    const double s = warp_sum(acc[v]);
    if (lane == 0) red[v][wid] = s;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int q = 0; q < DOT_THREADS / 32; q++) s += red[threadIdx.x][q];
    part[blockIdx.x * nv + threadIdx.x] = s;
  }
}

// out[v] = (accumulate ? out[v] : 0) + sum_blk part[blk * nv + v]
__global__ void reduce_parts_kernel(const double *part, int nv, int nblk, double *out, int accumulate) {
  const int v = threadIdx.x;
  if (v >= nv) return;
  double s = 0.0;
  for (int b = 0; b < nblk; b++) s += part[b * nv + v];
  out[v] = accumulate ? out[v] + s : s;
}

// w -= sum_v V[v] * h[v]
__global__ void __launch_bounds__(256) sub_comb_kernel(const double *V, int64_t ldv, int nv, const double *h,
                                                       double *w, int64_t n) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    double s = w[e];
    for (int v = 0; v < nv; v++) s -= V[v * ldv + e] * h[v];
    w[e] = s;
  }
}

// y = sum_v V[v] * c[v] (c on the device)
__global__ void __launch_bounds__(256) comb_kernel(const double *V, int64_t ldv, int nv, const double *c, double *y,
                                                   int64_t n) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int v = 0; v < nv; v++) s += V[v * ldv + e] * c[v];
    y[e] = s;
  }
}

// y = x * (1 / *s)   (s on the device), or y = a * x + b * y with host scalars
__global__ void __launch_bounds__(256) scale_kernel(const double *x, const double *s, double *y, int64_t n) {
  const double f = 1.0 / *s;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    y[e] = x[e] * f;
}

__global__ void __launch_bounds__(256) axpby_kernel(double a, const double *x, double b, double *y, int64_t n) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    y[e] = a * x[e] + b * y[e];
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

int num_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

struct IlutCfg {
  int warps, ctas, nwords;
  size_t smem;
  int64_t slots;
};

IlutCfg ilut_cfg(int64_t n) {
  IlutCfg c{};
  c.nwords = int((n + 31) / 32);
  const size_t per_warp = size_t(c.nwords) * 4 + 256 * 4;
  c.warps = int(std::max<size_t>(1, std::min<size_t>(8, (200u << 10) / per_warp)));
  c.smem = per_warp * c.warps;
  const int per_sm = std::max(1, 8 / c.warps);
  c.ctas = num_sms() * per_sm;
  c.slots = int64_t(c.ctas) * c.warps;
  return c;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct IlutWs {
  unsigned long long *ctr;  // cursor, ticket
  int32_t *status, *done;
  double *w, *cval;
  int32_t *ccol;
  size_t bytes;
};

IlutWs ilut_carve(unsigned char *base, int64_t n, int64_t slots) {
  IlutWs s{};
  size_t off = 0;
  auto take = [&](size_t b) {
    unsigned char *p = base ? base + off : nullptr;
    off += align256(b);
    return p;
  };
  s.ctr = reinterpret_cast<unsigned long long *>(take(16));
  s.status = reinterpret_cast<int32_t *>(take(8));
  s.done = reinterpret_cast<int32_t *>(take(size_t(n) * 4));
  s.w = reinterpret_cast<double *>(take(size_t(slots) * n * 8));
  s.cval = reinterpret_cast<double *>(take(size_t(slots) * n * 8));
  s.ccol = reinterpret_cast<int32_t *>(take(size_t(slots) * n * 4));
  s.bytes = off;
  return s;
}

struct TrsvWs {
  int32_t *flag;
  unsigned long long *ticket;
  size_t bytes;
};

TrsvWs trsv_carve(unsigned char *base, int64_t n) {
  TrsvWs s{};
  s.flag = reinterpret_cast<int32_t *>(base);
  s.ticket = reinterpret_cast<unsigned long long *>(base ? base + align256(size_t(n) * 4) : nullptr);
  s.bytes = align256(size_t(n) * 4) + 256;
  return s;
}

h2sp_status check_csr(const h2sp_csr *A) {
  if (!A || A->n < 0 || (A->n > 0 && (!A->rowptr || !A->col || !A->val)))
    return fail(H2SP_EINVAL, "CSR: NULL pointer or negative size");
  if (A->n >= (int64_t(1) << 31)) return fail(H2SP_EUNSUPPORTED, "CSR: n >= 2^31 (int32 columns)");
  return H2SP_OK;
}

h2sp_status check_factors(const h2sp_ilut_factors *F, int64_t n) {
  if (!F || F->n != n || (n > 0 && (!F->l_start || !F->u_start || !F->l_len || !F->u_len || !F->diag)))
    return fail(H2SP_EINVAL, "ILUT factors: NULL pointer or size mismatch");
  return H2SP_OK;
}

h2sp_status launch_trsv(const h2sp_ilut_factors *F, const double *b, double *x, unsigned char *ws, cudaStream_t st) {
  const int64_t n = F->n;
  if (n == 0) return H2SP_OK;
  TrsvWs t = trsv_carve(ws, n);
  KCK(cudaMemsetAsync(t.flag, 0, size_t(n) * 4, st));
  KCK(cudaMemsetAsync(t.ticket, 0, 16, st));
  TrsvArgs a{n, F->l_start, F->u_start, F->l_len, F->u_len, F->diag, F->pool_col, F->pool_val, b, x, t.flag, t.ticket};
  const int grid = num_sms() * 8;
  trsv_lower_kernel<<<grid, 256, 0, st>>>(a);
  KCK(cudaGetLastError());
  trsv_upper_kernel<<<grid, 256, 0, st>>>(a);
  KCK(cudaGetLastError());
  return H2SP_OK;
}

h2sp_status launch_spmv(const h2sp_csr *A, const double *x, double *y, cudaStream_t st) {
  if (A->n == 0) return H2SP_OK;
  const int grid = int(std::min<int64_t>(num_sms() * 8, (A->n + 7) / 8));
  spmv_kernel<<<grid, 256, 0, st>>>(A->n, A->rowptr, A->col, A->val, x, y);
  KCK(cudaGetLastError());
  return H2SP_OK;
}

int vec_grid(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>(num_sms() * 4, (n + 255) / 256))); }

}  // namespace

extern "C" {

int64_t h2sp_ilut_ws_bytes(int64_t n) {
  if (n < 0) return -1;
  const IlutCfg c = ilut_cfg(std::max<int64_t>(n, 1));
  return int64_t(ilut_carve(nullptr, n, c.slots).bytes);
}

h2sp_status h2sp_ilut(const h2sp_csr *A, double tau, int p, h2sp_ilut_factors *F, void *ws, size_t ws_bytes,
                      int64_t *pool_used, void *stream) {
  if (h2sp_status s = check_csr(A)) return s;
  if (h2sp_status s = check_factors(F, A->n)) return s;
  if (!(tau >= 0.0)) return fail(H2SP_EINVAL, "ILUT: tau must be >= 0");
  if (A->n > 0 && (!F->pool_col || !F->pool_val || F->pool_cap < 0))
    return fail(H2SP_EINVAL, "ILUT: NULL pool");
  const int64_t n = A->n;
  if (pool_used) *pool_used = 0;
  if (n == 0) return H2SP_OK;
  const IlutCfg c = ilut_cfg(n);
  if (c.smem > (227u << 10)) return fail(H2SP_EUNSUPPORTED, "ILUT: n too large for the shared-memory bitmap");
  IlutWs s = ilut_carve(static_cast<unsigned char *>(ws), n, c.slots);
  if (!ws || ws_bytes < s.bytes) return fail(H2SP_EINVAL, "ILUT: workspace too small (h2sp_ilut_ws_bytes)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KCK(cudaMemsetAsync(s.ctr, 0, 16, st));
  const int32_t status0[2] = {0, INT32_MAX};
  KCK(cudaMemcpyAsync(s.status, status0, 8, cudaMemcpyHostToDevice, st));
  KCK(cudaMemsetAsync(s.done, 0, size_t(n) * 4, st));
  // the work rows must start zero; they are left zero row after row
  KCK(cudaMemsetAsync(s.w, 0, size_t(c.slots) * n * 8, st));
  IlutArgs a{};
  a.n = n;
  a.rp = A->rowptr;
  a.ci = A->col;
  a.av = A->val;
  a.tau = tau;
  a.p = p;
  a.nwords = c.nwords;
  a.l_start = F->l_start;
  a.u_start = F->u_start;
  a.l_len = F->l_len;
  a.u_len = F->u_len;
  a.diag = F->diag;
  a.pool_col = F->pool_col;
  a.pool_val = F->pool_val;
  a.cap = F->pool_cap;
  a.cursor = s.ctr;
  a.ticket = s.ctr + 1;
  a.done = s.done;
  a.status = s.status;
  a.w = s.w;
  a.ccol = s.ccol;
  a.cval = s.cval;
  KCK(cudaFuncSetAttribute(ilut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c.smem)));
  ilut_kernel<<<c.ctas, 32 * c.warps, c.smem, st>>>(a, c.warps);
  KCK(cudaGetLastError());
  unsigned long long used = 0;
  int32_t status[2];
  KCK(cudaMemcpyAsync(&used, s.ctr, 8, cudaMemcpyDeviceToHost, st));
  KCK(cudaMemcpyAsync(status, s.status, 8, cudaMemcpyDeviceToHost, st));
  KCK(cudaStreamSynchronize(st));
  if (pool_used) *pool_used = int64_t(used);
  if (status[0] & 1)
    return fail(H2SP_ENOMEM, "ILUT: pool capacity " + std::to_string(F->pool_cap) + " exceeded (" +
                                 std::to_string(used) + " entries requested so far)");
  if (status[0] & 2) return fail(H2SP_EINVAL, "ILUT: zero pivot at row " + std::to_string(status[1]));
  return H2SP_OK;
}

int64_t h2sp_ilu_solve_ws_bytes(int64_t n) { return n < 0 ? -1 : int64_t(trsv_carve(nullptr, n).bytes); }

h2sp_status h2sp_ilu_solve(const h2sp_ilut_factors *F, const double *b, double *x, void *ws, size_t ws_bytes,
                           void *stream) {
  if (!F) return fail(H2SP_EINVAL, "ILU solve: NULL factors");
  if (h2sp_status s = check_factors(F, F->n)) return s;
  if (F->n > 0 && (!b || !x)) return fail(H2SP_EINVAL, "ILU solve: NULL vector");
  if (!ws || ws_bytes < trsv_carve(nullptr, F->n).bytes) return fail(H2SP_EINVAL, "ILU solve: workspace too small");
  return launch_trsv(F, b, x, static_cast<unsigned char *>(ws), static_cast<cudaStream_t>(stream));
}

h2sp_status h2sp_csr_spmv(const h2sp_csr *A, const double *x, double *y, void *stream) {
  if (h2sp_status s = check_csr(A)) return s;
  if (A->n > 0 && (!x || !y)) return fail(H2SP_EINVAL, "SpMV: NULL vector");
  return launch_spmv(A, x, y, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// ---------------------------------------------------------------------------
// GMRES
// ---------------------------------------------------------------------------

namespace {

struct GmresWs {
  double *V, *t1, *t2, *z, *w, *r, *part, *h, *hn, *c;
  unsigned char *trsv;
  size_t bytes;
};

GmresWs gmres_carve(unsigned char *base, int64_t n, int m) {
  GmresWs g{};
  size_t off = 0;
  auto take = [&](size_t b) {
    unsigned char *p = base ? base + off : nullptr;
    off += align256(b);
    return p;
  };
  g.V = reinterpret_cast<double *>(take(size_t(m + 1) * n * 8));
  g.t1 = reinterpret_cast<double *>(take(size_t(n) * 8));
  g.t2 = reinterpret_cast<double *>(take(size_t(n) * 8));
  g.z = reinterpret_cast<double *>(take(size_t(n) * 8));
  g.w = reinterpret_cast<double *>(take(size_t(n) * 8));
  g.r = reinterpret_cast<double *>(take(size_t(n) * 8));
  g.part = reinterpret_cast<double *>(take(size_t(DOT_BLOCKS) * DOT_MAXV * 8));
  g.h = reinterpret_cast<double *>(take(size_t(m + 2) * 8));
  g.hn = reinterpret_cast<double *>(take(size_t(m + 2) * 8));
  g.c = reinterpret_cast<double *>(take(size_t(m + 2) * 8));
  g.trsv = take(trsv_carve(nullptr, n).bytes);
  g.bytes = off;
  return g;
}

struct Ctx {
  const h2sp_sparsified *A, *M;
  const h2sp_ilut_factors *F;
  int64_t n;
  GmresWs g;
  cudaStream_t st;
  int64_t launches = 0;
};

// y = A x = U (S (U^T x))   (A = U S V^T, V = U: symmetric plan)
h2sp_status op_A(Ctx &c, const double *x, double *y) {
  const h2sp_sparsified *A = c.A;
  if (h2sp_status s = h2sp_apply_Ut(A->plan, A->q, x, c.n, c.g.t1, c.n, 1, A->apply_ws, A->apply_ws_bytes, c.st))
    return s;
  if (h2sp_status s = launch_spmv(&A->S, c.g.t1, c.g.t2, c.st)) return s;
  return h2sp_apply_V(A->plan, A->q, c.g.t2, c.n, y, c.n, 1, A->apply_ws, A->apply_ws_bytes, c.st);
}

// y = M^-1 x = U_M (L U)^-1 U_M^T x, or y = x without a preconditioner
h2sp_status op_M(Ctx &c, const double *x, double *y) {
  if (!c.M) {
    KCK(cudaMemcpyAsync(y, x, size_t(c.n) * 8, cudaMemcpyDeviceToDevice, c.st));
    return H2SP_OK;
  }
  const h2sp_sparsified *M = c.M;
  if (h2sp_status s = h2sp_apply_Ut(M->plan, M->q, x, c.n, c.g.t1, c.n, 1, M->apply_ws, M->apply_ws_bytes, c.st))
    return s;
  if (h2sp_status s = launch_trsv(c.F, c.g.t1, c.g.t2, c.g.trsv, c.st)) return s;
  return h2sp_apply_V(M->plan, M->q, c.g.t2, c.n, y, c.n, 1, M->apply_ws, M->apply_ws_bytes, c.st);
}

// out[0..nv) = V[0..nv)^T w (accumulate: +=)
h2sp_status dots(Ctx &c, const double *V, int nv, const double *w, double *out, bool accumulate) {
  for (int v0 = 0; v0 < nv; v0 += DOT_MAXV) {
    const int k = std::min(DOT_MAXV, nv - v0);
    dots_kernel<<<DOT_BLOCKS, DOT_THREADS, 0, c.st>>>(V + size_t(v0) * c.n, c.n, k, w, c.n, c.g.part);
    reduce_parts_kernel<<<1, 32, 0, c.st>>>(c.g.part, k, DOT_BLOCKS, out + v0, accumulate ? 1 : 0);
    c.launches += 2;
  }
  KCK(cudaGetLastError());
  return H2SP_OK;
}

}  // namespace

extern "C" {

int64_t h2sp_gmres_ws_bytes(int64_t n, int restart) {
  if (n < 0 || restart < 1) return -1;
  return int64_t(gmres_carve(nullptr, n, restart).bytes);
}

h2sp_status h2sp_gmres(const h2sp_sparsified *A, const h2sp_sparsified *M, const h2sp_ilut_factors *F,
                       const double *b, double *x, const h2sp_gmres_opts *opt, h2sp_gmres_info *info, void *ws,
                       size_t ws_bytes, void *stream) {
  if (!A || !opt || !info || !b || !x) return fail(H2SP_EINVAL, "GMRES: NULL argument");
  if ((M == nullptr) != (F == nullptr)) return fail(H2SP_EINVAL, "GMRES: the preconditioner needs both M and F");
  if (opt->restart < 1 || opt->maxiter < 0 || !(opt->tol > 0.0)) return fail(H2SP_EINVAL, "GMRES: bad options");
  const int64_t n = A->S.n;
  if (h2sp_status s = check_csr(&A->S)) return s;
  for (const h2sp_sparsified *o : {A, M}) {
    if (!o) continue;
    if (!o->plan || !o->q) return fail(H2SP_EINVAL, "GMRES: NULL plan / Q");
    if (!o->plan->sym) return fail(H2SP_EUNSUPPORTED, "GMRES: symmetric plans only (A = U S U^T)");
    if (o->plan->world != 1 || o->plan->n_rows_local != n || o->S.n != n)
      return fail(H2SP_EINVAL, "GMRES: operator sizes differ / sharded plan");
  }
  if (F && F->n != n) return fail(H2SP_EINVAL, "GMRES: factor size differs");
  const int m = opt->restart;
  Ctx c{A, M, F, n, gmres_carve(static_cast<unsigned char *>(ws), n, m), static_cast<cudaStream_t>(stream)};
  if (!ws || ws_bytes < c.g.bytes) return fail(H2SP_EINVAL, "GMRES: workspace too small (h2sp_gmres_ws_bytes)");
  const int vg = vec_grid(n);
  double *hist = info->history;
  const int hist_cap = info->history_cap;
  int nh = 0;
  auto push = [&](double v) {
    if (hist && nh < hist_cap) hist[nh] = v;
    nh++;
  };
  KCK(cudaMemsetAsync(x, 0, size_t(n) * 8, c.st));
  // ||b||
  if (h2sp_status s = dots(c, b, 1, b, c.g.h, false)) return s;
  double bb = 0.0;
  KCK(cudaMemcpyAsync(&bb, c.g.h, 8, cudaMemcpyDeviceToHost, c.st));
  KCK(cudaStreamSynchronize(c.st));
  const double bnorm = std::sqrt(bb);
  push(1.0);
  info->iters = 0;
  info->converged = 0;
  info->restarts = 0;
  if (bnorm == 0.0) {
    info->converged = 1;
    info->history_len = nh;
    return H2SP_OK;
  }
  std::vector<double> H(size_t(m + 1) * m), cs(m), sn(m), gv(m + 1), y(m), hcol(m + 2);
  int it = 0;
  bool converged = false;
  while (it < opt->maxiter && !converged) {
    // r = b - A x;  beta = ||r||
    if (h2sp_status s = op_A(c, x, c.g.r)) return s;
    axpby_kernel<<<vg, 256, 0, c.st>>>(1.0, b, -1.0, c.g.r, n);
    if (h2sp_status s = dots(c, c.g.r, 1, c.g.r, c.g.h, false)) return s;
    double rr = 0.0;
    KCK(cudaMemcpyAsync(&rr, c.g.h, 8, cudaMemcpyDeviceToHost, c.st));
    KCK(cudaStreamSynchronize(c.st));
    const double beta = std::sqrt(rr);
    if (beta <= opt->tol * bnorm) {
      converged = true;
      break;
    }
    KCK(cudaMemcpyAsync(c.g.hn, &beta, 8, cudaMemcpyHostToDevice, c.st));
    scale_kernel<<<vg, 256, 0, c.st>>>(c.g.r, c.g.hn, c.g.V, n);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int jd = 0;
    for (int j = 0; j < m; j++) {
      double *vj = c.g.V + size_t(j) * n, *vn = c.g.V + size_t(j + 1) * n;
      if (h2sp_status s = op_M(c, vj, c.g.z)) return s;
      if (h2sp_status s = op_A(c, c.g.z, c.g.w)) return s;
      // CGS2: h = V^T w, w -= V h, twice
      if (h2sp_status s = dots(c, c.g.V, j + 1, c.g.w, c.g.h, false)) return s;
      sub_comb_kernel<<<vg, 256, 0, c.st>>>(c.g.V, n, j + 1, c.g.h, c.g.w, n);
      if (h2sp_status s = dots(c, c.g.V, j + 1, c.g.w, c.g.c, false)) return s;
      sub_comb_kernel<<<vg, 256, 0, c.st>>>(c.g.V, n, j + 1, c.g.c, c.g.w, n);
      if (h2sp_status s = dots(c, c.g.w, 1, c.g.w, c.g.hn, false)) return s;
      KCK(cudaGetLastError());
      std::vector<double> h1(j + 2), h2(j + 1);
      KCK(cudaMemcpyAsync(h1.data(), c.g.h, size_t(j + 1) * 8, cudaMemcpyDeviceToHost, c.st));
      KCK(cudaMemcpyAsync(h2.data(), c.g.c, size_t(j + 1) * 8, cudaMemcpyDeviceToHost, c.st));
      KCK(cudaMemcpyAsync(&h1[j + 1], c.g.hn, 8, cudaMemcpyDeviceToHost, c.st));
      KCK(cudaStreamSynchronize(c.st));
      for (int i = 0; i <= j; i++) H[size_t(i) * m + j] = h1[i] + h2[i];
      const double hnext = std::sqrt(h1[j + 1]);
      H[size_t(j + 1) * m + j] = hnext;
      if (hnext != 0.0) {
        KCK(cudaMemcpyAsync(c.g.hn, &hnext, 8, cudaMemcpyHostToDevice, c.st));
        scale_kernel<<<vg, 256, 0, c.st>>>(c.g.w, c.g.hn, vn, n);
      }
      for (int i = 0; i < j; i++) {  // previous rotations on column j
        const double a = H[size_t(i) * m + j], bq = H[size_t(i + 1) * m + j];
        H[size_t(i) * m + j] = cs[i] * a + sn[i] * bq;
        H[size_t(i + 1) * m + j] = -sn[i] * a + cs[i] * bq;
      }
      const double hj = H[size_t(j) * m + j], hj1 = H[size_t(j + 1) * m + j];
      const double den = std::hypot(hj, hj1);
      cs[j] = hj / den;
      sn[j] = hj1 / den;
      H[size_t(j) * m + j] = den;
      H[size_t(j + 1) * m + j] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      it++;
      jd = j + 1;
      push(std::fabs(gv[j + 1]) / bnorm);
      if (std::fabs(gv[j + 1]) <= opt->tol * bnorm || it >= opt->maxiter) break;
    }
    for (int i = jd - 1; i >= 0; i--) {  // H[:jd, :jd] y = g[:jd]
      double s = gv[i];
      for (int q = i + 1; q < jd; q++) s -= H[size_t(i) * m + q] * y[q];
      y[i] = s / H[size_t(i) * m + i];
    }
    // x += M^-1 (V y)
    KCK(cudaMemcpyAsync(c.g.c, y.data(), size_t(jd) * 8, cudaMemcpyHostToDevice, c.st));
    comb_kernel<<<vg, 256, 0, c.st>>>(c.g.V, n, jd, c.g.c, c.g.w, n);
    if (h2sp_status s = op_M(c, c.g.w, c.g.z)) return s;
    axpby_kernel<<<vg, 256, 0, c.st>>>(1.0, c.g.z, 1.0, x, n);
    KCK(cudaGetLastError());
    info->restarts++;
    if (std::fabs(gv[jd]) <= opt->tol * bnorm) converged = true;
  }
  KCK(cudaStreamSynchronize(c.st));
  info->iters = it;
  info->converged = converged ? 1 : 0;
  info->history_len = nh;
  return H2SP_OK;
}

}  // extern "C"
