// The paper's preconditioning workload on the device (SURVEY §8(f) #3,
// "Sparsification method as a preconditioner") and the direct
// solve it shares its factorisation with (§8(f) #1, x = V S^-1 U^T b):
//
//   * ilut_cta_kernel -- ILUT(tau, p) of S (reading 25: Saad's
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
// One CTA (4 warps) factorises one row at a time; rows are handed out in increasing
// order by an atomic ticket, a row waits (acquire) on the completion flag of
// each U row it uses and publishes its own U row (release) BEFORE it selects
// and writes its L part -- the L part is off every other row's critical path.
// Tickets are taken only by running warps and a row waits only on smaller
// rows, so there is no deadlock whatever the grid size.  The work row w is a
// dense per-CTA vector in HBM (touched entries only: O(row) per row) with a
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
  int32_t *done;               // [n] 1 once u_ii is published, 2 once U row i is
  int32_t *status;             // [0] bit 1 = pool overflow, bit 2 = zero pivot; [1] first zero-pivot row
  double *w;                   // [slots][n] work rows (zero between rows)
  int32_t *ccol;               // [slots][n] candidate columns
  double *cval;                // [slots][n] candidate values
};

// Bitmap word wi restricted to columns [lo, hi] (0 outside the word range).
__device__ __forceinline__ uint32_t word_in(const uint32_t *bits, int64_t wi, int64_t lo, int64_t hi) {
  const int64_t l = lo - (wi << 5), h = hi - (wi << 5);
  if (l >= 32 || h < 0) return 0;
  uint32_t v = bits[wi];
  if (l > 0) v &= ~0u << l;
  if (h < 31) v &= (2u << h) - 1u;
  return v;
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

// ---------------------------------------------------------------------------
// ilut_cta_kernel: one CTA of IW warps per row.  Warp 0 runs the rule-1
// batches (lane q takes the q-th next present k and evaluates rule 1 on it;
// every k before the first kept one is dropped at once -- their values are
// final, no update lies between them --, the first kept one is applied and the
// batch restarts after it; rule 1 needs only u_kk (flag >= 1), the update U row
// k (flag >= 2), so a dropped k never waits for k's U row); a kept k's update
// with U row k, the gathers of the U and L parts (1024-column chunks, chunk c
// on warp c % IW, kept entries placed in chunk order through a shared-memory
// scan) and the clean-up use all IW warps -- the U gather is on the row-to-row
// chain whenever the next row keeps its l entry, so a row's publication comes
// IW times sooner (one warp per row: 2.37 -> 1.30 s at N = 131,072, DESIGN 9e).
// ---------------------------------------------------------------------------
constexpr int IW = 4;

__device__ int64_t gather_cta(const uint32_t *bits, const double *w, int64_t lo, int64_t hi, bool upper,
                              double taui, int32_t *ccol, double *cval, int lane, int warp, int *s_cnt) {
  int64_t cnt = 0;
  if (lo > hi) return 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t g = lo & ~int64_t(1023); g <= hi; g += 1024 * IW) {
    const int64_t base = g + 1024 * warp;
    double v[32];
    uint32_t keepm = 0;
    if (base <= hi) {
      const uint32_t wd = word_in(bits, (base >> 5) + lane, lo, hi);
      if (__ballot_sync(FULL, wd != 0)) {
#pragma unroll
        for (int q = 0; q < 32; q++) {
          const uint32_t wq = __shfl_sync(FULL, wd, q);
          const bool pq = (wq >> lane) & 1u;
          v[q] = pq ? w[base + 32 * q + lane] : 0.0;
          if (pq && (!upper || !(fabs(v[q]) < taui || v[q] == 0.0))) keepm |= 1u << q;
        }
      }
    }
    int mine = 0;
#pragma unroll
    for (int q = 0; q < 32; q++) mine += __popc(__ballot_sync(FULL, (keepm >> q) & 1u));
    if (lane == 0) s_cnt[warp] = mine;
    __syncthreads();
    int64_t off = cnt, tot = 0;
    for (int u = 0; u < IW; u++) {
      if (u < warp) off += s_cnt[u];
      tot += s_cnt[u];
    }
    if (keepm | __ballot_sync(FULL, keepm != 0)) {
#pragma unroll
      for (int q = 0; q < 32; q++) {
        const bool kq = (keepm >> q) & 1u;
        const unsigned m = __ballot_sync(FULL, kq);
        if (kq) {
          const int64_t pos = off + __popc(m & lt);
          ccol[pos] = int32_t(base + 32 * q + lane);
          cval[pos] = v[q];
        }
        off += __popc(m);
      }
    }
    cnt += tot;
    __syncthreads();
  }
  return cnt;
}

__global__ void __launch_bounds__(32 * IW) ilut_cta_kernel(IlutArgs A) {
  extern __shared__ uint32_t smem[];
  uint32_t *bits = smem;
  int *hist = reinterpret_cast<int *>(smem + A.nwords);
  int32_t *kbuf = hist + 256;
  __shared__ int s_cnt[IW];
  __shared__ long long s_row, s_kf, s_st;
  __shared__ double s_wkf, s_taui;
  __shared__ int s_lo, s_hi;
  __shared__ long long s_c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t slot = blockIdx.x;
  double *w = A.w + slot * A.n;
  int32_t *ccol = A.ccol + slot * A.n;
  double *cval = A.cval + slot * A.n;
  for (int i = tid; i < A.nwords; i += blockDim.x) bits[i] = 0;
  __syncthreads();
  for (;;) {
    if (tid == 0) s_row = static_cast<long long>(atomicAdd(A.ticket, 1ull));
    __syncthreads();
    const int64_t i = s_row;
    if (i >= A.n) break;
    const int64_t e0 = A.rp[i], e1 = A.rp[i + 1];
    if (tid == 0) {  // tau_i = tau * ||a_i||_2, the sum of squares in column order
      double sq = 0.0;
      for (int64_t e = e0; e < e1; e++) sq = __dadd_rn(sq, __dmul_rn(A.av[e], A.av[e]));
      s_taui = __dmul_rn(A.tau, sqrt(sq));
      s_lo = int(i);
      s_hi = int(i);
    }
    __syncthreads();
    {
      int lo = int(i), hi = int(i);
      for (int64_t e = e0 + tid; e < e1; e += blockDim.x) {
        const int32_t j = A.ci[e];
        w[j] = A.av[e];
        atomicOr(&bits[j >> 5], 1u << (j & 31));
        lo = min(lo, j);
        hi = max(hi, j);
      }
      atomicMin(&s_lo, lo);
      atomicMax(&s_hi, hi);
    }
    __syncthreads();
    const int64_t lo = s_lo;
    const double taui = s_taui;
    int64_t cur = lo;  // warp 0's cursor
    for (;;) {
      if (warp == 0) {  // rule-1 batches until a kept k (or the end)
        long long kf_out = -1;
        double wkf_out = 0.0;
        while (cur < i) {
          const int64_t wi0 = cur >> 5, wi = wi0 + lane;
          const int64_t wend = (i + 31) >> 5;
          const uint32_t wd = wi < wend ? word_in(bits, wi, cur, i - 1) : 0u;
          const int c = __popc(wd);
          int excl = c;
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, excl, o);
            if (lane >= o) excl += y;
          }
          const int total = __shfl_sync(FULL, excl, 31);
          excl -= c;
          if (total == 0) {
            cur = (wi0 + 32) << 5;
            continue;
          }
          {
            int r = excl;
            for (uint32_t t = wd; t && r < 32; t &= t - 1, r++) kbuf[r] = int32_t((wi << 5) + __ffs(t) - 1);
          }
          __syncwarp();
          const int nk = min(total, 32);
          const int64_t k = lane < nk ? int64_t(kbuf[lane]) : -1;
          bool drop = true;
          double wk = 0.0;
          if (k >= 0) {
            wait_flag(A.done + k, 1);
            wk = __ddiv_rn(w[k], __ldcg(A.diag + k));
            drop = fabs(wk) < taui || wk == 0.0;  // rule 1
          }
          const unsigned kept = __ballot_sync(FULL, !drop);
          const int f = kept ? __ffs(kept) - 1 : nk;
          __syncwarp();
          if (lane < f && k >= 0) {
            w[k] = 0.0;
            atomicAnd(&bits[k >> 5], ~(1u << (k & 31)));
          }
          if (f == nk) {
            cur = total > 32 ? int64_t(__shfl_sync(FULL, k, 31)) + 1 : int64_t((wi0 + 32) << 5);
            __syncwarp();
            continue;
          }
          const int64_t kf = __shfl_sync(FULL, k, f);
          const double wkf = __shfl_sync(FULL, wk, f);
          if (lane == f) {
            w[kf] = wkf;
            wait_flag(A.done + kf, 2);
          }
          __syncwarp();
          kf_out = kf;
          wkf_out = wkf;
          cur = kf + 1;
          break;
        }
        if (lane == 0) {
          s_kf = kf_out;
          s_wkf = wkf_out;
        }
      }
      __syncthreads();
      const int64_t kf = s_kf;
      if (kf < 0) break;
      const double wkf = s_wkf;
      const int64_t us = __ldcg(A.u_start + kf);
      const int32_t ul = __ldcg(A.u_len + kf);
      int hi = 0;
      for (int32_t e0u = 0; e0u < ul; e0u += 4 * 32 * IW) {
        int32_t j[4];
        double u[4], x[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int32_t e = e0u + 32 * IW * q + tid;
          j[q] = e < ul ? __ldcg(A.pool_col + us + e) : -1;
          u[q] = e < ul ? __ldcg(A.pool_val + us + e) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) x[q] = j[q] >= 0 ? w[j[q]] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (j[q] >= 0) {
            w[j[q]] = __dsub_rn(x[q], __dmul_rn(wkf, u[q]));
            atomicOr(&bits[j[q] >> 5], 1u << (j[q] & 31));
            hi = max(hi, j[q]);
          }
      }
      atomicMax(&s_hi, hi);
      __syncthreads();
    }
    const int64_t hi = s_hi;
    if (tid == 0) {  // u_ii is final: publish it (flag 1)
      A.diag[i] = w[i];
      __threadfence();
      st_release(A.done + i, 1);
    }
    // rule 2, U part
    int64_t cu = gather_cta(bits, w, i + 1, hi, true, taui, ccol, cval, lane, warp, s_cnt);
    if (A.p >= 0 && cu > A.p) {
      if (warp == 0) {
        const int64_t kept = keep_largest(ccol, cval, cu, A.p, hist, lane);
        if (lane == 0) s_c = kept;
      }
      __syncthreads();
      cu = s_c;
    }
    if (tid == 0) {
      unsigned long long st = 0;
      if (cu > 0) {
        st = atomicAdd(A.cursor, static_cast<unsigned long long>(cu));
        if (int64_t(st) + cu > A.cap) atomicOr(&A.status[0], 1);
      }
      s_st = static_cast<long long>(st);
    }
    __syncthreads();
    int64_t st = s_st;
    bool fits = st + cu <= A.cap;
    if (fits)
      for (int64_t a = tid; a < cu; a += blockDim.x) {
        A.pool_col[st + a] = ccol[a];
        A.pool_val[st + a] = cval[a];
      }
    __syncthreads();
    if (tid == 0) {
      const double uii = w[i];
      A.u_start[i] = st;
      A.u_len[i] = fits ? int32_t(cu) : 0;
      if (uii == 0.0) {
        atomicOr(&A.status[0], 2);
        atomicMin(&A.status[1], int32_t(i));
      }
      __threadfence();
      st_release(A.done + i, 2);
    }
    // L part (kept entries of rule 1)
    int64_t cl = gather_cta(bits, w, lo, i - 1, false, taui, ccol, cval, lane, warp, s_cnt);
    if (A.p >= 0 && cl > A.p) {
      if (warp == 0) {
        const int64_t kept = keep_largest(ccol, cval, cl, A.p, hist, lane);
        if (lane == 0) s_c = kept;
      }
      __syncthreads();
      cl = s_c;
    }
    if (tid == 0) {
      unsigned long long st2 = 0;
      if (cl > 0) {
        st2 = atomicAdd(A.cursor, static_cast<unsigned long long>(cl));
        if (int64_t(st2) + cl > A.cap) atomicOr(&A.status[0], 1);
      }
      s_st = static_cast<long long>(st2);
    }
    __syncthreads();
    st = s_st;
    fits = st + cl <= A.cap;
    if (fits)
      for (int64_t a = tid; a < cl; a += blockDim.x) {
        A.pool_col[st + a] = ccol[a];
        A.pool_val[st + a] = cval[a];
      }
    if (tid == 0) {
      A.l_start[i] = st;
      A.l_len[i] = fits ? int32_t(cl) : 0;
    }
    // clear the touched range of w, then the bitmap
    for (int64_t base = (lo & ~int64_t(255)) + 256 * warp; base <= hi; base += 256 * IW) {
      const int64_t wi = (base >> 5) + (lane & 7);
      const uint32_t wd = lane < 8 ? word_in(bits, wi, lo, hi) : 0u;
      if (!__ballot_sync(FULL, wd != 0)) continue;
#pragma unroll
      for (int q = 0; q < 8; q++)
        if ((__shfl_sync(FULL, wd, q) >> lane) & 1u) w[base + 32 * q + lane] = 0.0;
    }
    __syncthreads();
    for (int64_t wi = (lo >> 5) + tid; wi <= (hi >> 5); wi += blockDim.x) bits[wi] = 0;
    __syncthreads();
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
  double *y;                   // forward result (workspace), sentinel-initialised
  double *x;                   // result, sentinel-initialised before the backward pass
  unsigned long long *ticket;  // [0] forward, [1] backward
};

// A solved value is its own completion flag: the vectors start filled with a
// NaN payload no arithmetic produces, readers poll the value (relaxed, gpu
// scope: one L2 round trip, no separate flag / fence).
constexpr unsigned long long XSENT = 0x7ff4deadbeefcafeull;

__device__ __forceinline__ unsigned long long ld_rlx(const double *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double poll(const double *p, unsigned long long v) {
  while (v == XSENT) {
    __nanosleep(16);
    v = ld_rlx(p);
  }
  return __longlong_as_double(static_cast<long long>(v));
}

__device__ __forceinline__ void st_rlx(double *p, double v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}

__global__ void fill_sentinel_kernel(double *v, int64_t n) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    v[e] = __longlong_as_double(static_cast<long long>(XSENT));
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Rows are solved in blocks of TB = 32 consecutive rows (in solve order:
// ascending for L, descending for U -- the U solve is the L solve of the
// reversed index i' = n - 1 - i), one warp per block, blocks handed out in
// solve order by a ticket.  Lane r owns row r of the block: it walks its
// row's entries oldest first, summing those more than two blocks back (polling
// each value -- the oldest are long done) and scattering the rest into three
// dense 32 x 32 tiles in shared memory (two previous blocks, own block).  The
// chain from block to block is then: poll the 32 values of a previous block,
// 32 shuffle-FMAs per tile, the 32-step triangular solve of the own tile by
// shuffles, 32 stores -- no per-row global round trip.
constexpr int TB = 32;

template <bool UPPER>
__global__ void __launch_bounds__(32) trsv_block_kernel(TrsvArgs A) {
  __shared__ double T[3 * TB][TB];  // [c][r]: column jp - (r0 - 2 TB) of row r
  const int lane = threadIdx.x;
  const int64_t n = A.n, nb = (n + TB - 1) / TB;
  const double *src = UPPER ? A.y : A.b;
  double *dst = UPPER ? A.x : A.y;
  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(A.ticket + (UPPER ? 1 : 0), 1ull);
    const int64_t t = int64_t(__shfl_sync(FULL, tk, 0));
    if (t >= nb) return;
    for (int c = 0; c < 3 * TB; c++) T[c][lane] = 0.0;
    const int64_t r0 = t * TB, w0 = r0 - 2 * TB;
    const int64_t ip = r0 + lane;
    const bool live = ip < n;
    const int64_t i = UPPER ? n - 1 - ip : ip;
    double acc = 0.0;
    if (live) {
      const int64_t s0 = UPPER ? A.u_start[i] : A.l_start[i];
      const int32_t len = UPPER ? A.u_len[i] : A.l_len[i];
      // oldest first: ascending column for L, descending for U
      for (int32_t e0 = 0; e0 < len; e0 += 4) {
        int64_t jp[4], j[4];
        double v[4];
        unsigned long long xv[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int32_t e = e0 + q;
          const int64_t idx = s0 + (UPPER ? len - 1 - e : e);
          j[q] = e < len ? A.pool_col[idx] : 0;
          v[q] = e < len ? A.pool_val[idx] : 0.0;
          jp[q] = e < len ? (UPPER ? n - 1 - j[q] : j[q]) : INT64_MAX;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) xv[q] = jp[q] < w0 ? ld_rlx(dst + j[q]) : 0ull;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (jp[q] < w0)
            acc += v[q] * poll(dst + j[q], xv[q]);
          else if (jp[q] != INT64_MAX)
            T[jp[q] - w0][lane] = v[q];
        }
      }
    }
    __syncwarp();
    double rhs = live ? src[i] - acc : 0.0;
    const double dg = (UPPER && live) ? A.diag[i] : 1.0;
    for (int pb = 0; pb < 2; pb++) {  // blocks t - 2, t - 1
      const int64_t base = w0 + int64_t(pb) * TB;
      if (base < 0) continue;
      bool any = false;
      for (int c = 0; c < TB; c++) any |= T[pb * TB + c][lane] != 0.0;
      if (!__ballot_sync(FULL, any)) continue;
      const int64_t jq = base + lane;
      const double *px = dst + (UPPER ? n - 1 - jq : jq);
      const double xp = poll(px, ld_rlx(px));
      for (int c = 0; c < TB; c++) rhs -= T[pb * TB + c][lane] * __shfl_sync(FULL, xp, c);
    }
    double xr = 0.0;
    for (int c = 0; c < TB; c++) {
      if (lane == c) xr = UPPER ? rhs / dg : rhs;
      const double xc = __shfl_sync(FULL, xr, c);
      if (lane > c) rhs -= T[2 * TB + c][lane] * xc;
    }
    if (live) st_rlx(dst + i, xr);
    __syncwarp();
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

IlutCfg ilut_cfg(int64_t n) {  // ilut_cta_kernel: one row per CTA of IW warps, 2 CTAs per SM
  IlutCfg c{};
  c.nwords = int((n + 31) / 32);
  c.warps = IW;
  c.smem = size_t(c.nwords) * 4 + 288 * 4;
  c.ctas = num_sms() * 2;
  c.slots = c.ctas;
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
  double *y;
  unsigned long long *ticket;
  size_t bytes;
};

TrsvWs trsv_carve(unsigned char *base, int64_t n) {
  TrsvWs s{};
  const size_t yb = align256(size_t(n) * 8);
  s.y = reinterpret_cast<double *>(base);
  s.ticket = reinterpret_cast<unsigned long long *>(base ? base + yb : nullptr);
  s.bytes = yb + 256;
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
  const int64_t nb = (n + TB - 1) / TB;
  const int fg = int(std::min<int64_t>(int64_t(num_sms()) * 4, (n + 255) / 256));
  KCK(cudaMemsetAsync(t.ticket, 0, 16, st));
  fill_sentinel_kernel<<<fg, 256, 0, st>>>(t.y, n);
  TrsvArgs a{n, F->l_start, F->u_start, F->l_len, F->u_len, F->diag, F->pool_col, F->pool_val, b, t.y, x, t.ticket};
  const int grid = int(std::min<int64_t>(int64_t(num_sms()) * 16, nb));
  trsv_block_kernel<false><<<grid, 32, 0, st>>>(a);
  KCK(cudaGetLastError());
  fill_sentinel_kernel<<<fg, 256, 0, st>>>(x, n);  // b (possibly aliased by x) is consumed
  trsv_block_kernel<true><<<grid, 32, 0, st>>>(a);
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
  KCK(cudaFuncSetAttribute(ilut_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c.smem)));
  ilut_cta_kernel<<<c.ctas, 32 * IW, c.smem, st>>>(a);
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
