// Supernodal Cholesky of S on the device (the direct solve
// x = V S^-1 U^T b, Eq. sp0; the paper factorises S with CHOLMOD,
// P:804).  S is symmetric positive definite in symmetric mode
// (Proposition) and block-structured: its rows come in groups --
// the frozen rows of one cluster, S order off(k, t) -- whose rows
// share one column pattern, and every block of S joins two groups.  Those
// groups are the supernodes here, in S's own level-major order (leaves'
// frozen rows first, each level after the levels below: the upper levels play
// the separators of a nested dissection).
//
//   analysis (host, h2sp_chol_analyse): the block elimination tree and the
//     block structure struct(J) of every column of L by the supernodal
//     symbolic factorisation (struct(J) = A's blocks in column J ∪ the
//     structures of J's children minus themselves, parent(J) = the smallest
//     block below J), panel layout: supernode J owns a dense row-major panel
//     of (sum over I in struct(J) of m_I) x m_J doubles, block I at row
//     offset pos[J][I].
//   factor (device, right-looking, one supernode after another):
//     chol_potrf_kernel   L_JJ = chol(A_JJ)           (one CTA, shared memory)
//     chol_trsm_kernel    L_IJ = A_IJ L_JJ^-T         (one warp per row)
//     chol_schur_kernel   A_IK -= L_IJ L_KJ^T for I >= K in struct(J): 64 x 64
//                         output tiles on the FP64 tensor cores (DMMA), the
//                         result subtracted in place in panel K
//   solve: forward / backward substitution supernode by supernode.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "h2sp_internal.h"

using namespace h2sp;

#define CCK(x)                                                                                           \
  do {                                                                                                   \
    cudaError_t e_ = (x);                                                                                \
    if (e_ != cudaSuccess) return fail(H2SP_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct h2sp_chol_s {
  int64_t n = 0;
  int32_t ns = 0, mmax = 0;
  std::vector<int64_t> start;               // [ns + 1] first S row of supernode J
  std::vector<int32_t> m;                   // [ns]
  std::vector<int32_t> parent;              // [ns] block elimination tree, -1 = root
  std::vector<std::vector<int32_t>> st;     // struct(J), ascending, st[J][0] == J
  std::vector<int64_t> poff;                // [ns + 1] panel offsets (doubles)
  std::vector<int32_t> prows;               // [ns] panel rows
  std::vector<int64_t> roff;                // [ns + 1] per-panel-row arrays offset
  double flops = 0.0;
  // device meta image
  std::vector<unsigned char> meta;
  size_t o_start = 0, o_m = 0, o_poff = 0, o_prows = 0, o_roff = 0, o_pos = 0, o_blk = 0, o_grow = 0, o_sgrp = 0;
};

namespace {

constexpr unsigned FULL = 0xffffffffu;

struct CholMeta {
  int32_t ns;
  int64_t n;
  const int64_t *start;
  const int32_t *m;
  const int64_t *poff;
  const int32_t *prows;
  const int64_t *roff;
  const int32_t *pos;    // [ns * ns]: pos[K * ns + I] = row offset of block I in panel K, -1 if absent
  const int32_t *blk;    // per panel row: its block (supernode) I
  const int32_t *grow;   // per panel row: its S row
  const int32_t *sgrp;   // [n]: supernode of S row i
};

CholMeta meta_view(const h2sp_chol_s *c, const unsigned char *d) {
  CholMeta v;
  v.ns = c->ns;
  v.n = c->n;
  v.start = reinterpret_cast<const int64_t *>(d + c->o_start);
  v.m = reinterpret_cast<const int32_t *>(d + c->o_m);
  v.poff = reinterpret_cast<const int64_t *>(d + c->o_poff);
  v.prows = reinterpret_cast<const int32_t *>(d + c->o_prows);
  v.roff = reinterpret_cast<const int64_t *>(d + c->o_roff);
  v.pos = reinterpret_cast<const int32_t *>(d + c->o_pos);
  v.blk = reinterpret_cast<const int32_t *>(d + c->o_blk);
  v.grow = reinterpret_cast<const int32_t *>(d + c->o_grow);
  v.sgrp = reinterpret_cast<const int32_t *>(d + c->o_sgrp);
  return v;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// S (lower triangle, CSR) -> the panels (zeroed before): warp per S row
__global__ void __launch_bounds__(256) chol_scatter_kernel(CholMeta M, const int64_t *rp, const int32_t *ci,
                                                           const double *av, double *panel) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < M.n; i += nw) {
    const int32_t I = M.sgrp[i];
    const int64_t a = i - M.start[I];
    for (int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
      const int32_t j = ci[e];
      if (j > i) continue;
      const int32_t J = M.sgrp[j];
      const int32_t p = M.pos[int64_t(J) * M.ns + I];
      panel[M.poff[J] + (p + a) * M.m[J] + (j - M.start[J])] = av[e];
    }
  }
}

// L_JJ = chol(A_JJ) in shared memory (right-looking, column by column)
__global__ void __launch_bounds__(512) chol_potrf_kernel(CholMeta M, double *panel, int32_t J, int32_t *status) {
  extern __shared__ double sA[];
  const int m = M.m[J], ld = m + 1;
  double *P = panel + M.poff[J];
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sA[(e / m) * ld + e % m] = P[e];
  __syncthreads();
  for (int c = 0; c < m; c++) {
    if (threadIdx.x == 0) {
      const double d = sA[c * ld + c];
      if (!(d > 0.0)) atomicMin(status, J);
      sA[c * ld + c] = sqrt(d);
    }
    __syncthreads();
    const double piv = sA[c * ld + c];
    for (int r = c + 1 + threadIdx.x; r < m; r += blockDim.x) sA[r * ld + c] /= piv;
    __syncthreads();
    const int t = m - 1 - c;  // trailing size
    for (int e = threadIdx.x; e < t * t; e += blockDim.x) {
      const int r = c + 1 + e / t, s = c + 1 + e % t;
      if (s <= r) sA[r * ld + s] -= sA[r * ld + c] * sA[s * ld + c];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int r = e / m, s = e % m;
    P[e] = s <= r ? sA[r * ld + s] : 0.0;
  }
}

// rows below the diagonal block: x L_JJ^T = a (forward substitution), one warp
// per row, lane l holds columns l, l + 32, l + 64, l + 96
__global__ void __launch_bounds__(256) chol_trsm_kernel(CholMeta M, double *panel, int32_t J) {
  extern __shared__ double sL[];
  const int m = M.m[J], ld = m + 1;
  double *P = panel + M.poff[J];
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sL[(e / m) * ld + e % m] = P[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int rows = M.prows[J];
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t p = m + int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); p < rows; p += nw) {
    double *row = P + p * m;
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; u++) x[u] = lane + 32 * u < m ? row[lane + 32 * u] : 0.0;
    for (int c = 0; c < m; c++) {
      const int uc = c >> 5;
      double xc = 0.0;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (u == uc) xc = x[u];
      xc = __shfl_sync(FULL, xc, c & 31) / sL[c * ld + c];
      if ((c & 31) == lane) {
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (u == uc) x[u] = xc;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int s = lane + 32 * u;
        if (s > c && s < m) x[u] -= xc * sL[s * ld + c];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (lane + 32 * u < m) row[lane + 32 * u] = x[u];
  }
}

// Schur update of supernode J: C = L_below L_below^T on the lower triangle,
// 64 x 64 tiles (8 warps of 16 x 32, DMMA m8n8k4), subtracted into the panels.
constexpr int ST = 64;

__global__ void __launch_bounds__(256) chol_schur_kernel(CholMeta M, double *panel, int32_t J, int32_t R,
                                                         int32_t ntile) {
  extern __shared__ double sm[];
  const int m = M.m[J], m4 = (m + 3) & ~3, ldk = ((m4 + 15) & ~15) + 4;
  double *sA = sm, *sB = sm + ST * ldk;
  __shared__ int32_t rI[ST], ri[ST], cK[ST], ck[ST];
  // tile (ti, tk), tk <= ti, from the linear index
  const int x = blockIdx.x;
  int ti = int((sqrt(8.0 * x + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= x) ti++;
  while (ti * (ti + 1) / 2 > x) ti--;
  const int tk = x - ti * (ti + 1) / 2;
  const bool diag = ti == tk;
  const double *P = panel + M.poff[J] + int64_t(m) * m;  // below rows
  const int32_t *blk = M.blk + M.roff[J] + m, *grow = M.grow + M.roff[J] + m;
  // stage the two row blocks with 8-byte async copies (one round trip)
  for (int e = threadIdx.x; e < ST * m4; e += blockDim.x) {
    const int r = e / m4, k = e % m4;
    const int ra = ti * ST + r, rb = tk * ST + r;
    double *da = &sA[r * ldk + k];
    if (ra < R && k < m) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(unsigned(__cvta_generic_to_shared(da))),
                   "l"(P + int64_t(ra) * m + k));
    } else {
      *da = 0.0;
    }
    if (!diag) {
      double *db = &sB[r * ldk + k];
      if (rb < R && k < m)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(unsigned(__cvta_generic_to_shared(db))),
                     "l"(P + int64_t(rb) * m + k));
      else
        *db = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  for (int r = threadIdx.x; r < ST; r += blockDim.x) {
    const int ra = ti * ST + r, rb = tk * ST + r;
    if (ra < R) {
      rI[r] = blk[ra];
      ri[r] = grow[ra] - int32_t(M.start[rI[r]]);
    }
    if (rb < R) {
      cK[r] = blk[rb];
      ck[r] = grow[rb] - int32_t(M.start[cK[r]]);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const double *B = diag ? sA : sB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = lane >> 2, q = lane & 3;
  const int m0 = (warp >> 1) * 16, n0 = (warp & 1) * 32;
  if (diag && n0 > m0 + 15) return;  // strictly above the diagonal
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < m4; k0 += 4) {
    double a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; i++) a[i] = sA[(m0 + 8 * i + r) * ldk + k0 + q];
#pragma unroll
    for (int j = 0; j < 4; j++) b[j] = B[(n0 + 8 * j + r) * ldk + k0 + q];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) dmma(acc[i][j], a[i], b[j]);
  }
  // epilogue in three batches of independent loads: block offsets, targets, stores
  int32_t pv[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int lr = m0 + 8 * i + r, lc = n0 + 8 * j + 2 * q + e;
        const int ra = ti * ST + lr, rb = tk * ST + lc;
        pv[i][j][e] = (ra < R && rb <= ra) ? __ldg(M.pos + int64_t(cK[lc]) * M.ns + rI[lr]) : -1;
      }
  int64_t dst[2][4][2];
  double old[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int lr = m0 + 8 * i + r, lc = n0 + 8 * j + 2 * q + e;
        const int32_t K = cK[lc];
        dst[i][j][e] = pv[i][j][e] >= 0 ? M.poff[K] + int64_t(pv[i][j][e] + ri[lr]) * M.m[K] + ck[lc] : -1;
        old[i][j][e] = dst[i][j][e] >= 0 ? panel[dst[i][j][e]] : 0.0;
      }
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int e = 0; e < 2; e++)
        if (dst[i][j][e] >= 0) panel[dst[i][j][e]] = old[i][j][e] - acc[i][j][e];
}

// Solve, per supernode J.  Forward: (1) chol_diag_kernel<false>: x_J =
// L_JJ^-1 x_J (one warp); (2) chol_fwd_update_kernel: x[grow[p]] -= L_below[p]
// . x_J for the rows below (one warp per row, lanes over the columns).
// Backward: (1) chol_bwd_partial_kernel: per CTA, the partial sums
// sum_p L_below[p][c] x[grow[p]] over its rows (fixed grid, fixed order);
// (2) chol_diag_kernel<true>: x_J = L_JJ^-T (x_J - sum of the partials).
template <bool TRANS>
__global__ void __launch_bounds__(32) chol_diag_kernel(CholMeta M, const double *panel, double *x, int32_t J,
                                                       const double *part, int nparts) {
  const int m = M.m[J], lane = threadIdx.x;
  const double *P = panel + M.poff[J];
  const int64_t s0 = M.start[J];
  double v[4];
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const int c = lane + 32 * u;
    double t = 0.0;
    if (c < m) {
      t = x[s0 + c];
      if (TRANS)
        for (int w = 0; w < nparts; w++) t -= part[w * 128 + c];
    }
    v[u] = t;
  }
  if (!TRANS) {
    for (int c = 0; c < m; c++) {
      const int uc = c >> 5;
      double vc = 0.0;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (u == uc) vc = v[u];
      vc = __shfl_sync(FULL, vc, c & 31) / P[int64_t(c) * m + c];
      if (lane == (c & 31)) x[s0 + c] = vc;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int s = lane + 32 * u;
        if (s > c && s < m) v[u] -= vc * P[int64_t(s) * m + c];
      }
    }
  } else {
    for (int c = m - 1; c >= 0; c--) {
      const int uc = c >> 5;
      double vc = 0.0;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (u == uc) vc = v[u];
      vc = __shfl_sync(FULL, vc, c & 31) / P[int64_t(c) * m + c];
      if (lane == (c & 31)) x[s0 + c] = vc;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int s = lane + 32 * u;
        if (s < c) v[u] -= vc * P[int64_t(c) * m + s];
      }
    }
  }
}

__global__ void __launch_bounds__(256) chol_fwd_update_kernel(CholMeta M, const double *panel, double *x, int32_t J) {
  const int m = M.m[J], lane = threadIdx.x & 31;
  const double *P = panel + M.poff[J];
  const int64_t s0 = M.start[J];
  double xj[4];
#pragma unroll
  for (int u = 0; u < 4; u++) xj[u] = lane + 32 * u < m ? x[s0 + lane + 32 * u] : 0.0;
  const int rows = M.prows[J];
  const int32_t *grow = M.grow + M.roff[J];
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t p = m + int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); p < rows; p += nw) {
    const double *row = P + p * m;
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (lane + 32 * u < m) s += row[lane + 32 * u] * xj[u];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) x[grow[p]] -= s;
  }
}

constexpr int BWD_CTAS = 64;

__global__ void __launch_bounds__(256) chol_bwd_partial_kernel(CholMeta M, const double *panel, const double *x,
                                                               int32_t J, double *part) {
  __shared__ double red[8][128];
  const int m = M.m[J], lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double *P = panel + M.poff[J];
  const int rows = M.prows[J];
  const int32_t *grow = M.grow + M.roff[J];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t p = m + int64_t(blockIdx.x) * 8 + warp; p < rows; p += int64_t(gridDim.x) * 8) {
    const double xp = x[grow[p]];
    const double *row = P + p * m;
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (lane + 32 * u < m) acc[u] += row[lane + 32 * u] * xp;
  }
#pragma unroll
  for (int u = 0; u < 4; u++) red[warp][lane + 32 * u] = acc[u];
  __syncthreads();
  for (int c = threadIdx.x; c < 128; c += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < 8; w++) s += red[w][c];
    part[blockIdx.x * 128 + c] = s;
  }
}

int n_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

size_t schur_smem(int m) {
  const int m4 = (m + 3) & ~3, ldk = ((m4 + 15) & ~15) + 4;
  return size_t(2) * ST * ldk * sizeof(double);
}

// supernodal symbolic factorisation: struct(J) = A's column J (lower) U {J}
// U the structures of J's children minus themselves; parent(J) = the
// smallest block of struct(J) below J
void symbolic(int32_t ns, const std::vector<std::vector<int32_t>> &acol, std::vector<int32_t> &parent,
              std::vector<std::vector<int32_t>> &st) {
  parent.assign(ns, -1);
  st.assign(ns, {});
  std::vector<std::vector<int32_t>> children(ns);
  for (int32_t J = 0; J < ns; J++) {
    std::vector<int32_t> s = acol[J];
    s.push_back(J);
    for (int32_t ch : children[J]) s.insert(s.end(), st[ch].begin() + 1, st[ch].end());
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    st[J] = std::move(s);
    if (st[J].size() > 1) {
      parent[J] = st[J][1];
      children[parent[J]].push_back(J);
    }
  }
}

template <typename T>
size_t put(std::vector<unsigned char> &img, const std::vector<T> &v) {
  const size_t off = (img.size() + 255) & ~size_t(255);
  img.resize(off + v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(img.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

}  // namespace

extern "C" {

h2sp_status h2sp_chol_analyse(h2sp_plan P, int amalgamate, h2sp_chol *out, int64_t *panel_doubles,
                              int64_t *meta_bytes) {
  if (amalgamate > 128) return fail(H2SP_EINVAL, "chol: amalgamated supernodes are at most 128 wide");
  if (!P || !out) return fail(H2SP_EINVAL, "chol: NULL argument");
  *out = nullptr;
  if (!P->sym) return fail(H2SP_EUNSUPPORTED, "chol: symmetric plans only (S SPD, Proposition P:504-509)");
  if (P->world != 1) return fail(H2SP_EUNSUPPORTED, "chol: unsharded plans only");
  if (P->bench) return fail(H2SP_EUNSUPPORTED, "chol: stored-S plans only (no H2SP_PLAN_BENCH)");
  try {
    auto *c = new h2sp_chol_s();
    c->n = P->N;
    const auto *rows = reinterpret_cast<const CsrBlockRow *>(P->meta.data() + P->csr_rows_off);
    const auto *blocks = reinterpret_cast<const CsrBlock *>(P->meta.data() + P->csr_blocks_off);
    const int64_t nr = P->n_csr_rows;
    // supernodes = the row groups, in S order
    std::vector<int32_t> sgrp(size_t(c->n), -1);
    for (int64_t r = 0; r < nr; r++) {
      c->start.push_back(rows[r].row0);
      c->m.push_back(rows[r].m_r);
      if (rows[r].m_r > 128) {
        delete c;
        return fail(H2SP_EUNSUPPORTED, "chol: supernode wider than 128 rows");
      }
      for (int32_t a = 0; a < rows[r].m_r; a++) sgrp[size_t(rows[r].row0 + a)] = int32_t(r);
    }
    c->ns = int32_t(nr);
    c->start.push_back(c->n);
    for (int64_t i = 0; i < c->n; i++)
      if (sgrp[size_t(i)] < 0) {
        delete c;
        return fail(H2SP_EUNSUPPORTED, "chol: S row outside every group");
      }
    const int32_t ns0 = c->ns;
    // A's lower block pattern by column
    std::vector<std::vector<int32_t>> acol(ns0);
    for (int64_t r = 0; r < nr; r++)
      for (int32_t j = 0; j < rows[r].nblk; j++) {
        const CsrBlock &b = blocks[rows[r].blk_begin + j];
        const int32_t J = sgrp[size_t(b.col0)];
        if (c->start[J] != b.col0 || c->m[J] != b.m_c) {
          delete c;
          return fail(H2SP_EUNSUPPORTED, "chol: S block not aligned with the row groups");
        }
        if (J <= r) acol[J].push_back(int32_t(r));
      }
    symbolic(ns0, acol, c->parent, c->st);
    // relaxed amalgamation: a supernode J whose parent is J + 1 joins it (one
    // wider panel: one potrf / trsm / Schur pass instead of two, K = the summed
    // width) while the merged width stays <= amalgamate and the explicit zeros
    // it adds to J's columns (rows of struct(J + 1) not in struct(J)) stay
    // under a quarter of J's rows; then the same symbolic factorisation on the
    // coarser partition (its structures contain the zeros)
    if (amalgamate > 0) {
      auto rows_of = [&](int32_t J) {
        int64_t r = 0;
        for (int32_t I : c->st[J]) r += c->m[I];
        return r;
      };
      std::vector<int32_t> cgrp(ns0);
      std::vector<int64_t> cstart;
      std::vector<int32_t> cm;
      for (int32_t J = 0; J < ns0; J++) {
        bool join = false;
        if (J > 0 && c->parent[J - 1] == J && cm.back() + c->m[J] <= amalgamate) {
          const int64_t rj = rows_of(J - 1), rp = rows_of(J);
          join = rp + c->m[J - 1] - rj <= rj / 4;
        }
        if (join) {
          cm.back() += c->m[J];
        } else {
          cstart.push_back(c->start[J]);
          cm.push_back(c->m[J]);
        }
        cgrp[J] = int32_t(cm.size()) - 1;
      }
      const int32_t nc = int32_t(cm.size());
      std::vector<std::vector<int32_t>> ccol(nc);
      for (int32_t J = 0; J < ns0; J++)
        for (int32_t I : acol[J]) ccol[cgrp[J]].push_back(cgrp[I]);
      for (auto &v : ccol) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
      }
      for (int64_t i = 0; i < c->n; i++) sgrp[size_t(i)] = cgrp[sgrp[size_t(i)]];
      cstart.push_back(c->n);
      c->start = std::move(cstart);
      c->m = std::move(cm);
      c->ns = nc;
      symbolic(nc, ccol, c->parent, c->st);
    }
    const int32_t ns = c->ns;
    c->mmax = ns ? *std::max_element(c->m.begin(), c->m.end()) : 0;
    // layout
    c->poff.assign(size_t(ns) + 1, 0);
    c->prows.assign(ns, 0);
    c->roff.assign(size_t(ns) + 1, 0);
    std::vector<int32_t> pos(size_t(ns) * ns, -1), blk, grow;
    double fl = 0.0;
    for (int32_t J = 0; J < ns; J++) {
      int32_t rws = 0;
      for (int32_t I : c->st[J]) {
        pos[size_t(J) * ns + I] = rws;
        for (int32_t a = 0; a < c->m[I]; a++) {
          blk.push_back(I);
          grow.push_back(int32_t(c->start[I] + a));
        }
        rws += c->m[I];
      }
      c->prows[J] = rws;
      c->poff[J + 1] = c->poff[J] + int64_t(rws) * c->m[J];
      c->roff[J + 1] = c->roff[J] + rws;
      const double mj = c->m[J], R = rws - mj;
      fl += mj * mj * mj / 3.0 + R * mj * mj + R * R * mj;
    }
    c->flops = fl;
    std::vector<unsigned char> &img = c->meta;
    c->o_start = put(img, c->start);
    c->o_m = put(img, c->m);
    c->o_poff = put(img, c->poff);
    c->o_prows = put(img, c->prows);
    c->o_roff = put(img, c->roff);
    c->o_pos = put(img, pos);
    c->o_blk = put(img, blk);
    c->o_grow = put(img, grow);
    c->o_sgrp = put(img, sgrp);
    img.resize((img.size() + 255) & ~size_t(255));
    if (panel_doubles) *panel_doubles = c->poff[ns];
    if (meta_bytes) *meta_bytes = int64_t(img.size());
    *out = c;
    return H2SP_OK;
  } catch (const std::bad_alloc &) {
    return fail(H2SP_ENOMEM, "chol: host allocation failed");
  }
}

h2sp_status h2sp_chol_info(h2sp_chol c, int32_t *ns, int32_t *parent, int64_t *panel_rows, double *flops) {
  if (!c) return fail(H2SP_EINVAL, "chol: NULL handle");
  if (ns) *ns = c->ns;
  if (parent) std::memcpy(parent, c->parent.data(), c->parent.size() * sizeof(int32_t));
  if (panel_rows)
    for (int32_t J = 0; J < c->ns; J++) panel_rows[J] = c->prows[J];
  if (flops) *flops = c->flops;
  return H2SP_OK;
}

h2sp_status h2sp_chol_supernodes(h2sp_chol c, int64_t *start) {
  if (!c || !start) return fail(H2SP_EINVAL, "chol: NULL argument");
  std::memcpy(start, c->start.data(), c->start.size() * sizeof(int64_t));
  return H2SP_OK;
}

h2sp_status h2sp_chol_struct(h2sp_chol c, int32_t J, int32_t *blocks, int32_t cap, int32_t *count) {
  if (!c || J < 0 || J >= c->ns) return fail(H2SP_EINVAL, "chol: bad supernode");
  const auto &s = c->st[J];
  if (count) *count = int32_t(s.size());
  if (blocks) std::memcpy(blocks, s.data(), std::min<size_t>(s.size(), size_t(std::max(cap, 0))) * sizeof(int32_t));
  return H2SP_OK;
}

h2sp_status h2sp_chol_upload(h2sp_chol c, void *meta, size_t meta_bytes, void *stream) {
  if (!c || !meta || meta_bytes < c->meta.size()) return fail(H2SP_EINVAL, "chol: meta buffer too small");
  CCK(cudaMemcpyAsync(meta, c->meta.data(), c->meta.size(), cudaMemcpyHostToDevice,
                      static_cast<cudaStream_t>(stream)));
  return H2SP_OK;
}

h2sp_status h2sp_chol_factor(h2sp_chol c, const h2sp_csr *S, const void *meta, double *panel, void *stream) {
  if (!c || !S || !meta || !panel) return fail(H2SP_EINVAL, "chol: NULL argument");
  if (S->n != c->n) return fail(H2SP_EINVAL, "chol: S size differs from the plan");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const CholMeta M = meta_view(c, static_cast<const unsigned char *>(meta));
  int32_t *status = nullptr;
  CCK(cudaMallocAsync(reinterpret_cast<void **>(&status), sizeof(int32_t), st));
  const int32_t big = INT32_MAX;
  CCK(cudaMemcpyAsync(status, &big, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CCK(cudaMemsetAsync(panel, 0, size_t(c->poff[c->ns]) * sizeof(double), st));
  const int sms = n_sms();
  chol_scatter_kernel<<<sms * 8, 256, 0, st>>>(M, S->rowptr, S->col, S->val, panel);
  CCK(cudaGetLastError());
  const size_t pot_smem = size_t(c->mmax) * (c->mmax + 1) * sizeof(double);
  CCK(cudaFuncSetAttribute(chol_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pot_smem)));
  CCK(cudaFuncSetAttribute(chol_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pot_smem)));
  CCK(cudaFuncSetAttribute(chol_schur_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(schur_smem(c->mmax))));
  for (int32_t J = 0; J < c->ns; J++) {
    const int m = c->m[J];
    if (m == 0) continue;
    const size_t sm = size_t(m) * (m + 1) * sizeof(double);
    chol_potrf_kernel<<<1, 512, sm, st>>>(M, panel, J, status);
    const int32_t R = c->prows[J] - m;
    if (R > 0) {
      const int grid = int(std::min<int64_t>(int64_t(sms) * 4, (R + 7) / 8));
      chol_trsm_kernel<<<grid, 256, sm, st>>>(M, panel, J);
      const int64_t T = (R + ST - 1) / ST, nt = T * (T + 1) / 2;
      if (nt > INT32_MAX) return fail(H2SP_EUNSUPPORTED, "chol: Schur update too large");
      chol_schur_kernel<<<unsigned(nt), 256, schur_smem(m), st>>>(M, panel, J, R, int32_t(nt));
    }
  }
  CCK(cudaGetLastError());
  int32_t bad = 0;
  CCK(cudaMemcpyAsync(&bad, status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CCK(cudaFreeAsync(status, st));
  CCK(cudaStreamSynchronize(st));
  if (bad != INT32_MAX) return fail(H2SP_EINVAL, "chol: S not positive definite (supernode " + std::to_string(bad) + ")");
  return H2SP_OK;
}

h2sp_status h2sp_chol_solve(h2sp_chol c, const void *meta, const double *panel, const double *b, double *x,
                            void *stream) {
  if (!c || !meta || !panel || !b || !x) return fail(H2SP_EINVAL, "chol: NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const CholMeta M = meta_view(c, static_cast<const unsigned char *>(meta));
  if (x != b) CCK(cudaMemcpyAsync(x, b, size_t(c->n) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  double *part = nullptr;
  CCK(cudaMallocAsync(reinterpret_cast<void **>(&part), size_t(BWD_CTAS) * 128 * sizeof(double), st));
  const int sms = n_sms();
  for (int32_t J = 0; J < c->ns; J++) {
    chol_diag_kernel<false><<<1, 32, 0, st>>>(M, panel, x, J, nullptr, 0);
    const int32_t R = c->prows[J] - c->m[J];
    if (R > 0)
      chol_fwd_update_kernel<<<int(std::min<int64_t>(int64_t(sms) * 8, (R + 7) / 8)), 256, 0, st>>>(M, panel, x, J);
  }
  for (int32_t J = c->ns - 1; J >= 0; J--) {
    const int32_t R = c->prows[J] - c->m[J];
    const int np = R > 0 ? int(std::min<int64_t>(BWD_CTAS, (R + 7) / 8)) : 0;
    if (np) chol_bwd_partial_kernel<<<np, 256, 0, st>>>(M, panel, x, J, part);
    chol_diag_kernel<true><<<1, 32, 0, st>>>(M, panel, x, J, part, np);
  }
  CCK(cudaGetLastError());
  CCK(cudaFreeAsync(part, st));
  return H2SP_OK;
}

void h2sp_chol_destroy(h2sp_chol c) { delete c; }

}  // extern "C"
