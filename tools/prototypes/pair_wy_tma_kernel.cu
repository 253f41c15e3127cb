// PROTOTYPE (not compiled): level-0 congruence with the nn block and its mirror
// staged in shared memory and written by cp.async.bulk row copies.  Parity-green
// with all GPU tests (H2SP_WY_TMA=1) but 487 us vs 448 us alone on config 2
// (353 us with the stores skipped); see DESIGN.md §6.
// --------------------------------------------------------------------------
// Level-0 compact-WY congruence with TMA bulk stores (k <= 16; H2SP_WY_TMA=1).
// As pair_wy_kernel, but the frozen nn block of each pair (and its transpose,
// the mirror block) is staged in shared memory and written by one
// cp.async.bulk row copy per S row, issued by single threads and completed in
// the background while the CTA computes the next pair; only the small bb /
// row-strip / column-strip parts are stored from registers.  Pairs whose nn
// block is not 8-aligned, wider than 48, symmetric-diagonal or not 16-byte
// aligned in S fall back to the register scatter.  P aliases V_t (reloaded per
// pair) to make room for the two staging buffers.
// --------------------------------------------------------------------------
struct PairTmaCfg {
  static constexpr int KP = 16, NP = 64, LD = NP + 4, LDV = KP + 4, NN = 48, LDN = NN + 2;
  static constexpr int THREADS = 256;
  static constexpr int V_D = NP * LDV, M_D = KP * LD, G_D = NP * LD, N_D = NN * LDN;
  static_assert(KP * LD <= V_D, "P aliases V_t");
  static constexpr size_t SMEM = size_t(2 * V_D + 2 * M_D + G_D + 2 * N_D) * sizeof(double);
};

__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(PairTmaCfg::THREADS, 2) pair_wy_tma_kernel(PairArgs A, const double *wy_row,
                                                                             const double *wy_col) {
  using C = PairTmaCfg;
  constexpr int KP = C::KP, LD = C::LD, LDV = C::LDV, LDN = C::LDN, TN = 8;
  extern __shared__ __align__(16) double sm[];
  double *sVt = sm, *sMt = sVt + C::V_D, *sG = sMt + C::M_D, *sVs = sG + C::G_D, *sMs = sVs + C::V_D;
  double *sN = sMs + C::M_D, *sNt = sN + C::N_D;
  double *sP = sVt;
  __shared__ __align__(16) PairItem s_it[PAIR_CHUNK_MAX];
  const Chunk ch = A.chunks[blockIdx.x];
  stage_items(A.items, ch, s_it);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int m0 = warp * 8;
  const int src_lo = r * 4 + (q >> 1), src_hi = src_lo + 2;
  {
    const PairItem &i0 = s_it[0];
    wy_load<KP>(sVt, sMt, wy_row, i0.t);
    async_tile<64, 64, LD>(sG, A.close + i0.g_src[0], i0.nt, i0.ns, A.B, A.chunks);
    wy_load<KP>(sVs, sMs, wy_col, i0.s);
    cp_commit();
  }
  bool bulk_pending = false;  // thread-local: this thread issued bulk copies not yet waited for
  for (int p = ch.begin; p < ch.end; p++) {
    const PairItem &it = s_it[p - ch.begin];
    const bool more = p + 1 < ch.end && !(A.debug & 2);
    cp_wait_all();
    __syncthreads();
    // ---- step 1: P = V_t^T G
    double pacc[2][KP / 8][2];
#pragma unroll
    for (int i = 0; i < KP / 8; i++) pacc[0][i][0] = pacc[0][i][1] = pacc[1][i][0] = pacc[1][i][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 64; k0 += 4) {
      const double b = sG[(k0 + q) * LD + m0 + r];
#pragma unroll
      for (int i = 0; i < KP / 8; i++) dmma(pacc[(k0 >> 2) & 1][i], sVt[(k0 + q) * LDV + i * 8 + r], b);
    }
    __syncthreads();  // V_t is dead: P overwrites it
#pragma unroll
    for (int i = 0; i < KP / 8; i++) {
      sP[(i * 8 + r) * LD + m0 + 2 * q] = pacc[0][i][0] + pacc[1][i][0];
      sP[(i * 8 + r) * LD + m0 + 2 * q + 1] = pacc[0][i][1] + pacc[1][i][1];
    }
    __syncthreads();
    // ---- step 2: T1 = G - M_t^T P
    double H[TN][2];
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
    __syncthreads();  // G, P (= V_t), M_t dead
    if (more) {
      const PairItem &nx = s_it[p + 1 - ch.begin];
      async_tile<64, 64, LD>(sG, A.close + nx.g_src[0], nx.nt, nx.ns, A.B, A.chunks);
      if (nx.t != it.t) {
        wy_load<KP>(sVt, sMt, wy_row, nx.t);
      } else {
        const double *g = wy_row + int64_t(nx.t) * (2 * 64 * KP);
        async_tile<64, KP, LDV>(sVt, g, 64, KP, KP, g);
      }
      cp_commit();
    }
    // ---- step 3: R = T1 V_s
    double R[KP / 8][2], R2[KP / 8][2];
#pragma unroll
    for (int i = 0; i < KP / 8; i++) R[i][0] = R[i][1] = R2[i][0] = R2[i][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 64; k0 += 4) {
      const int jt = k0 >> 3;
      const int srcl = (k0 & 4) ? src_hi : src_lo;
      const double e0 = __shfl_sync(0xffffffffu, H[jt][0], srcl);
      const double e1 = __shfl_sync(0xffffffffu, H[jt][1], srcl);
      const double a = (q & 1) ? e1 : e0;
#pragma unroll
      for (int i = 0; i < KP / 8; i++) dmma((k0 & 4) ? R2[i] : R[i], a, sVs[(k0 + q) * LDV + i * 8 + r]);
    }
#pragma unroll
    for (int i = 0; i < KP / 8; i++) {
      R[i][0] += R2[i][0];
      R[i][1] += R2[i][1];
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
    // ---- stores
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
    const int mt = D.nt - D.kt, ms = D.ns - D.ks;
    const bool staged = !D.dsym && !(A.debug & 1) && ((D.kt | D.ks | D.nt | D.ns) & 7) == 0 && mt <= C::NN &&
                        ms <= C::NN && mt > 0 && ms > 0 &&
                        (D.s_dst < 0 || ((D.s_dst | int64_t(D.s_ld)) & 1) == 0) &&
                        (D.s_dst_m < 0 || ((D.s_dst_m | int64_t(D.s_ld_m)) & 1) == 0);
    if (staged) {
      // the previous pair's bulk copies must have read the staging buffers
      if (bulk_pending) {
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        bulk_pending = false;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < TN; j++) {
        const int row = m0 + r, col = j * 8 + 2 * q;
        if (m0 >= D.kt && j * 8 >= D.ks) {
          const int a = row - D.kt, b = col - D.ks;
          if (row < D.nt && col < D.ns) {
            sN[a * LDN + b] = H[j][0];
            sN[a * LDN + b + 1] = H[j][1];
            sNt[b * LDN + a] = H[j][0];
            sNt[(b + 1) * LDN + a] = H[j][1];
          }
        } else {
          scatter_pair2(A, D, m0, j * 8, row, col, H[j][0], H[j][1]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      const int t = threadIdx.x;
      if (t < mt && D.s_dst >= 0) {
        bulk_store(A.s_val + D.s_dst + int64_t(t) * D.s_ld, sN + t * LDN, unsigned(ms) * 8u);
        bulk_pending = true;
      } else if (t >= 128 && t - 128 < ms && D.s_dst_m >= 0) {
        const int b = t - 128;
        bulk_store(A.s_val + D.s_dst_m + int64_t(b) * D.s_ld_m, sNt + b * LDN, unsigned(mt) * 8u);
        bulk_pending = true;
      }
      if (bulk_pending) asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    } else if (!(A.debug & 1)) {
#pragma unroll
      for (int j = 0; j < TN; j++) scatter_pair2(A, D, m0, j * 8, m0 + r, j * 8 + 2 * q, H[j][0], H[j][1]);
    }
    __syncthreads();  // V_s / M_s dead
    if (more) {
      wy_load<KP>(sVs, sMs, wy_col, s_it[p + 1 - ch.begin].s);
      cp_commit();
    }
  }
  if (bulk_pending) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

static h2sp_status launch_pairs_tma(const PairArgs &a, const double *wy_row, const double *wy_col, int64_t nchunks,
                                    cudaStream_t st) {
  using C = PairTmaCfg;
  static bool attr = false;
  if (!attr) {
    H2SP_CK(cudaFuncSetAttribute(pair_wy_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)));
    attr = true;
  }
  pair_wy_tma_kernel<<<unsigned(nchunks), C::THREADS, C::SMEM, st>>>(a, wy_row, wy_col);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}

