// PROTOTYPE (not compiled): warp-specialised level-0 congruence, extracted from
// paper_1705_04601_b200/csrc/kernels.cu of round 1.  Parity-green with all GPU
// tests (H2SP_WY_WS=1).  Alone on config 2: 563 us with the even-k fast store
// pass and setmaxnreg 96/40 (775 us without the fast pass; 370 us with the
// stores skipped) vs 448 us for pair_wy_kernel<16> -- the 4-warp store group is
// the bottleneck.  Needs: async_tile / wy_load with a (tid, nthr)
// thread subset, and the dispatch in launch_build (k == 0 && wy_kp == 16).
// --------------------------------------------------------------------------
// Warp-specialised level-0 compact-WY congruence (k <= 16; H2SP_WY_WS=1):
// 8 DMMA warps compute the pairs of a chunk exactly as pair_wy_kernel, stage
// each finished H in shared memory and go on with the next pair, while a 4-warp
// store group writes the staged H out -- S rows, bb and row strips row-major,
// the mirror block and the column strips column-major (both coalesced).  Named
// barriers hand the staging buffer back and forth; setmaxnreg moves registers
// from the store warpgroup (32) to the DMMA warpgroups (104), so two CTAs
// (2 x 384 threads) still fit an SM.  P aliases V_t, which is reloaded per pair.
// --------------------------------------------------------------------------
struct PairWsCfg {
  static constexpr int KP = 16, NP = 64, LD = NP + 4, LDV = KP + 4, LDH = NP + 1;
  static constexpr int MMA_THREADS = 256, STORE_THREADS = 128, THREADS = MMA_THREADS + STORE_THREADS;
  static constexpr int V_D = NP * LDV, M_D = KP * LD, G_D = NP * LD, H_D = NP * LDH;
  static_assert(KP * LD <= V_D, "P aliases V_t");
  static constexpr size_t SMEM = size_t(2 * V_D + 2 * M_D + G_D + H_D) * sizeof(double);
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// The store group's half of the pipeline: write one staged H (sH, ld LDH).
__device__ __forceinline__ void ws_store_pair(const PairArgs &A, const PairItem &it, const double *sH, int tid) {
  constexpr int LDH = PairWsCfg::LDH;
  const int nt = it.nt, ns = it.ns, kt = it.kt, ks = it.ks;
  const bool dsym = A.sym && it.s == it.t;
  const int sw = tid >> 5, lane = tid & 31;
  // H_sym[i][j] = H[min][max] inside the symmetric diagonal block (nn and bb parts)
  auto hval = [&](int r, int c) -> double {
    if (dsym && ((r >= kt) == (c >= ks))) {
      const int a = (r >= kt) ? r - kt : r, b = (c >= ks) ? c - ks : c, off_r = (r >= kt) ? kt : 0,
                off_c = (c >= ks) ? ks : 0;
      return a <= b ? sH[(off_r + a) * LDH + off_c + b] : sH[(off_r + b) * LDH + off_c + a];
    }
    return sH[r * LDH + c];
  };
  if (!dsym && ((kt | ks) & 1) == 0) {
    // fast pass 1: even k_t, k_s -> a column pair never straddles a region edge;
    // the lane's column class is fixed, one 16-byte store per row
    const int c0 = 2 * lane;
    if (c0 < ns) {
      const bool two = c0 + 1 < ns;
      for (int row = sw; row < nt; row += 4) {
        double *d = nullptr;
        if (row < kt) {
          if (c0 < ks) {
            if (it.bb_dst >= 0) d = A.bb_out + it.bb_dst + row * ks + c0;
          } else if (it.yr_dst >= 0) {
            d = A.yr + it.yr_dst + int64_t(row) * it.yr_ld + (c0 - ks);
          }
        } else if (c0 >= ks && it.s_dst >= 0) {
          d = A.s_val + it.s_dst + int64_t(row - kt) * it.s_ld + (c0 - ks);
        }
        if (d) {
          const double v0 = sH[row * LDH + c0];
          if (two)
            store2(d, v0, sH[row * LDH + c0 + 1]);
          else
            *d = v0;
        }
      }
    }
  } else
  // pass 1, row-major: lane -> column pair (2 lane, 2 lane + 1)
  for (int row = sw; row < nt; row += 4) {
    const int c0 = 2 * lane;
    if (c0 >= ns) continue;
    const bool two = c0 + 1 < ns;
    const double v0 = hval(row, c0), v1 = two ? hval(row, c0 + 1) : 0.0;
    double *d0 = nullptr, *d1 = nullptr;
    for (int e = 0; e < (two ? 2 : 1); e++) {
      const int c = c0 + e;
      double *d = nullptr;
      if (row >= kt && c >= ks) {
        if (it.s_dst >= 0) d = A.s_val + it.s_dst + int64_t(row - kt) * it.s_ld + (c - ks);
      } else if (row < kt && c < ks) {
        if (it.bb_dst >= 0) d = A.bb_out + it.bb_dst + row * ks + c;
      } else if (row < kt) {
        if (it.yr_dst >= 0) d = A.yr + it.yr_dst + int64_t(row) * it.yr_ld + (c - ks);
      }
      (e ? d1 : d0) = d;
    }
    if (d0 && d1 == d0 + 1)
      store2(d0, v0, v1);
    else {
      if (d0) *d0 = v0;
      if (d1) *d1 = v1;
    }
  }
  // pass 2, column-major: lane -> rows lane, lane + 32 (mirror block, column strips)
  if (it.s_dst_m < 0 && it.yc_dst < 0) return;
  for (int c = sw; c < ns; c += 4) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int row = lane + 32 * h;
      if (row >= nt || row < kt) continue;
      const double v = sH[row * LDH + c];
      if (c >= ks) {
        if (it.s_dst_m >= 0) A.s_val[it.s_dst_m + int64_t(c - ks) * it.s_ld_m + (row - kt)] = v;
      } else if (it.yc_dst >= 0) {
        A.yc[it.yc_dst + int64_t(c) * it.yc_ld + (row - kt)] = v;
      }
    }
  }
}

__global__ void __launch_bounds__(PairWsCfg::THREADS, 2) pair_wy_ws_kernel(PairArgs A, const double *wy_row,
                                                                           const double *wy_col) {
  using C = PairWsCfg;
  constexpr int KP = C::KP, LD = C::LD, LDV = C::LDV, LDH = C::LDH, TN = 8;
  extern __shared__ __align__(16) double sm[];
  double *sVt = sm, *sMt = sVt + C::V_D, *sG = sMt + C::M_D, *sVs = sG + C::G_D, *sMs = sVs + C::V_D;
  double *sH = sMs + C::M_D;
  double *sP = sVt;  // after step 1
  __shared__ __align__(16) PairItem s_it[PAIR_CHUNK_MAX];
  const Chunk ch = A.chunks[blockIdx.x];
  stage_items(A.items, ch, s_it);  // all 384 threads
  const int warp = threadIdx.x >> 5;
  if (warp >= 8) {  // ---- store warpgroup
    // the CTA holds 80 registers / thread (2 CTAs x 384 threads); the store group
    // gives 48 back so the DMMA warps can grow to 104: (104 - 80) * 256 == (80 - 32) * 128
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n");
    const int tid = threadIdx.x - C::MMA_THREADS;
    named_arrive(3, C::THREADS);  // staging buffer starts empty
    for (int p = ch.begin; p < ch.end; p++) {
      named_sync(2, C::THREADS);  // H of pair p staged
      if (!(A.debug & 1)) ws_store_pair(A, s_it[p - ch.begin], sH, tid);
      named_arrive(3, C::THREADS);
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 96;\n");
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int m0 = warp * 8;
  const int src_lo = r * 4 + (q >> 1), src_hi = src_lo + 2;
  // prologue: V_t, M_t, G, V_s, M_s of the first pair
  {
    const PairItem &i0 = s_it[0];
    wy_load<KP>(sVt, sMt, wy_row, i0.t, threadIdx.x, C::MMA_THREADS);
    async_tile<64, 64, LD>(sG, A.close + i0.g_src[0], i0.nt, i0.ns, A.B, A.chunks, threadIdx.x, C::MMA_THREADS);
    wy_load<KP>(sVs, sMs, wy_col, i0.s, threadIdx.x, C::MMA_THREADS);
    cp_commit();
  }
  for (int p = ch.begin; p < ch.end; p++) {
    const PairItem &it = s_it[p - ch.begin];
    const bool more = p + 1 < ch.end && !(A.debug & 2);
    cp_wait_all();
    named_sync(1, C::MMA_THREADS);
    // ---- step 1: P = V_t^T G (KP x 64), warp w: columns 8w..8w+7
    double pacc[2][KP / 8][2];
#pragma unroll
    for (int i = 0; i < KP / 8; i++) pacc[0][i][0] = pacc[0][i][1] = pacc[1][i][0] = pacc[1][i][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 64; k0 += 4) {
      const double b = sG[(k0 + q) * LD + m0 + r];
#pragma unroll
      for (int i = 0; i < KP / 8; i++) dmma(pacc[(k0 >> 2) & 1][i], sVt[(k0 + q) * LDV + i * 8 + r], b);
    }
    named_sync(1, C::MMA_THREADS);  // every warp is done with V_t: P overwrites it
#pragma unroll
    for (int i = 0; i < KP / 8; i++) {
      sP[(i * 8 + r) * LD + m0 + 2 * q] = pacc[0][i][0] + pacc[1][i][0];
      sP[(i * 8 + r) * LD + m0 + 2 * q + 1] = pacc[0][i][1] + pacc[1][i][1];
    }
    named_sync(1, C::MMA_THREADS);
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
    named_sync(1, C::MMA_THREADS);  // G, P (= V_t) and M_t are dead
    if (more) {
      const PairItem &nx = s_it[p + 1 - ch.begin];
      async_tile<64, 64, LD>(sG, A.close + nx.g_src[0], nx.nt, nx.ns, A.B, A.chunks, threadIdx.x, C::MMA_THREADS);
      if (nx.t != it.t) {
        wy_load<KP>(sVt, sMt, wy_row, nx.t, threadIdx.x, C::MMA_THREADS);
      } else {  // same block row: V_t again (P overwrote it), M_t stays
        const double *g = wy_row + int64_t(nx.t) * (2 * 64 * KP);
        async_tile<64, KP, LDV>(sVt, g, 64, KP, KP, g, threadIdx.x, C::MMA_THREADS);
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
    named_sync(1, C::MMA_THREADS);  // V_s / M_s are dead
    if (more) {
      wy_load<KP>(sVs, sMs, wy_col, s_it[p + 1 - ch.begin].s, threadIdx.x, C::MMA_THREADS);
      cp_commit();
    }
    // ---- hand H to the store group
    named_sync(3, C::THREADS);  // staging buffer drained
#pragma unroll
    for (int j = 0; j < TN; j++) {
      sH[(m0 + r) * LDH + j * 8 + 2 * q] = H[j][0];
      sH[(m0 + r) * LDH + j * 8 + 2 * q + 1] = H[j][1];
    }
    named_arrive(2, C::THREADS);
  }
  named_sync(3, C::THREADS);  // pairs with the store group's last arrive
}

static h2sp_status launch_pairs_ws(const PairArgs &a, const double *wy_row, const double *wy_col, int64_t nchunks,
                                   cudaStream_t st) {
  using C = PairWsCfg;
  static bool attr = false;
  if (!attr) {
    H2SP_CK(cudaFuncSetAttribute(pair_wy_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)));
    attr = true;
  }
  pair_wy_ws_kernel<<<unsigned(nchunks), C::THREADS, C::SMEM, st>>>(a, wy_row, wy_col);
  H2SP_CK(cudaGetLastError());
  return H2SP_OK;
}

