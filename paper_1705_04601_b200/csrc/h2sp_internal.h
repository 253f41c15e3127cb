// Internal plan / work-list layout shared by the host plan (plan.cpp) and the
// sm_100a kernels (kernels.cu).  Every struct here is POD and lives verbatim in
// the device "meta" region at the start of the build workspace.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/h2sp.h"

namespace h2sp {

// Source kinds of the four quadrants of a merged close block G_ts (step (iv),
// P:238-250): children pair (t_a, s_b) is near -> its H basis x basis part;
// admissible -> its orthogonalised coupling D~.  "_T" = read the canonical
// (t <= s) block transposed (symmetric mode).
constexpr int STRIP_TN = 128;  // columns per strip tile (plan.cpp tiles, kernels.cu strip_kernel TN)
constexpr int STRIP_TN_SMALL = 64;  // narrower tiles for the small upper-level launches (more CTAs)
// tile width of the strip launches of level k (H2SP_STRIP_NARROW_FROM: first level
// with narrow tiles; default: none, measured no gain at levels >= 2, 3 or 4)
int strip_tn_of_level(int k);

enum GKind : int32_t { G_EMPTY = 0, G_BB = 1, G_BB_T = 2, G_DT = 3, G_DT_T = 4 };

// One congruence H_ts = Q^R_t^T G_ts Q^C_s for (t, s) in N_k (canonical t <= s
// when symmetric).  Offsets are element offsets (doubles) into the named
// buffers; -1 = not produced.
struct PairItem {
  int32_t t, s;          // level-major cluster ids (row side t, column side s)
  int32_t gkind;         // 4 x 4 bits (quadrant a*2+b at bits 4*(a*2+b)), level >= 1
  int32_t s_ld;          // row length (elements) of S block row (t@k)
  int32_t s_ld_m;        // row length of S block row (s@k) (mirror, symmetric)
  int32_t yr_ld;         // leading dimension of the row-strip panel receiving bn
  int32_t yc_ld;         // leading dimension of the panel receiving nb^T
  int32_t pad_;
  int16_t nt, ns, kt, ks;      // local sizes / ranks of t (row side) and s (column side)
  int16_t kr0, kr1, kc0, kc1;  // ranks of the children of t and of s (level >= 1)
  int64_t q_off_t, q_off_s;    // Q_t in q_row, Q_s in q_col
  int64_t g_src[4];      // level 0: g_src[0] = offset of C_ts in `close`; else slot offsets
  int64_t s_dst;         // S block (t@k, s@k): element (0,0) in s_val
  int64_t s_dst_m;       // symmetric: S block (s@k, t@k) (transpose), t != s
  int64_t bb_dst;        // H[:k_t, :k_s]      -> bb buffer (k_t x k_s)
  int64_t yr_dst;        // H[:k_t, k_s:]      -> row-strip panel of t (k_t rows, ld yr_ld)
  int64_t yc_dst;        // H[k_t:, :k_s]^T    -> column-strip panel of s (general) /
                         //                      row-strip panel of s (symmetric), ld yc_ld
  int64_t pad2_;
};
static_assert(sizeof(PairItem) == 144, "PairItem is staged into shared memory in 16-byte pieces");
constexpr int PAIR_CHUNK_MAX = 8;  // items per congruence CTA (staged in shared memory)

// Strips (Eq. u1v1).  All strips rotated by cluster q at level k
// are stored as one row-major panel (k_q rows; columns = the frozen groups
// (l, s), in S column order).  At level k+1 the parent p stacks its children's
// panels (union of their groups, child 2 rows at offset k_c1) into Z and
// computes W = Q_p^T Z: rows [k_p, n_p) of W are S row block (p@k+1),
// columns [0, width) -- contiguous in S --, rows [0, k_p) continue as p's panel.
struct StripPanel {
  int32_t q;             // rotating cluster (level-major id)
  int32_t width;         // columns of W (sum of the group widths)
  int32_t ld_c1, ld_c2;  // leading dimensions of the children's panels
  int64_t src_c1, src_c2;  // children's panels (k_c x ld_c), -1 if absent
  int64_t y_dst;         // W[:k_q] -> y[y_dst + i*y_ld + c], -1 if k_q == 0
  int64_t s_dst;         // W[k_q + a][c] -> S[s_dst + a*s_ld + c] (direct), -1 if none
  int32_t y_ld, s_ld;
  int32_t gbeg, gend;    // groups of this panel in the level's group array
};

struct StripGroup {      // one frozen group (l, s) of a panel
  int32_t col0, m;       // columns [col0, col0 + m) of the panel
  int32_t pos_c1, pos_c2;  // column of the group in the children's panels, -1 if absent
  int64_t s_dst_t;       // W[k_q + a][col0 + b] -> S[s_dst_t + b*s_ld_t + a] (transposed), -1 if none
                         // (bench mode: partial slot s_dst_t + b*s_ld_t of S row b of the fixed cluster)
  int32_t s_ld_t;
  int32_t wc0;           // S column index (column side) of the group's first column (bench mode weights)
};

static_assert(sizeof(StripGroup) == 32, "staged as 4 x 8 bytes");

struct StripTile {       // columns [c0, c1) of one panel; g0 = first group overlapping c0
  int32_t panel, c0, c1, g0;
};

// Kernel-side strip tile: the tile, its panel and the cluster sizes folded into
// one 96-byte record (staged with 16-byte async copies: one round trip).
struct StripTileX {
  int32_t q, c0, ncol, g0;     // rotating cluster, panel columns [c0, c0 + ncol), first group
  int32_t gend;                // end of the panel's groups
  int16_t n, kq, k1, k2;       // n_q, k_q, k_c1, k_c2
  int32_t ld_c1, ld_c2, y_ld, s_ld;
  int32_t wq0;                 // S column index (column side) of q's first frozen column (bench mode)
  int64_t q_off;               // Q_q in the side's Q array
  int64_t src_c1, src_c2, y_dst, s_dst;  // as StripPanel
  int64_t pad2_;
};
static_assert(sizeof(StripTileX) == 96, "staged as 6 x 16 bytes");

// A run of items that share the rotating cluster (Q kept in shared memory).
struct Chunk {
  int32_t begin, end;
};

struct CouplingItem {    // D~ = R^R_t D R^C_s^T (reading 11)
  int32_t t, s;          // level-major ids
  int64_t d_src;         // offset of D_ts in `coupling`
  int64_t dt_dst;        // slot offset in the dt buffer
};

struct CsrBlockRow {     // rows [row0, row0 + m_r) of S, all with the same column pattern
  int64_t row0;
  int64_t p_base;        // s_val offset of row row0
  int64_t pat_off;       // the block row's column pattern (rowlen int32) in the pattern array
  int32_t m_r;
  int32_t rowlen;
  int32_t blk_begin, nblk;
  int64_t grow0;         // global S row index of row0 (row side S order)
  int64_t part_base;     // bench mode: partial slot of (row0, block 0); row a, block j -> part_base + a*nblk + j
};

struct CsrBlock {        // columns [col0, col0 + m_c) at row positions [colpos, colpos + m_c)
  int32_t col0, m_c, colpos, pad_;
};

struct LevelPlan {
  int k;
  int np_row, np_col;    // max n_t at this level (row / column side)
  int mp;                // max strip width at this level
  int64_t n_pairs, n_pair_chunks;
  int64_t pair_split;    // level 0: chunks of the first half of the leaves (0 = no split)
  int64_t n_coup;
  size_t pairs_off, pair_chunks_off;          // byte offsets in meta
  size_t coup_off;
  struct StripSet {                           // strip panels of one set at this level (tiles = launch size)
    int64_t n_rtiles, n_ctiles;
    int64_t n_rtiles_a;  // set 0: row tiles of the first half of the clusters (0 = no split)
    size_t rtiles_off, rpanels_off, rgroups_off;
    size_t ctiles_off, cpanels_off, cgroups_off;
  } sp[2];                                    // [0]: groups born at level 0, [1]: born at a level >= 1
  int np_pair;           // padded tile size for the congruence at this level
  int np_rstrip, np_cstrip;
};

struct ClusterArrays {   // byte offsets in meta of per-cluster arrays
  size_t n_row, k_row, n_col, k_col;       // int32 [ncl]
  size_t q_off_row, q_off_col;             // int64 [ncl]
  size_t rh_off_row, rh_off_col;           // int64 [ncl]
  size_t leaf_off_row, leaf_off_col;       // int64 [n_leaves]
  size_t tr_off_row, tr_off_col;           // int64 [ncl]
  size_t s_off_row, s_off_col;             // int64 [ncl]
  size_t zb_off_row, zb_off_col;           // int64 [ncl]: apply basis-coefficient slots (per rhs)
  size_t loc_off_row, loc_off_col;         // int64 [ncl]: local S row offset of owned clusters, -1 otherwise
  size_t need_row, need_col;               // int8 [ncl]: Q needed by this shard
  size_t need_all;                         // int8 [ncl]: all ones (H2SP_QR_ALL builds)
};

}  // namespace h2sp

struct h2sp_plan_s {
  int32_t qr_mode = 0;                     // H2SP_QR_NEED / _ALL / _REUSE (h2sp_plan_set_qr_mode)
  int32_t L, B, sym;
  int32_t rank, world, part_level;         // sharding by top-level subtrees (world == 1: everything)
  int64_t first_leaf, n_leaves_local, n_rows_local, n_cols_local;
  std::vector<int64_t> loc_off_row, loc_off_col;
  std::vector<int8_t> need_r, need_c;
  int64_t N, ncl;
  std::vector<int32_t> n_row, k_row, n_col, k_col;
  std::vector<int64_t> q_off_row, q_off_col, s_off_row, s_off_col;
  int64_t q_row_len, q_col_len;
  int64_t leaf_row_len, leaf_col_len, tr_row_len, tr_col_len, close_len, coupling_len;
  int64_t rh_row_len, rh_col_len, dt_len, bb_len, yr_len, yc_len;
  int64_t zb_row_len, zb_col_len;          // per rhs
  int64_t s_nnz, s_blocks;
  int levels_active;
  double flops, bytes, flops_cong, flops_strip, flops_exec;
  std::vector<h2sp::LevelPlan> levels;
  h2sp::ClusterArrays ca;
  size_t csr_rows_off, csr_blocks_off, rowptr_off, csr_pat_off;
  int64_t n_csr_rows, n_csr_blocks;
  std::vector<unsigned char> meta;          // device image of all work lists
  size_t meta_bytes;
  // workspace layout after the meta region (byte offsets)
  size_t ws_rh_row, ws_rh_col, ws_dt, ws_bb, ws_yr, ws_yc, ws_total;
  // compact-WY form of the level-0 Q (0 = explicit Q everywhere): per leaf,
  // V (wy_n x wy_kp, row-major) then M = T V^T (wy_kp x wy_n), zero padded
  int32_t wy_kp, wy_n;                      // wy_n: padded leaf size of V / M (64 or 128)
  size_t ws_wy_row, ws_wy_col, ws_qr_end;
  int32_t nmax;                             // largest local size n_t
  int32_t bench;                            // H2SP_PLAN_BENCH: S reduced to S*w and row norms, never stored
  int32_t strip_aligned;                    // every frozen size m_t is a multiple of 32 (matrix-wide)
  int64_t n_part;                           // bench mode: partial slots (double2 {S*w, |S|^2} per block row x block)
  size_t ws_part;                           // bench mode: partial buffer in the workspace
  double flops_unique;                      // sharded: work attributed to this shard's own clusters only
  int64_t launches;
  std::vector<h2sp_launch_info> launch_info;
  uint64_t magic;                           // first 8 bytes of the meta image (checked on device)
};

namespace h2sp {
void set_error(const std::string &msg);
h2sp_status fail(h2sp_status s, const std::string &msg);

// kernels.cu
// meta: the plan's work lists on the device; scratch: the rest of the workspace
// (sizes.workspace_bytes - meta_bytes); ap_scratch: the applies' scratch (ap != NULL)
h2sp_status launch_build(const h2sp_plan_s *p, const h2sp_inputs *in, const h2sp_outputs *out,
                         const unsigned char *meta, unsigned char *scratch, void *stream, int64_t *launches,
                         void *const *events, int64_t n_events, const h2sp_apply_args *ap = nullptr,
                         unsigned char *ap_scratch = nullptr);
h2sp_status launch_csr_early(const h2sp_plan_s *p, unsigned char *ws, int64_t *d_rowptr, int32_t *d_col,
                             int64_t *h_rowptr, int32_t *h_col, void *stream);
h2sp_status launch_csr_early_join(const h2sp_plan_s *p, void *stream);
h2sp_status launch_cheb_construct(const h2sp_plan_s *P, const unsigned char *meta, int side, const h2sp_cheb_spec *s,
                                  const double *points, const double *box_lo, const double *box_hi, double *leaf,
                                  double *transfer, double *nodes, void *stream);
h2sp_status launch_kernel_blocks(const h2sp_close_gen *k, const double *xn, const double *yn,
                                 const h2sp_block_desc *blocks, int64_t n_blocks, double *out, void *stream);
h2sp_status launch_apply_Ut(const h2sp_plan_s *p, const double *q, const double *b, int64_t ldb, double *y,
                            int64_t ldy, int nrhs, const unsigned char *meta, unsigned char *scratch, void *stream,
                            bool col_side);
h2sp_status launch_apply_V(const h2sp_plan_s *p, const double *q, const double *y, int64_t ldy, double *x,
                           int64_t ldx, int nrhs, const unsigned char *meta, unsigned char *scratch, void *stream,
                           bool col_side);
}  // namespace h2sp
