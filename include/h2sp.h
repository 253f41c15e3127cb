/*
 * h2sp.h -- C ABI of the B200-native non-extensive sparsification of an H^2
 * matrix (arXiv 1705.04601, "PAPER.md" = P below).
 *
 * Given the parameters of an H^2 matrix (Def. "H^2 matrix":
 * A = C + sum_{b=(t,s) admissible} R_t D_b E_s^T, with nested cluster bases
 * R_p = diag(R_c1, R_c2) T_p), the library computes the exact
 * factorisation A = U S V^T (Eq. main_fact):
 *   - U, V orthogonal: products of level-wise block-diagonal factors whose
 *     blocks are the completed square bases Q_t = [W_t, W_t^perp]
 *      and of the basis/non-basis permutations P_rk, P_ck
 *     (P:219-223).  They are returned as the batch of Q_t blocks plus the
 *     S-order offsets (the permutation) of every cluster.
 *   - S sparse N x N ("non-extensive"), returned as CSR.
 * and applies y = U^T b, x = V y (Eq. sp0).
 *
 * Conventions shared by every entry point
 *   - Balanced binary cluster tree, level 0 = 2^L leaves of B indices each,
 *     level L = root.  Cluster (k, i) has the level-major id
 *     cid = (2^(L+1) - 2^(L-k+1)) + i; its children are (k-1, 2i), (k-1, 2i+1).
 *     Indices are in cluster-tree order: leaf i owns [iB, (i+1)B).
 *   - All dense blocks are row-major FP64.
 *   - Local size n_t = B (leaf) or k_c1 + k_c2 (internal); frozen count
 *     m_t = n_t - k_t; 0 <= k_t <= n_t, k_root = 0 (readings 3-5).
 *   - S order: off(k,t) = sum_{k'<k} sum_t' m_t' + sum_{t'<t at level k} m_t'
 *     (non-basis before basis, order preserved).  Row side uses
 *     m^R, column side m^C; sum m^R = sum m^C = N.
 *   - Q_t columns [0, k_t) span the orthogonalised basis; column k_t + a is the
 *     a-th non-basis direction, i.e. S index off(k,t) + a.  Householder
 *     convention H of DESIGN.md (LAPACK dgeqrf/dorg2r semantics).
 *   - Every call returns h2sp_status; nothing throws across the ABI; a
 *     thread-local message is kept for h2sp_last_error().
 *   - Device pointers are caller-owned (torch tensors in the Python binding).
 *     The plan owns only host memory.  No CPU fallback: a missing device or a
 *     CUDA error is reported as H2SP_ECUDA.
 */
#ifndef H2SP_H
#define H2SP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  H2SP_OK = 0,
  H2SP_EINVAL = 1,       /* bad argument (NULL pointer, size too small, ...)  */
  H2SP_ETREE = 2,        /* block cluster tree is not a partition / unsorted   */
  H2SP_ERANK = 3,        /* rank outside [0, n_t] or nonzero root rank          */
  H2SP_ENOMEM = 4,       /* host allocation failed                              */
  H2SP_ECUDA = 5,        /* CUDA launch / runtime error                         */
  H2SP_ENCCL = 6,        /* reserved for the multi-GPU halo exchange            */
  H2SP_EUNSUPPORTED = 7  /* shape outside what the kernels are built for        */
} h2sp_status;

const char *h2sp_status_str(h2sp_status s);
/* Detail of the last error raised on this host thread ("" if none). */
const char *h2sp_last_error(void);

typedef struct h2sp_plan_s *h2sp_plan;

/* Structure of the H^2 matrix (HOST pointers, read during plan_create only).
 *   rank_row/rank_col: [2^(L+1)-1] ranks k_t by level-major id; rank_col may be
 *     NULL iff symmetric (then the column side is the row side).
 *   near_ptr[2^L + 1], near_col[nnz]: N_0 (inadmissible leaf pairs) as CSR over
 *     leaves, columns strictly ascending within a row.
 *   adm_ptr[k][2^(L-k) + 1], adm_col[k][...]: A_k (admissible pairs at level
 *     k = 0..L-1) as CSR per level, columns strictly ascending.
 * Symmetric mode (symmetric != 0) requires both lists to be symmetric; the
 * numeric inputs must then satisfy C_st = C_ts^T and D_st = D_ts^T (only the
 * t <= s blocks are read).  The plan checks that the block tree is a partition
 * (P:613-649): every pair of N_k (k >= 1, N_k = parents of N_{k-1} u A_{k-1})
 * has its 4 children in N_{k-1} u A_{k-1}, no pair is both near and far, and
 * N_L = {(root, root)}. */
typedef struct {
  int32_t L;
  int32_t leaf_size;
  int32_t symmetric;
  const int32_t *rank_row;
  const int32_t *rank_col;
  const int64_t *near_ptr;
  const int32_t *near_col;
  const int64_t *const *adm_ptr;
  const int32_t *const *adm_col;
} h2sp_structure;

/* Sizes derived by the plan (all element counts are numbers of doubles unless
 * stated otherwise). */
typedef struct {
  int64_t n;                   /* N = B * 2^L                                  */
  int64_t n_clusters;          /* 2^(L+1) - 1                                  */
  int64_t leaf_row, transfer_row, leaf_col, transfer_col; /* input lengths    */
  int64_t close, coupling;     /* input lengths: n_near*B*B, sum k_t*k_s        */
  int64_t q_row, q_col;        /* output lengths of the Q batches (sum n_t^2)  */
  int64_t s_nnz;               /* nonzeros of S (of this shard's rows)         */
  int64_t s_rows;              /* rows of S held by this plan (N if world = 1) */
  int64_t rank, world;         /* shard of a sharded plan (0, 1 otherwise)     */
  int64_t first_leaf;          /* first leaf of this shard's subtree           */
  int64_t n_leaves_local;      /* leaves of this shard's subtree               */
  int64_t s_blocks;            /* blocks (t@i, s@j) of S                       */
  int64_t workspace_bytes;     /* device workspace for h2sp_build (incl. meta) */
  int64_t meta_bytes;          /* leading part of every workspace: work lists  */
  int64_t levels_active;       /* levels with any nonzero local size           */
  int64_t launches;            /* kernel launches issued by one h2sp_build     */
  double flops;                /* algorithmic FP64 flops of one build          */
  double bytes;                /* algorithmic HBM bytes of one build           */
  double flops_congruence;     /* of which: congruence H = Q^T G Q             */
  double flops_strips;         /* of which: strip rotations                    */
  double flops_executed;       /* FP64 flops actually issued (<= flops)        */
  double flops_unique;         /* sharded plan: the part of `flops` whose row /
                                  rotating cluster this shard owns (the shards'
                                  flops_unique add up to the unsharded flops;
                                  flops - flops_unique is halo / mirror work
                                  done twice).  = flops when world = 1.        */
  int64_t bench_parts;         /* H2SP_PLAN_BENCH: partial slots (16 B each) in
                                  the workspace; 0 otherwise                   */
} h2sp_sizes;

/* Matrix-free close blocks ("close_gen" mode, SURVEY §8(d) config-5 protocol
 * step 1): instead of reading C_ts from `close`, the level-0 congruence
 * evaluates C_ts[i][j] = K(x_{tB+i}, x_{sB+j}) from the points while it stages
 * G (P:238-250 with G = C_ts at level 0).  The paper materialises the close
 * blocks; this mode exists because config 5's 980 GB of close
 * blocks fit no GPU.  Kernels (r = Euclidean distance, "same" = the same
 * point, i.e. t == s and i == j):
 *   H2SP_KERNEL_EXP       exp(-r / p0) + p1 [same]        configs 1, 2, 5
 *   H2SP_KERNEL_INVSHIFT  1 / (r + p0) + p1 [same]        config 3
 *   H2SP_KERNEL_LAPLACE   1 / (4 pi r); p1 at [same]      config 4
 * points: DEVICE, N x dim row-major doubles in tree order (leaf i owns rows
 * [iB, (i+1)B)), N = B << L (a sharded plan reads its own and its neighbours'
 * leaves, so pass all N points).  dim in 1..3.  The diagonal blocks are
 * bitwise symmetric (|x-y| is evaluated from the squared differences). */
#define H2SP_KERNEL_EXP 1
#define H2SP_KERNEL_INVSHIFT 2
#define H2SP_KERNEL_LAPLACE 3
typedef struct {
  const double *points;
  int32_t dim;
  int32_t kernel;
  double p0;
  double p1;
  /* Matrix-free far couplings (optional, config-5 protocol): with
   * h2sp_inputs.coupling == NULL, D_b = K(nodes_t, nodes_s) is evaluated inside
   * the coupling step (D~ = R^_t D R^_s^T) -- the interpolation H^2
   * construction's couplings (SURVEY §8(d) generator), never stored (config 5:
   * 130 GB).  nodes_row: DEVICE, (sum_c k_row[c]) x dim doubles, the k_c nodes
   * of every cluster in level-major cluster order (rank-0 clusters have none);
   * nodes_col likewise for the column side (NULL if symmetric).  Same
   * arithmetic as h2sp_eval_kernel_blocks.  Both NULL: couplings are read. */
  const double *nodes_row;
  const double *nodes_col;
} h2sp_close_gen;

/* Kernel blocks on the device (first piece of GPU H^2
 * construction): out[b] (nx x ny, row-major at out_off) = K(x_i, y_j) with
 * x_i = x_nodes row x_off + i, y_j = y_nodes row y_off + j (dim columns each),
 * for the kernels of h2sp_close_gen, whose `points` is ignored here (the "same
 * point" term never applies).  With the Chebyshev nodes of the cluster boxes this is the
 * coupling D_b = K(nodes_t, nodes_s) of the interpolation H^2 construction
 * (configs 2-5), evaluated where the build consumes it instead of on the host.
 * All pointers DEVICE except `k` (host); asynchronous on `stream`. */
typedef struct {
  int64_t x_off, y_off, out_off;
  int32_t nx, ny;
} h2sp_block_desc;
h2sp_status h2sp_eval_kernel_blocks(const h2sp_close_gen *k, const double *x_nodes, const double *y_nodes,
                                    const h2sp_block_desc *blocks, int64_t n_blocks, double *out, void *stream);

/* GPU H^2 construction (the input side of the path,
 * P:601-602): nested cluster bases by tensor Chebyshev interpolation on each
 * cluster's box, the recipe of the synthetic inputs, so that no
 * numeric input of config 5 is built on the host.  For `side` (0 row, 1
 * column) of the plan and every cluster of rank k > 0 (k must equal
 * prod(orders)):
 *   box = [lo - pad, hi + pad], pad = max(1e-9 (hi - lo), 1e-12) per axis;
 *   axis a gets order orders[i] where a is the i-th axis by decreasing
 *   extent (stable); axis nodes mid + half * cheb_cos[(p-1)*8 + j] (p = 1: mid);
 *   nodes: the tensor grid, axis 0 slowest -> nodes[(zb(c) + j) * dim ...]
 *   (zb(c) = sum of the ranks of the clusters before c, level-major);
 *   leaf_basis (as h2sp_inputs.leaf_basis_*): row i of R_t = the tensor
 *     Lagrange basis of t at point i of t;
 *   transfer (as h2sp_inputs.transfer_*): row i of T_p = p's basis at node
 *     i of its children (child 1 first).
 * Every step is an explicitly rounded IEEE operation, so with the cosine table
 * of the numpy generator the arrays are bitwise equal to it.
 * points: DEVICE N x dim (tree order); box_lo / box_hi: DEVICE n_clusters x dim
 * tight boxes; `meta`: the plan's uploaded work lists (h2sp_plan_upload).
 * Outputs DEVICE, lengths as in the plan sizes; nodes: sum of ranks x dim.
 * Asynchronous on `stream`.  H2SP_ERANK if a rank is neither 0 nor prod(orders). */
typedef struct {
  int32_t dim;            /* 1..3 */
  int32_t orders[3];      /* base orders, largest-extent axis first; prod <= 64 */
  double cheb_cos[64];    /* [(p - 1) * 8 + j]: Chebyshev cosines of order p = 1..8 */
} h2sp_cheb_spec;
h2sp_status h2sp_cheb_construct(h2sp_plan plan, const void *meta, int side, const h2sp_cheb_spec *spec,
                                const double *points, const double *box_lo, const double *box_hi, double *leaf_basis,
                                double *transfer, double *nodes, void *stream);

/* Numeric inputs (DEVICE pointers, read-only, row-major FP64):
 *   leaf_basis_row: R_t of every leaf, B x k_t each, concatenated by leaf.
 *   transfer_row:   T_p of every internal cluster, (k_c1 + k_c2) x k_p each
 *                   (child 1 rows first), concatenated by level-major id.
 *   *_col: the column side (ignored, may be NULL, if symmetric).
 *   close:    C_ts (B x B) per N_0 pair in near_ptr/near_col order (or
 *             close_gen: the blocks are evaluated on the fly, see above).
 *   coupling: D_b (k_t x k_s) per A_k pair, level-major, CSR order. */
typedef struct {
  const double *leaf_basis_row;
  const double *transfer_row;
  const double *leaf_basis_col;
  const double *transfer_col;
  const double *close;         /* ignored (may be NULL) when close_gen != NULL  */
  const double *coupling;      /* NULL: evaluated from close_gen->nodes_*       */
  const h2sp_close_gen *close_gen;  /* HOST pointer to the descriptor, or NULL */
} h2sp_inputs;

/* Outputs (DEVICE pointers, caller-allocated with the lengths of h2sp_sizes):
 *   q_row[q_row], q_col[q_col]: Q_t (n_t x n_t, row-major) concatenated by
 *     level-major id (offsets from h2sp_plan_offsets); q_col ignored if
 *     symmetric (U == V, use q_row).
 *   s_rowptr[s_rows+1] (int64), s_col[s_nnz] (int32), s_val[s_nnz]: S in CSR,
 *     rows and columns in S order, columns ascending (a sharded plan holds its
 *     local rows only, see h2sp_plan_create_shard).  s_col / s_rowptr may be NULL
 *     to skip writing the (value-independent) index arrays. */
typedef struct {
  double *q_row;
  double *q_col;
  int64_t *s_rowptr;
  int32_t *s_col;
  double *s_val;
  /* Bench mode (plan flag H2SP_PLAN_BENCH, SURVEY §8(b)/(d) config-5 protocol
   * step 3): S is not stored (s_val / s_col ignored, may be NULL).  Every S
   * block is reduced, in the congruence and strip epilogues, to one partial
   * {sum_j S[i][j] w[j], sum_j S[i][j]^2} per block row i; a final pass sums a
   * row's partials in block order (no atomics: bitwise reproducible, and
   * independent of the shard count).  All DEVICE, global S order, N entries:
   *   bench_w  (in)  w, indexed by S column (column-side S order)
   *   bench_y  (out) y = S w at this plan's S rows (other rows untouched)
   *   bench_r2 (out) ||S[i, :]||_2^2 at this plan's S rows (may be NULL)     */
  const double *bench_w;
  double *bench_y;
  double *bench_r2;
} h2sp_outputs;

/* Symbolic phase (host, O(#blocks)): validates the structure and derives all
 * sizes, S offsets, the S block pattern, CSR row pointers and the per-level
 * work lists.  flags: 0 or any of H2SP_PLAN_EXPLICIT_Q, H2SP_PLAN_BENCH. */
h2sp_status h2sp_plan_create(const h2sp_structure *st, int flags, h2sp_plan *out);

/* Plan flags.  By default the level-0 congruence H = Q_t^T G Q_s (n_t = B <= 64,
 * k <= 24) applies each Q in its compact-WY form Q = I - V M, M = T V^T (the
 * Householder vectors of step (i)), costing 4 n_t n_s (k_t + k_s)
 * flops instead of 2 n_t n_s (n_t + n_s); equal to the explicit product up to
 * rounding (and exactly equal when every Q is a permutation).
 * H2SP_PLAN_EXPLICIT_Q forces the explicit-Q product at every level. */
#define H2SP_PLAN_EXPLICIT_Q 1
/* Bench mode: S is reduced to y = S w and the row norms ||S[i,:]||^2 (see
 * h2sp_outputs) instead of being stored -- config 5's S is ~2 TB.  The plan
 * builds no CSR column pattern; s_rowptr may still be written. */
#define H2SP_PLAN_BENCH 2
/* Sharded plan: rank `rank` of `world` (a power of two <= 2^L)
 * owns the top-level subtree of cluster `rank` at the partition level
 * Lp = L - log2(world): S rows of its clusters, the congruences whose row cluster
 * is owned (general mode) or whose row or column cluster is owned (symmetric:
 * cross pairs are computed by both owners, each keeping its rows), and the strip
 * columns landing in owned rows.  Q and the couplings are computed for every
 * cluster on every rank (no exchange needed).  S is returned with local rows:
 * the owned clusters' rows in S order (h2sp_plan_local_rows); column indices
 * stay global.  world = 1 is h2sp_plan_create.  H2SP_EUNSUPPORTED if any cluster
 * above Lp has a nonzero local size (the remainder gather is not implemented). */
h2sp_status h2sp_plan_create_shard(const h2sp_structure *st, int rank, int world, int flags, h2sp_plan *out);
/* Local S row offset of every cluster owned by the shard (-1 otherwise); row /
 * column side (host arrays of n_clusters entries, either may be NULL). */
h2sp_status h2sp_plan_local_rows(h2sp_plan plan, int64_t *loc_off_row, int64_t *loc_off_col);
h2sp_status h2sp_plan_sizes(h2sp_plan plan, h2sp_sizes *out);
/* Host copies of per-cluster data (each array has n_clusters entries; any
 * pointer may be NULL): S-order offsets (row / column side), offsets of Q_t in
 * q_row / q_col, local sizes n_t (row / column). */
h2sp_status h2sp_plan_offsets(h2sp_plan plan, int64_t *s_off_row, int64_t *s_off_col, int64_t *q_off_row,
                              int64_t *q_off_col, int64_t *n_row, int64_t *n_col);
/* Host copy of the symbolic CSR pattern of S: rowptr[s_rows+1] (int64) and, if
 * col != NULL, col[s_nnz] (int32) -- identical to what h2sp_build writes into
 * s_rowptr / s_col.  Host only (no device needed). */
h2sp_status h2sp_plan_pattern(h2sp_plan plan, int64_t *rowptr, int32_t *col);
void h2sp_plan_destroy(h2sp_plan plan);

/* Description of the kernel launches of one h2sp_build, in launch order
 * (kind: 0 QR row side, 1 QR column side, 2 couplings, 3 merge+congruence+
 * freeze, 4 row strips, 5 column strips, 6 CSR index expansion, 7 level-0 Q
 * formed from its compact-WY factors, both sides, 8 bench-mode row sums).  flops and
 * bytes are the algorithmic FP64 flops and HBM bytes of that launch
 * (SURVEY §8(d) per-unit figures x units in the launch); items = work units;
 * flops_exec = the FP64 flops the kernel actually issues (differs from flops
 * only for the compact-WY level-0 congruence, see H2SP_PLAN_EXPLICIT_Q). */
typedef struct {
  int32_t kind;
  int32_t level;
  int64_t items;
  double flops;
  double bytes;
  double flops_exec;
} h2sp_launch_info;
/* Writes min(max, count) records to out (may be NULL) and the count to *count. */
h2sp_status h2sp_plan_launches(h2sp_plan plan, h2sp_launch_info *out, int64_t max, int64_t *count);

/* Copies the plan's device work lists (sizes.meta_bytes bytes) into the first
 * part of a device workspace `ws` (256-byte aligned) on `stream`.  Must be
 * called once for every workspace before it is passed to h2sp_build or
 * h2sp_apply_*; the work lists stay valid as long as the caller does not
 * overwrite that region.  A workspace uploaded for another plan is detected
 * on the device (kernel trap -> H2SP_ECUDA at the next synchronisation). */
h2sp_status h2sp_plan_upload(h2sp_plan plan, void *ws, size_t ws_bytes, void *stream);

/* Numeric phase: computes Q (both sides) and S on `stream` (a cudaStream_t;
 * NULL = legacy default stream).  Asynchronous; errors of the launches are
 * returned, faults inside kernels surface at the next synchronising call.
 * ws: device workspace of at least sizes.workspace_bytes bytes, 256-byte
 * aligned, uploaded with h2sp_plan_upload.
 * Internally the build forks onto the library's side streams (one set per
 * device, created on first use) and joins back into `stream` with events, so
 * it is stream-ordered and CUDA-graph capturable.  Builds issued from several
 * host threads onto the same device must be serialised by the caller (they
 * share those side streams and events); different devices are independent. */
h2sp_status h2sp_build(h2sp_plan plan, const h2sp_inputs *in, const h2sp_outputs *out, void *ws,
                       size_t ws_bytes, void *stream);

/* h2sp_build that also records CUDA events for profiling: events[2i] and
 * events[2i+1] (cudaEvent_t) just before and just after launch i of
 * h2sp_plan_launches, on the stream that launch runs on (the build forks
 * independent chains -- QR/couplings of levels >= 1, CSR index expansion --
 * onto internal side streams joined back into `stream`); n_events >= 2*count. */
h2sp_status h2sp_build_ex(h2sp_plan plan, const h2sp_inputs *in, const h2sp_outputs *out, void *ws,
                          size_t ws_bytes, void *stream, void *const *events, int64_t n_events);

/* One pass of the whole hot path (BASELINE.json north_star: "the same pass also
 * applies U^T b and V y"): h2sp_build plus y = U^T b and x = V w.  The applies
 * depend only on Q, so they run on the build's side streams right after the
 * QR chain, overlapping the congruence and strips (V w beside U^T b when w is
 * not y; after it when w == y).  Either apply is skipped if
 * its input pointer is NULL; w may be y (then x = V U^T b).  `ws` of the apply
 * must be a DIFFERENT uploaded workspace (>= h2sp_apply_ws_bytes(nrhs)) than
 * the build's.  Layouts as in h2sp_apply_Ut / h2sp_apply_V.  `events` as in
 * h2sp_build_ex (may be NULL). */
typedef struct {
  const double *b;
  int64_t ldb;
  double *y;
  int64_t ldy;
  const double *w;
  int64_t ldw;
  double *x;
  int64_t ldx;
  int nrhs;
  void *ws;
  size_t ws_bytes;
} h2sp_apply_args;
h2sp_status h2sp_build_apply(h2sp_plan plan, const h2sp_inputs *in, const h2sp_outputs *out, void *ws,
                             size_t ws_bytes, const h2sp_apply_args *ap, void *stream, void *const *events,
                             int64_t n_events);

/* h2sp_build_apply with the plan's work lists and the rest of the workspace in
 * separate device buffers: `meta` (sizes.meta_bytes, filled by h2sp_plan_upload)
 * and `scratch` (>= sizes.workspace_bytes - sizes.meta_bytes bytes), both
 * 256-byte aligned.  Several plans -- the virtual shards of one matrix
 * (SURVEY §8(d) config-5 protocol step 2) -- can keep their work lists resident
 * and take turns on one scratch buffer (builds ordered on one stream).  `ap`
 * may be NULL (no applies); otherwise ap->ws is the applies' scratch only (no
 * meta at its head), >= h2sp_apply_ws_bytes(nrhs) - sizes.meta_bytes bytes. */
h2sp_status h2sp_build_meta(h2sp_plan plan, const h2sp_inputs *in, const h2sp_outputs *out, const void *meta,
                            void *scratch, size_t scratch_bytes, const h2sp_apply_args *ap, void *stream,
                            void *const *events, int64_t n_events);

/* QR sharing between the shard plans of ONE matrix that are built one after
 * another on one scratch buffer with one set of Q outputs (h2sp_build_meta; SURVEY
 * §8(d) config-5 protocol step 2: "QR/R^ for every cluster depends only on the
 * bases, so it runs first for all clusters").  The mode is host-side state of
 * the plan, read by the next h2sp_build* call:
 *   H2SP_QR_NEED  (default) QR completion of the clusters this plan
 *                 needs: its own subtree plus the halo closure over descendants
 *                 -- at the upper levels of a 3-D tree that closure is nearly
 *                 the whole tree, so every shard repeats almost the full chain;
 *   H2SP_QR_ALL   QR completion of EVERY cluster of the tree (what an unsharded
 *                 plan computes);
 *   H2SP_QR_REUSE no QR launch at all: the caller guarantees that the head of
 *                 `scratch` (R^ and the level-0 compact-WY factors; the same
 *                 offsets and sizes in every shard plan of one matrix, of the
 *                 same flags) and out->q_row / q_col still hold the results of
 *                 an H2SP_QR_ALL build of the same inputs.
 * Results are bitwise the same in every mode (each cluster's Q_t, R^_t depend on
 * its subtree's bases only).  H2SP_EINVAL: unknown mode. */
#define H2SP_QR_NEED 0
#define H2SP_QR_ALL 1
#define H2SP_QR_REUSE 2
h2sp_status h2sp_plan_set_qr_mode(h2sp_plan plan, int mode);

/* End-to-end variant with HOST buffers: copies the host inputs into the given
 * device input buffers, builds, and copies every output back into the host
 * output buffers (host pointers should be pinned for overlap).  All copies
 * are cudaMemcpyAsync on `stream`; the call returns after enqueueing them.
 * close_gen mode: host_in->close_gen->points (host) is copied into
 * dev_in->close_gen->points (device), N * dim doubles. */
h2sp_status h2sp_build_host(h2sp_plan plan, const h2sp_inputs *host_in, const h2sp_outputs *host_out,
                            const h2sp_inputs *dev_in, const h2sp_outputs *dev_out, void *ws, size_t ws_bytes,
                            void *stream);

/* Workspace bytes for h2sp_apply_Ut / h2sp_apply_V with nrhs right-hand sides
 * (meta region, then one half per direction -- basis coefficients and the
 * arrival counters of U^T b; basis coefficients, cluster flags and the ticket of
 * V y -- so the two applies may run side by side).  The build workspace may be reused
 * when it is at least this large (after the build has completed on the
 * stream); it must have been uploaded with h2sp_plan_upload. */
int64_t h2sp_apply_ws_bytes(h2sp_plan plan, int nrhs);

/* y = U^T b: b is N x nrhs column-major in tree order (leading
 * dimension ldb), y is N x nrhs column-major in S order (row side, ldy).
 * Sharded plan: b holds the shard's leaves only (n_leaves_local * B rows) and y
 * its local S rows (s_rows); likewise for h2sp_apply_V.
 * q_row as produced by h2sp_build.  Leaves to root: z = Q_t^T x_t,
 * z[k_t:] -> y, z[:k_t] -> parent's local vector. */
h2sp_status h2sp_apply_Ut(h2sp_plan plan, const double *q_row, const double *b, int64_t ldb, double *y,
                          int64_t ldy, int nrhs, void *ws, size_t ws_bytes, void *stream);
/* x = V y: y in S order (column side), x in tree order.  Root to leaves:
 * x_t = Q_t [z_basis; y_t], each cluster's product computed once (by the CTA of
 * its leftmost leaf) and handed down through the workspace.  q_col as produced
 * by h2sp_build (q_row if symmetric). */
h2sp_status h2sp_apply_V(h2sp_plan plan, const double *q_col, const double *y, int64_t ldy, double *x,
                         int64_t ldx, int nrhs, void *ws, size_t ws_bytes, void *stream);

/* Multi-GPU communicator: one process per GPU; NCCL over
 * NVLink, loaded with dlopen on first use (H2SP_ENCCL if unavailable -- no
 * fallback).  Bootstrap: rank 0 calls h2sp_comm_unique_id, the caller's
 * process group (torch.distributed) broadcasts the 128 bytes, every rank calls
 * h2sp_comm_init on its own device (the current CUDA device).  The sharded
 * build has no data-path exchange (each shard recomputes its halo Q / R^,
 * DESIGN.md §10); the collectives are the checks and the assembly of the
 * distributed results: h2sp_comm_allreduce sums (H2SP_SUM) or maximises
 * (H2SP_MAX) n doubles of a DEVICE buffer in place on `stream` -- e.g. the
 * bench-mode y = S w of all ranks (their rows are disjoint). */
typedef struct h2sp_comm_s *h2sp_comm;
#define H2SP_SUM 0
#define H2SP_MAX 1
h2sp_status h2sp_comm_unique_id(void *id /* 128 bytes out */);
h2sp_status h2sp_comm_init(const void *id, int rank, int world, h2sp_comm *out);
h2sp_status h2sp_comm_allreduce(h2sp_comm comm, double *buf, int64_t n, int op, void *stream);
h2sp_status h2sp_comm_info(h2sp_comm comm, int *rank, int *world);
void h2sp_comm_destroy(h2sp_comm comm);

/* ------------------------------------------------------------------------
 * The preconditioning workload ("Sparsification method as a
 * preconditioner") and the direct solve (§8(f) #1, x = V S^-1 U^T b,
 * Eq. sp0).  The paper solves A x = b by GMRES "for the matrix
 * approximated in H^2 format with accuracy 1e-9" and, "as a preconditioner,
 * the H^2 approximation of A with accuracy 1e-3 sparsified and factorized with
 * ILUt decomposition".  The operator's matvec here is
 * the exact sparse factorisation of that H^2 matrix, A x = U S U^T x
 * (symmetric plans, V = U); the preconditioner is
 * M^-1 = U_M (L U)^-1 U_M^T with L U = ILUT(S_M).  Vectors are in tree order
 * (h2sp_apply_Ut's b / h2sp_apply_V's x); S-order temporaries stay inside.
 * ------------------------------------------------------------------------ */

/* A square CSR matrix on the DEVICE: rowptr[n + 1] (int64), col (int32,
 * ascending and unique within a row), val (FP64).  S as h2sp_build writes it
 * (s_rowptr / s_col / s_val) is one. */
typedef struct {
  int64_t n;
  const int64_t *rowptr;
  const int32_t *col;
  const double *val;
} h2sp_csr;

/* ILUT factors in row-pool form, DEVICE, caller-owned (allocated with n and
 * pool_cap): row i of L (strict lower; unit diagonal implied) is
 * pool_col/pool_val[l_start[i] .. + l_len[i]), row i of U (strict upper) is
 * [u_start[i] .. + u_len[i]), both in ascending column order; diag[i] = u_ii.
 * Rows are placed in the pool in completion order (the pool holds L and U). */
typedef struct {
  int64_t n;
  int64_t *l_start, *u_start;
  int32_t *l_len, *u_len;
  double *diag;
  int32_t *pool_col;
  double *pool_val;
  int64_t pool_cap;
} h2sp_ilut_factors;

/* Device workspace of h2sp_ilut for an n x n matrix (per-warp work rows and
 * candidate lists, completion flags), or -1. */
int64_t h2sp_ilut_ws_bytes(int64_t n);
/* ILUT(tau, p) of A (reading 25: Saad's Algorithm 10.6, IKJ order,
 * dual dropping -- w_k / u_kk dropped if |.| < tau ||a_i||_2 or == 0; after the
 * row: entries below tau ||a_i||_2 dropped, then only the p largest of the L
 * part and of the U part kept (ties: smaller column; p < 0 keeps all); the
 * diagonal is always kept).  tau = 0, p < 0: the complete LU without pivoting
 * (the direct solve of §8(f) #1; S is SPD in symmetric mode, Proposition
 * P:504-509, so no pivot vanishes in exact arithmetic).  The factors are
 * bitwise those of the algorithm run row by row in this arithmetic order.
 * Synchronises the stream.  pool_used (HOST, may be NULL): entries written.
 * Errors: H2SP_ENOMEM if pool_cap is too small (pool_used = entries requested
 * so far -- a lower bound; retry with a larger pool), H2SP_EINVAL on a zero
 * pivot (message names the first row) or bad arguments, H2SP_EUNSUPPORTED if
 * n > ~1.6M (the per-warp presence bitmap lives in shared memory). */
h2sp_status h2sp_ilut(const h2sp_csr *A, double tau, int p, h2sp_ilut_factors *F, void *ws, size_t ws_bytes,
                      int64_t *pool_used, void *stream);
/* x = (L U)^-1 b (forward substitution with the unit L, then backward with
 * U), asynchronous on the stream; x may alias b. */
int64_t h2sp_ilu_solve_ws_bytes(int64_t n);
h2sp_status h2sp_ilu_solve(const h2sp_ilut_factors *F, const double *b, double *x, void *ws, size_t ws_bytes,
                           void *stream);
/* y = A x for a device CSR matrix (asynchronous). */
h2sp_status h2sp_csr_spmv(const h2sp_csr *A, const double *x, double *y, void *stream);

/* A sparsified symmetric H^2 matrix A = U S U^T: the plan, its Q batch (q_row
 * of h2sp_build), its stored S and an apply workspace (h2sp_apply_ws_bytes(plan,
 * 1), uploaded with h2sp_plan_upload).  All DEVICE pointers. */
typedef struct {
  h2sp_plan plan;
  const double *q;
  h2sp_csr S;
  void *apply_ws;
  size_t apply_ws_bytes;
} h2sp_sparsified;

typedef struct {
  int restart;   /* m of GMRES(m)                                      */
  int maxiter;   /* total Arnoldi steps                                */
  double tol;    /* stop when the residual estimate <= tol * ||b||_2   */
} h2sp_gmres_opts;

typedef struct {
  int iters;          /* Arnoldi steps taken                                       */
  int restarts;       /* cycles completed                                          */
  int converged;
  int history_len;    /* entries of history produced (may exceed history_cap)      */
  double *history;    /* HOST, caller-owned, history_cap doubles (may be NULL):
                         ||r_j|| / ||b|| -- 1, then the estimate after each step    */
  int history_cap;
} h2sp_gmres_info;

/* Device workspace of h2sp_gmres: the (restart + 1) Krylov vectors and
 * temporaries. */
int64_t h2sp_gmres_ws_bytes(int64_t n, int restart);
/* Solve A x = b by restarted GMRES(m) with right preconditioning (Saad,
 * Algorithm 9.5; x0 = 0), x = M^-1 u: A from `A`, M^-1 from `M` and `F` (the
 * ILUT of M's S) -- both NULL for no preconditioner.  Arnoldi by classical
 * Gram-Schmidt with one re-orthogonalisation; the Hessenberg least-squares
 * problem is reduced by Givens rotations on the host (a handful of scalars per
 * step; one device-to-host read of the step's dot products).  Synchronous.
 * Errors: H2SP_EUNSUPPORTED for nonsymmetric or sharded plans, H2SP_EINVAL on
 * size mismatches / bad options. */
h2sp_status h2sp_gmres(const h2sp_sparsified *A, const h2sp_sparsified *M, const h2sp_ilut_factors *F,
                       const double *b, double *x, const h2sp_gmres_opts *opt, h2sp_gmres_info *info, void *ws,
                       size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Supernodal Cholesky of S on the device (the direct solve
 * x = V S^-1 U^T b, Eq. sp0; the paper factorises S with CHOLMOD,
 * P:804).  Symmetric (SPD, Proposition), unsharded,
 * stored-S plans.  Supernodes = the row groups of S (the frozen rows of one
 * cluster, in S's own level-major order -- no reordering); S = L L^T with L in
 * dense row-major panels, one per supernode J: the blocks I of struct(J)
 * (ascending, J first) stacked, (sum m_I) x m_J doubles.
 * ------------------------------------------------------------------------ */
typedef struct h2sp_chol_s *h2sp_chol;
/* Host analysis from the plan's block pattern: block elimination tree,
 * struct(J) by the supernodal symbolic factorisation, panel layout.
 * amalgamate > 0: consecutive supernodes J, J + 1 with parent(J) = J + 1 are
 * merged while the merged width stays <= amalgamate (<= 128) and the explicit
 * zeros added to J's columns stay under a quarter of its rows; 0: the row
 * groups themselves.  Outputs (HOST, may be NULL): the panel length in doubles
 * and the device meta bytes.  Errors: H2SP_EUNSUPPORTED for nonsymmetric /
 * sharded / bench plans or a group wider than 128 rows. */
h2sp_status h2sp_chol_analyse(h2sp_plan plan, int amalgamate, h2sp_chol *out, int64_t *panel_doubles,
                              int64_t *meta_bytes);
/* Number of supernodes, elimination-tree parents [ns] (-1 = root), panel rows
 * [ns] and the factorisation's flops (any output may be NULL). */
h2sp_status h2sp_chol_info(h2sp_chol c, int32_t *ns, int32_t *parent, int64_t *panel_rows, double *flops);
/* First S row of every supernode and n: start[ns + 1] (HOST). */
h2sp_status h2sp_chol_supernodes(h2sp_chol c, int64_t *start);
/* struct(J) (ascending block ids, J first): *count entries, at most cap written. */
h2sp_status h2sp_chol_struct(h2sp_chol c, int32_t J, int32_t *blocks, int32_t cap, int32_t *count);
/* Copy the analysis tables to a DEVICE buffer of meta_bytes (asynchronous). */
h2sp_status h2sp_chol_upload(h2sp_chol c, void *meta, size_t meta_bytes, void *stream);
/* Numeric factorisation of S (the stored output of h2sp_build, h2sp_csr) into
 * `panel` (DEVICE, panel_doubles): scatter of S's lower triangle, then per
 * supernode in order the dense Cholesky of the diagonal block, the triangular
 * solve of the rows below and the Schur update of the later panels (64 x 64
 * FP64 tensor-core tiles).  Synchronises the stream.  H2SP_EINVAL if a pivot
 * is not positive (message names the supernode). */
h2sp_status h2sp_chol_factor(h2sp_chol c, const h2sp_csr *S, const void *meta, double *panel, void *stream);
/* x = S^-1 b = L^-T L^-1 b (S order, DEVICE; x may alias b), asynchronous. */
h2sp_status h2sp_chol_solve(h2sp_chol c, const void *meta, const double *panel, const double *b, double *x,
                            void *stream);
void h2sp_chol_destroy(h2sp_chol c);

#ifdef __cplusplus
}
#endif

#endif /* H2SP_H */
