// C-ABI entry points of the numeric phase (include/h2sp.h).  Argument checks,
// workspace carving and stream-ordered copies; all arithmetic is in kernels.cu.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "h2sp_internal.h"

using namespace h2sp;

namespace {
constexpr int L_MAX_CHEB = 30;
}

namespace {

h2sp_status check_ws(const h2sp_plan_s *P, const void *ws, size_t ws_bytes, size_t need) {
  if (!ws) return fail(H2SP_EINVAL, "workspace is NULL");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(H2SP_EINVAL, "workspace not 256-byte aligned");
  if (ws_bytes < need)
    return fail(H2SP_EINVAL, "workspace too small: " + std::to_string(ws_bytes) + " < " + std::to_string(need));
  (void)P;
  return H2SP_OK;
}

h2sp_status cuda_ok(cudaError_t e, const char *what) {
  if (e != cudaSuccess) return fail(H2SP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return H2SP_OK;
}

h2sp_status check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(H2SP_ECUDA, "no CUDA device (the library has no CPU fallback)");
  return H2SP_OK;
}

h2sp_status check_inputs(const h2sp_plan_s *P, const h2sp_inputs *in) {
  const h2sp_close_gen *g = in->close_gen;
  if (g) {
    if (!g->points) return fail(H2SP_EINVAL, "close_gen: NULL points");
    if (g->dim < 1 || g->dim > 3) return fail(H2SP_EINVAL, "close_gen: dim must be 1, 2 or 3");
    if (g->kernel < H2SP_KERNEL_EXP || g->kernel > H2SP_KERNEL_LAPLACE)
      return fail(H2SP_EINVAL, "close_gen: unknown kernel id " + std::to_string(g->kernel));
    if (g->kernel == H2SP_KERNEL_EXP && !(g->p0 > 0.0)) return fail(H2SP_EINVAL, "close_gen: exp length p0 <= 0");
  }
  const bool coup_gen = g && g->nodes_row && (P->sym || g->nodes_col);
  if (!in->leaf_basis_row || (P->tr_row_len && !in->transfer_row) || (P->close_len && !in->close && !g) ||
      (P->coupling_len && !in->coupling && !coup_gen))
    return fail(H2SP_EINVAL, "NULL input array (coupling: NULL needs close_gen->nodes_row / nodes_col)");
  if (!P->sym && ((P->leaf_col_len && !in->leaf_basis_col) || (P->tr_col_len && !in->transfer_col)))
    return fail(H2SP_EINVAL, "NULL column-side input array in general mode");
  return H2SP_OK;
}

h2sp_status check_outputs(const h2sp_plan_s *P, const h2sp_outputs *out) {
  if (!out->q_row || (!P->sym && !out->q_col)) return fail(H2SP_EINVAL, "NULL Q output array");
  if (P->bench) {
    if (P->n_csr_rows && (!out->bench_w || !out->bench_y))
      return fail(H2SP_EINVAL, "bench-mode plan: bench_w and bench_y are required");
  } else if (!out->s_val && P->s_nnz) {
    return fail(H2SP_EINVAL, "NULL s_val");
  }
  return H2SP_OK;
}

}  // namespace

extern "C" {

h2sp_status h2sp_plan_upload(h2sp_plan P, void *ws, size_t ws_bytes, void *stream) {
  if (!P) return fail(H2SP_EINVAL, "NULL plan");
  if (h2sp_status s = check_device()) return s;
  if (h2sp_status s = check_ws(P, ws, ws_bytes, P->meta_bytes)) return s;
  return cuda_ok(cudaMemcpyAsync(ws, P->meta.data(), P->meta_bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream),
                 "upload of plan work lists");
}

h2sp_status h2sp_build(h2sp_plan P, const h2sp_inputs *in, const h2sp_outputs *out, void *ws, size_t ws_bytes,
                       void *stream) {
  if (!P || !in || !out) return fail(H2SP_EINVAL, "NULL plan, inputs or outputs");
  if (h2sp_status s = check_ws(P, ws, ws_bytes, P->ws_total)) return s;
  if (h2sp_status s = check_inputs(P, in)) return s;
  if (h2sp_status s = check_outputs(P, out)) return s;
  if (h2sp_status s = check_device()) return s;
  int64_t nl = 0;
  unsigned char *w = static_cast<unsigned char *>(ws);
  return launch_build(P, in, out, w, w + P->meta_bytes, stream, &nl, nullptr, 0);
}

h2sp_status h2sp_build_ex(h2sp_plan P, const h2sp_inputs *in, const h2sp_outputs *out, void *ws, size_t ws_bytes,
                          void *stream, void *const *events, int64_t n_events) {
  if (!P || !in || !out) return fail(H2SP_EINVAL, "NULL plan, inputs or outputs");
  if (events && n_events < 2 * P->launches) return fail(H2SP_EINVAL, "need 2 * launches events");
  if (h2sp_status s = check_ws(P, ws, ws_bytes, P->ws_total)) return s;
  if (h2sp_status s = check_inputs(P, in)) return s;
  if (h2sp_status s = check_outputs(P, out)) return s;
  if (h2sp_status s = check_device()) return s;
  int64_t nl = 0;
  unsigned char *w = static_cast<unsigned char *>(ws);
  h2sp_status s = launch_build(P, in, out, w, w + P->meta_bytes, stream, &nl, events, n_events);
  if (s == H2SP_OK && nl != P->launches) return fail(H2SP_EINVAL, "internal: launch count mismatch");
  return s;
}

h2sp_status h2sp_build_apply(h2sp_plan P, const h2sp_inputs *in, const h2sp_outputs *out, void *ws, size_t ws_bytes,
                             const h2sp_apply_args *ap, void *stream, void *const *events, int64_t n_events) {
  if (!P || !in || !out || !ap) return fail(H2SP_EINVAL, "NULL plan, inputs, outputs or apply arguments");
  if (events && n_events < 2 * P->launches) return fail(H2SP_EINVAL, "need 2 * launches events");
  if (h2sp_status s = check_ws(P, ws, ws_bytes, P->ws_total)) return s;
  if (h2sp_status s = check_outputs(P, out)) return s;
  if (h2sp_status s = check_inputs(P, in)) return s;
  if (ap->ws == ws) return fail(H2SP_EINVAL, "the apply workspace must differ from the build workspace");
  if (ap->nrhs < 1) return fail(H2SP_EINVAL, "nrhs < 1");
  if (h2sp_status s = check_ws(P, ap->ws, ap->ws_bytes, size_t(h2sp_apply_ws_bytes(P, ap->nrhs)))) return s;
  if (ap->b && (!ap->y || ap->ldb < P->n_leaves_local * P->B || ap->ldy < P->n_rows_local))
    return fail(H2SP_EINVAL, "bad U^T b arguments");
  if (ap->w && (!ap->x || ap->ldx < P->n_leaves_local * P->B || ap->ldw < P->n_cols_local))
    return fail(H2SP_EINVAL, "bad V w arguments");
  if (h2sp_status s = check_device()) return s;
  int64_t nl = 0;
  unsigned char *w = static_cast<unsigned char *>(ws);
  h2sp_status s = launch_build(P, in, out, w, w + P->meta_bytes, stream, &nl, events, n_events, ap,
                               static_cast<unsigned char *>(ap->ws) + P->meta_bytes);
  if (s == H2SP_OK && nl != P->launches) return fail(H2SP_EINVAL, "internal: launch count mismatch");
  return s;
}

h2sp_status h2sp_build_meta(h2sp_plan P, const h2sp_inputs *in, const h2sp_outputs *out, const void *meta,
                            void *scratch, size_t scratch_bytes, const h2sp_apply_args *ap, void *stream,
                            void *const *events, int64_t n_events) {
  if (!P || !in || !out || !meta || !scratch) return fail(H2SP_EINVAL, "NULL plan, inputs, outputs, meta or scratch");
  if ((reinterpret_cast<uintptr_t>(meta) & 255) || (reinterpret_cast<uintptr_t>(scratch) & 255))
    return fail(H2SP_EINVAL, "meta / scratch not 256-byte aligned");
  if (scratch_bytes < P->ws_total - P->meta_bytes)
    return fail(H2SP_EINVAL, "scratch too small: " + std::to_string(scratch_bytes) + " < " +
                                 std::to_string(P->ws_total - P->meta_bytes));
  if (events && n_events < 2 * P->launches) return fail(H2SP_EINVAL, "need 2 * launches events");
  if (h2sp_status s = check_outputs(P, out)) return s;
  if (h2sp_status s = check_inputs(P, in)) return s;
  if (ap) {
    if (ap->nrhs < 1) return fail(H2SP_EINVAL, "nrhs < 1");
    if (!ap->ws || (reinterpret_cast<uintptr_t>(ap->ws) & 255)) return fail(H2SP_EINVAL, "apply scratch NULL / unaligned");
    if (ap->ws_bytes < size_t(h2sp_apply_ws_bytes(P, ap->nrhs)) - P->meta_bytes)
      return fail(H2SP_EINVAL, "apply scratch too small");
    if (ap->ws == scratch) return fail(H2SP_EINVAL, "the apply scratch must differ from the build scratch");
    if (ap->b && (!ap->y || ap->ldb < P->n_leaves_local * P->B || ap->ldy < P->n_rows_local))
      return fail(H2SP_EINVAL, "bad U^T b arguments");
    if (ap->w && (!ap->x || ap->ldx < P->n_leaves_local * P->B || ap->ldw < P->n_cols_local))
      return fail(H2SP_EINVAL, "bad V w arguments");
  }
  if (h2sp_status s = check_device()) return s;
  int64_t nl = 0;
  h2sp_status s = launch_build(P, in, out, static_cast<const unsigned char *>(meta), static_cast<unsigned char *>(scratch),
                               stream, &nl, events, n_events, ap, ap ? static_cast<unsigned char *>(ap->ws) : nullptr);
  if (s == H2SP_OK && nl != P->launches) return fail(H2SP_EINVAL, "internal: launch count mismatch");
  return s;
}

h2sp_status h2sp_build_host(h2sp_plan P, const h2sp_inputs *hi, const h2sp_outputs *ho, const h2sp_inputs *di,
                            const h2sp_outputs *dout, void *ws, size_t ws_bytes, void *stream) {
  if (!P || !hi || !ho || !di || !dout) return fail(H2SP_EINVAL, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  // every argument is validated before anything is enqueued (no fork is left
  // unjoined on an error return)
  if (h2sp_status s = check_ws(P, ws, ws_bytes, P->ws_total)) return s;
  if (h2sp_status s = check_inputs(P, di)) return s;
  if (h2sp_status s = check_outputs(P, dout)) return s;
  if (h2sp_status s = check_device()) return s;
  if (hi->close_gen || di->close_gen) {
    if (!hi->close_gen || !di->close_gen) return fail(H2SP_EINVAL, "close_gen set on one side only");
    if (hi->close_gen->dim != di->close_gen->dim) return fail(H2SP_EINVAL, "close_gen: dim differs");
    if (!hi->close_gen->points) return fail(H2SP_EINVAL, "close_gen: NULL host points");
  }
  {
    auto need = [&](const void *h, int64_t n) { return n == 0 || h != nullptr; };
    if (!need(hi->leaf_basis_row, P->leaf_row_len) || !need(hi->transfer_row, P->tr_row_len) ||
        (!P->sym && (!need(hi->leaf_basis_col, P->leaf_col_len) || !need(hi->transfer_col, P->tr_col_len))) ||
        (!hi->close_gen && !need(hi->close, P->close_len)) || (di->coupling && !need(hi->coupling, P->coupling_len)))
      return fail(H2SP_EINVAL, "NULL host input buffer");
  }
  // value-independent CSR indices: expanded and read back on a side stream that
  // overlaps the input copies and the build (joined on every path below)
  const bool early = !P->bench && dout->s_col && ho->s_col && dout->s_rowptr && ho->s_rowptr;
  if (early) {
    if (h2sp_status s = launch_csr_early(P, static_cast<unsigned char *>(ws), dout->s_rowptr, dout->s_col,
                                         ho->s_rowptr, ho->s_col, stream))
      return s;
  }
  h2sp_status rc = H2SP_OK;
  auto done = [&](h2sp_status s) -> h2sp_status {  // join the early fork whatever happened
    if (early) {
      h2sp_status j = launch_csr_early_join(P, stream);
      if (s == H2SP_OK) s = j;
    }
    return s;
  };
  auto h2d = [&](const double *d, const double *h, int64_t n) -> h2sp_status {
    if (n == 0) return H2SP_OK;
    return cuda_ok(cudaMemcpyAsync(const_cast<double *>(d), h, size_t(n) * 8, cudaMemcpyHostToDevice, st), "H2D");
  };
  const int64_t N = int64_t(P->B) << P->L;
  if ((rc = h2d(di->leaf_basis_row, hi->leaf_basis_row, P->leaf_row_len))) return done(rc);
  if ((rc = h2d(di->transfer_row, hi->transfer_row, P->tr_row_len))) return done(rc);
  if (!P->sym) {
    if ((rc = h2d(di->leaf_basis_col, hi->leaf_basis_col, P->leaf_col_len))) return done(rc);
    if ((rc = h2d(di->transfer_col, hi->transfer_col, P->tr_col_len))) return done(rc);
  }
  if (hi->close_gen) {
    if ((rc = h2d(di->close_gen->points, hi->close_gen->points, N * int64_t(hi->close_gen->dim)))) return done(rc);
    if (hi->close_gen->nodes_row && di->close_gen->nodes_row &&
        (rc = h2d(di->close_gen->nodes_row, hi->close_gen->nodes_row, P->zb_row_len * hi->close_gen->dim)))
      return done(rc);
    if (!P->sym && hi->close_gen->nodes_col && di->close_gen->nodes_col &&
        (rc = h2d(di->close_gen->nodes_col, hi->close_gen->nodes_col, P->zb_col_len * hi->close_gen->dim)))
      return done(rc);
  } else if ((rc = h2d(di->close, hi->close, P->close_len))) {
    return done(rc);
  }
  if (di->coupling && (rc = h2d(di->coupling, hi->coupling, P->coupling_len))) return done(rc);
  if (P->bench && (rc = h2d(dout->bench_w, ho->bench_w, N))) return done(rc);
  h2sp_outputs d2 = *dout;
  if (early) d2.s_col = nullptr, d2.s_rowptr = nullptr;  // already being produced on the side stream
  if ((rc = h2sp_build(P, di, &d2, ws, ws_bytes, stream))) return done(rc);
  auto d2h = [&](void *h, const void *d, size_t bytes) -> h2sp_status {
    if (bytes == 0 || !h) return H2SP_OK;
    if (!d) return fail(H2SP_EINVAL, "NULL device output");
    return cuda_ok(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st), "D2H");
  };
  if ((rc = d2h(ho->q_row, dout->q_row, size_t(P->q_row_len) * 8))) return done(rc);
  if (!P->sym && (rc = d2h(ho->q_col, dout->q_col, size_t(P->q_col_len) * 8))) return done(rc);
  if (P->bench) {
    if ((rc = d2h(ho->bench_y, dout->bench_y, size_t(N) * 8))) return done(rc);
    if ((rc = d2h(ho->bench_r2, dout->bench_r2, size_t(N) * 8))) return done(rc);
  } else if ((rc = d2h(ho->s_val, dout->s_val, size_t(P->s_nnz) * 8))) {
    return done(rc);
  }
  if (early) return done(H2SP_OK);
  if (dout->s_col && (rc = d2h(ho->s_col, dout->s_col, size_t(P->s_nnz) * 4))) return rc;
  if (dout->s_rowptr && (rc = d2h(ho->s_rowptr, dout->s_rowptr, size_t(P->n_rows_local + 1) * 8))) return rc;
  return H2SP_OK;
}

h2sp_status h2sp_eval_kernel_blocks(const h2sp_close_gen *k, const double *x_nodes, const double *y_nodes,
                                    const h2sp_block_desc *blocks, int64_t n_blocks, double *out, void *stream) {
  if (!k || n_blocks < 0) return fail(H2SP_EINVAL, "NULL kernel descriptor or n_blocks < 0");
  if (n_blocks > 0 && (!x_nodes || !y_nodes || !blocks || !out)) return fail(H2SP_EINVAL, "NULL device array");
  if (k->dim < 1 || k->dim > 3) return fail(H2SP_EINVAL, "kernel blocks: dim must be 1, 2 or 3");
  if (k->kernel < H2SP_KERNEL_EXP || k->kernel > H2SP_KERNEL_LAPLACE)
    return fail(H2SP_EINVAL, "kernel blocks: unknown kernel id " + std::to_string(k->kernel));
  if (k->kernel == H2SP_KERNEL_EXP && !(k->p0 > 0.0)) return fail(H2SP_EINVAL, "kernel blocks: exp length p0 <= 0");
  if (h2sp_status s = check_device()) return s;
  return launch_kernel_blocks(k, x_nodes, y_nodes, blocks, n_blocks, out, stream);
}

h2sp_status h2sp_cheb_construct(h2sp_plan P, const void *meta, int side, const h2sp_cheb_spec *spec,
                                const double *points, const double *box_lo, const double *box_hi, double *leaf_basis,
                                double *transfer, double *nodes, void *stream) {
  if (!P || !meta || !spec || !points || !box_lo || !box_hi || !leaf_basis || !nodes)
    return fail(H2SP_EINVAL, "NULL argument");
  if (side != 0 && side != 1) return fail(H2SP_EINVAL, "side must be 0 (row) or 1 (column)");
  if (spec->dim < 1 || spec->dim > 3) return fail(H2SP_EINVAL, "dim must be 1, 2 or 3");
  int r = 1;
  for (int a = 0; a < spec->dim; a++) {
    if (spec->orders[a] < 1 || spec->orders[a] > 8) return fail(H2SP_EINVAL, "orders must lie in [1, 8]");
    r *= spec->orders[a];
  }
  if (r > 64) return fail(H2SP_EINVAL, "prod(orders) > 64");
  const auto &k = (side && !P->sym) ? P->k_col : P->k_row;
  for (int64_t c = 0; c < P->ncl; c++)
    if (k[c] != 0 && k[c] != r)
      return fail(H2SP_ERANK, "cluster " + std::to_string(c) + ": rank " + std::to_string(k[c]) +
                                  " is neither 0 nor prod(orders) = " + std::to_string(r));
  if (P->ncl > (int64_t(1) << L_MAX_CHEB)) return fail(H2SP_EUNSUPPORTED, "too many clusters");
  if ((side ? P->tr_col_len : P->tr_row_len) > 0 && !transfer && !(side && P->sym))
    return fail(H2SP_EINVAL, "NULL transfer");
  if (h2sp_status s = check_device()) return s;
  return launch_cheb_construct(P, static_cast<const unsigned char *>(meta), side, spec, points, box_lo, box_hi,
                               leaf_basis, transfer, nodes, stream);
}

h2sp_status h2sp_plan_set_qr_mode(h2sp_plan P, int mode) {
  if (!P) return fail(H2SP_EINVAL, "NULL plan");
  if (mode != H2SP_QR_NEED && mode != H2SP_QR_ALL && mode != H2SP_QR_REUSE) return fail(H2SP_EINVAL, "unknown QR mode");
  P->qr_mode = mode;
  return H2SP_OK;
}

int64_t h2sp_apply_ws_bytes(h2sp_plan P, int nrhs) {
  if (!P || nrhs < 0) return -1;
  int64_t z = P->zb_row_len > P->zb_col_len ? P->zb_row_len : P->zb_col_len;
  // meta | upward pass: basis coefficients (256-aligned), arrival counters (256-aligned)
  //      | downward pass: basis coefficients (256-aligned), cluster flags + ticket
  const int64_t zb = (z * int64_t(nrhs) * 8 + 255) / 256 * 256, ab = (P->ncl * 4 + 255) / 256 * 256;
  return int64_t(P->meta_bytes) + 2 * zb + ab + (P->ncl + 1) * 4;
}

static h2sp_status apply_common(h2sp_plan P, const double *q, const void *a, int64_t lda, void *b, int64_t ldb,
                                int nrhs, void *ws, size_t ws_bytes) {
  if (!P || !q || !a || !b) return fail(H2SP_EINVAL, "NULL argument");
  if (nrhs < 1) return fail(H2SP_EINVAL, "nrhs < 1");
  const int64_t ntree = P->n_leaves_local * P->B;  // tree-order rows of this shard
  const int64_t nrows = P->n_rows_local;
  (void)ntree;
  (void)nrows;
  if (lda < 1 || ldb < 1) return fail(H2SP_EINVAL, "leading dimension < 1");
  if (h2sp_status s = check_ws(P, ws, ws_bytes, size_t(h2sp_apply_ws_bytes(P, nrhs)))) return s;
  return check_device();
}

h2sp_status h2sp_apply_Ut(h2sp_plan P, const double *q_row, const double *b, int64_t ldb, double *y, int64_t ldy,
                          int nrhs, void *ws, size_t ws_bytes, void *stream) {
  if (h2sp_status s = apply_common(P, q_row, b, ldb, y, ldy, nrhs, ws, ws_bytes)) return s;
  if (ldb < P->n_leaves_local * P->B || ldy < P->n_rows_local) return fail(H2SP_EINVAL, "leading dimension too small");
  unsigned char *w = static_cast<unsigned char *>(ws);
  return launch_apply_Ut(P, q_row, b, ldb, y, ldy, nrhs, w, w + P->meta_bytes, stream, false);
}

h2sp_status h2sp_apply_V(h2sp_plan P, const double *q_col, const double *y, int64_t ldy, double *x, int64_t ldx,
                         int nrhs, void *ws, size_t ws_bytes, void *stream) {
  if (h2sp_status s = apply_common(P, q_col, y, ldy, x, ldx, nrhs, ws, ws_bytes)) return s;
  if (ldx < P->n_leaves_local * P->B || ldy < P->n_cols_local) return fail(H2SP_EINVAL, "leading dimension too small");
  unsigned char *w = static_cast<unsigned char *>(ws);
  return launch_apply_V(P, q_col, y, ldy, x, ldx, nrhs, w, w + P->meta_bytes, stream, !P->sym);
}

}  // extern "C"
