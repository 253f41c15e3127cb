// Host symbolic phase ("plan"): validates the block cluster
// tree, derives local sizes, the S order (the permutations P_rk / P_ck,
// P:219-223), the block pattern of S, CSR row pointers
// and every per-level device work list.  Integer work only, O(#blocks log).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2sp_internal.h"

namespace h2sp {
static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }
h2sp_status fail(h2sp_status s, const std::string &m) {
  g_err = m;
  return s;
}
}  // namespace h2sp

using namespace h2sp;

namespace {

struct PlanError : std::runtime_error {
  h2sp_status code;
  PlanError(h2sp_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

inline int64_t lvl_off(int L, int k) { return (int64_t(1) << (L + 1)) - (int64_t(1) << (L - k + 1)); }
}  // namespace
namespace h2sp {
int strip_tn_of_level(int k) {
  static const int from = getenv("H2SP_STRIP_NARROW_FROM") ? atoi(getenv("H2SP_STRIP_NARROW_FROM")) : 1 << 20;
  return k >= from ? STRIP_TN_SMALL : STRIP_TN;
}
}  // namespace h2sp
namespace {
inline int level_of(int L, int64_t c) {  // level of level-major cluster id c
  int k = 0;
  while (k < L && c >= lvl_off(L, k + 1)) k++;
  return k;
}
inline uint64_t pkey(int64_t t, int64_t s) { return (uint64_t(uint32_t(t)) << 32) | uint64_t(uint32_t(s)); }
inline int32_t kt(uint64_t k) { return int32_t(k >> 32); }
inline int32_t ks(uint64_t k) { return int32_t(k & 0xffffffffu); }

int64_t find(const std::vector<uint64_t> &v, uint64_t key) {
  auto it = std::lower_bound(v.begin(), v.end(), key);
  if (it == v.end() || *it != key) return -1;
  return int64_t(it - v.begin());
}

std::vector<uint64_t> read_csr(const int64_t *ptr, const int32_t *col, int64_t M, const char *what) {
  std::vector<uint64_t> out;
  if (M == 0) return out;
  if (!ptr) throw PlanError(H2SP_EINVAL, std::string(what) + ": NULL row pointer");
  if (ptr[0] != 0) throw PlanError(H2SP_ETREE, std::string(what) + ": ptr[0] != 0");
  for (int64_t t = 0; t < M; t++) {
    if (ptr[t + 1] < ptr[t]) throw PlanError(H2SP_ETREE, std::string(what) + ": decreasing row pointer");
    for (int64_t j = ptr[t]; j < ptr[t + 1]; j++) {
      int32_t s = col[j];
      if (s < 0 || s >= M) throw PlanError(H2SP_ETREE, std::string(what) + ": column out of range");
      if (j > ptr[t] && col[j - 1] >= s) throw PlanError(H2SP_ETREE, std::string(what) + ": columns not strictly ascending");
      out.push_back(pkey(t, s));
    }
  }
  return out;
}

struct Grp {  // a frozen column group (l, s) of a strip panel, at columns [col0, col0 + m)
  int32_t l, s, m, col0;
};


struct BlockRec {
  int64_t roff, coff;
  int64_t grow;  // global S row of roff (row side)
  int32_t mr, mc;
  int32_t kind;  // 0 pair direct, 1 pair mirror, 2 rstrip direct, 3 rstrip transposed, 4 cstrip transposed
  int32_t level;
  int64_t idx;   // item index within its level list
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct MetaBuilder {
  std::vector<unsigned char> buf;
  template <class T>
  size_t put(const std::vector<T> &v) {
    size_t off = align_up(buf.size(), 256);
    buf.resize(off + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(buf.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  }
};

int round8(int x) { return (x + 7) / 8 * 8; }

}  // namespace

extern "C" {

const char *h2sp_status_str(h2sp_status s) {
  switch (s) {
    case H2SP_OK: return "ok";
    case H2SP_EINVAL: return "invalid argument";
    case H2SP_ETREE: return "invalid block cluster tree";
    case H2SP_ERANK: return "invalid rank distribution";
    case H2SP_ENOMEM: return "out of host memory";
    case H2SP_ECUDA: return "CUDA error";
    case H2SP_ENCCL: return "NCCL error";
    case H2SP_EUNSUPPORTED: return "unsupported shape";
  }
  return "unknown status";
}

const char *h2sp_last_error(void) { return g_err.c_str(); }

void h2sp_plan_destroy(h2sp_plan p) { delete p; }

h2sp_status h2sp_plan_create(const h2sp_structure *st, int flags, h2sp_plan *out) {
  return h2sp_plan_create_shard(st, 0, 1, flags, out);
}

h2sp_status h2sp_plan_create_shard(const h2sp_structure *st, int rank, int world, int flags, h2sp_plan *out) {
  if (flags & ~(H2SP_PLAN_EXPLICIT_Q | H2SP_PLAN_BENCH)) return fail(H2SP_EINVAL, "unknown plan flags");
  if (!st || !out) return fail(H2SP_EINVAL, "NULL structure or output pointer");
  *out = nullptr;
  h2sp_plan_s *P = nullptr;
  try {
    const int L = st->L, B = st->leaf_size;
    if (world < 1 || (world & (world - 1)) != 0) throw PlanError(H2SP_EINVAL, "world must be a power of two");
    if (rank < 0 || rank >= world) throw PlanError(H2SP_EINVAL, "rank outside [0, world)");
    if (L >= 0 && L <= 24 && int64_t(world) > (int64_t(1) << L)) throw PlanError(H2SP_EINVAL, "world > number of leaves");
    if (L < 0 || L > 24) throw PlanError(H2SP_EINVAL, "L out of range [0, 24]");
    if (B < 1) throw PlanError(H2SP_EINVAL, "leaf_size < 1");
    if (!st->rank_row) throw PlanError(H2SP_EINVAL, "rank_row is NULL");
    if (!st->symmetric && !st->rank_col) throw PlanError(H2SP_EINVAL, "rank_col is NULL in general mode");
    P = new h2sp_plan_s();
    P->L = L;
    P->B = B;
    P->sym = st->symmetric ? 1 : 0;
    P->bench = (flags & H2SP_PLAN_BENCH) ? 1 : 0;
    const bool bench = P->bench != 0;
    P->N = int64_t(B) << L;
    const int64_t ncl = (int64_t(1) << (L + 1)) - 1;
    const int64_t nleaf = int64_t(1) << L;
    P->ncl = ncl;
    auto &nr = P->n_row, &kr = P->k_row, &nc = P->n_col, &kc = P->k_col;
    kr.assign(st->rank_row, st->rank_row + ncl);
    if (P->sym) {
      if (st->rank_col)
        for (int64_t c = 0; c < ncl; c++)
          if (st->rank_col[c] != st->rank_row[c]) throw PlanError(H2SP_ERANK, "symmetric mode needs rank_col == rank_row");
      kc = kr;
    } else {
      kc.assign(st->rank_col, st->rank_col + ncl);
    }
    auto local = [&](const std::vector<int32_t> &k, std::vector<int32_t> &n, const char *side) {
      n.assign(ncl, 0);
      for (int64_t i = 0; i < nleaf; i++) n[i] = B;
      for (int k_ = 1; k_ <= L; k_++)
        for (int64_t i = 0; i < (int64_t(1) << (L - k_)); i++)
          n[lvl_off(L, k_) + i] = k[lvl_off(L, k_ - 1) + 2 * i] + k[lvl_off(L, k_ - 1) + 2 * i + 1];
      for (int64_t c = 0; c < ncl; c++)
        if (k[c] < 0 || k[c] > n[c])
          throw PlanError(H2SP_ERANK, std::string(side) + " rank outside [0, n_t] at cluster " + std::to_string(c));
      if (k[ncl - 1] != 0) throw PlanError(H2SP_ERANK, std::string(side) + " root rank must be 0");
    };
    local(kr, nr, "row");
    local(kc, nc, "column");
    P->nmax = 0;
    for (int64_t c = 0; c < ncl; c++) {
      P->nmax = std::max(P->nmax, std::max(nr[c], nc[c]));
      if (c < nleaf ? (nr[c] > 128 || nc[c] > 128) : (nr[c] > 64 || nc[c] > 64))
        throw PlanError(H2SP_EUNSUPPORTED, "local size n_t > 128 at a leaf or > 64 above (kernels are built for B <= 128, 2r <= 64)");
    }
    // ---- sharding by top-level subtrees: rank g owns cluster g of the
    //      partition level Pl = L - log2(world) and all of its descendants
    int lw = 0;
    while ((1 << lw) < world) lw++;
    const int Pl = L - lw;
    P->rank = rank;
    P->world = world;
    P->part_level = Pl;
    if (world > 1)
      for (int k = Pl + 1; k <= L; k++)
        for (int64_t i = 0; i < (int64_t(1) << (L - k)); i++)
          if (nr[lvl_off(L, k) + i] > 0 || nc[lvl_off(L, k) + i] > 0)
            throw PlanError(H2SP_EUNSUPPORTED,
                            "sharded plan: work above the partition level (gather of the remainder not implemented)");
    // mine(k, i): cluster (k, i) belongs to this rank's subtree (levels above Pl are empty)
    auto mine = [&](int k, int64_t i) -> bool {
      if (world == 1) return true;
      if (k > Pl) return rank == 0;
      return (i >> (Pl - k)) == rank;
    };
    P->first_leaf = world == 1 ? 0 : int64_t(rank) << Pl;
    P->n_leaves_local = world == 1 ? nleaf : (int64_t(1) << Pl);

    // ---------------------------------------------------------------- block tree
    std::vector<std::vector<uint64_t>> near(L + 1), adm(L + 1);
    if (!st->near_col && st->near_ptr && st->near_ptr[nleaf] > 0) throw PlanError(H2SP_EINVAL, "near_col is NULL");
    near[0] = read_csr(st->near_ptr, st->near_col, nleaf, "near");
    std::vector<int64_t> adm_in_off(L + 1, 0);  // CSR order index base per level (coupling offsets)
    for (int k = 0; k < L; k++) {
      if (!st->adm_ptr || !st->adm_col) throw PlanError(H2SP_EINVAL, "adm_ptr/adm_col is NULL");
      adm[k] = read_csr(st->adm_ptr[k], st->adm_col[k], int64_t(1) << (L - k), "adm");
    }
    if (P->sym) {
      auto check_sym = [&](const std::vector<uint64_t> &v, const char *w) {
        for (uint64_t x : v)
          if (find(v, pkey(ks(x), kt(x))) < 0) throw PlanError(H2SP_ETREE, std::string(w) + " list not symmetric");
      };
      check_sym(near[0], "near");
      for (int k = 0; k < L; k++) check_sym(adm[k], "adm");
    }
    for (int k = 1; k <= L; k++) {
      std::vector<uint64_t> par;
      par.reserve(near[k - 1].size() / 2 + adm[k - 1].size() / 2 + 1);
      for (uint64_t x : near[k - 1]) par.push_back(pkey(kt(x) / 2, ks(x) / 2));
      for (uint64_t x : adm[k - 1]) par.push_back(pkey(kt(x) / 2, ks(x) / 2));
      std::sort(par.begin(), par.end());
      par.erase(std::unique(par.begin(), par.end()), par.end());
      near[k] = std::move(par);
      for (uint64_t x : near[k]) {
        if (k < L && find(adm[k], x) >= 0) throw PlanError(H2SP_ETREE, "pair is both near and admissible");
        for (int a = 0; a < 2; a++)
          for (int b = 0; b < 2; b++) {
            uint64_t ch = pkey(2 * kt(x) + a, 2 * ks(x) + b);
            bool inn = find(near[k - 1], ch) >= 0, ina = find(adm[k - 1], ch) >= 0;
            if (inn == ina) throw PlanError(H2SP_ETREE, "children of a close block are not partitioned by N u A at level " + std::to_string(k - 1));
          }
      }
    }
    if (L == 0) {
      if (near[0].size() != 1) throw PlanError(H2SP_ETREE, "L = 0 needs the single near pair (0, 0)");
    } else if (near[L].size() != 1 || near[L][0] != pkey(0, 0)) {
      throw PlanError(H2SP_ETREE, "block tree does not cover the matrix (N_L != {(root, root)})");
    }

    // ---------------------------------------------------------------- offsets
    auto mr = [&](int64_t c) { return nr[c] - kr[c]; };
    auto mc = [&](int64_t c) { return nc[c] - kc[c]; };
    P->s_off_row.assign(ncl, 0);
    P->s_off_col.assign(ncl, 0);
    {
      int64_t a = 0, b = 0;
      for (int64_t c = 0; c < ncl; c++) {  // level-major order == S order
        P->s_off_row[c] = a;
        a += mr(c);
        P->s_off_col[c] = b;
        b += mc(c);
      }
      if (a != P->N || b != P->N) throw PlanError(H2SP_ERANK, "sum of frozen sizes != N");
    }
    // frozen group widths are frozen sizes m: all multiples of 32 -> the strip
    // kernels' bench epilogue can reduce straight from the accumulators (a
    // property of the whole matrix, so every shard of it agrees)
    P->strip_aligned = 1;
    for (int64_t c = 0; c < ncl; c++)
      if (mr(c) % 32 || mc(c) % 32) P->strip_aligned = 0;
    // local S rows of this shard: the owned clusters' rows, in S order (== s_off for one rank)
    std::vector<int64_t> loc_off(ncl, -1), loc_off_c(ncl, -1);
    {
      int64_t a = 0, b = 0;
      for (int k = 0; k <= L; k++)
        for (int64_t i = 0; i < (int64_t(1) << (L - k)); i++) {
          const int64_t c = lvl_off(L, k) + i;
          if (!mine(k, i)) continue;
          loc_off[c] = a;
          a += mr(c);
          loc_off_c[c] = b;
          b += mc(c);
        }
      P->n_rows_local = a;
      P->n_cols_local = b;
    }
    P->loc_off_row = loc_off;
    P->loc_off_col = loc_off_c;
    std::vector<int64_t> rh_off_row(ncl), rh_off_col(ncl), tr_off_row(ncl, 0), tr_off_col(ncl, 0), zb_row(ncl),
        zb_col(ncl);
    std::vector<int64_t> leaf_off_row(nleaf), leaf_off_col(nleaf);
    P->q_off_row.assign(ncl, 0);
    P->q_off_col.assign(ncl, 0);
    {
      int64_t q1 = 0, q2 = 0, r1 = 0, r2 = 0, t1 = 0, t2 = 0, z1 = 0, z2 = 0, l1 = 0, l2 = 0;
      for (int64_t c = 0; c < ncl; c++) {
        P->q_off_row[c] = q1;
        q1 += int64_t(nr[c]) * nr[c];
        P->q_off_col[c] = q2;
        q2 += int64_t(nc[c]) * nc[c];
        rh_off_row[c] = r1;
        r1 += int64_t(kr[c]) * kr[c];
        rh_off_col[c] = r2;
        r2 += int64_t(kc[c]) * kc[c];
        zb_row[c] = z1;
        z1 += kr[c];
        zb_col[c] = z2;
        z2 += kc[c];
        if (c >= nleaf) {
          tr_off_row[c] = t1;
          t1 += int64_t(nr[c]) * kr[c];
          tr_off_col[c] = t2;
          t2 += int64_t(nc[c]) * kc[c];
        } else {
          leaf_off_row[c] = l1;
          l1 += int64_t(B) * kr[c];
          leaf_off_col[c] = l2;
          l2 += int64_t(B) * kc[c];
        }
      }
      P->q_row_len = q1;
      P->q_col_len = P->sym ? 0 : q2;
      P->rh_row_len = r1;
      P->rh_col_len = P->sym ? 0 : r2;
      P->tr_row_len = t1;
      P->tr_col_len = P->sym ? 0 : t2;
      P->leaf_row_len = l1;
      P->leaf_col_len = P->sym ? 0 : l2;
      P->zb_row_len = z1;
      P->zb_col_len = z2;
    }
    P->close_len = int64_t(near[0].size()) * B * B;
    std::vector<std::vector<int64_t>> coup_in(L + 1);  // input offset of D per adm pair
    {
      int64_t o = 0;
      for (int k = 0; k < L; k++) {
        coup_in[k].resize(adm[k].size());
        for (size_t j = 0; j < adm[k].size(); j++) {
          coup_in[k][j] = o;
          o += int64_t(kr[lvl_off(L, k) + kt(adm[k][j])]) * kc[lvl_off(L, k) + ks(adm[k][j])];
        }
      }
      P->coupling_len = o;
    }

    // ---------------------------------------------------------------- work lists
    const bool sym = P->sym;
    double flops_qr = 0, flops_coup = 0, flops_cong = 0, flops_strip = 0;
    double uniq_qr = 0, uniq_coup = 0, uniq_cong = 0, uniq_strip = 0;  // owned work only (sharded plans)
    double flops_strip_exec = 0;
    // strip kernels skip the k range of an absent child when every panel column
    // of a warp's slab has the same children present (aligned plans, kernels.cu)
    const bool strip_skip = bench && P->strip_aligned;
    int64_t dt_len = 0, bb_len = 0, yr_len = 0, yc_len = 0;
    std::vector<std::vector<PairItem>> pairs(L + 1);
    // strip panels, index set * (L+1) + level (set 0: groups born at level 0, set 1: later)
    std::vector<std::vector<StripPanel>> rpan(2 * (L + 1)), cpan(2 * (L + 1));
    std::vector<std::vector<StripGroup>> rgrp(2 * (L + 1)), cgrp(2 * (L + 1));
    std::vector<std::vector<StripTile>> rtil(2 * (L + 1)), ctil(2 * (L + 1));
    std::vector<std::vector<int64_t>> rgrp_direct(2 * (L + 1));   // direct S dst of each row group (checked below)
    std::vector<std::vector<CouplingItem>> coup(L + 1);
    std::vector<std::vector<int64_t>> dt_slot(L + 1), bb_slot(L + 1);
    std::vector<std::vector<int64_t>> pair_index(L + 1);   // near index -> item index (canonical) or -1
    std::vector<BlockRec> blocks;
    std::vector<std::vector<Grp>> R_prev[2], C_prev[2];   // groups of each panel at level k-1, per set
    std::vector<int64_t> Rb_prev[2], Cb_prev[2];          // panel bases at level k-1, per set
    for (int k = 0; k <= L; k++) {
      const int64_t base = lvl_off(L, k);
      const int64_t M = int64_t(1) << (L - k);
      // QR flops (approximate Householder count)
      for (int64_t i = 0; i < M; i++) {
        double n = nr[base + i], kk = kr[base + i];
        double f = 2 * n * kk * kk + 4 * n * n * kk;
        if (!sym) {
          n = nc[base + i];
          kk = kc[base + i];
          f += 2 * n * kk * kk + 4 * n * n * kk;
        }
        flops_qr += f;
        if (mine(k, i)) uniq_qr += f;
      }
      // couplings
      if (k < L) {
        dt_slot[k].assign(adm[k].size(), -1);
        for (size_t j = 0; j < adm[k].size(); j++) {
          int32_t t = kt(adm[k][j]), s = ks(adm[k][j]);
          if (sym && t > s) continue;
          int64_t ct = base + t, cs = base + s;
          int64_t sz = int64_t(kr[ct]) * kc[cs];
          if (sz == 0) continue;
          // sharded: only the couplings feeding a congruence of this shard at level k+1
          if (!(mine(k + 1, t / 2) || (sym && mine(k + 1, s / 2)))) continue;
          dt_slot[k][j] = dt_len;
          coup[k].push_back(CouplingItem{int32_t(ct), int32_t(cs), coup_in[k][j], dt_len});
          dt_len += sz;
          flops_coup += 2.0 * kr[ct] * kc[cs] * (kr[ct] + kc[cs]);
          if (mine(k + 1, t / 2)) uniq_coup += 2.0 * kr[ct] * kc[cs] * (kr[ct] + kc[cs]);
        }
      }
      // near pairs: items for canonical pairs
      const auto &Nk = near[k];
      pair_index[k].assign(Nk.size(), -1);
      bb_slot[k].assign(Nk.size(), -1);
      for (size_t j = 0; j < Nk.size(); j++) {
        int32_t t = kt(Nk[j]), s = ks(Nk[j]);
        if (sym && t > s) continue;
        int64_t ct = base + t, cs = base + s;
        if (nr[ct] == 0 || nc[cs] == 0) continue;  // empty block: nothing to compute
        // sharded: rows of t are ours, or (symmetric) the mirror rows of s are
        if (!(mine(k, t) || (sym && mine(k, s)))) continue;
        PairItem it{};
        it.t = int32_t(ct);
        it.s = int32_t(cs);
        it.nt = int16_t(nr[ct]);
        it.ns = int16_t(nc[cs]);
        it.kt = int16_t(kr[ct]);
        it.ks = int16_t(kc[cs]);
        if (k > 0) {
          const int64_t t1 = lvl_off(L, k - 1) + 2 * int64_t(t), s1 = lvl_off(L, k - 1) + 2 * int64_t(s);
          it.kr0 = int16_t(kr[t1]);
          it.kr1 = int16_t(kr[t1 + 1]);
          it.kc0 = int16_t(kc[s1]);
          it.kc1 = int16_t(kc[s1 + 1]);
        }
        it.q_off_t = P->q_off_row[ct];
        it.q_off_s = sym ? P->q_off_row[cs] : P->q_off_col[cs];
        it.s_dst = it.s_dst_m = it.bb_dst = it.yr_dst = it.yc_dst = -1;
        for (int q = 0; q < 4; q++) it.g_src[q] = -1;
        if (k == 0) {
          it.g_src[0] = int64_t(j) * B * B;
        } else {
          int32_t gk = 0;
          for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) {
              int32_t ca = 2 * t + a, db = 2 * s + b;
              int64_t kca = kr[lvl_off(L, k - 1) + ca], kdb = kc[lvl_off(L, k - 1) + db];
              int kind = G_EMPTY;
              int64_t src = -1;
              if (kca > 0 && kdb > 0) {
                bool tr = sym && ca > db;
                uint64_t key = tr ? pkey(db, ca) : pkey(ca, db);
                int64_t jn = find(near[k - 1], key);
                if (jn >= 0) {
                  kind = tr ? G_BB_T : G_BB;
                  src = bb_slot[k - 1][jn];
                } else {
                  int64_t ja = find(adm[k - 1], key);
                  if (ja < 0) throw PlanError(H2SP_ETREE, "internal: child pair neither near nor admissible");
                  kind = tr ? G_DT_T : G_DT;
                  src = dt_slot[k - 1][ja];
                }
                if (src < 0) throw PlanError(H2SP_ETREE, "internal: missing child block slot");
              }
              gk |= kind << (4 * (a * 2 + b));
              it.g_src[a * 2 + b] = src;
            }
          it.gkind = gk;
        }
        if (k < L && kr[ct] > 0 && kc[cs] > 0) {
          bb_slot[k][j] = bb_len;
          it.bb_dst = bb_len;
          bb_len += int64_t(kr[ct]) * kc[cs];
        }
        pair_index[k][j] = int64_t(pairs[k].size());
        pairs[k].push_back(it);
        flops_cong += 2.0 * nr[ct] * nc[cs] * (nr[ct] + nc[cs]);
        if (mine(k, t)) uniq_cong += 2.0 * nr[ct] * nc[cs] * (nr[ct] + nc[cs]);
      }
      // ---- strips arriving from level k-1 (Eq. u1v1): one panel per rotating cluster
      //      and per panel set: set 0 = groups born at level 0 (they depend on the
      //      level-0 congruence only and run concurrently with the upper levels),
      //      set 1 = groups born at a level >= 1.  Index of (set, level): set*(L+1)+k.
      std::vector<std::vector<Grp>> R_cur[2] = {std::vector<std::vector<Grp>>(M), std::vector<std::vector<Grp>>(M)};
      std::vector<std::vector<Grp>> C_cur[2] = {std::vector<std::vector<Grp>>(M), std::vector<std::vector<Grp>>(M)};
      auto merge = [&](std::vector<std::vector<Grp>> &prev, std::vector<int64_t> &prev_base, bool row_side,
                       int sidx, std::vector<StripPanel> &pans, std::vector<StripGroup> &grps,
                       std::vector<StripTile> &tils, std::vector<std::vector<Grp>> &cur) {
        const auto &kq = row_side ? kr : kc;
        const auto &nq = row_side ? nr : nc;
        for (int64_t p = 0; p < M; p++) {
          const auto &A = prev[2 * p], &Bv = prev[2 * p + 1];
          if (A.empty() && Bv.empty()) continue;
          const int64_t cq = base + p;
          const int64_t c1 = lvl_off(L, k - 1) + 2 * p;
          const int32_t mq = nq[cq] - kq[cq];
          StripPanel pn{};
          pn.q = int32_t(cq);
          pn.ld_c1 = A.empty() ? 0 : A.back().col0 + A.back().m;
          pn.ld_c2 = Bv.empty() ? 0 : Bv.back().col0 + Bv.back().m;
          pn.src_c1 = A.empty() ? -1 : prev_base[2 * p];
          pn.src_c2 = Bv.empty() ? -1 : prev_base[2 * p + 1];
          pn.y_dst = pn.s_dst = -1;
          pn.gbeg = int32_t(grps.size());
          size_t i = 0, j = 0;
          int32_t col = 0;
          const int64_t pidx = int64_t(pans.size());
          while (i < A.size() || j < Bv.size()) {
            bool takeA, takeB;
            if (i < A.size() && j < Bv.size()) {
              const bool eq = A[i].l == Bv[j].l && A[i].s == Bv[j].s;
              const bool lt = A[i].l < Bv[j].l || (A[i].l == Bv[j].l && A[i].s < Bv[j].s);
              takeA = eq || lt;
              takeB = eq || !lt;
            } else {
              takeA = i < A.size();
              takeB = !takeA;
            }
            const Grp &g = takeA ? A[i] : Bv[j];
            StripGroup sg{};
            sg.col0 = col;
            sg.m = g.m;
            sg.pos_c1 = takeA ? A[i].col0 : -1;
            sg.pos_c2 = takeB ? Bv[j].col0 : -1;
            sg.s_dst_t = -1;
            const int64_t gi = int64_t(grps.size());
            const int64_t cf = lvl_off(L, g.l) + g.s;  // fixed cluster
            sg.wc0 = row_side ? int32_t(P->s_off_col[cf]) : 0;
            if (mq > 0) {
              if (row_side) {
                if (mine(k, p))
                  blocks.push_back(BlockRec{loc_off[cq], P->s_off_col[cf], P->s_off_row[cq], mq, g.m, 2, sidx, gi});
                if (sym && mine(g.l, g.s))
                  blocks.push_back(BlockRec{loc_off[cf], P->s_off_col[cq], P->s_off_row[cf], g.m, mq, 3, sidx, gi});
              } else if (mine(g.l, g.s)) {
                blocks.push_back(BlockRec{loc_off[cf], P->s_off_col[cq], P->s_off_row[cf], g.m, mq, 4, sidx, gi});
              }
            }
            const double rows = (takeA ? kq[c1] : 0) + (takeB ? kq[c1 + 1] : 0);
            flops_strip += 2.0 * nq[cq] * rows * g.m;
            flops_strip_exec += 2.0 * nq[cq] * nq[cq] * g.m;  // the kernels multiply by all of Q_p
            // a row panel's groups all sit with its rotating cluster's owner (the
            // symmetric halo copies elsewhere are duplicates); a column-strip group
            // exists only with its fixed row cluster's owner
            if (!row_side || mine(k, p)) uniq_strip += 2.0 * nq[cq] * rows * g.m;
            grps.push_back(sg);
            if (kq[cq] > 0) cur[p].push_back(Grp{g.l, g.s, g.m, col});
            col += g.m;
            if (takeA) i++;
            if (takeB) j++;
          }
          pn.width = col;
          pn.gend = int32_t(grps.size());
          const int tn = strip_tn_of_level(k);
          if (bench) {
            // bench mode: tiles hold whole groups (each group's partial sums come
            // from one CTA, so no two CTAs add into one slot)
            int32_t g = pn.gbeg;
            while (g < pn.gend) {
              int32_t e = g, w = 0;
              while (e < pn.gend && w + grps[e].m <= tn) w += grps[e++].m;
              if (e == g) throw PlanError(H2SP_EUNSUPPORTED, "bench mode: frozen group wider than a strip tile");
              tils.push_back(StripTile{int32_t(pidx), grps[g].col0, grps[g].col0 + w, g});
              g = e;
            }
          } else {
            for (int32_t c0 = 0; c0 < col; c0 += tn) {
              int32_t g0 = pn.gbeg;
              while (g0 + 1 < pn.gend && grps[g0 + 1].col0 <= c0) g0++;
              tils.push_back(StripTile{int32_t(pidx), c0, std::min(col, c0 + tn), g0});
            }
          }
          pans.push_back(pn);
        }
      };
      if (k > 0)
        for (int set = 0; set < 2; set++) {
          const int sidx = set * (L + 1) + k;
          merge(R_prev[set], Rb_prev[set], true, sidx, rpan[sidx], rgrp[sidx], rtil[sidx], R_cur[set]);
          if (!sym) merge(C_prev[set], Cb_prev[set], false, sidx, cpan[sidx], cgrp[sidx], ctil[sidx], C_cur[set]);
        }
      // ---- strips started at this level (from every pair of N_k) and S blocks of pairs
      const int nset = k == 0 ? 0 : 1;  // the panel set new strips of this level belong to
      struct NewStrip { int64_t item; int which; int64_t c; int32_t col0; };  // which: 0 yr, 1 yc
      std::vector<NewStrip> newr, newc;
      for (size_t j = 0; j < Nk.size(); j++) {
        int32_t t = kt(Nk[j]), s = ks(Nk[j]);
        int64_t ct = base + t, cs = base + s;
        bool canon = !sym || t <= s;
        int64_t item = canon ? pair_index[k][j] : pair_index[k][find(Nk, pkey(s, t))];
        const bool row_ok = mine(k, t) || (sym && mine(k, s));
        if (kr[ct] > 0 && mc(cs) > 0 && row_ok) {
          auto &lst = R_cur[nset][t];
          const int32_t col0 = lst.empty() ? 0 : lst.back().col0 + lst.back().m;
          lst.push_back(Grp{k, s, mc(cs), col0});
          // H_ts = H_st^T when t > s (symmetric): row strip of (t,s) = (nb part of H_st)^T
          newr.push_back(NewStrip{item, canon ? 0 : 1, t, col0});
        }
        if (!sym && mr(ct) > 0 && kc[cs] > 0 && mine(k, t)) {
          auto &lst = C_cur[nset][s];
          const int32_t col0 = lst.empty() ? 0 : lst.back().col0 + lst.back().m;
          lst.push_back(Grp{k, t, mr(ct), col0});
          newc.push_back(NewStrip{item, 1, s, col0});
        }
        if (canon && mr(ct) > 0 && mc(cs) > 0) {
          if (mine(k, t))
            blocks.push_back(BlockRec{loc_off[ct], P->s_off_col[cs], P->s_off_row[ct], mr(ct), mc(cs), 0, k, item});
          if (sym && t != s && mine(k, s))
            blocks.push_back(BlockRec{loc_off[cs], P->s_off_col[ct], P->s_off_row[cs], mc(cs), mr(ct), 1, k, item});
        }
      }
      // ---- panel bases of level k, and the destinations that point into them
      auto bases = [&](std::vector<std::vector<Grp>> &cur, const std::vector<int32_t> &kq, int64_t &ylen) {
        std::vector<int64_t> b(M, -1);
        for (int64_t c = 0; c < M; c++) {
          if (cur[c].empty()) continue;
          b[c] = ylen;
          ylen += int64_t(kq[base + c]) * (cur[c].back().col0 + cur[c].back().m);
        }
        return b;
      };
      std::vector<int64_t> Rb[2], Cb[2];
      for (int set = 0; set < 2; set++) {
        Rb[set] = bases(R_cur[set], kr, yr_len);
        Cb[set] = sym ? std::vector<int64_t>(M, -1) : bases(C_cur[set], kc, yc_len);
      }
      auto width = [](const std::vector<Grp> &g) { return g.empty() ? 0 : g.back().col0 + g.back().m; };
      for (const NewStrip &ns : newr) {
        PairItem &it = pairs[k][ns.item];
        if (ns.which == 0) {
          it.yr_dst = Rb[nset][ns.c] + ns.col0;
          it.yr_ld = width(R_cur[nset][ns.c]);
        } else {
          it.yc_dst = Rb[nset][ns.c] + ns.col0;
          it.yc_ld = width(R_cur[nset][ns.c]);
        }
      }
      for (const NewStrip &ns : newc) {
        PairItem &it = pairs[k][ns.item];
        it.yc_dst = Cb[nset][ns.c] + ns.col0;
        it.yc_ld = width(C_cur[nset][ns.c]);
      }
      for (int set = 0; set < 2; set++) {
        const int sidx = set * (L + 1) + k;
        for (auto &pn : rpan[sidx])
          if (kr[pn.q] > 0) {
            pn.y_dst = Rb[set][pn.q - base];
            pn.y_ld = width(R_cur[set][pn.q - base]);
          }
        for (auto &pn : cpan[sidx])
          if (kc[pn.q] > 0) {
            pn.y_dst = Cb[set][pn.q - base];
            pn.y_ld = width(C_cur[set][pn.q - base]);
          }
        R_prev[set].swap(R_cur[set]);
        C_prev[set].swap(C_cur[set]);
        Rb_prev[set].swap(Rb[set]);
        Cb_prev[set].swap(Cb[set]);
      }
    }

    // ---------------------------------------------------------------- Q needed by this shard
    // Q_t (and the R^ chain below it) is needed for every cluster a kept item
    // rotates with, and for the owned clusters (apply); closure over descendants.
    std::vector<int8_t> need_r(ncl, world == 1 ? 1 : 0), need_c(ncl, world == 1 ? 1 : 0);
    if (world > 1) {
      for (int k = 0; k <= L; k++) {
        for (const auto &it : pairs[k]) {
          need_r[it.t] = 1;
          need_c[it.s] = 1;
        }
        for (int set = 0; set < 2; set++) {
          for (const auto &pn : rpan[set * (L + 1) + k]) need_r[pn.q] = 1;
          for (const auto &pn : cpan[set * (L + 1) + k]) need_c[pn.q] = 1;
        }
        for (const auto &ci : coup[k]) {
          need_r[ci.t] = 1;
          need_c[ci.s] = 1;
        }
        for (int64_t i = 0; i < (int64_t(1) << (L - k)); i++)
          if (mine(k, i)) need_r[lvl_off(L, k) + i] = need_c[lvl_off(L, k) + i] = 1;
      }
      for (int k = L; k >= 1; k--)
        for (int64_t i = 0; i < (int64_t(1) << (L - k)); i++) {
          const int64_t c = lvl_off(L, k) + i, c1 = lvl_off(L, k - 1) + 2 * i;
          if (need_r[c]) need_r[c1] = need_r[c1 + 1] = 1;
          if (need_c[c]) need_c[c1] = need_c[c1 + 1] = 1;
        }
      if (sym)
        for (int64_t c = 0; c < ncl; c++) need_r[c] = need_c[c] = (need_r[c] | need_c[c]);
      // QR flops of this shard
      flops_qr = 0;
      for (int64_t c = 0; c < ncl; c++) {
        if (need_r[c]) flops_qr += 2.0 * nr[c] * kr[c] * kr[c] + 4.0 * nr[c] * nr[c] * kr[c];
        if (!sym && need_c[c]) flops_qr += 2.0 * nc[c] * kc[c] * kc[c] + 4.0 * nc[c] * nc[c] * kc[c];
      }
    }
    P->need_r = need_r;
    P->need_c = need_c;

    // ---------------------------------------------------------------- S pattern, CSR
    std::sort(blocks.begin(), blocks.end(), [](const BlockRec &a, const BlockRec &b) {
      return a.roff != b.roff ? a.roff < b.roff : a.coff < b.coff;
    });
    for (size_t j = 1; j < blocks.size(); j++)
      if (blocks[j].roff == blocks[j - 1].roff && blocks[j].coff == blocks[j - 1].coff)
        throw PlanError(H2SP_ETREE, "internal: S block produced twice");
    std::vector<CsrBlockRow> csr_rows;
    std::vector<CsrBlock> csr_blocks;
    const int64_t NR_loc = P->n_rows_local;
    std::vector<int64_t> rowptr(NR_loc + 1, 0);
    std::vector<int32_t> row_nblk(bench ? NR_loc : 0, 0);  // bench: blocks per local row (partial slot stride)
    int64_t nnz = 0, n_part = 0;
    {
      size_t j = 0;
      int64_t row = 0;  // next S row without a pointer
      while (j < blocks.size()) {
        size_t e = j;
        int64_t rowlen = 0;
        while (e < blocks.size() && blocks[e].roff == blocks[j].roff) rowlen += blocks[e++].mc;
        if (rowlen > INT32_MAX) throw PlanError(H2SP_EUNSUPPORTED, "S row longer than 2^31");
        const int64_t r0 = blocks[j].roff, m_r = blocks[j].mr;
        for (; row < r0; row++) rowptr[row] = nnz;  // empty rows
        const int32_t nblk = int32_t(e - j);
        CsrBlockRow br{r0, nnz, 0, int32_t(m_r), int32_t(rowlen), int32_t(csr_blocks.size()), nblk,
                       blocks[j].grow, n_part};
        csr_rows.push_back(br);
        int64_t colpos = 0;
        // S block -> its destination: the S values (stored mode, row length ld) or
        // the block's partial slot in every row (bench mode, stride nblk)
        const int32_t ld = bench ? nblk : int32_t(rowlen);
        for (size_t x = j; x < e; x++) {
          const BlockRec &b = blocks[x];
          if (b.mr != m_r) throw PlanError(H2SP_ETREE, "internal: inconsistent block row height");
          if (b.grow != blocks[j].grow) throw PlanError(H2SP_ETREE, "internal: inconsistent block row start");
          csr_blocks.push_back(CsrBlock{int32_t(b.coff), b.mc, int32_t(colpos), 0});
          const int64_t dst = bench ? n_part + int64_t(x - j) : nnz + colpos;
          switch (b.kind) {
            case 0: pairs[b.level][b.idx].s_dst = dst; pairs[b.level][b.idx].s_ld = ld; break;
            case 1: pairs[b.level][b.idx].s_dst_m = dst; pairs[b.level][b.idx].s_ld_m = ld; break;
            case 2:
              if (rgrp_direct[b.level].empty()) rgrp_direct[b.level].assign(rgrp[b.level].size(), -1);
              rgrp_direct[b.level][b.idx] = dst;
              break;
            case 3: rgrp[b.level][b.idx].s_dst_t = dst; rgrp[b.level][b.idx].s_ld_t = ld; break;
            case 4: cgrp[b.level][b.idx].s_dst_t = dst; cgrp[b.level][b.idx].s_ld_t = ld; break;
          }
          colpos += b.mc;
        }
        for (int64_t a = 0; a < m_r; a++) rowptr[r0 + a] = nnz + a * rowlen;
        if (bench)
          for (int64_t a = 0; a < m_r; a++) row_nblk[r0 + a] = nblk;
        n_part += m_r * nblk;
        row = r0 + m_r;
        nnz += m_r * rowlen;
        j = e;
      }
      for (; row <= NR_loc; row++) rowptr[row] = nnz;
    }
    P->s_nnz = nnz;
    P->n_part = bench ? n_part : 0;
    P->s_blocks = int64_t(blocks.size());
    // direct strip output of a panel: its groups are consecutive blocks of S row
    // block (q@k) (set 0 at the row start, set 1 right after), so contiguous in S
    for (int sidx = 0; sidx < 2 * (L + 1); sidx++)
      for (auto &pn : rpan[sidx]) {
        const int32_t mq = nr[pn.q] - kr[pn.q];
        if (mq == 0 || pn.gend == pn.gbeg || loc_off[pn.q] < 0) continue;
        const int64_t d0 = rgrp_direct[sidx][pn.gbeg];
        const int64_t r0 = loc_off[pn.q];
        if (!bench && sidx <= L && d0 != rowptr[r0])
          throw PlanError(H2SP_ETREE, "internal: strip panel not at the start of its S row");
        for (int32_t g = pn.gbeg; g < pn.gend; g++)
          if (rgrp_direct[sidx][g] != d0 + (bench ? int64_t(g - pn.gbeg) : int64_t(rgrp[sidx][g].col0)))
            throw PlanError(H2SP_ETREE, "internal: strip panel not contiguous in S");
        pn.s_dst = d0;
        pn.s_ld = bench ? row_nblk[r0] : int32_t(rowptr[r0 + 1] - rowptr[r0]);
      }

    // ---------------------------------------------------------------- meta image
    MetaBuilder mb;
    mb.buf.resize(256, 0);
    P->magic = 0x4832535050000000ull ^ (uint64_t(P->N) << 8) ^ uint64_t(nnz & 0xffffff) ^ (uint64_t(blocks.size()) << 40) ^
               (uint64_t(rank) << 32) ^ (uint64_t(world) << 36) ^ (uint64_t(P->bench) << 60);
    std::memcpy(mb.buf.data(), &P->magic, 8);
    P->ca.n_row = mb.put(nr);
    P->ca.k_row = mb.put(kr);
    P->ca.n_col = mb.put(sym ? nr : nc);
    P->ca.k_col = mb.put(sym ? kr : kc);
    P->ca.q_off_row = mb.put(P->q_off_row);
    P->ca.q_off_col = mb.put(sym ? P->q_off_row : P->q_off_col);
    P->ca.rh_off_row = mb.put(rh_off_row);
    P->ca.rh_off_col = mb.put(sym ? rh_off_row : rh_off_col);
    P->ca.leaf_off_row = mb.put(leaf_off_row);
    P->ca.leaf_off_col = mb.put(sym ? leaf_off_row : leaf_off_col);
    P->ca.tr_off_row = mb.put(tr_off_row);
    P->ca.tr_off_col = mb.put(sym ? tr_off_row : tr_off_col);
    P->ca.s_off_row = mb.put(P->s_off_row);
    P->ca.s_off_col = mb.put(P->s_off_col);
    P->ca.zb_off_row = mb.put(zb_row);
    P->ca.zb_off_col = mb.put(zb_col);
    P->ca.loc_off_row = mb.put(loc_off);
    P->ca.loc_off_col = mb.put(sym ? loc_off : loc_off_c);
    P->ca.need_row = mb.put(need_r);
    P->ca.need_col = mb.put(sym ? need_r : need_c);
    P->ca.need_all = mb.put(std::vector<int8_t>(size_t(ncl), int8_t(1)));
    P->levels.resize(L + 1);
    int levels_active = 0;
    int64_t launches = 0;
    // items per CTA chunk sharing one rotating cluster: up to 8 (reuse of the
    // resident Q), fewer when a level has too few items to fill ~4 CTAs/SM
    auto chunk = [&](const auto &items, auto qof) {
      static const int CHMAX =
          std::max(1, std::min(PAIR_CHUNK_MAX, getenv("H2SP_CHUNK") ? atoi(getenv("H2SP_CHUNK")) : 6));
      const int CH = int(std::max<int64_t>(1, std::min<int64_t>(CHMAX, int64_t(items.size()) / (148 * 4))));
      std::vector<Chunk> ch;
      size_t j = 0;
      while (j < items.size()) {
        size_t e = j + 1;
        while (e < items.size() && qof(items[e]) == qof(items[j]) && int(e - j) < CH) e++;
        ch.push_back(Chunk{int32_t(j), int32_t(e)});
        j = e;
      }
      return ch;
    };
    auto flat_tiles = [&](const std::vector<StripTile> &tils, const std::vector<StripPanel> &pans, bool row_side) {
      const auto &n = row_side ? nr : nc;
      const auto &kk = row_side ? kr : kc;
      const auto &qoff = (row_side || sym) ? P->q_off_row : P->q_off_col;
      std::vector<StripTileX> out(tils.size());
      for (size_t i = 0; i < tils.size(); i++) {
        const StripTile &t = tils[i];
        const StripPanel &pn = pans[t.panel];
        const int64_t q = pn.q;
        const int k = level_of(L, q);
        const int64_t c1 = lvl_off(L, k - 1) + 2 * (q - lvl_off(L, k));
        StripTileX &x = out[i];
        x = StripTileX{};
        x.q = pn.q;
        x.c0 = t.c0;
        x.ncol = t.c1 - t.c0;
        x.g0 = t.g0;
        x.gend = pn.gend;
        x.n = int16_t(n[q]);
        x.kq = int16_t(kk[q]);
        x.k1 = int16_t(kk[c1]);
        x.k2 = int16_t(kk[c1 + 1]);
        x.ld_c1 = pn.ld_c1;
        x.ld_c2 = pn.ld_c2;
        x.y_ld = pn.y_ld;
        x.s_ld = pn.s_ld;
        x.q_off = qoff[q];
        x.src_c1 = pn.src_c1;
        x.src_c2 = pn.src_c2;
        x.y_dst = pn.y_dst;
        x.s_dst = pn.s_dst;
        // bench mode: tiles start on a group boundary; slot of the tile's first group
        if (bench && pn.s_dst >= 0) x.s_dst = pn.s_dst + (t.g0 - pn.gbeg);
        x.wq0 = int32_t(P->s_off_col[q]);
      }
      return out;
    };
    for (int k = 0; k <= L; k++) {
      LevelPlan &lp = P->levels[k];
      lp = LevelPlan{};
      lp.k = k;
      const int64_t base = lvl_off(L, k), M = int64_t(1) << (L - k);
      int npr = 0, npc = 0;
      for (int64_t i = 0; i < M; i++) {
        npr = std::max(npr, int(nr[base + i]));
        npc = std::max(npc, int(nc[base + i]));
      }
      lp.np_row = npr;
      lp.np_col = npc;
      if (npr > 0 || npc > 0) levels_active++;
      lp.mp = strip_tn_of_level(k);
      lp.np_pair = round8(std::max(npr, npc));
      if (k == 0) {
        // compact-WY congruence at level 0 (kernels.cu pair_wy_kernel): n <= 64
        // tiles padded to 64, every k <= 24; pays off for k <= n / 2
        int kmx = 0;
        for (int64_t i = 0; i < M; i++) kmx = std::max(kmx, int(std::max(kr[base + i], kc[base + i])));
        P->wy_kp = 0;
        P->wy_n = 64;
        if (lp.np_pair > 64) {  // 128-point leaves: only the compact-WY kernel exists (k <= 32)
          if ((flags & H2SP_PLAN_EXPLICIT_Q) || kmx > 32)
            throw PlanError(H2SP_EUNSUPPORTED, "leaves with n_t > 64 need the compact-WY congruence (k_t <= 32, "
                                               "no H2SP_PLAN_EXPLICIT_Q)");
          P->wy_n = 128;
          P->wy_kp = kmx <= 16 ? 16 : 32;
        } else if (!(flags & H2SP_PLAN_EXPLICIT_Q) && lp.np_pair > 48 && kmx >= 1 && kmx <= 24) {
          P->wy_kp = kmx <= 16 ? 16 : 24;
        }
      }
      lp.np_rstrip = round8(npr);
      lp.np_cstrip = round8(npc);
      lp.n_pairs = int64_t(pairs[k].size());
      lp.pairs_off = mb.put(pairs[k]);
      auto pc = chunk(pairs[k], [](const PairItem &x) { return x.t; });
      lp.n_pair_chunks = int64_t(pc.size());
      // split the level-0 congruence and the level-0-born row strips at the middle
      // of the tree: the strips of the first half only need the first half's pairs
      // (canonical pairs have their row <= both clusters), so their level chain
      // starts while the second half of the level-0 congruence still runs
      static const bool split = !getenv("H2SP_SPLIT") || atoi(getenv("H2SP_SPLIT")) != 0;
      // first part = leaves [0, lsplit) (H2SP_SPLIT_FRAC of them, default 1/2); at level
      // k the clusters entirely inside it are p < lsplit >> k
      static const double frac = getenv("H2SP_SPLIT_FRAC") ? atof(getenv("H2SP_SPLIT_FRAC")) : 0.5;
      const int64_t lsplit = int64_t(double(int64_t(1) << L) * frac);
      const int64_t bound = lsplit >> k;
      const bool do_split = split && world == 1 && M >= 2 && lsplit > 0 && lsplit < (int64_t(1) << L);
      lp.pair_split = 0;
      if (k == 0 && do_split) {
        while (lp.pair_split < int64_t(pc.size()) && pairs[0][pc[lp.pair_split].begin].t < bound) lp.pair_split++;
        if (lp.pair_split == int64_t(pc.size())) lp.pair_split = 0;
      }
      lp.pair_chunks_off = mb.put(pc);
      for (int set = 0; set < 2; set++) {
        const int sidx = set * (L + 1) + k;
        lp.sp[set].n_rtiles = int64_t(rtil[sidx].size());
        lp.sp[set].n_rtiles_a = 0;
        static const int split_max = getenv("H2SP_SPLIT_MAXLEVEL") ? atoi(getenv("H2SP_SPLIT_MAXLEVEL")) : 1 << 20;
        if (set == 0 && do_split && P->levels[0].pair_split > 0 && k <= split_max) {
          auto &na = lp.sp[set].n_rtiles_a;
          while (na < int64_t(rtil[sidx].size()) && rpan[sidx][rtil[sidx][na].panel].q - base < bound) na++;
          if (na == int64_t(rtil[sidx].size())) na = 0;  // nothing left for the second half: no split
        }
        lp.sp[set].rtiles_off = mb.put(flat_tiles(rtil[sidx], rpan[sidx], true));
        lp.sp[set].rpanels_off = mb.put(rpan[sidx]);
        lp.sp[set].rgroups_off = mb.put(rgrp[sidx]);
        lp.sp[set].n_ctiles = int64_t(ctil[sidx].size());
        lp.sp[set].ctiles_off = mb.put(flat_tiles(ctil[sidx], cpan[sidx], false));
        lp.sp[set].cpanels_off = mb.put(cpan[sidx]);
        lp.sp[set].cgroups_off = mb.put(cgrp[sidx]);
      }
      lp.n_coup = int64_t(coup[k].size());
      lp.coup_off = mb.put(coup[k]);
      // launches issued by launch_build (kept in sync with kernels.cu), with
      // their algorithmic flops / HBM bytes
      double qbytes_row = 0, qbytes_col = 0;
      for (int64_t i = 0; i < M; i++) {
        qbytes_row += 8.0 * nr[base + i] * nr[base + i];
        qbytes_col += 8.0 * nc[base + i] * nc[base + i];
      }
      auto qr_info = [&](const std::vector<int32_t> &n, const std::vector<int32_t> &kk, int kind) {
        h2sp_launch_info li{kind, k, 0, 0.0, 0.0, 0.0};
        const auto &need = (kind == 0) ? need_r : need_c;
        for (int64_t i = 0; i < M; i++) {
          const int64_t c = base + i;
          const double nn = n[c], k_ = kk[c];
          if (nn == 0 || !need[c]) continue;
          li.items++;
          li.flops += 2 * nn * k_ * k_ + 4 * nn * nn * k_;
          double in_ = (k == 0) ? double(B) * k_ : nn * k_;
          if (k > 0) {
            const int64_t c1 = lvl_off(L, k - 1) + 2 * i;
            in_ += double(kk[c1]) * kk[c1] + double(kk[c1 + 1]) * kk[c1 + 1];
          }
          li.bytes += 8.0 * (in_ + nn * nn + k_ * k_);
        }
        return li;
      };
      if (npr > 0) {
        launches++;
        P->launch_info.push_back(qr_info(nr, kr, 0));
      }
      if (!sym && npc > 0) {
        launches++;
        P->launch_info.push_back(qr_info(nc, kc, 1));
      }
      if (lp.n_coup) {
        launches++;
        h2sp_launch_info li{2, k, lp.n_coup, 0.0, 0.0, 0.0};
        for (const auto &c : coup[k]) {
          const double a = kr[c.t], b = kc[c.s];
          li.flops += 2 * a * b * (a + b);
          li.bytes += 8.0 * (2 * a * b + a * a + b * b);
        }
        P->launch_info.push_back(li);
      }
      if (lp.n_pairs) {
        launches++;
        h2sp_launch_info li{3, k, lp.n_pairs, 0.0, qbytes_row + (sym ? 0.0 : qbytes_col), 0.0};
        for (const auto &it : pairs[k]) {
          const double a = nr[it.t], b = nc[it.s];
          li.flops += 2 * a * b * (a + b);
          li.flops_exec += (k == 0 && P->wy_kp) ? 4 * a * b * (kr[it.t] + kc[it.s]) : 2 * a * b * (a + b);
          double outb = a * b;  // nn + bb + bn + nb
          if (it.s_dst_m >= 0) outb += double(nr[it.t] - kr[it.t]) * (nc[it.s] - kc[it.s]);
          li.bytes += 8.0 * (a * b + outb);
        }
        P->launch_info.push_back(li);
      }
      auto strip_info = [&](const std::vector<StripPanel> &pans, const std::vector<StripGroup> &grps,
                            const std::vector<StripTile> &tils, const std::vector<int32_t> &n,
                            const std::vector<int32_t> &kk, int kind, double qb, int half) {
        h2sp_launch_info li{kind, k, int64_t(tils.size()), 0.0, qb, 0.0};
        for (const auto &pn : pans) {
          if (half >= 0 && (pn.q - base < bound) != (half == 0)) continue;
          const int64_t c1 = lvl_off(L, k - 1) + 2 * (pn.q - base);
          const double nq = n[pn.q], kq = kk[pn.q];
          for (int32_t g = pn.gbeg; g < pn.gend; g++) {
            const StripGroup &sg = grps[g];
            const double rows = (sg.pos_c1 >= 0 ? kk[c1] : 0) + (sg.pos_c2 >= 0 ? kk[c1 + 1] : 0);
            const double m = sg.m;
            li.flops += 2 * nq * rows * m;
            li.flops_exec += 2 * nq * (strip_skip ? rows : nq) * m;  // the kernel's k range
            const double outb = (pn.y_dst >= 0 ? kq * m : 0.0) + (pn.s_dst >= 0 ? (nq - kq) * m : 0.0) +
                                (sg.s_dst_t >= 0 ? (nq - kq) * m : 0.0);
            li.bytes += 8.0 * (rows * m + outb);
          }
        }
        return li;
      };
      for (int set = 0; set < 2; set++) {
        const int sidx = set * (L + 1) + k;
        const int64_t na = lp.sp[set].n_rtiles_a;
        if (na > 0) {  // two launches: first half (A), second half (B)
          launches += 2;
          h2sp_launch_info a = strip_info(rpan[sidx], rgrp[sidx], rtil[sidx], nr, kr, 4, qbytes_row / 2, 0);
          h2sp_launch_info b = strip_info(rpan[sidx], rgrp[sidx], rtil[sidx], nr, kr, 4, qbytes_row / 2, 1);
          a.items = na;
          b.items = lp.sp[set].n_rtiles - na;
          P->launch_info.push_back(a);
          P->launch_info.push_back(b);
        } else if (lp.sp[set].n_rtiles) {
          launches++;
          P->launch_info.push_back(strip_info(rpan[sidx], rgrp[sidx], rtil[sidx], nr, kr, 4, qbytes_row, -1));
        }
        if (lp.sp[set].n_ctiles) {
          launches++;
          P->launch_info.push_back(strip_info(cpan[sidx], cgrp[sidx], ctil[sidx], nc, kc, 5, qbytes_col, -1));
        }
      }
    }
    P->n_csr_rows = int64_t(csr_rows.size());
    P->n_csr_blocks = int64_t(csr_blocks.size());
    // per block row column pattern (value-independent), 16-byte aligned rows
    // (bench mode: no column indices, no pattern)
    std::vector<int32_t> csr_pat;
    for (auto &br : csr_rows) {
      br.pat_off = int64_t(csr_pat.size());
      if (bench) continue;
      for (int32_t j = 0; j < br.nblk; j++) {
        const CsrBlock &b = csr_blocks[br.blk_begin + j];
        for (int32_t e = 0; e < b.m_c; e++) csr_pat.push_back(b.col0 + e);
      }
      while (csr_pat.size() % 4) csr_pat.push_back(0);
    }
    P->csr_pat_off = mb.put(csr_pat);
    P->csr_rows_off = mb.put(csr_rows);
    P->csr_blocks_off = mb.put(csr_blocks);
    P->rowptr_off = mb.put(rowptr);
    if (P->n_csr_rows && !bench) {  // CSR column expansion (+ the rowptr D2D copy)
      launches++;
      P->launch_info.push_back(h2sp_launch_info{6, L, P->n_csr_rows, 0.0, 4.0 * double(nnz) + 16.0 * double(NR_loc + 1), 0.0});
    }
    if (P->n_csr_rows && bench) {  // bench mode: row sums of the partial slots -> S w, row norms
      launches++;
      P->launch_info.push_back(
          h2sp_launch_info{8, L, P->n_csr_rows, 0.0, 16.0 * double(n_part) + 16.0 * double(NR_loc), 0.0});
    }
    if (P->wy_kp) {  // level-0 Q formed from V / M (kernels.cu wy_form_q_kernel), after the CSR entry
      launches++;
      h2sp_launch_info li{7, 0, 0, 0.0, 0.0, 0.0};
      for (int side = 0; side < (sym ? 1 : 2); side++) {
        const auto &n = side ? nc : nr;
        const auto &kk = side ? kc : kr;
        const auto &need = side ? need_c : need_r;
        for (int64_t c = 0; c < nleaf; c++) {
          if (n[c] == 0 || !need[c]) continue;
          li.items++;
          li.flops += 2.0 * n[c] * n[c] * kk[c];
          li.bytes += 8.0 * (n[c] * n[c] + 2.0 * P->wy_n * P->wy_kp);
        }
      }
      P->launch_info.push_back(li);
      // the QR launches of level 0 no longer form Q: move those flops (keeps the total)
      for (auto &x : P->launch_info)
        if (x.level == 0 && (x.kind == 0 || x.kind == 1)) {
          const auto &n = x.kind ? nc : nr;
          const auto &kk = x.kind ? kc : kr;
          const auto &need = x.kind ? need_c : need_r;
          for (int64_t c = 0; c < nleaf; c++)
            if (n[c] && need[c]) x.flops -= 2.0 * n[c] * n[c] * kk[c];
        }
    }
    P->launches = launches;
    P->levels_active = levels_active;
    P->flops_exec = 0;
    for (auto &x : P->launch_info) {
      if (x.kind != 3 && x.kind != 4 && x.kind != 5) x.flops_exec = x.flops;
      P->flops_exec += x.flops_exec;
    }
    P->meta_bytes = align_up(mb.buf.size(), 256);
    mb.buf.resize(P->meta_bytes, 0);
    P->meta.swap(mb.buf);
    // workspace layout
    size_t o = P->meta_bytes;
    auto carve = [&](int64_t n_doubles) {
      size_t r = o;
      o = align_up(o + size_t(n_doubles) * 8, 256);
      return r;
    };
    P->dt_len = dt_len;
    P->bb_len = bb_len;
    P->yr_len = yr_len;
    P->yc_len = yc_len;
    // the QR results (R^ chain, level-0 compact-WY factors) first: their sizes
    // depend on the tree and ranks only, so they sit at the same scratch offsets
    // in every shard plan of one matrix (h2sp_plan_set_qr_mode: H2SP_QR_REUSE)
    P->ws_rh_row = carve(P->rh_row_len);
    P->ws_rh_col = carve(P->rh_col_len);
    P->ws_wy_row = P->ws_wy_col = 0;
    if (P->wy_kp) {
      const int64_t per = int64_t(2) * P->wy_n * P->wy_kp;
      P->ws_wy_row = carve(per * nleaf);
      P->ws_wy_col = sym ? P->ws_wy_row : carve(per * nleaf);
    }
    P->ws_qr_end = o;
    P->ws_dt = carve(dt_len);
    P->ws_bb = carve(bb_len);
    P->ws_yr = carve(yr_len);
    P->ws_yc = carve(yc_len);
    P->ws_part = bench ? carve(2 * n_part) : 0;
    P->ws_total = o;
    // algorithmic work
    double close_read = 0;
    for (uint64_t x : near[0])
      if (!sym || kt(x) <= ks(x)) close_read += double(B) * B;
    double coup_read = 0;
    for (int k = 0; k < L; k++)
      for (size_t j = 0; j < adm[k].size(); j++)
        if (!sym || kt(adm[k][j]) <= ks(adm[k][j]))
          coup_read += double(kr[lvl_off(L, k) + kt(adm[k][j])]) * kc[lvl_off(L, k) + ks(adm[k][j])];
    double in_bytes = 8.0 * (close_read + coup_read + P->leaf_row_len + P->leaf_col_len + P->tr_row_len + P->tr_col_len);
    // stored mode: S as CSR; bench mode: S w and the row norms (16 B per row) plus the partials
    double out_bytes = 8.0 * (P->q_row_len + P->q_col_len) +
                       (bench ? 16.0 * double(NR_loc) + 32.0 * double(n_part) : 12.0 * double(nnz) + 8.0 * double(NR_loc + 1));
    double mid_bytes = 2.0 * 8.0 * double(P->rh_row_len + P->rh_col_len + dt_len + bb_len + yr_len + yc_len);
    P->flops = flops_qr + flops_coup + flops_cong + flops_strip;
    P->flops_unique = world == 1 ? P->flops : uniq_qr + uniq_coup + uniq_cong + uniq_strip;
    P->flops_cong = flops_cong;
    P->flops_strip = flops_strip;
    P->bytes = in_bytes + out_bytes + mid_bytes;
    *out = P;
    return H2SP_OK;
  } catch (const PlanError &e) {
    delete P;
    return fail(e.code, e.what());
  } catch (const std::bad_alloc &) {
    delete P;
    return fail(H2SP_ENOMEM, "host allocation failed in plan_create");
  } catch (const std::exception &e) {
    delete P;
    return fail(H2SP_EINVAL, e.what());
  }
}

h2sp_status h2sp_plan_sizes(h2sp_plan P, h2sp_sizes *o) {
  if (!P || !o) return fail(H2SP_EINVAL, "NULL plan or output");
  std::memset(o, 0, sizeof(*o));
  o->n = P->N;
  o->n_clusters = P->ncl;
  o->leaf_row = P->leaf_row_len;
  o->transfer_row = P->tr_row_len;
  o->leaf_col = P->leaf_col_len;
  o->transfer_col = P->tr_col_len;
  o->close = P->close_len;
  o->coupling = P->coupling_len;
  o->q_row = P->q_row_len;
  o->q_col = P->q_col_len;
  o->s_nnz = P->s_nnz;
  o->s_rows = P->n_rows_local;
  o->rank = P->rank;
  o->world = P->world;
  o->first_leaf = P->first_leaf;
  o->n_leaves_local = P->n_leaves_local;
  o->s_blocks = P->s_blocks;
  o->workspace_bytes = int64_t(P->ws_total);
  o->meta_bytes = int64_t(P->meta_bytes);
  o->levels_active = P->levels_active;
  o->launches = P->launches;
  o->flops = P->flops;
  o->bytes = P->bytes;
  o->flops_congruence = P->flops_cong;
  o->flops_strips = P->flops_strip;
  o->flops_executed = P->flops_exec;
  o->flops_unique = P->flops_unique;
  o->bench_parts = P->n_part;
  return H2SP_OK;
}

h2sp_status h2sp_plan_offsets(h2sp_plan P, int64_t *s_off_row, int64_t *s_off_col, int64_t *q_off_row,
                              int64_t *q_off_col, int64_t *n_row, int64_t *n_col) {
  if (!P) return fail(H2SP_EINVAL, "NULL plan");
  for (int64_t c = 0; c < P->ncl; c++) {
    if (s_off_row) s_off_row[c] = P->s_off_row[c];
    if (s_off_col) s_off_col[c] = P->s_off_col[c];
    if (q_off_row) q_off_row[c] = P->q_off_row[c];
    if (q_off_col) q_off_col[c] = P->sym ? P->q_off_row[c] : P->q_off_col[c];
    if (n_row) n_row[c] = P->n_row[c];
    if (n_col) n_col[c] = P->n_col[c];
  }
  return H2SP_OK;
}

h2sp_status h2sp_plan_local_rows(h2sp_plan P, int64_t *loc_off_row, int64_t *loc_off_col) {
  if (!P) return fail(H2SP_EINVAL, "NULL plan");
  for (int64_t c = 0; c < P->ncl; c++) {
    if (loc_off_row) loc_off_row[c] = P->loc_off_row[c];
    if (loc_off_col) loc_off_col[c] = P->sym ? P->loc_off_row[c] : P->loc_off_col[c];
  }
  return H2SP_OK;
}

h2sp_status h2sp_plan_launches(h2sp_plan P, h2sp_launch_info *out, int64_t max, int64_t *count) {
  if (!P || !count) return fail(H2SP_EINVAL, "NULL plan or count");
  *count = int64_t(P->launch_info.size());
  if (out)
    for (int64_t i = 0; i < max && i < *count; i++) out[i] = P->launch_info[i];
  return H2SP_OK;
}

h2sp_status h2sp_plan_pattern(h2sp_plan P, int64_t *rowptr, int32_t *col) {
  if (!P || !rowptr) return fail(H2SP_EINVAL, "NULL plan or rowptr");
  std::memcpy(rowptr, P->meta.data() + P->rowptr_off, size_t(P->n_rows_local + 1) * sizeof(int64_t));
  if (col && P->bench) return fail(H2SP_EINVAL, "bench-mode plan: no column pattern");
  if (col) {
    const CsrBlockRow *rows = reinterpret_cast<const CsrBlockRow *>(P->meta.data() + P->csr_rows_off);
    const CsrBlock *blks = reinterpret_cast<const CsrBlock *>(P->meta.data() + P->csr_blocks_off);
    for (int64_t r = 0; r < P->n_csr_rows; r++)
      for (int32_t a = 0; a < rows[r].m_r; a++) {
        int32_t *dst = col + rows[r].p_base + int64_t(a) * rows[r].rowlen;
        for (int32_t j = 0; j < rows[r].nblk; j++) {
          const CsrBlock &b = blks[rows[r].blk_begin + j];
          for (int32_t e = 0; e < b.m_c; e++) dst[b.colpos + e] = b.col0 + e;
        }
      }
  }
  return H2SP_OK;
}

}  // extern "C"
