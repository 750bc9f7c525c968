// setup.cpp — host-side PSLR setup, native C++ (the reference does this in
// pure Python; the north star keeps it on the host).  Two routines, both
// bit-identical to the reference so the hot path sees exactly the same
// factors and the same reordered system:
//
//   pslr_partition_bisect  — partition.py:72-132 (recursive BFS level-set
//                            bisection, smallest-index roots, depth-first ids)
//   pslr_ilut_blocks       — ilu.py:35-138 + ilu.py:167-184 (per-block row-wise
//                            IKJ ILUT, drop |l| < droptol*||a_i||_2, pivot
//                            repair, optional fill cap), blocks factored in
//                            parallel on host threads (blocks are independent,
//                            so threading cannot change a single bit).
//
// Compiled without FMA contraction (-ffp-contract=off): numpy never fuses.
#include "pslr_internal.h"

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace pslr {

// numpy float64 add.reduce over a contiguous run (used by scipy's
// csr.sum(axis=1) via np.add.reduceat): acc = a[0]; acc += pairwise(a[1:]).
static double numpy_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double acc[8];
    for (int k = 0; k < 8; ++k) acc[k] = a[k];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) acc[k] += a[i + k];
    double r = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    for (; i < n; ++i) r += a[i];
    return r;
  }
  int64_t half = n / 2;
  half -= half % 8;
  return numpy_pairwise(a, half) + numpy_pairwise(a + half, n - half);
}

double numpy_sum(const double* a, int64_t n) {
  if (n <= 0) return 0.0;
  return a[0] + numpy_pairwise(a + 1, n - 1);
}

// ---------------------------------------------------------------- ILUT of one block
struct Kept {
  int64_t col;
  double val;
  int64_t order;  // discovery order: decides fill_cap ties (Python's sort is stable)
};

struct BlockFactor {
  int64_t n = 0;
  std::vector<int64_t> Lp, Up;
  std::vector<int32_t> Li, Ui;
  std::vector<double> Lx, Ux;
  int64_t repairs = 0;
};

// Factor the square block rows [lo, hi) of the CSR matrix (columns outside the
// block are ignored — the caller passes a block-diagonal matrix).
static void ilut_block(const int64_t* ip, const int32_t* ix, const double* ax, int64_t lo,
                       int64_t hi, double droptol, int64_t fill_cap, BlockFactor& out) {
  const int64_t n = hi - lo;
  out.n = n;
  out.Lp.assign(n + 1, 0);
  out.Up.assign(n + 1, 0);
  if (n == 0) return;
  std::vector<double> rnorm(n);
  std::vector<double> sq;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = ip[lo + i], b = ip[lo + i + 1];
    sq.resize(b - a);
    for (int64_t k = a; k < b; ++k) sq[k - a] = ax[k] * ax[k];
    rnorm[i] = std::sqrt(numpy_sum(sq.data(), b - a));
  }
  std::vector<double> work(n, 0.0), diag(n, 0.0);
  std::vector<char> hit(n, 0);
  std::vector<int64_t> seen;      // columns touched by row i, in discovery order
  std::vector<int64_t> pending;   // columns < i still to eliminate, kept sorted
  std::vector<Kept> lrow, urow;
  seen.reserve(64);
  // U rows as produced: diag first, then ascending upper columns (local indices)
  std::vector<int64_t> ucol;
  std::vector<double> uval;
  std::vector<int64_t> ustart(n + 1, 0);

  for (int64_t i = 0; i < n; ++i) {
    seen.clear();
    pending.clear();
    lrow.clear();
    urow.clear();
    for (int64_t k = ip[lo + i]; k < ip[lo + i + 1]; ++k) {
      const int64_t c = (int64_t)ix[k] - lo;
      if (c < 0 || c >= n) continue;  // not in the block (cannot happen for block-diagonal input)
      work[c] = ax[k];
      hit[c] = 1;
      seen.push_back(c);
      if (c < i) pending.push_back(c);  // CSR columns are sorted: pending stays sorted
    }
    const double tau = droptol * rnorm[i];
    size_t head = 0;
    while (head < pending.size()) {
      const int64_t k = pending[head++];
      const double mult = work[k] / diag[k];
      work[k] = 0.0;
      if (std::fabs(mult) < tau) continue;
      lrow.push_back({k, mult, (int64_t)lrow.size()});
      const int64_t ua = ustart[k], ub = ustart[k + 1];
      for (int64_t t = ua; t < ub; ++t) {
        const int64_t c = ucol[t];
        if (!hit[c]) {
          hit[c] = 1;
          seen.push_back(c);
          if (c < i) {
            // new fill below the diagonal: c > k, insert in order after head
            auto pos = std::upper_bound(pending.begin() + head, pending.end(), c);
            pending.insert(pos, c);
          }
        }
      }
      for (int64_t t = ua; t < ub; ++t) {
        const double prod = mult * uval[t];
        work[ucol[t]] = work[ucol[t]] - prod;
      }
    }
    double piv = work[i];
    if (piv == 0.0) {
      const double base = rnorm[i] > 0 ? rnorm[i] : 1.0;
      piv = droptol * base;
      if (piv == 0.0) piv = DBL_EPSILON * base;
      out.repairs++;
    }
    for (int64_t c : seen) {
      const double v = work[c];
      if (c > i && std::fabs(v) >= tau && v != 0.0) urow.push_back({c, v, (int64_t)urow.size()});
    }
    auto by_mag = [](const Kept& a, const Kept& b) {
      const double x = std::fabs(a.val), y = std::fabs(b.val);
      if (x != y) return x > y;
      return a.order < b.order;
    };
    auto by_col = [](const Kept& a, const Kept& b) { return a.col < b.col; };
    if (fill_cap >= 0) {
      if ((int64_t)lrow.size() > fill_cap) {
        std::sort(lrow.begin(), lrow.end(), by_mag);
        lrow.resize(fill_cap);
      }
      if ((int64_t)urow.size() > fill_cap) {
        std::sort(urow.begin(), urow.end(), by_mag);
        urow.resize(fill_cap);
      }
    }
    std::sort(lrow.begin(), lrow.end(), by_col);
    std::sort(urow.begin(), urow.end(), by_col);
    for (const Kept& e : lrow) {
      out.Li.push_back((int32_t)(e.col + lo));
      out.Lx.push_back(e.val);
    }
    out.Li.push_back((int32_t)(i + lo));  // unit diagonal stored last (ilu.py:128-131)
    out.Lx.push_back(1.0);
    out.Lp[i + 1] = (int64_t)out.Li.size();
    ustart[i] = (int64_t)ucol.size();
    ucol.push_back(i);
    uval.push_back(piv);
    for (const Kept& e : urow) {
      ucol.push_back(e.col);
      uval.push_back(e.val);
    }
    ustart[i + 1] = (int64_t)ucol.size();
    diag[i] = piv;
    for (int64_t c : seen) {
      work[c] = 0.0;
      hit[c] = 0;
    }
  }
  out.Ui.resize(ucol.size());
  for (size_t t = 0; t < ucol.size(); ++t) out.Ui[t] = (int32_t)(ucol[t] + lo);
  out.Ux.swap(uval);
  for (int64_t i = 0; i <= n; ++i) out.Up[i] = ustart[i];
}

}  // namespace pslr

struct pslr_factors {
  int64_t n = 0, nblocks = 0;
  std::vector<pslr::BlockFactor> blocks;
};

extern "C" {

int pslr_ilut_blocks(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data,
                     int64_t nblocks, const int64_t* offsets, double droptol, int64_t fill_cap,
                     int nthreads, pslr_factors** out, int64_t* nnz_L, int64_t* nnz_U,
                     int64_t* pivot_repairs) {
  if (droptol < 0) return pslr::fail(PSLR_EDIM, "droptol must be >= 0");
  if (nblocks < 0 || (nblocks > 0 && (offsets[0] != 0 || offsets[nblocks] != n)))
    return pslr::fail(PSLR_EDIM, "block sizes do not tile the matrix");
  for (int64_t b = 0; b < nblocks; ++b)
    if (offsets[b + 1] < offsets[b]) return pslr::fail(PSLR_EDIM, "negative block size");
  auto* f = new pslr_factors();
  f->n = n;
  f->nblocks = nblocks;
  f->blocks.resize(nblocks);
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  nthreads = (int)std::min<int64_t>(nthreads, std::max<int64_t>(nblocks, 1));
  // largest blocks first so the tail of the schedule is short
  std::vector<int64_t> order(nblocks);
  for (int64_t b = 0; b < nblocks; ++b) order[b] = b;
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return offsets[a + 1] - offsets[a] > offsets[b + 1] - offsets[b];
  });
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      const int64_t t = next.fetch_add(1);
      if (t >= nblocks) break;
      const int64_t b = order[t];
      pslr::ilut_block(indptr, indices, data, offsets[b], offsets[b + 1], droptol, fill_cap,
                       f->blocks[b]);
    }
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < nthreads; ++k) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  int64_t nl = 0, nu = 0, rep = 0;
  for (auto& bf : f->blocks) {
    nl += (int64_t)bf.Li.size();
    nu += (int64_t)bf.Ui.size();
    rep += bf.repairs;
  }
  *out = f;
  *nnz_L = nl;
  *nnz_U = nu;
  *pivot_repairs = rep;
  return PSLR_OK;
}

int pslr_factors_fetch(const pslr_factors* f, int64_t* Lp, int32_t* Li, double* Lx, int64_t* Up,
                       int32_t* Ui, double* Ux, int64_t* block_nnz, int64_t* block_repairs) {
  int64_t row = 0, lpos = 0, upos = 0;
  Lp[0] = 0;
  Up[0] = 0;
  for (int64_t b = 0; b < f->nblocks; ++b) {
    const auto& bf = f->blocks[b];
    for (int64_t i = 0; i < bf.n; ++i) {
      Lp[row + i + 1] = lpos + bf.Lp[i + 1];
      Up[row + i + 1] = upos + bf.Up[i + 1];
    }
    std::memcpy(Li + lpos, bf.Li.data(), bf.Li.size() * sizeof(int32_t));
    std::memcpy(Lx + lpos, bf.Lx.data(), bf.Lx.size() * sizeof(double));
    std::memcpy(Ui + upos, bf.Ui.data(), bf.Ui.size() * sizeof(int32_t));
    std::memcpy(Ux + upos, bf.Ux.data(), bf.Ux.size() * sizeof(double));
    if (block_nnz) {
      block_nnz[2 * b] = (int64_t)bf.Li.size();
      block_nnz[2 * b + 1] = (int64_t)bf.Ui.size();
    }
    if (block_repairs) block_repairs[b] = bf.repairs;
    row += bf.n;
    lpos += (int64_t)bf.Li.size();
    upos += (int64_t)bf.Ui.size();
  }
  return PSLR_OK;
}

void pslr_factors_free(pslr_factors* f) { delete f; }

int pslr_row_norms(int64_t n, const int64_t* indptr, const double* data, double* out) {
  std::vector<double> sq;
  for (int64_t i = 0; i < n; ++i) {
    sq.resize(indptr[i + 1] - indptr[i]);
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) sq[k - indptr[i]] = data[k] * data[k];
    out[i] = std::sqrt(pslr::numpy_sum(sq.data(), (int64_t)sq.size()));
  }
  return PSLR_OK;
}

// ---------------------------------------------------------------- BFS bisection
int pslr_partition_bisect(int64_t n, const int64_t* adj_indptr, const int64_t* adj_indices,
                          int64_t parts, int64_t* assignment) {
  if (parts < 1) return pslr::fail(PSLR_EDIM, "number of subdomains must be >= 1");
  if (parts > n) return pslr::fail(PSLR_EDIM, "cannot split the vertices into that many subdomains");
  std::vector<uint32_t> stamp(n, 0);   // membership epoch of the current subset
  std::vector<uint32_t> visit(n, 0);   // visited epoch
  uint32_t epoch = 0;
  std::vector<int64_t> verts(n), bfs(n);
  for (int64_t i = 0; i < n; ++i) verts[i] = i;
  struct Task { int64_t lo, cnt, parts; };
  // explicit depth-first stack: left subtree ids precede right subtree ids
  std::vector<Task> stack{{0, n, parts}};
  int64_t next_id = 0;
  while (!stack.empty()) {
    Task t = stack.back();
    stack.pop_back();
    int64_t* V = verts.data() + t.lo;
    if (t.parts == 1) {
      for (int64_t k = 0; k < t.cnt; ++k) assignment[V[k]] = next_id;
      ++next_id;
      continue;
    }
    ++epoch;
    for (int64_t k = 0; k < t.cnt; ++k) stamp[V[k]] = epoch;
    int64_t tail = 0;
    for (int64_t r = 0; r < t.cnt; ++r) {  // roots: smallest unvisited index first
      const int64_t root = V[r];
      if (visit[root] == epoch) continue;
      visit[root] = epoch;
      int64_t head = tail;
      bfs[tail++] = root;
      while (head < tail) {
        const int64_t v = bfs[head++];
        for (int64_t e = adj_indptr[v]; e < adj_indptr[v + 1]; ++e) {
          const int64_t u = adj_indices[e];
          if (stamp[u] == epoch && visit[u] != epoch) {
            visit[u] = epoch;
            bfs[tail++] = u;
          }
        }
      }
    }
    const int64_t lp = (t.parts + 1) / 2, rp = t.parts - lp;
    // Python round(len*lp/parts): correctly rounded quotient, ties to even
    int64_t cut = (int64_t)std::nearbyint((double)(t.cnt * lp) / (double)t.parts);
    cut = std::min(std::max(cut, lp), t.cnt - rp);
    std::memcpy(V, bfs.data(), t.cnt * sizeof(int64_t));
    std::sort(V, V + cut);
    std::sort(V + cut, V + t.cnt);
    stack.push_back({t.lo + cut, t.cnt - cut, rp});  // right after left
    stack.push_back({t.lo, cut, lp});
  }
  return PSLR_OK;
}

}  // extern "C"
