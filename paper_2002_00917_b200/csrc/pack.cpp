// pack.cpp — host packer: level-schedules every block of a block-diagonal
// triangular factor and emits the streamed device format the sm_100a solve
// kernel consumes (see kernels.cu: tri_phase).
//
// Per block the rows are ordered by (dependency level, entry count desc, row),
// which defines the row's "position".  Positions are global (block b owns
// [off_b, off_{b+1}) in both row and position space).  Each level is cut into
// segments (jagged-diagonal layout: slab k holds the k-th entry of every row
// that has one, so within a row the reference's ascending-column summation
// order is kept), segments are grouped into chunks of <= stage_bytes that the
// kernel streams into shared memory with TMA bulk copies.
//
// A dependency is read from the shared-memory ring (slot = local position mod W)
// when fewer than W positions separate it from the end of the reading row's
// level; otherwise ("far") it is read from the global position-ordered array.
#include "pslr_internal.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <set>
#include <tuple>

namespace pslr {

namespace {

inline int64_t a4(int64_t x) { return (x + 3) & ~int64_t(3); }
inline int64_t a2(int64_t x) { return (x + 1) & ~int64_t(1); }

}  // namespace

// List scheduling of a block's rows into steps of at most `cap` rows (cap = the consumer
// threads of a launch).  The ASAP dependency levels cost ceil(width / cap) steps each: cfg5's
// L_B levels are ~500 rows wide, i.e. two steps per level, the second one nearly empty
// (block 19: 118 levels, 215 steps).  Any schedule that keeps a row after its dependencies
// computes the same bits, so rows with slack move to later steps: each step takes up to cap
// ready rows, most urgent first (deadline = min(latest start that keeps the critical path,
// ASAP level + max_delay): the bound keeps a delayed row's dependencies within reach of the
// solution ring).  lev (ASAP levels on entry) is replaced by the step of each row when that
// takes fewer steps; returns the number of levels of the result.
static int32_t list_schedule(const pslr_csr& M, int64_t lo, int64_t nr, bool upper, int64_t cap, int64_t max_delay,
                             std::vector<int32_t>& lev) {
  int32_t depth = 0;
  for (int64_t i = 0; i < nr; ++i) depth = std::max(depth, lev[i] + 1);
  if (cap <= 0 || nr == 0) return depth;
  std::vector<int64_t> width(depth, 0);
  for (int64_t i = 0; i < nr; ++i) ++width[lev[i]];
  int64_t steps_asap = 0;
  for (int64_t w : width) steps_asap += (w + cap - 1) / cap;
  if (steps_asap == depth) return depth;  // every level fits one step already
  // successors (the transpose pattern) and the unscheduled-dependency count of each row
  std::vector<int64_t> sptr(nr + 1, 0);
  std::vector<int32_t> indeg(nr, 0);
  for (int64_t i = 0; i < nr; ++i)
    for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
      const int64_t j = M.indices[e] - lo;
      if (j != i) {
        ++sptr[j + 1];
        ++indeg[i];
      }
    }
  for (int64_t i = 0; i < nr; ++i) sptr[i + 1] += sptr[i];
  std::vector<int32_t> succ(sptr[nr]);
  {
    std::vector<int64_t> fill(sptr.begin(), sptr.end() - 1);
    for (int64_t i = 0; i < nr; ++i)
      for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
        const int64_t j = M.indices[e] - lo;
        if (j != i) succ[fill[j]++] = (int32_t)i;
      }
  }
  // height: the longest chain of dependents below a row (reverse topological order)
  std::vector<int32_t> height(nr, 0);
  for (int64_t t = 0; t < nr; ++t) {
    const int64_t i = upper ? t : nr - 1 - t;
    int32_t h = 0;
    for (int64_t e = sptr[i]; e < sptr[i + 1]; ++e) h = std::max(h, height[succ[e]] + 1);
    height[i] = h;
  }
  auto deadline = [&](int64_t i) {
    return std::min<int64_t>((int64_t)depth - 1 - height[i], (int64_t)lev[i] + max_delay);
  };
  using Key = std::pair<int64_t, int32_t>;  // (deadline, row): most urgent first, then row order
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
  for (int64_t i = 0; i < nr; ++i)
    if (indeg[i] == 0) ready.push({deadline(i), (int32_t)i});
  std::vector<int32_t> step(nr, 0), batch, freed;
  int64_t done = 0;
  int32_t t = 0;
  while (done < nr) {
    batch.clear();
    freed.clear();
    while (!ready.empty() && (int64_t)batch.size() < cap) {
      batch.push_back(ready.top().second);
      ready.pop();
    }
    if (batch.empty()) return depth;  // (a cycle: cannot happen for a triangular factor)
    for (int32_t i : batch) {
      step[i] = t;
      for (int64_t e = sptr[i]; e < sptr[i + 1]; ++e)
        if (--indeg[succ[e]] == 0) freed.push_back(succ[e]);
    }
    for (int32_t i : freed) ready.push({deadline(i), i});
    done += (int64_t)batch.size();
    ++t;
  }
  if ((int64_t)t >= steps_asap) return depth;  // no gain: keep the ASAP levels
  lev.swap(step);
  return t;
}

int analyze_factor(const pslr_csr& M, const std::vector<int64_t>& off, bool upper, TriAnalysis& A,
                   const char* name, int64_t sched_cap, int64_t sched_delay) {
  const int64_t n = M.nrows;
  const int64_t nb = (int64_t)off.size() - 1;
  A.upper = upper;
  A.pos_of_row.assign(n, 0);
  A.row_at_pos.assign(n, 0);
  A.level_end.assign(n, 0);
  A.diag.assign(upper ? n : 0, 0.0);
  A.depth_max = 0;
  A.levels = 0;
  A.reach = 0;
  A.level_of_row.assign(n, 0);
  A.len.assign(n, 0);
  A.blk_depth.assign(nb, 0);
  for (int64_t r = 0; r < n; ++r) {
    int32_t c = 0;
    for (int64_t e = M.indptr[r]; e < M.indptr[r + 1]; ++e) c += (M.indices[e] != r);
    A.len[r] = c;
  }
  std::vector<int32_t> lev;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = off[b], hi = off[b + 1], nr = hi - lo;
    lev.assign(nr, 0);
    for (int64_t t = 0; t < nr; ++t) {
      const int64_t i = upper ? nr - 1 - t : t;
      int32_t lv = 0;
      bool has_diag = false;
      for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
        const int64_t jg = M.indices[e];
        if (jg < lo || jg >= hi) return fail(PSLR_EINVAL, std::string(name) + " is not block diagonal");
        const int64_t j = jg - lo;
        if (upper ? (j < i) : (j > i))
          return fail(PSLR_EINVAL, std::string(name) + (upper ? " is not upper" : " is not lower") +
                                       " triangular");
        if (j == i) {
          has_diag = true;
          if (upper) A.diag[lo + i] = M.data[e];
        } else {
          lv = std::max(lv, lev[j] + 1);
        }
      }
      if (upper && (!has_diag || A.diag[lo + i] == 0.0))
        return fail(PSLR_ESINGULAR, std::string(name) + ": A is singular: zero entry on diagonal.");
      lev[i] = lv;
    }
    const int32_t depth = list_schedule(M, lo, nr, upper, sched_cap, sched_delay, lev);
    A.depth_max = std::max<int64_t>(A.depth_max, depth);
    A.blk_depth[b] = depth;
    A.levels += depth;
    std::vector<int64_t> order(nr);
    std::iota(order.begin(), order.end(), 0);
    auto len = [&](int64_t i) { return A.len[lo + i]; };
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t c) {
      if (lev[a] != lev[c]) return lev[a] < lev[c];
      return len(a) > len(c);
    });
    // level boundaries in position space
    std::vector<int64_t> lvl_end(depth, 0);
    for (int64_t k = 0; k < nr; ++k) lvl_end[lev[order[k]]] = lo + k + 1;
    for (int64_t k = 0; k < nr; ++k) {
      const int64_t i = order[k];
      A.pos_of_row[lo + i] = (int32_t)(lo + k);
      A.row_at_pos[lo + k] = (int32_t)(lo + i);
      A.level_end[lo + i] = (int32_t)lvl_end[lev[i]];
    }
    for (int64_t i = 0; i < nr; ++i) A.level_of_row[lo + i] = lev[i];
    // reach: positions between a dependency and the end of the reading row's level
    for (int64_t i = 0; i < nr; ++i)
      for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
        const int64_t j = M.indices[e] - lo;
        if (j == i) continue;
        A.reach = std::max<int64_t>(A.reach, A.level_end[lo + i] - A.pos_of_row[lo + j]);
      }
  }
  return PSLR_OK;
}

// Emit the streamed format.  far_index[row] gives the global index a far dependency
// is read from (the U-position of the row, where the kernel keeps every value).
// info_of_row[row]: the per-row int the kernel needs (L: U-position, U: row id).
int emit_factor(const pslr_csr& M, const std::vector<int64_t>& off, const TriAnalysis& A, int64_t W,
                int64_t stage_bytes, int64_t seg_rows, const std::vector<int32_t>& far_index,
                const std::vector<int32_t>& info_of_row, int64_t far_slots_max, int64_t rhs_row_bytes,
                TriHost& out, const char* name, bool alt_groups) {
  const int64_t nb = (int64_t)off.size() - 1;
  const bool upper = A.upper;
  out.data.clear();
  out.chunks.clear();
  out.blk_chunk.assign(nb + 1, 0);
  out.far = 0;
  out.nnz_offdiag = 0;
  out.segments = 0;
  std::vector<uint8_t> seg;
  // ELL segment, S = a4(nrows) row slots, G = ceil(w/4) groups of 4 entries per row:
  //   hdr int32[12] {nrows | w << 16, flags | tb << 8, pos0, bytes, S, far_off, rbase, 0, 0, 0, 0, 0}
  //   info int32[S]     L: U-position ; U: row id, bit 31 set when sd = 1 - 2^-53
  //   U: invd f64[S], and only for flags bit 2 ("explicit sd"): sd f64[S], rcp f64[S]
  //   slot u16[G][S][4] near: ring slot (< W), W = zero slot; far: 0x8000 | far-list index
  //   val  f64[G][2][S][2]
  //   far  int32[a4(nfar)] U-positions of the segment's far dependencies
  // Entries past a row's length are exact no-ops (value 0, slot W).  scipy's scaled
  // diagonal sd = d * (1/d) is 1 or 1 - 2^-53 for every diagonal met so far; the flag bit
  // carries it (rcp = RN(1/sd) is then a constant), other values switch the segment to
  // explicit sd / rcp arrays.
  constexpr double kSdLow = 0x1.fffffffffffffp-1;  // 1 - 2^-53
  auto seg_bytes = [&](int64_t nrows, int64_t w, int64_t nfar, bool explicit_sd, bool has_fr) {
    const int64_t S = a4(nrows), G = std::max<int64_t>(1, (w + 3) / 4);
    int64_t b = 48 + 4 * S;
    if (has_fr) b += (2 * S + 15) & ~int64_t(15);
    if (upper) b += (explicit_sd ? 24 : 8) * S;
    b += 40 * G * S;
    b += 4 * a4(nfar);
    return b;
  };
  // a chunk's rhs slice lands in its stage right behind the data: at most (rows + 2) rows
  // (the slice starts at an even position) of rhs_row_bytes each
  auto rhs_bytes = [&](int64_t rows) { return (rows + 2) * rhs_row_bytes; };
  auto sd_of = [&](int64_t r) { return A.diag[r] * (1.0 / A.diag[r]); };
  const bool force_explicit = std::getenv("PSLR_EXPLICIT_SD") != nullptr;  // tests: general layout
  auto sd_plain = [&](int64_t r) {
    const double v = sd_of(r);
    return !force_explicit && (v == 1.0 || (v == kSdLow && 1.0 / v == 0x1.0000000000001p+0));
  };
  // Far-ring: a row read as a far dependency (more than W positions behind the end of the
  // reading row's level) keeps its value in a shared-memory slot beside the ring (ring index
  // W + 1 + slot) from its level to the level of its last far reader, instead of being read
  // back from global memory inside the reader's dependent chain (round 2: those L2 reads cost
  // ~8 % of the single-vector apply).  Slots are reused greedily per block: a target whose
  // last far reader is at level L frees its slot for targets written at levels > L (the level
  // barrier orders the read before the overwrite).  Targets beyond far_slots_max stay global.
  std::vector<int32_t> tend(M.nrows, -1), fslot(M.nrows, -1);
  for (int64_t r = 0; r < M.nrows; ++r) {
    const int64_t lend_r = A.level_end[r];
    for (int64_t e = M.indptr[r]; e < M.indptr[r + 1]; ++e) {
      const int64_t j = M.indices[e];
      if (j != r && lend_r - A.pos_of_row[j] > W) tend[j] = std::max(tend[j], A.level_of_row[r]);
    }
  }
  out.far_slots = 0;
  if (far_slots_max > 0) {
    // When the ring is full, the live target whose last reader comes latest gives up its
    // slot to a new target with an earlier last reader (earliest-end-first keeps the most
    // intervals in a capacity-C interval set); the demoted target is read from global.
    for (int64_t b = 0; b < nb; ++b) {
      std::set<std::tuple<int32_t, int32_t, int32_t>> busy;  // (last reader level, slot, row)
      std::vector<int32_t> freed;
      int32_t next_new = 0, cur = -1;
      for (int64_t k = off[b]; k < off[b + 1]; ++k) {
        const int32_t j = A.row_at_pos[k], lv = A.level_of_row[j];
        if (lv != cur) {
          cur = lv;
          while (!busy.empty() && std::get<0>(*busy.begin()) < lv) {
            freed.push_back(std::get<1>(*busy.begin()));
            busy.erase(busy.begin());
          }
        }
        if (tend[j] < 0) continue;
        int32_t sl = -1;
        if (!freed.empty()) {
          sl = freed.back();
          freed.pop_back();
        } else if (next_new < far_slots_max) {
          sl = next_new++;
        } else if (!busy.empty() && std::get<0>(*busy.rbegin()) > tend[j]) {
          const auto victim = *busy.rbegin();
          busy.erase(std::prev(busy.end()));
          fslot[std::get<2>(victim)] = -1;  // its readers go to global memory
          sl = std::get<1>(victim);
        }
        if (sl < 0) continue;  // the far-ring is full of earlier-ending targets: global
        fslot[j] = sl;
        busy.insert({tend[j], sl, j});
      }
      out.far_slots = std::max<int64_t>(out.far_slots, next_new);
    }
  }
  // far dependencies of the row at position s1 within a level ending at lend that are read
  // from global memory (the segment's far list)
  auto row_far = [&](int64_t s1, int64_t lend) {
    const int64_t r = A.row_at_pos[s1];
    int64_t f = 0;
    for (int64_t e = M.indptr[r]; e < M.indptr[r + 1]; ++e) {
      const int64_t j = M.indices[e];
      if (j != r && lend - A.pos_of_row[j] > W && fslot[j] < 0) ++f;
    }
    return f;
  };
  if (W + 1 + out.far_slots >= 0x8000) return fail(PSLR_EINVAL, std::string(name) + ": ring too large for 16-bit slots");
  // U rows whose value some later row reads as a far dependency: only they need their
  // value in the global position-ordered array (info bit 30); the others stay in the ring
  std::vector<uint8_t> far_target;
  if (upper) {
    far_target.assign(M.nrows, 0);
    for (int64_t r = 0; r < M.nrows; ++r) {
      const int64_t lend_r = A.level_end[r];
      for (int64_t e = M.indptr[r]; e < M.indptr[r + 1]; ++e) {
        const int64_t j = M.indices[e];
        if (j != r && lend_r - A.pos_of_row[j] > W && fslot[j] < 0) far_target[j] = 1;
      }
    }
  }
  // current chunk being filled
  int64_t chunk_start = 0, chunk_nseg = 0, chunk_pos0 = 0, chunk_rows = 0, last_seg = 0;
  auto close_chunk = [&]() {
    if (chunk_nseg == 0) return;
    // the chunk's last segment carries flag bit 3 (the consumers move to the next stage)
    reinterpret_cast<int32_t*>(out.data.data() + last_seg)[1] |= 8;
    ChunkDesc d;
    d.off16 = (uint32_t)(chunk_start / 16);
    d.bytes = (uint32_t)((int64_t)out.data.size() - chunk_start);
    const int64_t p0 = chunk_pos0 & ~int64_t(1);
    d.rpos = (int32_t)p0;
    d.rbytes = (uint32_t)(((chunk_pos0 + chunk_rows - p0 + 1) & ~int64_t(1)) * 8);
    chunk_rows = 0;
    // the base position of the chunk's rhs slice: first segment, word 6 (even: 16-B TMA alignment)
    reinterpret_cast<int32_t*>(out.data.data() + chunk_start)[6] = (int32_t)(chunk_pos0 & ~int64_t(1));
    // word 7: the chunk's data bytes = where its rhs slice starts in the stage
    reinterpret_cast<int32_t*>(out.data.data() + chunk_start)[7] = (int32_t)d.bytes;
    out.chunks.push_back(d);
    chunk_nseg = 0;
    chunk_start = (int64_t)out.data.size();
  };
  // Alternating warp groups (PSLR_ALT_GROUPS, capi.cu): a level that fits the upper consumer
  // warps (threads [hi_tb, seg_rows)) goes there when the previous level did not, so
  // consecutive narrow levels belong to different warps.  A warp loads its row operands one
  // segment ahead, in program order behind its current row's chain; with the levels
  // alternating, the group that idles through level l loads its operands for level l + 1
  // meanwhile, and the level's critical path is barrier -> gathers -> chain -> publish.
  const int64_t hi_tb = ((seg_rows / 2 + 31) / 32) * 32;  // 480 rows: 256 (8 + 7 warps)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = off[b], hi = off[b + 1];
    close_chunk();
    out.blk_chunk[b] = (int32_t)out.chunks.size();
    int64_t k = lo;
    bool prev_upper = true;
    while (k < hi) {
      // one level: positions [k, level_end)
      const int64_t row0 = A.row_at_pos[k];
      const int64_t lend = A.level_end[row0];
      const bool to_upper = alt_groups && !prev_upper && lend - k <= seg_rows - hi_tb;
      const int64_t tb0 = to_upper ? hi_tb : 0;
      prev_upper = to_upper || lend - k > hi_tb;  // (a wide level occupies both groups)
      int64_t s0 = k;
      while (s0 < lend) {
        // Segments of one level run side by side: the segment's rows go to consumer
        // threads [tb, tb + nrows), tb = rows of the level emitted before, mod seg_rows.
        const int64_t tb = (tb0 + s0 - k) % seg_rows;
        // grow a segment while it fits a stage
        int64_t s1 = s0, nnz = 0, w = 0, nfar = 0;
        bool expl = false, hfr = false;
        auto grow = [&](int64_t cap) {
          s1 = s0, nnz = 0, w = 0, nfar = 0;
          expl = false;
          hfr = false;
          while (s1 < lend && s1 - s0 < cap) {
            const int64_t len = A.len[A.row_at_pos[s1]];
            const int64_t w2 = std::max(w, len);
            const int64_t f2 = nfar + row_far(s1, lend);
            const bool e2 = expl || (upper && !sd_plain(A.row_at_pos[s1]));
            const bool h2 = hfr || fslot[A.row_at_pos[s1]] >= 0;
            if (seg_bytes(s1 - s0 + 1, w2, f2, e2, h2) + rhs_bytes(s1 - s0 + 1) > stage_bytes || f2 >= 0x8000) break;
            w = w2;
            nnz += len;
            nfar = f2;
            expl = e2;
            hfr = h2;
            ++s1;
          }
        };
        grow(seg_rows - tb);
        if (s1 == s0)
          return fail(PSLR_EINVAL, std::string(name) + ": a row is too long for the streaming format");
        // A segment cut by the stage size ends on a warp boundary (tb + nrows a multiple
        // of 32), so the level's next segment starts on a fresh warp: no warp owns rows
        // of both, and every warp still takes one step per 480 rows of the level (a
        // straddling warp would take two, and the level ends with its slowest warp).
        if (s1 < lend && s1 - s0 < seg_rows - tb) {
          const int64_t end_t = ((tb + (s1 - s0)) / 32) * 32;
          if (end_t > tb && end_t - tb < s1 - s0) grow(end_t - tb);
        }
        const int64_t nrows = s1 - s0;
        const int64_t bytes = seg_bytes(nrows, w, nfar, expl, hfr);
        if ((int64_t)out.data.size() - chunk_start + bytes + rhs_bytes(chunk_rows + nrows) > stage_bytes ||
            chunk_rows + nrows > kChunkRows)
          close_chunk();
        if (chunk_nseg == 0) chunk_pos0 = s0;
        chunk_rows += nrows;
        seg.assign(bytes, 0);
        int32_t* h = reinterpret_cast<int32_t*>(seg.data());
        if (w > 0xffff) return fail(PSLR_EINVAL, std::string(name) + ": a row is too long for the streaming format");
        h[0] = (int32_t)(nrows | (w << 16));
        h[1] = ((s1 == lend) ? 1 : 0) | (expl ? 4 : 0) | (hfr ? 16 : 0) |
               (int32_t)(tb << 8);  // bit0 level end, bit2 explicit sd, bit4 far-ring targets
        const int64_t S = a4(nrows);
        const int64_t G = std::max<int64_t>(1, (w + 3) / 4);
        h[2] = (int32_t)s0;
        h[3] = (int32_t)bytes;
        h[4] = (int32_t)S;
        last_seg = (int64_t)out.data.size();
        int32_t* info = h + 12;
        uint8_t* p = reinterpret_cast<uint8_t*>(info + S);
        uint16_t* fsl = nullptr;  // far-ring slot + 1 of each row (0: not a far-ring target)
        if (hfr) {
          fsl = reinterpret_cast<uint16_t*>(p);
          p += (2 * S + 15) & ~int64_t(15);
        }
        double* invd = nullptr;
        double* sd = nullptr;
        double* rcp = nullptr;
        if (upper) {
          invd = reinterpret_cast<double*>(p);
          p += 8 * S;
          if (expl) {
            sd = reinterpret_cast<double*>(p);
            rcp = sd + S;
            p += 16 * S;
          }
        }
        uint16_t* slot = reinterpret_cast<uint16_t*>(p);
        double* val = reinterpret_cast<double*>(p + 8 * G * S);
        int32_t* far = reinterpret_cast<int32_t*>(p + 40 * G * S);
        h[5] = (int32_t)(reinterpret_cast<uint8_t*>(far) - seg.data());
        auto slot_at = [&](int64_t t, int64_t kk) -> uint16_t& { return slot[((kk >> 2) * S + t) * 4 + (kk & 3)]; };
        auto val_at = [&](int64_t t, int64_t kk) -> double& {
          return val[(((kk >> 2) * 2 + ((kk >> 1) & 1)) * S + t) * 2 + (kk & 1)];
        };
        for (int64_t t = 0; t < S; ++t)
          for (int64_t kk = 0; kk < 4 * G; ++kk) {  // padding (incl. rows nrows..S-1): exact no-ops
            val_at(t, kk) = 0.0;
            slot_at(t, kk) = (uint16_t)W;
          }
        for (int64_t t = 0; t < nrows; ++t) {
          const int64_t r = A.row_at_pos[s0 + t];
          info[t] = info_of_row[r];
          if (fsl) fsl[t] = (uint16_t)(fslot[r] + 1);
          if (upper) {
            const double dinv = 1.0 / A.diag[r];
            const double sdv = A.diag[r] * dinv;  // scipy: (U @ diags(1/diag)) diagonal
            invd[t] = dinv;
            if (expl) {
              sd[t] = sdv;
              rcp[t] = 1.0 / sdv;
            } else if (sdv != 1.0) {
              info[t] = (int32_t)((uint32_t)info[t] | 0x80000000u);
            }
            if (far_target[r]) info[t] = (int32_t)((uint32_t)info[t] | 0x40000000u);
          }
        }
        int64_t nf = 0;
        for (int64_t t = 0; t < nrows; ++t) {
          const int64_t r = A.row_at_pos[s0 + t];
          int64_t kk = 0;
          for (int64_t e = M.indptr[r]; e < M.indptr[r + 1]; ++e) {
            const int64_t j = M.indices[e];
            if (j == r) continue;
            double v = M.data[e];
            if (upper) v = v * (1.0 / A.diag[j]);  // scipy pre-scales U's columns by 1/diag
            val_at(t, kk) = v;
            const int64_t pj = A.pos_of_row[j];
            if (lend - pj > W && fslot[j] >= 0) {
              slot_at(t, kk) = (uint16_t)(W + 1 + fslot[j]);  // far-ring: a shared-memory read
            } else if (lend - pj <= W) {
              slot_at(t, kk) = (uint16_t)((pj - lo) & (W - 1));
            } else {
              far[nf] = far_index[j];
              slot_at(t, kk) = (uint16_t)(0x8000 | nf);
              ++nf;
              out.far++;
              h[1] |= 2;  // the segment has far dependencies (kernel gather variant)
            }
            ++kk;
          }
        }
        out.data.insert(out.data.end(), seg.begin(), seg.end());
        chunk_nseg++;
        out.segments++;
        out.nnz_offdiag += nnz;
        s0 = s1;
      }
      k = lend;
    }
    close_chunk();
  }
  out.blk_chunk[nb] = (int32_t)out.chunks.size();
  if ((uint64_t)out.data.size() / 16 > 0xffffffffull)
    return fail(PSLR_EINVAL, std::string(name) + ": packed factor exceeds 64 GiB");
  return PSLR_OK;
}

}  // namespace pslr

namespace pslr {

// Level merging (depth halving) of a block-diagonal triangular factor.
//
// A row i at an odd dependency level l has its dependencies at level l - 1 substituted by
// their own rows (rows at level l - 1 are at an even level and keep theirs):
//   L (unit lower):  z_i = b_i - sum_k L_ik z_k,  z_j = b_j - sum_k L_jk z_k
//     L'_ik = L_ik [k not adjacent] - sum_j L_ij L_jk ,   b'_i = b_i - sum_j L_ij b_j
//   U (upper):       U_ii x_i = y_i - sum_k U_ik x_k,  c_ij = U_ij / U_jj
//     U'_ik = U_ik [k not adjacent] - sum_j c_ij U_jk ,   y'_i = y_i - sum_j c_ij y_j
// over the adjacent-level dependencies j of i.  Every dependency of a merged row then sits
// at level <= l - 2, so a row at level l lands at level ceil(l / 2): the level count halves
// at ~1.5x the off-diagonal entries (cfg5: L 156 -> 78, U 370 -> 185 levels on the deepest
// block).  Same operator, different rounding: the solve is exact up to fp64 round-off, not
// bit-identical with the reference's row-by-row substitution (north star: 1e-10).
//
// The right-hand-side transform of the merged rows is returned as records of at most
// kXfWidth terms (i, j0..j2; c0..c2): rhs'_i = rhs_i - (c0 rhs_j0 + c1 rhs_j1 + c2 rhs_j2).
// It reads only unmerged (even-level) rows and writes only merged ones, so it runs in place.
// A row with more adjacent dependencies than kXfWidth keeps the rest (still correct; that
// row's level just does not halve).  wmax > 0 merges only the level pairs of at most wmax
// rows (the narrow, latency-bound levels): fewer levels at a few more streamed bytes.
int merge_levels(const pslr_csr& M, const std::vector<int64_t>& off, bool upper, int64_t wmax, HostCsr& out,
                 MergeXf& X, const char* name) {
  const int64_t n = M.nrows, nb = (int64_t)off.size() - 1;
  out.nrows = n;
  out.ncols = M.ncols;
  out.indptr.assign(n + 1, 0);
  out.indices.clear();
  out.data.clear();
  out.indices.reserve((size_t)(M.nnz * 3 / 2));
  out.data.reserve((size_t)(M.nnz * 3 / 2));
  X.rows.clear();
  X.c.clear();
  X.blk.assign(nb + 1, 0);
  std::vector<int32_t> lev;
  std::vector<double> acc;        // dense accumulator over the block's columns
  std::vector<uint8_t> used;
  std::vector<int32_t> cols;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = off[b], hi = off[b + 1], nr = hi - lo;
    X.blk[b] = (int32_t)(X.rows.size() / kXfWidth1);
    lev.assign(nr, 0);
    for (int64_t t = 0; t < nr; ++t) {
      const int64_t i = upper ? nr - 1 - t : t;
      int32_t lv = 0;
      for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
        const int64_t jg = M.indices[e];
        if (jg < lo || jg >= hi) return fail(PSLR_EINVAL, std::string(name) + " is not block diagonal");
        const int64_t j = jg - lo;
        if (upper ? (j < i) : (j > i))
          return fail(PSLR_EINVAL, std::string(name) + (upper ? " is not upper" : " is not lower") + " triangular");
        if (j != i) lv = std::max(lv, lev[j] + 1);
      }
      lev[i] = lv;
    }
    // level pair (l - 1, l), l odd, is merged when its rows fit one pass of the consumer
    // threads (wmax > 0): wider pairs would take two row steps per level, and their merged
    // rows reach past the ring (far dependencies) while saving no barrier on the critical path
    int32_t depth = 0;
    for (int64_t i = 0; i < nr; ++i) depth = std::max(depth, lev[i] + 1);
    std::vector<int64_t> width(depth + 1, 0);
    for (int64_t i = 0; i < nr; ++i) ++width[lev[i]];
    auto merge_level = [&](int32_t l) { return (l & 1) && (wmax <= 0 || width[l] + width[l - 1] <= wmax); };
    acc.assign(nr, 0.0);
    used.assign(nr, 0);
    auto diag_of = [&](int64_t r) -> double {  // r global
      for (int64_t e = M.indptr[r]; e < M.indptr[r + 1]; ++e)
        if (M.indices[e] == r) return M.data[e];
      return 0.0;
    };
    for (int64_t i = 0; i < nr; ++i) {
      const int64_t ig = lo + i;
      const int64_t e0 = M.indptr[ig], e1 = M.indptr[ig + 1];
      int nadj = 0;
      int32_t adj[kXfWidth];
      double cadj[kXfWidth];
      if (merge_level(lev[i])) {
        for (int64_t e = e0; e < e1 && nadj < kXfWidth; ++e) {
          const int64_t j = M.indices[e] - lo;
          if (j != i && lev[j] == lev[i] - 1) {
            double c = M.data[e];
            if (upper) {
              const double dj = diag_of(lo + j);
              if (dj == 0.0) return fail(PSLR_ESINGULAR, std::string(name) + ": A is singular: zero entry on diagonal.");
              c = c / dj;
            }
            adj[nadj] = (int32_t)j;
            cadj[nadj] = c;
            ++nadj;
          }
        }
      }
      if (nadj == 0) {  // copied as is
        for (int64_t e = e0; e < e1; ++e) {
          out.indices.push_back(M.indices[e]);
          out.data.push_back(M.data[e]);
        }
        out.indptr[ig + 1] = (int64_t)out.indices.size();
        continue;
      }
      cols.clear();
      auto add = [&](int64_t j, double v) {
        if (!used[j]) {
          used[j] = 1;
          acc[j] = 0.0;
          cols.push_back((int32_t)j);
        }
        acc[j] += v;
      };
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t j = M.indices[e] - lo;
        bool is_adj = false;
        for (int a = 0; a < nadj; ++a) is_adj |= (adj[a] == j);
        if (!is_adj) add(j, M.data[e]);
      }
      for (int a = 0; a < nadj; ++a) {
        const int64_t jg = lo + adj[a];
        for (int64_t e = M.indptr[jg]; e < M.indptr[jg + 1]; ++e) {
          const int64_t k = M.indices[e] - lo;
          if (k == adj[a]) continue;
          add(k, -cadj[a] * M.data[e]);
        }
      }
      std::sort(cols.begin(), cols.end());
      for (int32_t j : cols) {
        used[j] = 0;
        if (acc[j] == 0.0 && j != i) continue;  // exact cancellation: no entry
        out.indices.push_back((int32_t)(lo + j));
        out.data.push_back(acc[j]);
      }
      out.indptr[ig + 1] = (int64_t)out.indices.size();
      X.rows.push_back((int32_t)ig);
      for (int a = 0; a < kXfWidth; ++a) {
        X.rows.push_back(a < nadj ? (int32_t)(lo + adj[a]) : (int32_t)ig);
        X.c.push_back(a < nadj ? cadj[a] : 0.0);
      }
      X.c.push_back(0.0);
    }
  }
  X.blk[nb] = (int32_t)(X.rows.size() / kXfWidth1);
  out.nnz = (int64_t)out.indices.size();
  return PSLR_OK;
}

}  // namespace pslr
