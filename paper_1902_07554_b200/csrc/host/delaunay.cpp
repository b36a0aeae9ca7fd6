#include "delaunay.hpp"

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <string>
#include <numeric>

#include "../common/predicates.hpp"
#include "rng.hpp"

namespace sbdt_host {
namespace {

template <int D>
struct Cell {
  std::uint32_t v[D + 1];
  std::uint32_t n[D + 1];
  std::int8_t parity;
  std::uint8_t alive;
};

// Morton key with 21 bits (3D) / 32 bits (2D) per axis.
inline std::uint64_t spread3(std::uint64_t x) {
  x &= 0x1fffff;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}
inline std::uint64_t spread2(std::uint64_t x) {
  x &= 0xffffffffULL;
  x = (x | x << 16) & 0x0000ffff0000ffffULL;
  x = (x | x << 8) & 0x00ff00ff00ff00ffULL;
  x = (x | x << 4) & 0x0f0f0f0f0f0f0f0fULL;
  x = (x | x << 2) & 0x3333333333333333ULL;
  x = (x | x << 1) & 0x5555555555555555ULL;
  return x;
}

// Incremental Bowyer-Watson over a slot array of cells. The result is
// determined only by the conflict rules (restated from the reference's
// contract, see delaunay.hpp); the search structure below — bootstrap by
// exact affine-independence tests, a deterministic visibility walk with a
// linear-scan fallback, a depth-first cavity search with per-cell marks, and
// the new cells' mutual links through a small open-addressing ridge table —
// is this repo's own.
template <int D>
class Builder {
 public:
  Builder(const double* coords, std::uint64_t seed) : xyz_(coords), rng_(seed) {}

  TriSoA run(const std::uint32_t* ids, std::size_t n) {
    if (n < D + 1) throw DegenerateInputError("need at least " + std::to_string(D + 1) + " points");
    brio_order(ids, n);
    std::vector<char> used(order_.size(), 0);
    first_simplex(used);
    for (std::size_t i = 0; i < order_.size(); ++i)
      if (!used[i]) insert(order_[i]);
    return compact();
  }

 private:
  const double* P(std::uint32_t id) const { return xyz_ + std::size_t(id) * D; }

  int orient(const double* const* p) const {
    if constexpr (D == 2) return sbdt_pred::orient2(p[0], p[1], p[2]);
    else return sbdt_pred::orient3(p[0], p[1], p[2], p[3]);
  }

  int in_sphere(const double* const* p, const double* q) const {
    if constexpr (D == 2) {
      const int s = sbdt_pred::in_sphere2_filtered(p[0], p[1], p[2], q);
      if (s != 2) return s;
      scratch_.resize(sbdt_pred::kInSphere2Scratch);
      return sbdt_pred::in_sphere2_exact_buf(p[0], p[1], p[2], q, scratch_.data());
    } else {
      const int s = sbdt_pred::in_sphere3_filtered(p[0], p[1], p[2], p[3], q);
      if (s != 2) return s;
      scratch_.resize(sbdt_pred::kInSphere3Scratch);
      return sbdt_pred::in_sphere3_exact_buf(p[0], p[1], p[2], p[3], q, scratch_.data());
    }
  }

  void brio_order(const std::uint32_t* ids, std::size_t n) {
    order_.assign(ids, ids + n);
    // Seeded shuffle, then rounds of doubling size, each sorted on a Morton curve.
    for (std::size_t i = n - 1; i > 0; --i) std::swap(order_[i], order_[uniform_index(rng_, i + 1)]);
    double lo[D], hi[D];
    for (int d = 0; d < D; ++d) lo[d] = hi[d] = P(order_[0])[d];
    for (std::size_t i = 1; i < n; ++i)
      for (int d = 0; d < D; ++d) {
        lo[d] = std::min(lo[d], P(order_[i])[d]);
        hi[d] = std::max(hi[d], P(order_[i])[d]);
      }
    for (int d = 0; d < D; ++d) blo_[d] = lo[d], bhi_[d] = hi[d];
    const double bits = (D == 3) ? 2097151.0 : 4294967295.0;
    std::vector<std::pair<std::uint64_t, std::uint32_t>> keyed(n);
    for (std::size_t i = 0; i < n; ++i) {
      std::uint64_t key = 0;
      for (int d = 0; d < D; ++d) {
        const double ext = hi[d] - lo[d];
        const double t = ext > 0 ? (P(order_[i])[d] - lo[d]) / ext : 0.0;
        const std::uint64_t q = static_cast<std::uint64_t>(std::min(bits, std::max(0.0, t * bits)));
        key |= (D == 3 ? spread3(q) : spread2(q)) << d;
      }
      keyed[i] = {key, order_[i]};
    }
    // rounds: [0, n/2^r) ... ; the last round is the upper half.
    std::vector<std::size_t> bounds;
    std::size_t end = n;
    while (end > 64) {
      bounds.push_back(end);
      end /= 2;
    }
    bounds.push_back(end);
    std::reverse(bounds.begin(), bounds.end());
    std::size_t begin = 0;
    for (std::size_t b : bounds) {
      std::sort(keyed.begin() + begin, keyed.begin() + b);
      begin = b;
    }
    for (std::size_t i = 0; i < n; ++i) order_[i] = keyed[i].second;
  }

  std::uint32_t new_cell(const Cell<D>& c) {
    std::uint32_t id;
    if (free_.empty()) {
      id = static_cast<std::uint32_t>(cells_.size());
      cells_.push_back(c);
      mark_.push_back(0);
    } else {
      id = free_.back();
      free_.pop_back();
      cells_[id] = c;
    }
    cells_[id].alive = 1;
    return id;
  }

  int parity_of(const std::uint32_t* v) const {
    const double* p[D + 1];
    for (int i = 0; i <= D; ++i) p[i] = P(v[i]);
    return orient(p);
  }

  // Rank of the affine hull of {q} and the already chosen points (exact).
  bool extends_hull(const std::vector<std::uint32_t>& chosen, std::uint32_t q) const {
    const double* c = P(q);
    if (chosen.size() == 1) {
      const double* a = P(chosen[0]);
      for (int d = 0; d < D; ++d)
        if (a[d] != c[d]) return true;
      return false;
    }
    const double* a = P(chosen[0]);
    const double* b = P(chosen[1]);
    if (chosen.size() == 2) {
      if constexpr (D == 2) {
        return sbdt_pred::orient2(a, b, c) != 0;
      } else {
        // collinear in 3-D iff all three coordinate-plane projections are
        for (int u = 0; u < 3; ++u) {
          const int v = (u + 1) % 3;
          const double pa[2] = {a[u], a[v]}, pb[2] = {b[u], b[v]}, pc[2] = {c[u], c[v]};
          if (sbdt_pred::orient2(pa, pb, pc) != 0) return true;
        }
        return false;
      }
    }
    if constexpr (D == 3) return sbdt_pred::orient3(a, b, P(chosen[2]), c) != 0;
    return false;
  }

  // The first D+1 affinely independent points of the insertion order form
  // the first cell, closed by one infinite cell per facet.
  void first_simplex(std::vector<char>& used) {
    std::vector<std::uint32_t> chosen;
    for (std::size_t i = 0; i < order_.size() && chosen.size() <= D; ++i) {
      if (chosen.empty() || extends_hull(chosen, order_[i])) {
        chosen.push_back(order_[i]);
        used[i] = 1;
      }
    }
    if (chosen.size() < D + 1) throw DegenerateInputError("all points affinely dependent");
    std::sort(chosen.begin(), chosen.end());
    Cell<D> f;
    for (int i = 0; i <= D; ++i) f.v[i] = chosen[i], f.n[i] = kNone;
    f.parity = static_cast<std::int8_t>(parity_of(f.v));
    const std::uint32_t fid = new_cell(f);
    // the hull star: cell opposite vertex d = facet d + infinity, linked to
    // the finite cell through slot D and to each other through their ridges
    std::vector<std::uint32_t> made;
    for (int d = 0; d <= D; ++d) {
      Cell<D> h;
      int w = 0;
      for (int i = 0; i <= D; ++i)
        if (i != d) h.v[w++] = chosen[i];
      h.v[D] = kInf;
      h.parity = 0;
      for (int i = 0; i <= D; ++i) h.n[i] = kNone;
      h.n[D] = fid;
      const std::uint32_t hid = new_cell(h);
      cells_[fid].n[d] = hid;
      made.push_back(hid);
    }
    link_by_ridges(made, kInf);
    hint_ = fid;
  }

  // conflict of q with an infinite cell: q strictly on the outer side of its
  // hull facet, or on the facet's plane with a facet vertex of lower id
  bool hull_conflict(const Cell<D>& s, const double* q, std::uint32_t qid) const {
    const Cell<D>& inside = cells_[s.n[D]];
    std::uint32_t apex = kInf;  // the inside cell's vertex off the facet
    for (int i = 0; i <= D && apex == kInf; ++i) {
      const std::uint32_t v = inside.v[i];
      if (std::find(s.v, s.v + D, v) == s.v + D) apex = v;
    }
    const double* f[D + 1];
    for (int i = 0; i < D; ++i) f[i] = P(s.v[i]);
    f[D] = q;
    const int side_q = orient(f);
    if (side_q == 0) return *std::min_element(s.v, s.v + D) < qid;
    f[D] = P(apex);
    return side_q == -orient(f);
  }

  // conflict of q with a cell (in_sphere, tie toward "lowest id is outside")
  bool in_conflict(std::uint32_t id, const double* q, std::uint32_t qid) const {
    const Cell<D>& s = cells_[id];
    if (s.v[D] == kInf) return hull_conflict(s, q, qid);
    const double* p[D + 1];
    for (int i = 0; i <= D; ++i) p[i] = P(s.v[i]);
    if (s.parity < 0) std::swap(p[0], p[1]);
    const int r = in_sphere(p, q);
    if (r != 0) return r > 0;
    return *std::min_element(s.v, s.v + D + 1) < qid;
  }

  // Visibility walk from the hint: leave through the first facet (in slot
  // order, not back through the facet just crossed) that separates q from
  // the cell's apex; a cell with no such facet contains q. A hull cell ends
  // the walk when q conflicts with it. The walk terminates in a Delaunay
  // triangulation; the step budget only guards the degenerate ties, after
  // which every live cell is scanned for a conflict.
  std::uint32_t locate(const double* q, std::uint32_t qid) const {
    std::uint32_t cur = hint_, came = kNone;
    const std::size_t budget = 8 * cells_.size() + 64;
    for (std::size_t step = 0; step < budget; ++step) {
      const Cell<D>& s = cells_[cur];
      if (s.v[D] == kInf) {
        if (hull_conflict(s, q, qid)) return cur;
        came = cur;
        cur = s.n[D];
        continue;
      }
      const double* c[D + 1];
      for (int i = 0; i <= D; ++i) c[i] = P(s.v[i]);
      int leave = -1;
      for (int d = 0; d <= D && leave < 0; ++d) {
        if (s.n[d] == came) continue;
        const double* keep = c[d];
        c[d] = q;
        const int o = orient(c);
        c[d] = keep;
        if (o != 0 && o != s.parity) leave = d;
      }
      if (leave < 0) return cur;
      came = cur;
      cur = s.n[leave];
    }
    for (std::uint32_t id = 0; id < cells_.size(); ++id)
      if (cells_[id].alive && in_conflict(id, q, qid)) return id;
    throw DegenerateInputError("point location failed");
  }

  // Pairs the facets through q of the cells in `made`: every ridge (a facet
  // minus `pivot`) is shared by exactly two of them.
  void link_by_ridges(const std::vector<std::uint32_t>& made, std::uint32_t pivot) {
    std::size_t cap = 16;
    while (cap < 4 * made.size() * D) cap <<= 1;
    table_.assign(cap, Slot{~0ull, kNone, 0});
    for (std::uint32_t cid : made) {
      const Cell<D>& c = cells_[cid];
      for (int d = 0; d <= D; ++d) {
        if (c.v[d] == pivot) continue;
        std::uint64_t key = 0;  // the D-1 ridge ids, ascending (the cell's order minus v[d], pivot)
        for (int i = 0; i <= D; ++i)
          if (i != d && c.v[i] != pivot) key = key * 0x100000000ull + c.v[i];
        std::size_t h = (key * 0x9E3779B97F4A7C15ull) >> 7 & (cap - 1);
        for (;; h = (h + 1) & (cap - 1)) {
          Slot& sl = table_[h];
          if (sl.cell == kNone) {
            sl = Slot{key, cid, d};
            break;
          }
          if (sl.key == key) {
            cells_[cid].n[d] = sl.cell;
            cells_[sl.cell].n[sl.slot] = cid;
            sl.key = ~0ull - 1;  // consumed: a third owner would be a defect
            break;
          }
        }
      }
    }
  }

  void insert(std::uint32_t qid) {
    const double* q = P(qid);
    const std::uint32_t start = locate(q, qid);
    // depth-first cavity search; mark_: 1 = in the cavity, 2 = checked outside
    std::vector<std::uint32_t>& stack = stack_;
    stack.assign(1, start);
    mark_[start] = 1;
    touched_.assign(1, start);
    shell_.clear();
    while (!stack.empty()) {
      const std::uint32_t id = stack.back();
      stack.pop_back();
      for (int d = 0; d <= D; ++d) {
        const std::uint32_t nb = cells_[id].n[d];
        if (mark_[nb] == 0) {
          mark_[nb] = in_conflict(nb, q, qid) ? 1 : 2;
          touched_.push_back(nb);
          if (mark_[nb] == 1) stack.push_back(nb);
        }
        if (mark_[nb] == 2) shell_.push_back(Face{id, d, nb});
      }
    }
    // the cavity's boundary facets, each coned to q; the outside cell's
    // back link is found before any cavity slot is recycled
    std::vector<std::uint32_t>& made = made_;
    made.clear();
    for (Face& f : shell_) {
      const Cell<D>& inner = cells_[f.cell];
      const Cell<D>& outer = cells_[f.outside];
      f.back = -1;
      for (int j = 0; j <= D; ++j)
        if (outer.n[j] == f.cell) f.back = j;
      Cell<D> c;
      std::uint32_t vs[D + 1];
      int w = 0;
      for (int i = 0; i <= D; ++i)
        if (i != f.slot) vs[w++] = inner.v[i];
      vs[D] = qid;
      std::sort(vs, vs + D + 1);  // ascending, the infinite id last
      for (int i = 0; i <= D; ++i) c.v[i] = vs[i], c.n[i] = kNone;
      const int at_q = static_cast<int>(std::find(vs, vs + D + 1, qid) - vs);
      c.n[at_q] = f.outside;
      if (c.v[D] == kInf) {
        c.parity = 0;
      } else {
        c.parity = static_cast<std::int8_t>(parity_of(c.v));
        if (c.parity == 0) throw DegenerateInputError("affinely dependent points beyond the tie-break's scope");
      }
      made.push_back(0);
      pending_.push_back(c);
    }
    for (std::uint32_t id : touched_) {
      if (mark_[id] == 1) {
        cells_[id].alive = 0;
        free_.push_back(id);
      }
      mark_[id] = 0;
    }
    for (std::size_t i = 0; i < shell_.size(); ++i) {
      made[i] = new_cell(pending_[i]);
      cells_[shell_[i].outside].n[shell_[i].back] = made[i];
    }
    pending_.clear();
    link_by_ridges(made, qid);
    hint_ = made.back();
    if (cells_[hint_].v[D] == kInf) hint_ = cells_[hint_].n[D];
  }

  // Morton key of a cell's position (centroid of its finite vertices) in the
  // bounding box of the inserted points.
  std::uint64_t cell_key(const Cell<D>& c) const {
    const double bits = (D == 3) ? 2097151.0 : 4294967295.0;
    double ctr[D] = {};
    int nf = 0;
    for (int j = 0; j <= D; ++j)
      if (c.v[j] != kInf) {
        for (int d = 0; d < D; ++d) ctr[d] += P(c.v[j])[d];
        ++nf;
      }
    std::uint64_t key = 0;
    for (int d = 0; d < D; ++d) {
      const double ext = bhi_[d] - blo_[d];
      const double t = ext > 0 ? (ctr[d] / nf - blo_[d]) / ext : 0.0;
      const std::uint64_t q = static_cast<std::uint64_t>(std::min(bits, std::max(0.0, t * bits)));
      key |= (D == 3 ? spread3(q) : spread2(q)) << d;
    }
    return key;
  }

  // Output rows in the order of a Morton curve through the cells' positions
  // (ties by slot): consecutive rows of the SoA are neighbours in space, which
  // is the layout the device kernels' coordinate gathers want.
  // Any row order is a valid Triangulation; SBDT_HOST_ROW_ORDER=slot keeps the
  // slot order of the construction (what the bench's row-order leg compares).
  TriSoA compact() {
    std::vector<std::uint32_t> remap(cells_.size(), kNone);
    std::size_t cnt = 0;
    const char* ord = std::getenv("SBDT_HOST_ROW_ORDER");
    if (ord && std::string(ord) == "slot") {
      for (std::size_t i = 0; i < cells_.size(); ++i)
        if (cells_[i].alive) remap[i] = static_cast<std::uint32_t>(cnt++);
    } else {
      std::vector<std::pair<std::uint64_t, std::uint32_t>> keyed;
      keyed.reserve(cells_.size());
      for (std::size_t i = 0; i < cells_.size(); ++i)
        if (cells_[i].alive) keyed.emplace_back(cell_key(cells_[i]), static_cast<std::uint32_t>(i));
      std::sort(keyed.begin(), keyed.end());
      for (const auto& kv : keyed) remap[kv.second] = static_cast<std::uint32_t>(cnt++);
    }
    TriSoA t;
    t.dim = D;
    t.count = cnt;
    t.verts.resize((D + 1) * cnt);
    t.nbrs.resize((D + 1) * cnt);
    t.parity.resize(cnt);
    for (std::size_t i = 0; i < cells_.size(); ++i) {
      if (!cells_[i].alive) continue;
      const std::size_t s = remap[i];
      for (int j = 0; j <= D; ++j) {
        t.verts[j * cnt + s] = cells_[i].v[j];
        t.nbrs[j * cnt + s] = cells_[i].n[j] == kNone ? kNone : remap[cells_[i].n[j]];
      }
      t.parity[s] = cells_[i].parity;
    }
    return t;
  }

  struct Face {
    std::uint32_t cell;     // the cavity cell
    int slot;               // its slot facing `outside`
    std::uint32_t outside;  // the kept cell across that facet
    int back = -1;          // outside's slot facing the cavity
  };
  struct Slot {
    std::uint64_t key;
    std::uint32_t cell;
    int slot;
  };

  const double* xyz_;
  Rng rng_;
  std::vector<std::uint32_t> order_;
  std::vector<Cell<D>> cells_;
  std::vector<std::uint8_t> mark_;
  std::vector<std::uint32_t> free_, stack_, touched_, made_;
  std::vector<Face> shell_;
  std::vector<Cell<D>> pending_;
  std::vector<Slot> table_;
  std::uint32_t hint_ = 0;
  double blo_[D] = {}, bhi_[D] = {};
  mutable std::vector<double> scratch_;
};

}  // namespace

TriSoA triangulate(int dim, const double* coords, const std::uint32_t* ids, std::size_t n,
                   std::uint64_t seed) {
  if (dim == 2) {
    Builder<2> b(coords, seed);
    return b.run(ids, n);
  }
  if (dim == 3) {
    Builder<3> b(coords, seed);
    return b.run(ids, n);
  }
  throw std::invalid_argument("dim must be 2 or 3");
}

}  // namespace sbdt_host
