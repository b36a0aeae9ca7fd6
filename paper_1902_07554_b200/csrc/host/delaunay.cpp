#include "delaunay.hpp"

#include <algorithm>
#include <array>
#include <cstring>
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

template <int D>
class Builder {
 public:
  Builder(const double* coords, std::uint64_t seed) : xyz_(coords), rng_(seed) {}

  TriSoA run(const std::uint32_t* ids, std::size_t n) {
    if (n < D + 1) throw DegenerateInputError("need at least " + std::to_string(D + 1) + " points");
    brio_order(ids, n);
    bootstrap();
    for (std::size_t i = D + 1; i < order_.size(); ++i) insert(order_[i]);
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

  static bool collinear3(const double* a, const double* b, const double* c) {
    const double ux = b[0] - a[0], uy = b[1] - a[1], uz = b[2] - a[2];
    const double vx = c[0] - a[0], vy = c[1] - a[1], vz = c[2] - a[2];
    return (uy * vz - uz * vy) == 0.0 && (uz * vx - ux * vz) == 0.0 && (ux * vy - uy * vx) == 0.0;
  }

  static bool same_point(const double* a, const double* b) {
    for (int d = 0; d < D; ++d)
      if (a[d] != b[d]) return false;
    return true;
  }

  std::uint32_t create(const Cell<D>& c) {
    if (!free_.empty()) {
      const std::uint32_t id = free_.back();
      free_.pop_back();
      cells_[id] = c;
      cells_[id].alive = 1;
      return id;
    }
    cells_.push_back(c);
    cells_.back().alive = 1;
    return static_cast<std::uint32_t>(cells_.size() - 1);
  }

  int parity_of(const std::uint32_t* v) const {
    const double* p[D + 1];
    for (int i = 0; i <= D; ++i) p[i] = P(v[i]);
    return orient(p);
  }

  void bootstrap() {
    std::vector<std::size_t> pick{0};
    for (std::size_t i = 1; i < order_.size() && pick.size() <= D; ++i) {
      bool independent = false;
      if (pick.size() == 1) {
        independent = !same_point(P(order_[pick[0]]), P(order_[i]));
      } else if (pick.size() == 2) {
        if constexpr (D == 2)
          independent = sbdt_pred::orient2(P(order_[pick[0]]), P(order_[pick[1]]), P(order_[i])) != 0;
        else
          independent = !collinear3(P(order_[pick[0]]), P(order_[pick[1]]), P(order_[i]));
      } else {
        if constexpr (D == 3)
          independent = sbdt_pred::orient3(P(order_[pick[0]]), P(order_[pick[1]]),
                                           P(order_[pick[2]]), P(order_[i])) != 0;
      }
      if (independent) pick.push_back(i);
    }
    if (pick.size() < D + 1) throw DegenerateInputError("all points affinely dependent");
    std::vector<std::uint32_t> reordered;
    reordered.reserve(order_.size());
    for (std::size_t j = 0; j <= D; ++j) reordered.push_back(order_[pick[j]]);
    std::size_t next_pick = 0;
    for (std::size_t r = 0; r < order_.size(); ++r) {
      if (next_pick < pick.size() && pick[next_pick] == r) {
        ++next_pick;
        continue;
      }
      reordered.push_back(order_[r]);
    }
    order_ = std::move(reordered);

    Cell<D> s0;
    for (int i = 0; i <= D; ++i) s0.v[i] = order_[i];
    std::sort(s0.v, s0.v + D + 1);
    s0.parity = static_cast<std::int8_t>(parity_of(s0.v));
    for (int i = 0; i <= D; ++i) s0.n[i] = kNone;
    const std::uint32_t fid = create(s0);
    std::uint32_t inf_ids[D + 1];
    for (int d = 0; d <= D; ++d) {
      Cell<D> inf;
      int idx = 0;
      for (int i = 0; i <= D; ++i)
        if (i != d) inf.v[idx++] = cells_[fid].v[i];
      inf.v[D] = kInf;
      inf.parity = 0;
      for (int i = 0; i <= D; ++i) inf.n[i] = kNone;
      inf.n[D] = fid;
      inf_ids[d] = create(inf);
      cells_[fid].n[d] = inf_ids[d];
    }
    for (int d = 0; d <= D; ++d) {
      Cell<D>& inf = cells_[inf_ids[d]];
      for (int j = 0; j < D; ++j)
        for (int i = 0; i <= D; ++i)
          if (cells_[fid].v[i] == inf.v[j]) {
            inf.n[j] = inf_ids[i];
            break;
          }
    }
    hint_ = fid;
  }

  bool infinite_conflict(const Cell<D>& s, const double* q, std::uint32_t qid) const {
    const Cell<D>& owner = cells_[s.n[D]];
    const double* pts[D + 1];
    for (int i = 0; i < D; ++i) pts[i] = P(s.v[i]);
    std::uint32_t inner = kInf;
    for (int i = 0; i <= D; ++i) {
      const std::uint32_t v = owner.v[i];
      bool on_facet = false;
      for (int f = 0; f < D; ++f) on_facet |= (s.v[f] == v);
      if (!on_facet) {
        inner = v;
        break;
      }
    }
    pts[D] = P(inner);
    const int inner_sign = orient(pts);
    pts[D] = q;
    const int q_sign = orient(pts);
    if (q_sign == 0) {
      for (int f = 0; f < D; ++f)
        if (s.v[f] < qid) return true;
      return false;
    }
    return q_sign == -inner_sign;
  }

  bool conflict(std::uint32_t id, const double* q, std::uint32_t qid) const {
    const Cell<D>& s = cells_[id];
    if (s.v[D] == kInf) return infinite_conflict(s, q, qid);
    const double* p[D + 1];
    for (int i = 0; i <= D; ++i) p[i] = P(s.v[i]);
    if (s.parity < 0) std::swap(p[0], p[1]);
    const int r = in_sphere(p, q);
    if (r != 0) return r > 0;
    for (int i = 0; i <= D; ++i)
      if (s.v[i] < qid) return true;
    return false;
  }

  std::uint32_t random_alive() {
    for (int t = 0; t < 64; ++t) {
      const std::uint32_t id = static_cast<std::uint32_t>(uniform_index(rng_, cells_.size()));
      if (cells_[id].alive) return id;
    }
    for (std::uint32_t id = 0; id < cells_.size(); ++id)
      if (cells_[id].alive) return id;
    return kNone;
  }

  std::uint32_t locate(const double* q, std::uint32_t qid) {
    std::uint32_t cur = (hint_ < cells_.size() && cells_[hint_].alive) ? hint_ : random_alive();
    std::uint32_t prev = kNone;
    std::size_t steps = 0;
    const std::size_t budget = 4 * (cells_.size() - free_.size()) + 16;
    for (;;) {
      if (steps++ > budget) {
        cur = random_alive();
        prev = kNone;
        steps = 0;
      }
      const Cell<D>& s = cells_[cur];
      if (s.v[D] == kInf) {
        if (infinite_conflict(s, q, qid)) return cur;
        prev = cur;
        cur = s.n[D];
        continue;
      }
      const double* c[D + 1];
      for (int i = 0; i <= D; ++i) c[i] = P(s.v[i]);
      const unsigned rot = static_cast<unsigned>(rng_() % (D + 1));
      int exit_facet = -1;
      for (int k = 0; k <= D; ++k) {
        const int d = static_cast<int>((k + rot) % (D + 1));
        if (prev != kNone && s.n[d] == prev) continue;
        const double* saved = c[d];
        c[d] = q;
        const int o = orient(c);
        c[d] = saved;
        if (o != 0 && o != s.parity) {
          exit_facet = d;
          break;
        }
      }
      if (exit_facet < 0) return cur;
      prev = cur;
      cur = s.n[exit_facet];
    }
  }

  struct Boundary {
    std::uint32_t outside;
    int outside_slot;  // index in outside.n pointing back into the cavity
    std::uint32_t verts[D];
  };
  struct Ridge {
    std::uint64_t key;
    std::uint32_t simplex;
    int slot;
    bool operator<(const Ridge& o) const {
      return key < o.key || (key == o.key && simplex < o.simplex);
    }
  };

  void insert(std::uint32_t qid) {
    const double* q = P(qid);
    const std::uint32_t seed = locate(q, qid);
    if (stamp_.size() < cells_.size()) stamp_.resize(cells_.size() + cells_.size() / 2 + 16, 0);
    epoch_ += 2;
    if (epoch_ == 0 || epoch_ == 1) {
      std::fill(stamp_.begin(), stamp_.end(), 0);
      epoch_ = 2;
    }
    cavity_.clear();
    boundary_.clear();
    bfs_.clear();
    bfs_.push_back(seed);
    stamp_[seed] = epoch_ | 1;
    while (!bfs_.empty()) {
      const std::uint32_t id = bfs_.back();
      bfs_.pop_back();
      cavity_.push_back(id);
      const Cell<D>& s = cells_[id];
      for (int d = 0; d <= D; ++d) {
        const std::uint32_t nb = s.n[d];
        bool in_cavity;
        if (stamp_[nb] >= epoch_) {
          in_cavity = (stamp_[nb] & 1u) != 0;
        } else {
          in_cavity = conflict(nb, q, qid);
          stamp_[nb] = epoch_ | (in_cavity ? 1u : 0u);
          if (in_cavity) bfs_.push_back(nb);
        }
        if (!in_cavity) {
          Boundary bf;
          bf.outside = nb;
          bf.outside_slot = -1;
          const Cell<D>& o = cells_[nb];
          for (int j = 0; j <= D; ++j)
            if (o.n[j] == id) {
              bf.outside_slot = j;
              break;
            }
          int idx = 0;
          for (int i = 0; i <= D; ++i)
            if (i != d) bf.verts[idx++] = s.v[i];
          boundary_.push_back(bf);
        }
      }
    }
    for (std::uint32_t id : cavity_) {
      cells_[id].alive = 0;
      free_.push_back(id);
    }
    ridges_.clear();
    for (const Boundary& bf : boundary_) {
      Cell<D> ns;
      int idx = 0, q_slot = -1;
      for (int i = 0; i < D; ++i) {
        if (q_slot < 0 && qid < bf.verts[i]) {
          q_slot = idx;
          ns.v[idx++] = qid;
        }
        ns.v[idx++] = bf.verts[i];
      }
      if (q_slot < 0) {
        q_slot = idx;
        ns.v[idx++] = qid;
      }
      for (int i = 0; i <= D; ++i) ns.n[i] = kNone;
      ns.n[q_slot] = bf.outside;
      if (ns.v[D] == kInf) {
        ns.parity = 0;
      } else {
        ns.parity = static_cast<std::int8_t>(parity_of(ns.v));
        if (ns.parity == 0) throw DegenerateInputError("affinely dependent points beyond the tie-break's scope");
      }
      const std::uint32_t nid = create(ns);
      cells_[bf.outside].n[bf.outside_slot] = nid;
      for (int d = 0; d <= D; ++d) {
        if (ns.v[d] == qid) continue;
        // ridge = all vertices except v[d] and q
        std::uint64_t key = 0;
        for (int i = 0; i <= D; ++i) {
          if (i == d || ns.v[i] == qid) continue;
          key = (key << 32) | ns.v[i];
        }
        ridges_.push_back(Ridge{key, nid, d});
      }
      hint_ = nid;
    }
    std::sort(ridges_.begin(), ridges_.end());
    for (std::size_t i = 0; i + 1 < ridges_.size(); i += 2) {
      const Ridge& a = ridges_[i];
      const Ridge& b = ridges_[i + 1];
      if (a.key != b.key) throw DegenerateInputError("unpaired cavity ridge");
      cells_[a.simplex].n[a.slot] = b.simplex;
      cells_[b.simplex].n[b.slot] = a.simplex;
    }
    // prefer a finite hint
    if (cells_[hint_].v[D] == kInf) hint_ = cells_[hint_].n[D];
  }

  TriSoA compact() {
    std::vector<std::uint32_t> remap(cells_.size(), kNone);
    std::size_t cnt = 0;
    for (std::size_t i = 0; i < cells_.size(); ++i)
      if (cells_[i].alive) remap[i] = static_cast<std::uint32_t>(cnt++);
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

  const double* xyz_;
  Rng rng_;
  std::vector<std::uint32_t> order_;
  std::vector<Cell<D>> cells_;
  std::vector<std::uint32_t> free_;
  std::vector<std::uint32_t> stamp_;
  std::uint32_t epoch_ = 0;
  std::uint32_t hint_ = 0;
  std::vector<std::uint32_t> cavity_, bfs_;
  std::vector<Boundary> boundary_;
  std::vector<Ridge> ridges_;
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
