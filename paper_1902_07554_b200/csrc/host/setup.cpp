#include "setup.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <thread>

#include "rng.hpp"

namespace sbdt_host {

// ---------------------------------------------------------------------------
// Workload generators (BASELINE.json configs 1-5)
// ---------------------------------------------------------------------------
std::vector<double> generate(Distribution kind, int dim, std::size_t n, std::uint64_t seed,
                             const double* params, int nparams) {
  auto param = [&](int i, double dflt) { return (params && i < nparams) ? params[i] : dflt; };
  std::vector<double> out(n * dim);
  Rng rng(derive_seed(seed, kTagPoints));
  switch (kind) {
    case Distribution::kUniform:
      for (std::size_t i = 0; i < n * dim; ++i) out[i] = uniform01(rng);
      break;
    case Distribution::kNormal: {
      const double mean = param(0, 0.5), sigma = param(1, 0.1);
      NormalStream ns(rng);
      for (std::size_t i = 0; i < n * dim; ++i) out[i] = mean + sigma * ns.next();
      break;
    }
    case Distribution::kBubbles: {
      if (dim != 3) throw std::invalid_argument("bubbles is a 3D distribution");
      const int count = static_cast<int>(param(0, 64));
      const double rmin = param(1, 0.02), rmax = param(2, 0.1), jitter = param(3, 0.002);
      std::vector<double> centers(count * 3), radii(count);
      for (int b = 0; b < count; ++b) {
        for (int d = 0; d < 3; ++d) centers[b * 3 + d] = uniform01(rng);
        radii[b] = rmin + (rmax - rmin) * uniform01(rng);
      }
      NormalStream ns(rng);
      for (std::size_t i = 0; i < n; ++i) {
        const int b = static_cast<int>(i % count);
        double g[3];
        double norm;
        do {
          for (double& v : g) v = ns.next();
          norm = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
        } while (norm == 0.0);
        const double r = radii[b] + jitter * ns.next();
        for (int d = 0; d < 3; ++d) out[i * 3 + d] = centers[b * 3 + d] + r * g[d] / norm;
      }
      break;
    }
    case Distribution::kLines: {
      if (dim != 2) throw std::invalid_argument("lines is a 2D distribution");
      const int count = static_cast<int>(param(0, 1000));
      const double jitter = param(1, 1e-4);
      std::vector<double> seg(count * 4);
      for (double& v : seg) v = uniform01(rng);
      NormalStream ns(rng);
      for (std::size_t i = 0; i < n; ++i) {
        const std::size_t s = uniform_index(rng, count);
        const double t = uniform01(rng);
        const double ax = seg[s * 4], ay = seg[s * 4 + 1], bx = seg[s * 4 + 2], by = seg[s * 4 + 3];
        const double dx = bx - ax, dy = by - ay;
        const double len = std::sqrt(dx * dx + dy * dy);
        const double nx = len > 0 ? -dy / len : 0.0, ny = len > 0 ? dx / len : 1.0;
        const double off = jitter * ns.next();
        out[i * 2] = ax + t * dx + off * nx;
        out[i * 2 + 1] = ay + t * dy + off * ny;
      }
      break;
    }
  }
  return out;
}

std::vector<std::uint32_t> deduplicate(int dim, std::vector<double>& coords) {
  const std::size_t n = coords.size() / dim;
  std::vector<std::uint32_t> remap(n);
  std::size_t cap = 16;
  while (cap < 2 * n) cap <<= 1;
  std::vector<std::uint32_t> table(cap, 0xFFFFFFFFu);
  std::size_t next = 0;
  for (std::size_t i = 0; i < n; ++i) {
    const double* p = coords.data() + i * dim;
    std::uint64_t h = 0x9e3779b97f4a7c15ULL;
    for (int d = 0; d < dim; ++d) {
      std::uint64_t bits;
      std::memcpy(&bits, &p[d], 8);
      h = mix64(h ^ bits);
    }
    std::size_t slot = h & (cap - 1);
    std::uint32_t found = 0xFFFFFFFFu;
    while (table[slot] != 0xFFFFFFFFu) {
      const double* o = coords.data() + std::size_t(table[slot]) * dim;
      if (std::equal(p, p + dim, o)) {
        found = table[slot];
        break;
      }
      slot = (slot + 1) & (cap - 1);
    }
    if (found != 0xFFFFFFFFu) {
      remap[i] = found;
    } else {
      if (next != i) std::memmove(coords.data() + next * dim, p, sizeof(double) * dim);
      table[slot] = static_cast<std::uint32_t>(next);
      remap[i] = static_cast<std::uint32_t>(next);
      ++next;
    }
  }
  coords.resize(next * dim);
  return remap;
}

std::vector<std::uint32_t> draw_sample(std::size_t n, std::size_t m, std::uint64_t seed) {
  if (m > n) throw std::invalid_argument("sample larger than input");
  Rng rng(derive_seed(seed, kTagSample));
  std::vector<std::uint32_t> ids(n);
  std::iota(ids.begin(), ids.end(), 0u);
  for (std::size_t i = 0; i < m; ++i) {
    const std::size_t j = i + uniform_index(rng, n - i);
    std::swap(ids[i], ids[j]);
  }
  ids.resize(m);
  return ids;
}

// ---------------------------------------------------------------------------
// Sample graph: one edge per distinct finite DT edge,
// real weight per the weight table, mapped affinely to integers in [1,1000].
// ---------------------------------------------------------------------------
SampleGraph build_sample_graph(int dim, const double* coords, const std::uint32_t* sample_ids,
                               std::size_t m, const TriSoA& dt, WeightFn fn) {
  // DT vertices are global ids; map them to sample-local indices.
  std::vector<std::pair<std::uint32_t, std::uint32_t>> gid_to_local(m);
  for (std::size_t i = 0; i < m; ++i) gid_to_local[i] = {sample_ids[i], static_cast<std::uint32_t>(i)};
  std::sort(gid_to_local.begin(), gid_to_local.end());
  auto local = [&](std::uint32_t g) {
    auto it = std::lower_bound(gid_to_local.begin(), gid_to_local.end(),
                               std::make_pair(g, 0u));
    return it->second;
  };
  std::vector<std::uint64_t> edges;
  const std::size_t S = dt.count;
  edges.reserve(S * (dim == 2 ? 3 : 6));
  for (std::size_t s = 0; s < S; ++s) {
    if (dt.verts[dim * S + s] == kInf) continue;
    std::uint32_t v[4];
    for (int j = 0; j <= dim; ++j) v[j] = local(dt.verts[j * S + s]);
    for (int a = 0; a <= dim; ++a)
      for (int b = a + 1; b <= dim; ++b) {
        const std::uint32_t x = std::min(v[a], v[b]), y = std::max(v[a], v[b]);
        edges.push_back((std::uint64_t(x) << 32) | y);
      }
  }
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());

  // d_star = maximum diagonal of the sample bounding box.
  std::vector<double> lo(dim, INFINITY), hi(dim, -INFINITY);
  for (std::size_t i = 0; i < m; ++i)
    for (int d = 0; d < dim; ++d) {
      const double c = coords[std::size_t(sample_ids[i]) * dim + d];
      lo[d] = std::min(lo[d], c);
      hi[d] = std::max(hi[d], c);
    }
  double dstar2 = 0;
  for (int d = 0; d < dim; ++d) dstar2 += (hi[d] - lo[d]) * (hi[d] - lo[d]);
  const double dstar = std::sqrt(dstar2);
  std::vector<double> r(edges.size());
  double rmin = INFINITY, rmax = -INFINITY;
  for (std::size_t e = 0; e < edges.size(); ++e) {
    const std::uint32_t a = edges[e] >> 32, b = edges[e] & 0xFFFFFFFFu;
    double s2 = 0;
    for (int d = 0; d < dim; ++d) {
      const double t = coords[std::size_t(sample_ids[a]) * dim + d] -
                       coords[std::size_t(sample_ids[b]) * dim + d];
      s2 += t * t;
    }
    double dn = std::sqrt(s2) / dstar;
    dn = std::min(1.0, std::max(1e-12, dn));
    double val = 1.0;
    switch (fn) {
      case WeightFn::kConstant: val = 1.0; break;
      case WeightFn::kInverse: val = 1.0 / dn; break;
      case WeightFn::kLogarithmic: val = -std::log(dn); break;
      case WeightFn::kLinear: val = 1.0 - dn; break;
    }
    r[e] = val;
    rmin = std::min(rmin, val);
    rmax = std::max(rmax, val);
  }
  SampleGraph g;
  g.n = m;
  std::vector<std::uint32_t> deg(m, 0);
  for (std::uint64_t e : edges) {
    ++deg[e >> 32];
    ++deg[e & 0xFFFFFFFFu];
  }
  g.xadj.assign(m + 1, 0);
  for (std::size_t i = 0; i < m; ++i) g.xadj[i + 1] = g.xadj[i] + deg[i];
  g.adj.resize(g.xadj[m]);
  g.w.resize(g.xadj[m]);
  std::vector<std::uint32_t> pos(g.xadj.begin(), g.xadj.end() - 1);
  for (std::size_t e = 0; e < edges.size(); ++e) {
    const std::uint32_t a = edges[e] >> 32, b = edges[e] & 0xFFFFFFFFu;
    std::int32_t w = 1;
    if (rmax > rmin) w = static_cast<std::int32_t>(std::lround(1.0 + 999.0 * (r[e] - rmin) / (rmax - rmin)));
    g.adj[pos[a]] = b;
    g.w[pos[a]++] = w;
    g.adj[pos[b]] = a;
    g.w[pos[b]++] = w;
  }
  return g;
}

std::uint64_t cut_weight(const SampleGraph& g, const std::vector<std::uint32_t>& labels) {
  std::uint64_t c = 0;
  for (std::size_t v = 0; v < g.n; ++v)
    for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e)
      if (g.adj[e] > v && labels[g.adj[e]] != labels[v]) c += g.w[e];
  return c;
}

// ---------------------------------------------------------------------------
// Multilevel recursive bisection (SPEC.md:257-266 algorithm contract):
// heavy-edge matching coarsening to <= 200 vertices, greedy graph growing
// initial bisection, boundary FM refinement on every level.
// ---------------------------------------------------------------------------
namespace {

struct WGraph {
  std::vector<std::uint32_t> xadj, adj;
  std::vector<std::int64_t> w;   // edge weights
  std::vector<std::int64_t> vw;  // vertex weights
  std::size_t n() const { return vw.size(); }
};

WGraph coarsen(const WGraph& g, Rng& rng, std::vector<std::uint32_t>& cmap, std::int64_t maxvw) {
  const std::size_t n = g.n();
  std::vector<std::uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  for (std::size_t i = n; i > 1; --i) std::swap(order[i - 1], order[uniform_index(rng, i)]);
  std::vector<std::uint32_t> match(n, 0xFFFFFFFFu);
  for (std::uint32_t v : order) {
    if (match[v] != 0xFFFFFFFFu) continue;
    std::uint32_t best = v;
    std::int64_t bw = -1;
    for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) {
      const std::uint32_t u = g.adj[e];
      if (match[u] != 0xFFFFFFFFu || u == v) continue;
      if (g.vw[u] + g.vw[v] > maxvw) continue;
      if (g.w[e] > bw) {
        bw = g.w[e];
        best = u;
      }
    }
    match[v] = best;
    match[best] = v;
  }
  cmap.assign(n, 0xFFFFFFFFu);
  std::uint32_t nc = 0;
  for (std::uint32_t v = 0; v < n; ++v) {
    if (cmap[v] != 0xFFFFFFFFu) continue;
    cmap[v] = nc;
    cmap[match[v]] = nc;
    ++nc;
  }
  WGraph c;
  c.vw.assign(nc, 0);
  for (std::uint32_t v = 0; v < n; ++v) c.vw[cmap[v]] += g.vw[v];
  // members of each coarse vertex
  std::vector<std::uint32_t> first(nc, 0xFFFFFFFFu), second(nc, 0xFFFFFFFFu);
  for (std::uint32_t v = 0; v < n; ++v) {
    const std::uint32_t cv = cmap[v];
    if (first[cv] == 0xFFFFFFFFu) first[cv] = v;
    else second[cv] = v;
  }
  std::vector<std::int64_t> acc(nc, 0);
  std::vector<std::uint32_t> touched;
  c.xadj.assign(nc + 1, 0);
  for (std::uint32_t cv = 0; cv < nc; ++cv) {
    touched.clear();
    for (std::uint32_t mem : {first[cv], second[cv]}) {
      if (mem == 0xFFFFFFFFu) continue;
      for (std::uint32_t e = g.xadj[mem]; e < g.xadj[mem + 1]; ++e) {
        const std::uint32_t cu = cmap[g.adj[e]];
        if (cu == cv) continue;
        if (acc[cu] == 0) touched.push_back(cu);
        acc[cu] += g.w[e];
      }
    }
    std::sort(touched.begin(), touched.end());
    for (std::uint32_t cu : touched) {
      c.adj.push_back(cu);
      c.w.push_back(acc[cu]);
      acc[cu] = 0;
    }
    c.xadj[cv + 1] = static_cast<std::uint32_t>(c.adj.size());
  }
  return c;
}

// Boundary FM refinement for a bisection. side[v] in {0,1}.
void fm_refine(const WGraph& g, std::vector<std::uint8_t>& side, std::int64_t max0, std::int64_t max1,
               int passes) {
  const std::size_t n = g.n();
  std::vector<std::int64_t> gain(n);
  std::vector<std::uint8_t> locked(n);
  std::vector<std::uint32_t> moved;
  for (int pass = 0; pass < passes; ++pass) {
    std::int64_t wpart[2] = {0, 0};
    for (std::size_t v = 0; v < n; ++v) wpart[side[v]] += g.vw[v];
    auto compute_gain = [&](std::uint32_t v) {
      std::int64_t ext = 0, in = 0;
      for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e)
        (side[g.adj[e]] == side[v] ? in : ext) += g.w[e];
      return ext - in;
    };
    using Item = std::pair<std::int64_t, std::uint32_t>;
    std::priority_queue<Item> pq[2];
    for (std::uint32_t v = 0; v < n; ++v) {
      gain[v] = compute_gain(v);
      locked[v] = 0;
      bool boundary = false;
      for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e)
        if (side[g.adj[e]] != side[v]) boundary = true;
      if (boundary) pq[side[v]].push({gain[v], v});
    }
    moved.clear();
    std::int64_t cur = 0, best = 0;
    std::size_t best_len = 0;
    const std::int64_t maxw[2] = {max0, max1};
    int since_best = 0;
    while (since_best < 200) {
      // choose the side whose top move is feasible with the larger gain
      int pick = -1;
      std::int64_t pg = 0;
      for (int s = 0; s < 2; ++s) {
        while (!pq[s].empty()) {
          const auto [gv, v] = pq[s].top();
          if (locked[v] || side[v] != s || gv != gain[v]) {
            pq[s].pop();
            continue;
          }
          break;
        }
        if (pq[s].empty()) continue;
        const auto [gv, v] = pq[s].top();
        if (wpart[1 - s] + g.vw[v] > maxw[1 - s]) continue;
        if (pick < 0 || gv > pg) {
          pick = s;
          pg = gv;
        }
      }
      if (pick < 0) break;
      const std::uint32_t v = pq[pick].top().second;
      pq[pick].pop();
      locked[v] = 1;
      side[v] = static_cast<std::uint8_t>(1 - pick);
      wpart[pick] -= g.vw[v];
      wpart[1 - pick] += g.vw[v];
      cur += gain[v];
      moved.push_back(v);
      for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) {
        const std::uint32_t u = g.adj[e];
        if (locked[u]) continue;
        gain[u] += (side[u] == side[v]) ? -2 * g.w[e] : 2 * g.w[e];
        pq[side[u]].push({gain[u], u});
      }
      if (cur > best) {
        best = cur;
        best_len = moved.size();
        since_best = 0;
      } else {
        ++since_best;
      }
    }
    for (std::size_t i = moved.size(); i > best_len; --i) side[moved[i - 1]] ^= 1;
    if (best <= 0) break;
  }
}

std::int64_t bisect_cut(const WGraph& g, const std::vector<std::uint8_t>& side) {
  std::int64_t c = 0;
  for (std::uint32_t v = 0; v < g.n(); ++v)
    for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e)
      if (g.adj[e] > v && side[g.adj[e]] != side[v]) c += g.w[e];
  return c;
}

// Greedy graph growing from a seed until part 0 reaches target0.
std::vector<std::uint8_t> grow(const WGraph& g, std::uint32_t seed, std::int64_t target0) {
  const std::size_t n = g.n();
  std::vector<std::uint8_t> side(n, 1);
  std::vector<std::int64_t> conn(n, 0);
  using Item = std::pair<std::int64_t, std::uint32_t>;
  std::priority_queue<Item> pq;
  std::int64_t w0 = 0;
  std::uint32_t next_unvisited = 0;
  pq.push({0, seed});
  while (w0 < target0) {
    std::uint32_t v = 0xFFFFFFFFu;
    while (!pq.empty()) {
      const auto [c, u] = pq.top();
      pq.pop();
      if (side[u] == 0 || c != conn[u]) continue;
      v = u;
      break;
    }
    if (v == 0xFFFFFFFFu) {  // disconnected: take any remaining vertex
      while (next_unvisited < n && side[next_unvisited] == 0) ++next_unvisited;
      if (next_unvisited >= n) break;
      v = next_unvisited;
    }
    side[v] = 0;
    w0 += g.vw[v];
    for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) {
      const std::uint32_t u = g.adj[e];
      if (side[u] == 0) continue;
      conn[u] += g.w[e];
      pq.push({conn[u], u});
    }
  }
  return side;
}

std::vector<std::uint8_t> multilevel_bisect(const WGraph& g0, std::int64_t target0, std::int64_t max0,
                                            std::int64_t max1, Rng& rng) {
  std::vector<WGraph> levels;
  std::vector<std::vector<std::uint32_t>> maps;
  levels.push_back(g0);
  std::int64_t total = 0;
  for (auto w : g0.vw) total += w;
  while (levels.back().n() > 200) {
    std::vector<std::uint32_t> cmap;
    const std::int64_t maxvw = std::max<std::int64_t>(1, total / 100);
    WGraph c = coarsen(levels.back(), rng, cmap, maxvw);
    if (c.n() > levels.back().n() * 0.95) break;
    maps.push_back(std::move(cmap));
    levels.push_back(std::move(c));
  }
  const WGraph& cg = levels.back();
  std::vector<std::uint8_t> best;
  std::int64_t best_cut = -1;
  const int tries = 8;
  for (int t = 0; t < tries; ++t) {
    const std::uint32_t seed = static_cast<std::uint32_t>(uniform_index(rng, cg.n()));
    auto side = grow(cg, seed, target0);
    fm_refine(cg, side, max0, max1, 4);
    std::int64_t w0 = 0, w1 = 0;
    for (std::uint32_t v = 0; v < cg.n(); ++v) (side[v] ? w1 : w0) += cg.vw[v];
    const bool feasible = w0 <= max0 && w1 <= max1;
    const std::int64_t cut = bisect_cut(cg, side) + (feasible ? 0 : (std::int64_t(1) << 50));
    if (best_cut < 0 || cut < best_cut) {
      best_cut = cut;
      best = side;
    }
  }
  for (std::size_t l = levels.size() - 1; l > 0; --l) {
    const auto& cmap = maps[l - 1];
    std::vector<std::uint8_t> fine(levels[l - 1].n());
    for (std::size_t v = 0; v < fine.size(); ++v) fine[v] = best[cmap[v]];
    best = std::move(fine);
    fm_refine(levels[l - 1], best, max0, max1, 3);
  }
  return best;
}

WGraph subgraph(const WGraph& g, const std::vector<std::uint32_t>& verts,
                std::vector<std::uint32_t>& local_of) {
  WGraph s;
  s.vw.resize(verts.size());
  for (std::size_t i = 0; i < verts.size(); ++i) local_of[verts[i]] = static_cast<std::uint32_t>(i);
  s.xadj.assign(verts.size() + 1, 0);
  for (std::size_t i = 0; i < verts.size(); ++i) {
    const std::uint32_t v = verts[i];
    s.vw[i] = g.vw[v];
    for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) {
      const std::uint32_t lu = local_of[g.adj[e]];
      if (lu == 0xFFFFFFFFu) continue;
      s.adj.push_back(lu);
      s.w.push_back(g.w[e]);
    }
    s.xadj[i + 1] = static_cast<std::uint32_t>(s.adj.size());
  }
  for (std::uint32_t v : verts) local_of[v] = 0xFFFFFFFFu;
  return s;
}

void recurse(const WGraph& g, const std::vector<std::uint32_t>& verts, std::uint32_t k,
             std::uint32_t label0, double eps_level, Rng& rng, std::vector<std::uint32_t>& labels,
             std::vector<std::uint32_t>& scratch_local) {
  if (k == 1) {
    for (std::uint32_t v : verts) labels[v] = label0;
    return;
  }
  WGraph s = subgraph(g, verts, scratch_local);
  std::int64_t total = 0;
  for (auto w : s.vw) total += w;
  const std::uint32_t k0 = k / 2, k1 = k - k0;
  const std::int64_t target0 = static_cast<std::int64_t>(std::llround(double(total) * k0 / k));
  const std::int64_t max0 = static_cast<std::int64_t>(std::floor(double(total) * k0 / k * (1.0 + eps_level)));
  const std::int64_t max1 = static_cast<std::int64_t>(std::floor(double(total) * k1 / k * (1.0 + eps_level)));
  auto side = multilevel_bisect(s, target0, std::max<std::int64_t>(max0, target0),
                                std::max<std::int64_t>(max1, total - target0), rng);
  std::vector<std::uint32_t> a, b;
  for (std::size_t i = 0; i < verts.size(); ++i) (side[i] ? b : a).push_back(verts[i]);
  recurse(g, a, k0, label0, eps_level, rng, labels, scratch_local);
  recurse(g, b, k1, label0 + k0, eps_level, rng, labels, scratch_local);
}

// Final k-way balance repair so |V_i| <= (1+eps) ceil(|V|/k) holds exactly.
void rebalance(const WGraph& g, std::uint32_t k, double eps, std::vector<std::uint32_t>& labels) {
  const std::size_t n = g.n();
  const std::int64_t cap = static_cast<std::int64_t>(std::floor((1.0 + eps) * double((n + k - 1) / k)));
  std::vector<std::int64_t> size(k, 0);
  for (std::size_t v = 0; v < n; ++v) size[labels[v]] += g.vw[v];
  for (int round = 0; round < 64; ++round) {
    bool any = false;
    for (std::uint32_t v = 0; v < n; ++v) {
      const std::uint32_t p = labels[v];
      if (size[p] <= cap) continue;
      std::uint32_t best = p;
      std::int64_t best_conn = -1;
      for (std::uint32_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) {
        const std::uint32_t q = labels[g.adj[e]];
        if (q == p || size[q] + g.vw[v] > cap) continue;
        if (g.w[e] > best_conn) {
          best_conn = g.w[e];
          best = q;
        }
      }
      if (best != p) {
        labels[v] = best;
        size[p] -= g.vw[v];
        size[best] += g.vw[v];
        any = true;
      }
    }
    if (!any) break;
  }
}

}  // namespace

std::vector<std::uint32_t> partition_graph(const SampleGraph& sg, std::uint32_t k, double eps,
                                           std::uint64_t seed) {
  if (k == 0) throw std::invalid_argument("k must be >= 1");
  if (sg.n < k) throw std::invalid_argument("InfeasibleBalance: |V| < k");
  std::vector<std::uint32_t> labels(sg.n, 0);
  if (k == 1) return labels;
  WGraph g;
  g.xadj = sg.xadj;
  g.adj = sg.adj;
  g.w.assign(sg.w.begin(), sg.w.end());
  g.vw.assign(sg.n, 1);
  Rng rng(derive_seed(seed, kTagPartitioner));
  int levels = 0;
  while ((1u << levels) < k) ++levels;
  const double eps_level = eps / levels;
  std::vector<std::uint32_t> all(sg.n);
  std::iota(all.begin(), all.end(), 0u);
  std::vector<std::uint32_t> scratch(sg.n, 0xFFFFFFFFu);
  recurse(g, all, k, 0, eps_level, rng, labels, scratch);
  rebalance(g, k, eps, labels);
  return labels;
}

// ---------------------------------------------------------------------------
// Partial DTs (Alg. 1 "parallel triangulation"), one task per part.
// ---------------------------------------------------------------------------
Partials build_partials(int dim, const double* coords, std::size_t n, const std::uint32_t* labels,
                        std::uint32_t k, std::uint64_t seed, unsigned threads) {
  std::vector<std::vector<std::uint32_t>> parts(k);
  for (std::size_t i = 0; i < n; ++i) {
    if (labels[i] >= k) throw std::invalid_argument("label " + std::to_string(labels[i]) + " >= k");
    parts[labels[i]].push_back(static_cast<std::uint32_t>(i));
  }
  std::vector<TriSoA> tris(k);
  std::atomic<std::uint32_t> next{0};
  std::vector<std::string> errors(k);
  auto worker = [&]() {
    for (;;) {
      const std::uint32_t p = next.fetch_add(1);
      if (p >= k) return;
      try {
        tris[p] = triangulate(dim, coords, parts[p].data(), parts[p].size(),
                              derive_seed(seed, kTagPartialDt + p));
      } catch (const std::exception& e) {
        errors[p] = e.what();
      }
    }
  };
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = std::min<unsigned>(threads, k);
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  for (std::uint32_t p = 0; p < k; ++p)
    if (!errors[p].empty()) throw DegenerateInputError("part " + std::to_string(p) + ": " + errors[p]);
  Partials out;
  out.dim = dim;
  out.k = k;
  out.offsets.assign(k + 1, 0);
  for (std::uint32_t p = 0; p < k; ++p) out.offsets[p + 1] = out.offsets[p] + tris[p].count;
  const std::size_t S = out.total();
  out.verts.resize((dim + 1) * S);
  out.nbrs.resize((dim + 1) * S);
  out.parity.resize(S);
  for (std::uint32_t p = 0; p < k; ++p) {
    const std::size_t off = out.offsets[p], c = tris[p].count;
    for (int j = 0; j <= dim; ++j) {
      std::memcpy(out.verts.data() + j * S + off, tris[p].verts.data() + j * c, c * 4);
      std::memcpy(out.nbrs.data() + j * S + off, tris[p].nbrs.data() + j * c, c * 4);
    }
    std::memcpy(out.parity.data() + off, tris[p].parity.data(), c);
    tris[p] = TriSoA();
  }
  return out;
}

}  // namespace sbdt_host
