// TEST INFRASTRUCTURE — CPU restatement of dc-engine `merge` and
// `update_neighbors` (Alg. 1 merging and
// neighbourhood blocks), the checker for the GPU merge (merge.cu). Never on
// the product path.
//
// Restated as the SPEC states it, on a slot array in the manner of the
// reference's Triangulation<D> (triangulation.hpp:162-247):
//   1. every partial simplex becomes a slot (part-local neighbour ids turned
//      into slot ids); border simplices and infinite simplices are killed
//      (tombstones, ids stay stable: append_slot, triangulation.hpp:190-195;
//      "Infinite simplices are always stripped at merge");
//   2. the finite simplices of T_B are scanned in row order; s_b is appended
//      if its vertices span >= 2 partitions, or if a border simplex with the
//      identical vertex tuple existed (tuple set built once);
//      appended slots start with absent links and go to the repair queue Q;
//      inserting a tuple that is already alive is InconsistentMerge;
//   3. update_neighbors: a FacetIndex (key = facet_key of the D facet ids,
//      triangulation.hpp:73-94; entries sorted by key, candidates verified by
//      vertex sharing, triangulation.hpp:96-146) over every live slot; each
//      queued slot scans the candidates of its facets whose neighbour is dead
//      or absent; the candidate sharing exactly D vertices becomes the
//      neighbour on both sides and is itself queued (each slot claimed once);
//   4. the merged hull is re-derived from the facets with a single finite
//      owner: after compaction (triangulation.hpp:224), one
//      infinite simplex per hull facet, in (owner row, facet) order, linked
//      to its owner and, through the shared ridges, to each other.
// Output order (compaction of the slot array): kept partial rows in row order,
// then the inserted T_B rows in T_B row order, then the hull rows.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <deque>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace sbdt_oracle {

constexpr std::uint32_t kMergeNone = 0xFFFFFFFFu;
constexpr std::uint32_t kMergeInf = 0xFFFFFFFFu;

// splitmix64 finalizer (common.hpp:69-74) and the order-independent facet key
// (triangulation.hpp:68-94), restated.
inline std::uint64_t merge_mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

template <int D>
std::uint64_t merge_facet_key(const std::array<std::uint32_t, D + 1>& v, int opposite) {
  std::uint64_t sum = 0, xr = 0;
  for (int i = 0; i <= D; ++i) {
    if (i == opposite) continue;
    const std::uint64_t m = merge_mix64(v[i]);
    sum += m;
    xr ^= m;
  }
  return sum ^ (xr << 32 | xr >> 32);
}

struct MergeOut {
  std::vector<std::uint32_t> verts, nbrs;  // vertex-major, stride = rows
  std::vector<std::int8_t> parity;
  std::vector<std::uint64_t> offsets;      // k+3
  std::uint64_t rows = 0;
  std::string error;                       // "" = ok
};

template <int D>
MergeOut merge_oracle(std::uint32_t k, const std::uint64_t* offsets, const std::uint32_t* verts,
                      const std::uint32_t* nbrs, const std::int8_t* parity, const std::uint8_t* border,
                      const std::uint32_t* tb_verts, const std::uint32_t* tb_nbrs, const std::int8_t* tb_parity,
                      std::uint64_t SB, const std::uint32_t* labels, bool hull) {
  using Tup = std::array<std::uint32_t, D + 1>;
  struct Slot {
    Tup v, nb;
    std::int8_t par;
    bool alive;
  };
  MergeOut out;
  const std::uint64_t S = offsets[k];
  std::vector<Slot> slots(S);
  std::set<Tup> border_tuples, alive_tuples;
  // 1. partial simplices -> slots; strip border and infinite simplices
  for (std::uint32_t p = 0; p < k; ++p) {
    for (std::uint64_t s = offsets[p]; s < offsets[p + 1]; ++s) {
      Slot& sl = slots[s];
      for (int j = 0; j <= D; ++j) {
        sl.v[j] = verts[std::uint64_t(j) * S + s];
        const std::uint32_t nb = nbrs[std::uint64_t(j) * S + s];
        sl.nb[j] = nb == kMergeNone ? kMergeNone : static_cast<std::uint32_t>(offsets[p] + nb);
      }
      sl.par = parity[s];
      const bool finite = sl.v[D] != kMergeInf;
      sl.alive = finite && !border[s];
      if (finite && border[s]) border_tuples.insert(sl.v);
      if (sl.alive) alive_tuples.insert(sl.v);
    }
  }
  // 2. T_B insertion scan
  std::vector<std::uint32_t> Q;
  for (std::uint64_t t = 0; t < SB; ++t) {
    Tup v;
    for (int j = 0; j <= D; ++j) v[j] = tb_verts[std::uint64_t(j) * SB + t];
    if (v[D] == kMergeInf) continue;
    bool spans = false;
    for (int j = 1; j <= D; ++j) spans |= labels[v[j]] != labels[v[0]];
    if (!spans && !border_tuples.count(v)) continue;
    if (!alive_tuples.insert(v).second) {
      out.error = "InconsistentMerge: simplex inserted twice";
      return out;
    }
    Slot sl;
    sl.v = v;
    sl.nb.fill(kMergeNone);
    sl.par = tb_parity[t];
    sl.alive = true;
    Q.push_back(static_cast<std::uint32_t>(slots.size()));
    slots.push_back(sl);
  }
  const std::uint64_t n_inserted = Q.size();
  // 3. update_neighbors over a frozen facet index of the live slots
  std::vector<std::pair<std::uint64_t, std::uint32_t>> index;
  for (std::uint32_t s = 0; s < slots.size(); ++s)
    if (slots[s].alive)
      for (int d = 0; d <= D; ++d) index.emplace_back(merge_facet_key<D>(slots[s].v, d), s);
  std::sort(index.begin(), index.end());
  auto dead = [&](std::uint32_t nb) { return nb == kMergeNone || !slots[nb].alive; };
  std::vector<std::uint8_t> claimed(slots.size(), 0);
  std::deque<std::uint32_t> queue(Q.begin(), Q.end());
  for (std::uint32_t s : Q) claimed[s] = 1;
  while (!queue.empty()) {
    const std::uint32_t s = queue.front();
    queue.pop_front();
    for (int d = 0; d <= D; ++d) {
      if (!dead(slots[s].nb[d])) continue;
      const std::uint64_t key = merge_facet_key<D>(slots[s].v, d);
      auto it = std::lower_bound(index.begin(), index.end(), std::make_pair(key, std::uint32_t(0)));
      std::uint32_t found = kMergeNone;
      int hits = 0;
      for (; it != index.end() && it->first == key; ++it) {
        const std::uint32_t c = it->second;
        if (c == s) continue;
        int common = 0;  // shared_vertex_count (triangulation.hpp:49-66): both tuples ascending
        for (int i = 0, j = 0; i <= D && j <= D;) {
          if (slots[s].v[i] == slots[c].v[j]) ++common, ++i, ++j;
          else if (slots[s].v[i] < slots[c].v[j]) ++i;
          else ++j;
        }
        // sharing exactly D vertices AND not the opposite vertex of facet d
        if (common != D) continue;
        bool has_opp = false;
        for (int j = 0; j <= D; ++j) has_opp |= slots[c].v[j] == slots[s].v[d];
        if (has_opp) continue;
        found = c;
        ++hits;
      }
      if (hits > 1) {
        out.error = "InconsistentMerge: facet shared by more than two simplices";
        return out;
      }
      if (found == kMergeNone) continue;
      slots[s].nb[d] = found;
      Slot& c = slots[found];
      for (int j = 0; j <= D; ++j) {
        bool in_s = false;
        for (int i = 0; i <= D; ++i) in_s |= slots[s].v[i] == c.v[j];
        if (!in_s) {
          c.nb[j] = s;
          break;
        }
      }
      if (!claimed[found]) {
        claimed[found] = 1;
        queue.push_back(found);
      }
    }
  }
  // 4. compaction and hull re-derivation
  std::vector<std::uint32_t> newid(slots.size(), kMergeNone);
  std::uint64_t M = 0;
  out.offsets.assign(k + 3, 0);
  for (std::uint32_t p = 0; p < k; ++p) {
    out.offsets[p] = M;
    for (std::uint64_t s = offsets[p]; s < offsets[p + 1]; ++s)
      if (slots[s].alive) newid[s] = static_cast<std::uint32_t>(M++);
  }
  out.offsets[k] = M;
  for (std::uint64_t s = S; s < slots.size(); ++s) newid[s] = static_cast<std::uint32_t>(M++);
  out.offsets[k + 1] = M;
  std::vector<Tup> rv, rn;
  std::vector<std::int8_t> rp;
  rv.reserve(M);
  for (std::uint64_t s = 0; s < slots.size(); ++s) {
    if (!slots[s].alive) continue;
    Tup nb;
    for (int j = 0; j <= D; ++j) nb[j] = dead(slots[s].nb[j]) ? kMergeNone : newid[slots[s].nb[j]];
    rv.push_back(slots[s].v);
    rn.push_back(nb);
    rp.push_back(slots[s].par);
  }
  (void)n_inserted;
  if (hull) {
    std::map<std::array<std::uint32_t, D - 1>, std::vector<std::pair<std::uint32_t, int>>> ridges;
    for (std::uint64_t o = 0; o < M; ++o) {
      for (int d = 0; d <= D; ++d) {
        if (rn[o][d] != kMergeNone) continue;
        const std::uint32_t h = static_cast<std::uint32_t>(rv.size());
        Tup hv, hn;
        for (int j = 0, q = 0; j <= D; ++j)
          if (j != d) hv[q++] = rv[o][j];
        hv[D] = kMergeInf;
        hn.fill(kMergeNone);
        hn[D] = static_cast<std::uint32_t>(o);
        rn[o][d] = h;
        rv.push_back(hv);
        rn.push_back(hn);
        rp.push_back(0);
        for (int i = 0; i < D; ++i) {
          std::array<std::uint32_t, D - 1> r;
          for (int j = 0, q = 0; j < D; ++j)
            if (j != i) r[q++] = hv[j];
          ridges[r].emplace_back(h, i);
        }
      }
    }
    for (auto& [r, owners] : ridges) {
      if (owners.size() != 2) {
        out.error = "DanglingFacet: hull ridge without exactly two hull facets";
        return out;
      }
      rn[owners[0].first][owners[0].second] = owners[1].first;
      rn[owners[1].first][owners[1].second] = owners[0].first;
    }
  }
  const std::uint64_t R = rv.size();
  out.offsets[k + 2] = R;
  out.rows = R;
  out.verts.resize((D + 1) * R);
  out.nbrs.resize((D + 1) * R);
  for (std::uint64_t s = 0; s < R; ++s)
    for (int j = 0; j <= D; ++j) {
      out.verts[j * R + s] = rv[s][j];
      out.nbrs[j * R + s] = rn[s][j];
    }
  out.parity = rp;
  return out;
}

}  // namespace sbdt_oracle
