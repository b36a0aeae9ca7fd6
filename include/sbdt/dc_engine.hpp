// sbdt/dc_engine.hpp — drop-in dc-engine `merge` + `update_neighbors`
// backed by libsbdt_gpu.so.
//
// The reference specifies these operations (Alg. 1 merging and neighbourhood
// blocks, PAPER.md) but ships no source for them (dc_engine.cpp,
// proj/src/CMakeLists.txt:8). The signature below is the SPEC's, in the style
// of the shipped headers; the partial triangulations and T_B are the
// reference's own Triangulation<D> (proj/include/sbdt/triangulation.hpp:162-258;
// tombstoned slots are skipped), the border set is find_border's BorderSet
// (sbdt/border.hpp).
//
// merge() returns the merged triangulation with its neighbour structure
// already rebuilt — SPEC update_neighbors' postcondition (full neighbour
// symmetry) is met by the device's facet-hash join, so the
// repair queue Q of the SPEC never materialises — and, with `hull`, the
// merged hull re-derived as infinite simplices. Slot order:
// the kept partial simplices (partition by partition, slot order), then the
// inserted T_B simplices (T_B slot order), then the hull simplices ((owner,
// facet) order). Bit-identical to the CPU oracle (tests/test_merge.py).
// Errors: sbdt::InconsistentMerge (a simplex inserted twice / a facet with
// three owners), sbdt::DanglingFacet (a hull ridge without two hull facets).
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sbdt/border.hpp"
#include "sbdt/triangulation.hpp"

namespace sbdt {

namespace gpu_detail {

// Live slots of a triangulation as the C ABI's vertex-major rows [row0, ...)
// of a row set with stride S; neighbour slot ids become row ids local to the
// triangulation (kNoSimplex stays kNoSimplex).
template <int D>
void append_rows(const Triangulation<D>& t, std::uint64_t S, std::uint64_t row0, std::vector<SimplexId>& slot_of,
                 std::vector<std::uint32_t>& verts, std::vector<std::uint32_t>& nbrs,
                 std::vector<std::int8_t>& parity) {
  std::vector<SimplexId> local(t.slot_count(), kNoSimplex);
  std::uint64_t r = row0;
  t.for_each_alive([&](SimplexId id, const Simplex<D>&) { local[id] = static_cast<SimplexId>(r++ - row0); });
  r = row0;
  t.for_each_alive([&](SimplexId id, const Simplex<D>& s) {
    slot_of.push_back(id);
    for (int j = 0; j <= D; ++j) {
      verts[std::uint64_t(j) * S + r] = s.vertices[j];
      nbrs[std::uint64_t(j) * S + r] = s.neighbors[j] == kNoSimplex ? kNoSimplex : local[s.neighbors[j]];
    }
    parity[r] = s.parity;
    ++r;
  });
}

template <int D>
std::uint64_t alive_rows(const Triangulation<D>& t) {
  std::uint64_t c = 0;
  t.for_each_alive([&](SimplexId, const Simplex<D>&) { ++c; });
  return c;
}

}  // namespace gpu_detail

// SPEC.md:497-505 merge (+ SPEC.md:506-514 update_neighbors, fused).
template <int D>
Triangulation<D> merge(std::span<const Triangulation<D>> partials, const BorderSet& border,
                       const Triangulation<D>& T_B, std::span<const PartitionId> partition_labels,
                       bool hull = true, TaskPool* pool = nullptr) {
  (void)pool;
  static_assert(D == 2 || D == 3, "D must be 2 or 3");
  const std::uint32_t k = static_cast<std::uint32_t>(partials.size());
  if (k == 0) throw std::invalid_argument("merge: no partial triangulations");
  if (border.simplices.size() != k) throw std::invalid_argument("merge: BorderSet must hold one list per partition");
  const PointSet& ps = partials[0].points();
  const std::uint64_t n = ps.size();
  if (partition_labels.size() != n) throw std::invalid_argument("merge: one partition label per point");
  // the partials as one vertex-major row set with part offsets
  std::vector<std::uint64_t> offsets(k + 1, 0);
  for (std::uint32_t p = 0; p < k; ++p) offsets[p + 1] = offsets[p] + gpu_detail::alive_rows<D>(partials[p]);
  const std::uint64_t S = offsets[k];
  std::vector<std::uint32_t> verts((D + 1) * S), nbrs((D + 1) * S);
  std::vector<std::int8_t> parity(S);
  std::vector<std::vector<SimplexId>> slot_of(k);
  std::vector<std::uint8_t> bflags(S, 0);
  for (std::uint32_t p = 0; p < k; ++p) {
    gpu_detail::append_rows<D>(partials[p], S, offsets[p], slot_of[p], verts, nbrs, parity);
    // nbrs of part p are part-local row ids: append_rows numbers them from 0
    std::vector<SimplexId> row_of(partials[p].slot_count(), kNoSimplex);
    for (std::size_t i = 0; i < slot_of[p].size(); ++i) row_of[slot_of[p][i]] = static_cast<SimplexId>(i);
    for (SimplexId s : border.simplices[p]) {
      if (s >= row_of.size() || row_of[s] == kNoSimplex) throw std::invalid_argument("merge: border simplex is not alive");
      bflags[offsets[p] + row_of[s]] = 1;
    }
  }
  const std::uint64_t SB = gpu_detail::alive_rows<D>(T_B);
  std::vector<std::uint32_t> tv((D + 1) * SB), tn((D + 1) * SB);
  std::vector<std::int8_t> tp(SB);
  std::vector<SimplexId> tb_slots;
  gpu_detail::append_rows<D>(T_B, SB, 0, tb_slots, tv, tn, tp);
  std::vector<std::uint32_t> labels(partition_labels.begin(), partition_labels.end());

  sbdt_gpu_ctx* ctx = gpu_detail::thread_context();
  std::uint64_t cap = S + SB + (S + SB) / 8 + 1024, rows = 0;
  std::vector<std::uint32_t> ov, on;
  std::vector<std::int8_t> op;
  std::vector<std::uint64_t> oo(k + 3);
  for (int attempt = 0;; ++attempt) {
    ov.resize((D + 1) * cap);
    on.resize((D + 1) * cap);
    op.resize(cap);
    const int rc = sbdt_gpu_merge(ctx, D, labels.data(), n, k, offsets.data(), verts.data(), nbrs.data(),
                                  parity.data(), bflags.data(), tv.data(), tn.data(), tp.data(), SB,
                                  hull ? SBDT_MERGE_HULL : 0u, cap, ov.data(), on.data(), op.data(), oo.data(),
                                  &rows);
    if (rc == SBDT_ERR_RANGE && attempt == 0 && rows > cap) {
      cap = rows;
      continue;
    }
    if (rc == SBDT_ERR_MERGE) {
      const std::string msg = std::string("merge: ") + sbdt_gpu_last_error(ctx);
      if (msg.find("angling") != std::string::npos) throw DanglingFacet(msg);
      throw InconsistentMerge(msg);
    }
    gpu_detail::check(ctx, rc, "merge");
    break;
  }
  // rows come back compact (row stride = rows)
  Triangulation<D> out(&ps);
  std::uint32_t p = 0;  // kept partial rows of part p are [oo[p], oo[p+1]); then T_B and hull rows
  for (std::uint64_t r = 0; r < rows; ++r) {
    while (p < k && r >= oo[p + 1]) ++p;
    Simplex<D> s;
    for (int j = 0; j <= D; ++j) {
      s.vertices[j] = ov[std::uint64_t(j) * rows + r];
      s.neighbors[j] = on[std::uint64_t(j) * rows + r];
    }
    s.parity = op[r];
    s.origin_partition = p < k ? p : kNoPartition;
    out.append_slot(s);
  }
  return out;
}

}  // namespace sbdt
