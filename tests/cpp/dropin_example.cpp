// Drop-in check of the C++ layer (include/sbdt/*.hpp) on the reference's own
// types: reads an instance (points, sample, labels, partial triangulations,
// optionally the border triangulation T_B), calls sbdt::assign_points,
// sbdt::find_border and sbdt::merge exactly as delaunay_dc would
// (SPEC.md:479-505), and writes the results for tests/test_cpp_dropin.py.
//
// Input file (little-endian): u32 dim, u64 n, u32 m, u32 k, u64 S; f64 points
// [n*dim]; u32 sample_ids[m]; u32 sample_labels[m]; u64 offsets[k+1];
// u32 verts[(dim+1)*S]; u32 nbrs[(dim+1)*S]; i8 parity[S]; optionally
// u64 S_B; u32 tb_verts[(dim+1)*S_B]; u32 tb_nbrs[(dim+1)*S_B]; i8 tb_parity[S_B].
// Output file: u32 labels[n]; u8 positive[S]; u8 border[S]; u64 nv;
// u32 positive_vertex_ids[nv]; u64 nb; u32 border_vertex_ids[nb]; with T_B:
// u64 rows; u32 verts[(dim+1)*rows]; u32 nbrs[(dim+1)*rows]; i8 parity[rows]
// (the merged triangulation, slot order, vertex-major).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <vector>

#include "sbdt/dc_engine.hpp"

using namespace sbdt;

template <class T>
static void rd(std::ifstream& f, T* p, std::size_t count) {
  f.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(sizeof(T) * count));
  if (!f) throw std::runtime_error("short input");
}
template <class T>
static void wr(std::ofstream& f, const T* p, std::size_t count) {
  f.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(sizeof(T) * count));
}

template <int D>
static int run(std::ifstream& in, std::uint64_t n, std::uint32_t m, std::uint32_t k, std::uint64_t S,
               const char* out_path) {
  PointSet P(D);
  std::vector<double> xyz(n * D);
  rd(in, xyz.data(), xyz.size());
  for (std::uint64_t i = 0; i < n; ++i) P.add(xyz.data() + i * D);
  std::vector<PointId> sid(m);
  std::vector<PartitionId> slab(m);
  rd(in, sid.data(), m);
  rd(in, slab.data(), m);
  std::vector<std::uint64_t> offsets(k + 1);
  rd(in, offsets.data(), k + 1);
  std::vector<std::uint32_t> verts((D + 1) * S), nbrs((D + 1) * S);
  std::vector<std::int8_t> parity(S);
  rd(in, verts.data(), verts.size());
  rd(in, nbrs.data(), nbrs.size());
  rd(in, parity.data(), S);

  // SPEC.md:342-350 through the drop-in
  const Partitioning part = assign_points<D>(P, sid, slab, k);
  // the partial triangulations as the reference's Triangulation<D> objects
  std::vector<Triangulation<D>> partials;
  partials.reserve(k);
  for (std::uint32_t p = 0; p < k; ++p) {
    partials.emplace_back(&P);
    for (std::uint64_t r = offsets[p]; r < offsets[p + 1]; ++r) {
      Simplex<D> s;
      for (int j = 0; j <= D; ++j) {
        s.vertices[j] = verts[std::uint64_t(j) * S + r];
        s.neighbors[j] = nbrs[std::uint64_t(j) * S + r];
      }
      s.parity = parity[r];
      s.origin_partition = p;
      partials.back().append_slot(s);
    }
  }
  Box<D> bbox = Box<D>::empty();
  for (std::uint64_t i = 0; i < n; ++i) bbox.expand(P.template at<D>(static_cast<PointId>(i)));
  std::vector<GridIndex<D>> idx;
  for (std::uint32_t p = 0; p < k; ++p) idx.push_back(build_grid_index<D>(P, part.parts[p], bbox, n, 1.0));
  IntersectionPolicy pol;
  pol.kind = IntersectionPolicy::Grid;
  pol.c_G = 1.0;
  const BorderSet B = find_border<D>(std::span<const Triangulation<D>>(partials), std::span<const GridIndex<D>>(idx),
                                     pol);

  std::vector<std::uint8_t> pos(S, 0), bor(S, 0);
  for (std::uint32_t p = 0; p < k; ++p) {
    for (SimplexId s : B.positive[p]) pos[offsets[p] + s] = 1;
    for (SimplexId s : B.simplices[p]) bor[offsets[p] + s] = 1;
  }
  std::ofstream out(out_path, std::ios::binary);
  wr(out, part.labels.data(), n);
  wr(out, pos.data(), S);
  wr(out, bor.data(), S);
  const std::uint64_t nv = B.positive_vertex_ids.size(), nb = B.border_vertex_ids.size();
  wr(out, &nv, 1);
  wr(out, B.positive_vertex_ids.data(), nv);
  wr(out, &nb, 1);
  wr(out, B.border_vertex_ids.data(), nb);
  // merge the partials with T_B (the DT of B's vertices)
  std::uint64_t SB = 0;
  in.read(reinterpret_cast<char*>(&SB), sizeof(SB));
  if (in) {
    std::vector<std::uint32_t> tv((D + 1) * SB), tn((D + 1) * SB);
    std::vector<std::int8_t> tp(SB);
    rd(in, tv.data(), tv.size());
    rd(in, tn.data(), tn.size());
    rd(in, tp.data(), SB);
    Triangulation<D> TB(&P);
    for (std::uint64_t r = 0; r < SB; ++r) {
      Simplex<D> s;
      for (int j = 0; j <= D; ++j) {
        s.vertices[j] = tv[std::uint64_t(j) * SB + r];
        s.neighbors[j] = tn[std::uint64_t(j) * SB + r];
      }
      s.parity = tp[r];
      TB.append_slot(s);
    }
    const Triangulation<D> T = merge<D>(std::span<const Triangulation<D>>(partials), B, TB,
                                        std::span<const PartitionId>(part.labels));
    const std::uint64_t rows = T.slot_count();
    std::vector<std::uint32_t> ov((D + 1) * rows), on((D + 1) * rows);
    std::vector<std::int8_t> op(rows);
    for (std::uint64_t r = 0; r < rows; ++r) {
      const Simplex<D>& s = T.at(static_cast<SimplexId>(r));
      for (int j = 0; j <= D; ++j) {
        ov[std::uint64_t(j) * rows + r] = s.vertices[j];
        on[std::uint64_t(j) * rows + r] = s.neighbors[j];
      }
      op[r] = s.parity;
    }
    wr(out, &rows, 1);
    wr(out, ov.data(), ov.size());
    wr(out, on.data(), on.size());
    wr(out, op.data(), rows);
  }
  return out ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc != 3) {
    std::cerr << "usage: dropin_example <instance.bin> <result.bin>\n";
    return 2;
  }
  try {
    std::ifstream in(argv[1], std::ios::binary);
    std::uint32_t dim = 0, m = 0, k = 0;
    std::uint64_t n = 0, S = 0;
    rd(in, &dim, 1);
    rd(in, &n, 1);
    rd(in, &m, 1);
    rd(in, &k, 1);
    rd(in, &S, 1);
    return dim == 2 ? run<2>(in, n, m, k, S, argv[2]) : run<3>(in, n, m, k, S, argv[2]);
  } catch (const std::exception& e) {
    std::cerr << "dropin_example: " << e.what() << "\n";
    return 1;
  }
}
