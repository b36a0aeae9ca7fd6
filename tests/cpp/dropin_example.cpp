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
//
//   --level L   a recursion level of delaunay_dc: only the
//               first L partitions and their points take part; their indices
//               keep the full set's bbox and size (build_grid_index post,
//               SPEC.md:410). Flags cover the rows of those L partials.
//   --bench R   instead: R timed steps (after one warm-up) of assign_points
//               + build_grid_index + find_border on a TaskPool(--threads T),
//               no BFS, points resident from assign_points; prints one JSON
//               line with the per-call wall times.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <thread>
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

struct Args {
  std::uint32_t level = 0;  // 0: all partitions
  int bench = 0;
  unsigned threads = 0;
};

template <int D>
static int run(std::ifstream& in, std::uint64_t n, std::uint32_t m, std::uint32_t k, std::uint64_t S,
               const char* out_path, const Args& args) {
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
  const std::uint32_t L = args.level ? args.level : k;

  // the partial triangulations as the reference's Triangulation<D> objects
  std::vector<Triangulation<D>> partials;
  partials.reserve(k);
  for (std::uint32_t p = 0; p < L; ++p) {
    partials.emplace_back(&P);
    partials.back().raw_simplices().reserve(offsets[p + 1] - offsets[p]);
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
  IntersectionPolicy pol;
  pol.kind = IntersectionPolicy::Grid;
  pol.c_G = 1.0;

  if (args.bench > 0) {
    const unsigned T = args.threads ? args.threads : std::max(1u, std::thread::hardware_concurrency());
    TaskPool pool(T);
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    double t_assign = 0, t_index = 0, t_border = 0, t_total = 0;
    gpu_detail::PhaseTimes pa{}, pb{};  // summed phases of assign_points / find_border
    std::uint64_t n_pos = 0;
    for (int rep = -1; rep < args.bench; ++rep) {  // rep -1: warm-up (allocations, pinned staging)
      const auto t0 = now();
      const Partitioning part = assign_points<D>(P, sid, slab, k, &pool);
      const auto t1 = now();
      const gpu_detail::PhaseTimes ha = gpu_detail::last_phases();
      std::vector<GridIndex<D>> idx(k);
      pool.parallel_for(k, 1, [&](std::size_t b, std::size_t e) {
        for (std::size_t p = b; p < e; ++p) idx[p] = build_grid_index<D>(P, part.parts[p], bbox, n, 1.0);
      });
      const auto t2 = now();
      BorderOptions o;
      o.hull_bfs = false;
      o.labels = part.labels;
      o.points_resident = true;
      const BorderSet B = find_border<D>(std::span<const Triangulation<D>>(partials),
                                         std::span<const GridIndex<D>>(idx), pol, &pool, o);
      const auto t3 = now();
      if (rep >= 0) {
        const gpu_detail::PhaseTimes& hb = gpu_detail::last_phases();
        pa.prepare_ms += ha.prepare_ms, pa.device_ms += ha.device_ms, pa.finish_ms += ha.finish_ms;
        pb.prepare_ms += hb.prepare_ms, pb.device_ms += hb.device_ms, pb.finish_ms += hb.finish_ms;
        t_assign += secs(t0, t1), t_index += secs(t1, t2), t_border += secs(t2, t3), t_total += secs(t0, t3);
        n_pos = 0;
        for (const auto& v : B.positive) n_pos += v.size();
      }
    }
    const double r = args.bench;
    std::printf("{\"steps\": %d, \"threads\": %u, \"ms_per_step\": %.3f, \"assign_points_ms\": %.3f, "
                "\"build_grid_index_ms\": %.3f, \"find_border_ms\": %.3f, \"positive_simplices\": %llu, "
                "\"phases_ms\": {\"assign_prepare\": %.3f, \"assign_abi\": %.3f, \"assign_finish\": %.3f, "
                "\"border_prepare\": %.3f, \"border_abi\": %.3f, \"border_finish\": %.3f}}\n",
                args.bench, T, 1e3 * t_total / r, 1e3 * t_assign / r, 1e3 * t_index / r, 1e3 * t_border / r,
                static_cast<unsigned long long>(n_pos), pa.prepare_ms / r, pa.device_ms / r, pa.finish_ms / r,
                pb.prepare_ms / r, pb.device_ms / r, pb.finish_ms / r);
    return 0;
  }

  // SPEC.md:342-350 through the drop-in
  const Partitioning part = assign_points<D>(P, sid, slab, k);
  std::vector<GridIndex<D>> idx;
  for (std::uint32_t p = 0; p < L; ++p) idx.push_back(build_grid_index<D>(P, part.parts[p], bbox, n, 1.0));
  const BorderSet B = find_border<D>(std::span<const Triangulation<D>>(partials), std::span<const GridIndex<D>>(idx),
                                     pol);
  const std::uint64_t SL = offsets[L];
  std::vector<std::uint8_t> pos(SL, 0), bor(SL, 0);
  for (std::uint32_t p = 0; p < L; ++p) {
    for (SimplexId s : B.positive[p]) pos[offsets[p] + s] = 1;
    for (SimplexId s : B.simplices[p]) bor[offsets[p] + s] = 1;
  }
  std::ofstream out(out_path, std::ios::binary);
  wr(out, part.labels.data(), n);
  wr(out, pos.data(), SL);
  wr(out, bor.data(), SL);
  const std::uint64_t nv = B.positive_vertex_ids.size(), nb = B.border_vertex_ids.size();
  wr(out, &nv, 1);
  wr(out, B.positive_vertex_ids.data(), nv);
  wr(out, &nb, 1);
  wr(out, B.border_vertex_ids.data(), nb);
  // merge the partials with T_B (the DT of B's vertices)
  std::uint64_t SB = 0;
  in.read(reinterpret_cast<char*>(&SB), sizeof(SB));
  if (in && L == k) {
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
  if (argc < 3) {
    std::cerr << "usage: dropin_example <instance.bin> <result.bin> [--level L] [--bench R] [--threads T]\n";
    return 2;
  }
  Args args;
  for (int i = 3; i + 1 < argc; i += 2) {
    if (!std::strcmp(argv[i], "--level")) args.level = static_cast<std::uint32_t>(std::atoi(argv[i + 1]));
    else if (!std::strcmp(argv[i], "--bench")) args.bench = std::atoi(argv[i + 1]);
    else if (!std::strcmp(argv[i], "--threads")) args.threads = static_cast<unsigned>(std::atoi(argv[i + 1]));
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
    return dim == 2 ? run<2>(in, n, m, k, S, argv[2], args) : run<3>(in, n, m, k, S, argv[2], args);
  } catch (const std::exception& e) {
    std::cerr << "dropin_example: " << e.what() << "\n";
    return 1;
  }
}
