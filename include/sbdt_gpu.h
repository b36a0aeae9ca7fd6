/*
 * sbdt_gpu.h — C ABI of libsbdt_gpu.so, the B200 (sm_100a) implementation of
 * the sample-based divide step's data-parallel core (arXiv 1902.07554):
 *
 *   sbdt_gpu_assign_points*  replaces  sample-partition `assign_points`
 *       (Alg. 2 lines "find nearest
 *       sample point" / "assign p to v_n's partition") and the
 *       Partitioning.parts bucketing.
 *   sbdt_gpu_merge*          replaces  dc-engine `merge` + `update_neighbors`
 *       (Alg. 1 merging / neighbourhood blocks), the
 *       step after the border triangulation.
 *   sbdt_gpu_find_border*    replaces  dc-engine `find_border` with the
 *       border-geom `GridIndex` / `intersects_{bbox,grid}` queries
 *       (Alg. 1 border block) on the
 *       reference's Triangulation<D> records (proj/include/sbdt/triangulation.hpp:17-68).
 *
 * Neither reference operation ships as code; the C++
 * drop-in headers include/sbdt/sample_partition.hpp and include/sbdt/border.hpp
 * declare them with the SPEC's signatures and call this ABI. Conventions:
 *   - plain pointers and sizes only; no exception crosses the ABI;
 *   - status 0 = ok; nonzero codes below map to the reference's exception
 *     types (common.hpp:22-65) in the C++ wrapper; sbdt_gpu_last_error() has
 *     the message;
 *   - *_dev entry points take DEVICE pointers and are asynchronous on the
 *     context's stream; the plain entry points take HOST buffers (H2D/D2H
 *     inside) and are synchronous;
 *   - one host thread per context.
 * Results are bit-identical to the CPU oracle: labels, positive flags,
 * hull-reachable border flags and border-vertex ids; circumcentres/radii are
 * the reference's binary64 expressions evaluated in the same order.
 */
#ifndef SBDT_GPU_H_
#define SBDT_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sbdt_gpu_ctx sbdt_gpu_ctx;

enum sbdt_status {
  SBDT_OK = 0,
  SBDT_ERR_INVALID = 1,    /* std::invalid_argument                     */
  SBDT_ERR_DEGENERATE = 2, /* sbdt::DegenerateSimplex (geometry.cpp:281) */
  SBDT_ERR_CUDA = 3,       /* std::runtime_error                        */
  SBDT_ERR_OOM = 4,        /* std::bad_alloc                            */
  SBDT_ERR_RANGE = 5,      /* grid larger than 4 n / c_G^D cells; output
                              capacity too small (merge)                 */
  SBDT_ERR_MERGE = 6       /* sbdt InconsistentMerge / DanglingFacet
                                                      */
};

/* IntersectionPolicy::Kind */
enum sbdt_policy { SBDT_POLICY_BBOX = 0, SBDT_POLICY_GRID = 1, SBDT_POLICY_EXACT = 2 };

/* find_border flags */
enum sbdt_border_flags {
  SBDT_BORDER_HULL_BFS = 1u, /* also compute the SPEC find_border BFS subset (border_out) */
  /* host-buffer call only: coords and labels are the buffers of the last
   * sbdt_gpu_assign_points call on this context (coords as passed, labels as
   * written to labels_out) and are unchanged since; their device copies are
   * reused instead of uploaded again (checked: same pointers, n and dim). */
  SBDT_BORDER_RESIDENT_POINTS = 2u
};

int sbdt_gpu_create(int device, sbdt_gpu_ctx** out);
void sbdt_gpu_destroy(sbdt_gpu_ctx* ctx);
const char* sbdt_gpu_last_error(const sbdt_gpu_ctx* ctx);
/* Launch on an external cudaStream_t from now on (e.g.
 * torch.cuda.current_stream().cuda_stream); the handle is used as given, so
 * NULL selects the legacy default stream. */
int sbdt_gpu_set_stream(sbdt_gpu_ctx* ctx, void* cuda_stream);
int sbdt_gpu_synchronize(sbdt_gpu_ctx* ctx);
/* Number of kernels launched by this context so far. */
unsigned long long sbdt_gpu_launch_count(const sbdt_gpu_ctx* ctx);
/* Reads and clears the device status word; returns the mapped status. */
int sbdt_gpu_check_status(sbdt_gpu_ctx* ctx);
/* enable bit 0: per-stage CUDA-event timing on the context stream; bit 1:
 * pipeline census counters (extra atomics: not for timed runs). Off by
 * default. sbdt_gpu_stage_times synchronizes, writes up to max_stages
 * durations (ms) and '\n'-separated stage names, clears the record and
 * returns the count. */
int sbdt_gpu_set_timing(sbdt_gpu_ctx* ctx, int enable);
int sbdt_gpu_stage_times(sbdt_gpu_ctx* ctx, char* names, int names_len, float* ms, int max_stages);
/* Voronoi-label-table census of the last assign with the census enabled:
 * out6 = {uniform records, short-list records, ring-search records,
 * long-list records, queued points (long lists + ring searches), coarse cells
 * built by the dense pass}. */
int sbdt_gpu_assign_table_stats(sbdt_gpu_ctx* ctx, unsigned* out6);
/* Border pipeline census of the last find_border with the census enabled:
 * the first `count` (<= 20) of {0 rows scanned by the prefilter, 1 rows that
 * reached the binary64 exact stage, 2 of those through its flattened cell
 * scan, 3 wide rows forwarded by the exact stage, 4 wide rows routed by the
 * prefilter, 5 (candidate, cell row) pairs of the binary64 flattened scan,
 * 6 wide-stage block expansions, 7 positives of the binary64 flattened scan,
 * 8 positives proven by the prefilter's own sphere test, 9 positives of the
 * wide stage, 10 positives proven by the prefilter's neighbour proofs
 * (foreign mask / near octant), 11 candidate-queue slots left unused (holes
 * of the per-warp chunks), 12 rows whose binary32 sphere failed (exact
 * orientation checked), 13 orientation predicates escalated to expansion
 * arithmetic, 14 in_sphere predicates escalated to expansion arithmetic
 * (exact policy), 15 negatives proven by the foreign mask, 16 rows of the
 * binary32 cell scan, 17 positives of the binary32 cell scan, 18 rows it
 * left to the binary64 exact stage, 19 0}. */
int sbdt_gpu_border_stats(sbdt_gpu_ctx* ctx, unsigned long long* out, int count);

/* Page-locked host memory for the host-buffer entry points' inputs and
 * outputs (transfers from/to pageable memory are staged by the driver and
 * fault in fresh pages). */
int sbdt_gpu_host_alloc(uint64_t bytes, void** out);
void sbdt_gpu_host_free(void* p);

/* Producer hook of sbdt_gpu_find_border (host buffers): when set, the call
 * invokes fill(user, SBDT_FILL_ROWS, r0, r1) right before it uploads the
 * simplex rows [r0, r1) of verts / nbrs / parity, in increasing order, so
 * the caller can write those rows into the (page-locked) buffers it passed
 * while the previous chunk is in flight (e.g. converting the reference's
 * Triangulation<D> records). A non-zero return aborts the call with
 * SBDT_ERR_INVALID. fill == NULL removes the hook. The hook applies to the
 * context's host-buffer find_border calls until removed. */
#define SBDT_FILL_ROWS 1
typedef int (*sbdt_fill_fn)(void* user, int what, uint64_t begin, uint64_t end);
int sbdt_gpu_set_fill(sbdt_gpu_ctx* ctx, sbdt_fill_fn fill, void* user);

/* ---- assign_points -------------------------------------
 * coords: n points, AoS binary64 (PointSet::raw(), geometry.hpp:94-95).
 * sample_ids: m global PointIds; sample_labels: m labels < k.
 * labels_out[i] = sample_labels[argmin_s squared_distance(p_i, p_s)], ties
 * toward the lowest sample PointId.
 * part_offsets_out (k+1, optional) and part_ids_out (n, optional) receive
 * Partitioning.parts as CSR, ids ascending within each part.
 * bbox_out (optional, 2*dim doubles: lo[], hi[]) receives the global point
 * bounding box, fused into the same pass. */
int sbdt_gpu_assign_points(sbdt_gpu_ctx* ctx, int dim, const double* coords, uint64_t n,
                           const uint32_t* sample_ids, const uint32_t* sample_labels, uint32_t m,
                           uint32_t k, uint32_t* labels_out, uint64_t* part_offsets_out,
                           uint32_t* part_ids_out, double* bbox_out);

/* Device-pointer variant. d_bbox_ordered_out (optional) receives 2*dim
 * order-preserving uint64 keys of the bbox (input of sbdt_gpu_find_border_dev).
 * Precondition (not re-checked on the host: the labels stay on the device):
 * every sample id < n and every sample label < k. A label >= k is detected
 * by the bucketing pass when part_offsets / part_ids are requested and then
 * fails the next synchronizing call with SBDT_ERR_INVALID. */
int sbdt_gpu_assign_points_dev(sbdt_gpu_ctx* ctx, int dim, const double* d_coords, uint64_t n,
                               const uint32_t* d_sample_ids, const uint32_t* d_sample_labels,
                               uint32_t m, uint32_t k, uint32_t* d_labels_out,
                               uint64_t* d_part_offsets_out, uint32_t* d_part_ids_out,
                               uint64_t* d_bbox_ordered_out);

/* ---- find_border ---------------------------------------
 * The k partial triangulations are concatenated: part p owns simplex rows
 * [offsets[p], offsets[p+1]). Per row s, in vertex-major SoA (row j holds
 * Simplex::vertices[j] / neighbors[j] of every simplex):
 *   verts[j*S + s]  global PointId, ascending, kInfiniteVertex (0xFFFFFFFF) last
 *   nbrs[j*S + s]   part-local SimplexId sharing the facet opposite verts[j]
 *   parity[s]       Simplex::parity (orientation sign of the stored order);
 *                   read by the exact policy only (in_sphere_oriented), may be
 *                   NULL otherwise: a simplex whose vertices have zero exact
 *                   orientation fails the call with SBDT_ERR_DEGENERATE, as the
 *                   reference's circumsphere throws DegenerateSimplex
 * labels[i] is the partition of point i (the GridIndex of part j is built from
 * the points labelled j; cell edge c_G (V/n)^(1/D) over the global bbox).
 * Outputs (caller buffers):
 *   positive_out[s]  1 iff the (inflated) circumsphere / hull halfspace of s
 *                    reaches a cell occupied by another part (full scan);
 *   border_out[s]    (optional; needs SBDT_BORDER_HULL_BFS) the SPEC BFS
 *                    subset: positive simplices connected through positive
 *                    simplices to a hull simplex (hull_simplices,
 *                    triangulation.cpp:34-53);
 *   vertex_ids_out   sorted unique finite vertices of positive simplices
 *                    (capacity n), count in *n_vertices_out;
 *   bfs_vertex_ids_out / n_bfs_vertices_out (optional): same for border_out;
 *   spheres_out      (optional) (dim+1) doubles per row: inflated centre, r^2
 *                    (zeros for infinite rows). */
/* Recursion levels of delaunay_dc: the GridIndex of a
 * level's partitions keeps the cell edge of the TOP level,
 * c_G (vol(global bbox) / n_total)^(1/D) with origin global bbox lo
 * (build_grid_index post). grid_bbox (2*dim doubles lo[], hi[],
 * or NULL: the bbox of the n coords) and grid_n_total (0: n) give those
 * values; points of `coords` outside the level carry the label
 * SBDT_UNINDEXED (they occupy no cell and are nobody's points). */
#define SBDT_UNINDEXED 0xFFFFFFFFu

int sbdt_gpu_find_border(sbdt_gpu_ctx* ctx, int dim, const double* coords, uint64_t n,
                         const uint32_t* labels, uint32_t k, const uint64_t* offsets,
                         const uint32_t* verts, const uint32_t* nbrs, const int8_t* parity,
                         int policy, double c_G, uint32_t flags, uint8_t* positive_out,
                         uint8_t* border_out, uint32_t* vertex_ids_out, uint64_t* n_vertices_out,
                         uint32_t* bfs_vertex_ids_out, uint64_t* n_bfs_vertices_out,
                         double* spheres_out, const double* grid_bbox, uint64_t grid_n_total);

typedef struct sbdt_border_args {
  int dim;
  const double* d_xyz;
  uint64_t n;
  const uint32_t* d_labels;
  uint32_t k;
  const uint64_t* d_offsets; /* k+1 */
  const uint32_t* d_verts;
  const uint32_t* d_nbrs;
  const int8_t* d_parity;
  uint64_t S;
  int policy;
  double c_G;
  uint32_t flags;
  const uint64_t* d_bbox_ordered; /* optional: from sbdt_gpu_assign_points_dev */
  uint8_t* d_positive;            /* S */
  uint8_t* d_border;              /* S, optional (HULL_BFS) */
  uint8_t* d_vertex_flags;        /* n scratch */
  uint32_t* d_vertex_ids;         /* n */
  uint64_t* d_vertex_count;       /* 1 */
  uint8_t* d_bfs_vertex_flags;    /* n scratch, optional */
  uint32_t* d_bfs_vertex_ids;     /* n, optional */
  uint64_t* d_bfs_vertex_count;   /* 1, optional */
  double* d_spheres;              /* S*(dim+1), optional */
  const double* grid_bbox;        /* optional HOST array 2*dim (lo[], hi[]): the grid's global bbox (SBDT_UNINDEXED) */
  uint64_t grid_n_total;          /* 0: n */
  uint64_t grid_max_cells;        /* owner-grid capacity in cells; 0: 4 n / c_G^dim. A grid that needs more
                                     (a bbox far from cubical) fails with SBDT_ERR_RANGE; the host-buffer
                                     entry point then retries once with the capacity the grid needs
                                     (up to 2^31 cells) */
} sbdt_border_args;

int sbdt_gpu_find_border_dev(sbdt_gpu_ctx* ctx, const sbdt_border_args* args);

/* ---- merge + update_neighbors --------------------------
 * Inputs: the k partial triangulations (layout of sbdt_gpu_find_border), the
 * border flags B (border[s] != 0: row s is a border simplex — find_border's
 * border_out or positive_out), the border triangulation T_B over B's vertices
 * (tb_verts / tb_nbrs (dim+1) x S_B vertex-major, T_B-local neighbour ids,
 * tb_parity) and labels[i], the partition of point i.
 * Result (SPEC merge): the finite partial rows not in B, then the finite T_B
 * rows whose vertices span >= 2 partitions or whose vertex tuple is a finite
 * row of B, each group in row order; neighbour links rebuilt over the merged
 * set (update_neighbors); facets with a single finite owner are hull facets:
 * kNone (0xFFFFFFFF) links, or, with SBDT_MERGE_HULL, one infinite row per
 * hull facet appended in (owner row, facet) order ({facet ids, 0xFFFFFFFF},
 * parity 0, neighbours[dim] = owner), linked among themselves through their
 * ridges — the reference's Triangulation layout.
 * out_offsets (k+3): rows of part p are [out_offsets[p], out_offsets[p+1]),
 * the inserted T_B rows [out_offsets[k], out_offsets[k+1]), the hull rows
 * [out_offsets[k+1], out_offsets[k+2]).
 * Errors: SBDT_ERR_MERGE (a facet with three owners = InconsistentMerge; a
 * hull ridge without two hull facets = DanglingFacet); SBDT_ERR_RANGE when the
 * result exceeds `capacity` rows (*rows_out then holds the rows needed, or a
 * lower bound of them). Synchronizes the context stream (table sizing). */
enum sbdt_merge_flags { SBDT_MERGE_HULL = 1u };

typedef struct sbdt_merge_args {
  int dim;
  uint32_t k;
  const uint32_t* d_labels;   /* n */
  uint64_t n;
  const uint64_t* d_offsets;  /* k+1 */
  const uint32_t* d_verts;    /* (dim+1) x S */
  const uint32_t* d_nbrs;     /* (dim+1) x S, part-local */
  const int8_t* d_parity;     /* S */
  uint64_t S;
  const uint8_t* d_border;    /* S */
  const uint32_t* d_tb_verts; /* (dim+1) x S_B */
  const uint32_t* d_tb_nbrs;  /* (dim+1) x S_B */
  const int8_t* d_tb_parity;  /* S_B */
  uint64_t S_B;
  uint32_t flags;             /* sbdt_merge_flags */
} sbdt_merge_args;

/* Device outputs, vertex-major with row stride `capacity`. */
int sbdt_gpu_merge_dev(sbdt_gpu_ctx* ctx, const sbdt_merge_args* args, uint64_t capacity, uint32_t* d_out_verts,
                       uint32_t* d_out_nbrs, int8_t* d_out_parity, uint64_t* d_out_offsets, uint64_t* rows_out);

/* Host buffers; outputs vertex-major with row stride *rows_out (compact):
 * out_verts[j * rows + s]. Each out array holds (dim+1) * capacity entries
 * (out_parity: capacity). */
int sbdt_gpu_merge(sbdt_gpu_ctx* ctx, int dim, const uint32_t* labels, uint64_t n, uint32_t k,
                   const uint64_t* offsets, const uint32_t* verts, const uint32_t* nbrs, const int8_t* parity,
                   const uint8_t* border, const uint32_t* tb_verts, const uint32_t* tb_nbrs,
                   const int8_t* tb_parity, uint64_t S_B, uint32_t flags, uint64_t capacity,
                   uint32_t* out_verts, uint32_t* out_nbrs, int8_t* out_parity, uint64_t* out_offsets,
                   uint64_t* rows_out);

/* ---- diagnostics (tests and bench only; not on the path) ----------------- */

/* The device predicates on host arrays (synchronous): op 0 = orient, `pts`
 * holds count x (dim+1) points of dim coordinates, out = sign of
 * orient2/orient3 (geometry.cpp:150-189 / geometry.hpp:112-121 convention);
 * op 1 = in_sphere, count x (dim+2) points (the simplex, then q), out = sign
 * of in_sphere2/in_sphere3 (geometry.cpp:191-277). Binary64 filter, then
 * expansion arithmetic where the filter cannot decide; *n_escalated (may be
 * NULL) = how many cases took the exact path. Replaces no reference entry
 * point: it exposes what find_border evaluates internally so tests can pin it
 * case by case (SPEC.md acceptance criterion 2). */
int sbdt_gpu_predicates(sbdt_gpu_ctx* ctx, int op, int dim, const double* pts, uint64_t count, int8_t* out,
                        uint64_t* n_escalated);

/* Binding-ceiling microbenchmarks on the context's device: kind 0 = DFMA
 * throughput (FLOP/s, 2 per DFMA); kind 1 = random 8-byte gathers from a table
 * of `bytes` bytes (gathers/s). Best of 4 timed launches (CUDA events). */
int sbdt_gpu_microbench(sbdt_gpu_ctx* ctx, int kind, uint64_t bytes, double* result);

#ifdef __cplusplus
}
#endif

#endif /* SBDT_GPU_H_ */
