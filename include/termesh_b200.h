/*
 * termesh_b200.h -- C ABI of the B200 (sm_100a) mesh -> polygons path.
 *
 * Drop-in boundary for the reference `termesh` package's phase functions
 * (paths relative to /root/reference/pkg/src/termesh):
 *
 *   tm_label            replaces labeling.label_all        (labeling.py:118-145)
 *                       + mesh_core.compute_trivertex      (mesh_core.py:171-178)
 *                       + the twin/back-slot searches      (mesh_core.py:132-149,
 *                         labeling.py:84,110, traversal.py:250-256)
 *   tm_check_neighbors  the neighbor-reciprocity part of   mesh_core.validate (mesh_core.py:237-263)
 *   tm_traverse         replaces traversal.build_polygon_mesh (traversal.py:303-347)
 *   tm_repair           replaces reparation.repair_all     (reparation.py:343-377)
 *   tm_mesh_to_polygons_host
 *                       the timed part of pipeline.execute (pipeline.py:137-148)
 *                       from host arrays in the reference dtypes.
 *
 * Conventions
 *   - Pointers named d_* are device pointers owned by the caller (e.g. torch
 *     tensors); the library never frees caller memory.  Internal scratch is
 *     owned by the tm_ctx.  `stream` is a cudaStream_t (NULL = legacy stream).
 *   - Triangles: corners CCW, half-edge h = 3t + j is the edge opposite corner
 *     j, origin corner (j+1)%3, target (j+2)%3 (mesh_core.py:1-14).
 *   - Packed half-edge word (int32[3T]): (twin << 1) | frontier, border = -1.
 *   - Polygon meshes are CSR: offsets int64[P+1], verts int32[offsets[P]];
 *     polygon i = verts[offsets[i] .. offsets[i+1]), CCW, in the reference's
 *     SEQUENTIAL raw order and rotation.
 *   - Every call returns a status code.  Messages: tm_ctx_last_error();
 *     per-kind defect counts / first element: tm_ctx_defects().
 *     Status codes map onto the reference's exceptions:
 *       TM_ERR_STRUCTURAL -> errors.StructuralError  (errors.py:8-16)
 *       TM_ERR_VALIDATION -> errors.ValidationError  (errors.py:19-25)
 *       TM_ERR_ARGUMENT   -> ValueError
 */
#ifndef TERMESH_B200_H
#define TERMESH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TM_OK 0
#define TM_ERR_STRUCTURAL 1
#define TM_ERR_VALIDATION 2
#define TM_ERR_CAPACITY 3
#define TM_ERR_CUDA 4
#define TM_ERR_ARGUMENT 5

/* defect kinds reported by tm_ctx_defects (index into the 16-entry arrays);
 * 0..6 are the kinds of mesh_core.ValidationReport (mesh_core.py:28-35) */
#define TM_KIND_INDEX_RANGE 0
#define TM_KIND_ORIENTATION 1
#define TM_KIND_DEGENERATE 2
#define TM_KIND_DUPLICATE 3
#define TM_KIND_RECIPROCITY 4
#define TM_KIND_EDGE_COUNT 5
#define TM_KIND_TRIVERTEX 6
#define TM_KIND_NEIGHBORS 7
#define TM_KIND_WALK 8
#define TM_KIND_NO_FRONTIER 9
#define TM_KIND_NO_CONVERGE 10
#define TM_KIND_SPLIT_LAW 11
#define TM_KIND_POOL 12
#define TM_KIND_BARRIER 13
#define TM_KIND_NO_INTERNAL 14
#define TM_KIND_STRUCT 15
#define TM_NUM_KINDS 16

/* repair statistics (tm_repair / tm_mesh_to_polygons* `stats`, int64[TM_NUM_STATS]);
 * 0..3 are repair_all's stats_out keys (reparation.py:372-376) */
#define TM_STAT_ROUNDS 0
#define TM_STAT_SPLITS 1
#define TM_STAT_INITIAL_TIPS 2
#define TM_STAT_UNREPAIRED 3
#define TM_STAT_NONSIMPLE 4 /* pipeline.py:150 nonsimple_after_traversal */
#define TM_STAT_TIP_SPLITS 5
#define TM_STAT_PINCH_SPLITS 6
#define TM_STAT_WORK_ITEMS 7
/* the pinch pass's round guard (reparation.py:322) is GLOBAL: extra visits of
 * the tip-phase output + 1.  A seed partition (tm_ctx_set_partition) knows only
 * its own share (PINCH_EXTRA): items that reach the local guard with pinched
 * polygons left are parked (PINCH_DEFERRED); after the ranks exchange their
 * PINCH_EXTRA, tm_resume_pinch finishes them under the global guard, so the
 * stitched result equals the single-GPU one.  PINCH_TRUNCATED counts the items
 * the (final) guard cut off. */
#define TM_STAT_PINCH_EXTRA 8
#define TM_STAT_PINCH_TRUNCATED 9
/* seed partition only: items parked at the final LOCAL guard; when > 0 the
 * call's output is provisional and tm_resume_pinch must follow */
#define TM_STAT_PINCH_DEFERRED 10
#define TM_NUM_STATS 11

typedef struct tm_ctx tm_ctx;

int tm_version(void);
int tm_ctx_create(tm_ctx **out);
void tm_ctx_destroy(tm_ctx *ctx);
const char *tm_ctx_last_error(const tm_ctx *ctx);
int tm_ctx_defects(const tm_ctx *ctx, int64_t *counts, int64_t *first); /* TM_NUM_KINDS each */
/* per-phase device milliseconds of the last tm_mesh_to_polygons* call:
 * [0] label (K0+K1+K2), [1] traversal (K3), [2] reparation + stitch (K4) */
int tm_ctx_phase_ms(const tm_ctx *ctx, double *ms3);
/* device milliseconds of the last tm_label call: [0] pass A (twin insert +
 * LabelMax, labeling.py:46-62), [1] pass B (twin lookup + LabelSeed and
 * LabelFrontier fused, labeling.py:65-115) -- the reference's kernel_seconds */
int tm_ctx_label_ms(const tm_ctx *ctx, double *ms2);

/* Optional per-kernel device timing: CUDA events around each kernel group on
 * the launching stream.  tm_ctx_segment_ms flushes and returns the number of
 * segments; names from tm_segment_name(k).  tm_launch_count() counts this
 * library's own kernel launches (process-wide). */
int tm_ctx_set_profiling(tm_ctx *ctx, int on);
int tm_ctx_segment_ms(tm_ctx *ctx, double *ms, int64_t *counts, int n, int reset);
const char *tm_segment_name(int k);
int64_t tm_launch_count(void);
/* Seed partition for multi-GPU runs: traversal, repair and
 * stitch of this context only cover the polygons whose seed triangle lies in
 * [t_begin, t_end) (t_end = -1: up to T); labels always cover the whole mesh.
 * With ranks owning consecutive ranges, the concatenation of their outputs in
 * rank order is the single-GPU output (seed order = raw order, F13). */
int tm_ctx_set_partition(tm_ctx *ctx, int64_t t_begin, int64_t t_end);
/* Seed partition, second phase: finish the items the last tm_mesh_to_polygons*
 * call parked at its local pinch guard, under the global guard
 * extra_total + 1 (extra_total = sum of every rank's TM_STAT_PINCH_EXTRA), and
 * rewrite the output CSR.  off_out / v_out are device buffers after
 * tm_mesh_to_polygons, host buffers after tm_mesh_to_polygons_host; the
 * capacities are those of the first call.  Reference: reparation.py:315-340. */
int tm_resume_pinch(tm_ctx *ctx, int64_t extra_total, int64_t *off_out, int32_t *v_out, int64_t cap_polys,
                    int64_t cap_slots, int64_t *n_polys, int64_t *n_slots, int64_t *stats, void *stream);
/* Seed-partitioned labels ("each GPU labels its own edge
 * range").  tm_label_range labels triangles [t_begin, t_end) into the
 * context's own buffers with a range-local twin table (and converts the
 * corners of the whole mesh) and lists the range's still-unpaired half-edges
 * -- border or partner in another range -- as boundary entries (key
 * (lo << 32) | hi, value (h << 1) | longest-edge flag, into caller buffers of
 * `cap` entries; a padding key ~0 is ignored by tm_label_resolve).  After the ranks all-gather their entries
 * (this rank's at [own_begin, own_begin + own_count) of the concatenation),
 * tm_label_resolve labels the cross-range pairs of this rank's half-edges.
 * Once the ranks' hw / seed / max_edge chunks are all-gathered into the
 * context buffers, tm_polygons_from_labels runs the traversal, repair and
 * stitch of the context's seed partition (no label phase). */
int tm_label_range(tm_ctx *ctx, const double *d_xy, int64_t n_vertices, const void *d_tri, int tri_bits, int64_t T,
                   int64_t t_begin, int64_t t_end, uint64_t *d_boundary_keys, int32_t *d_boundary_vals, int64_t cap,
                   int64_t *n_boundary, void *stream);
int tm_ctx_label_buffers(tm_ctx *ctx, int32_t **d_tri32, int32_t **d_halfedge, int8_t **d_max_edge, uint8_t **d_seed);
/* copy the label state of triangles [t_begin, t_end) between caller arrays of
 * the whole mesh (hw int32[3T], seed uint8[T], max_edge int8[T]; any may be
 * NULL) and the context's: to_ctx = 1 caller -> context, 0 context -> caller */
int tm_ctx_copy_labels(tm_ctx *ctx, int to_ctx, int32_t *d_halfedge, uint8_t *d_seed, int8_t *d_max_edge,
                       int64_t t_begin, int64_t t_end, void *stream);
int tm_label_resolve(tm_ctx *ctx, const uint64_t *d_keys_all, const int32_t *d_vals_all, int64_t n_all,
                     int64_t own_begin, int64_t own_count, void *stream);
int tm_polygons_from_labels(tm_ctx *ctx, int64_t n_vertices, int64_t T, int64_t *d_offsets, int32_t *d_verts,
                            int64_t cap_polys, int64_t cap_slots, int64_t *n_polys, int64_t *n_slots, int64_t *stats,
                            void *stream);
/* d_offsets[0..n_polys] += delta: places a rank's CSR at its global slot base
 * (the exclusive prefix of the all-gathered per-rank slot counts). */
int tm_shift_offsets(int64_t *d_offsets, int64_t n_polys, int64_t delta, void *stream);
/* kernel debug timestamps (ns, %globaltimer) of the last run: repair lineage trace */
int tm_ctx_debug(const tm_ctx *ctx, uint64_t *out, int n);
/* Debug hook (determinism hunts): copy an internal buffer of the last whole-path
   run to device memory dst -- which: 0 pre-repair offsets, 1 pre-repair
   vertices, 2 packed half-edge words, 3 slot half-edges, 4 seed flags. */
int tm_ctx_debug_copy(const tm_ctx *ctx, int which, void *dst, size_t bytes);

/* Labels.  tri_bits = 32 or 64 (reference triangles are int64).  check != 0
 * also reports index_range / orientation / degenerate / edge_count /
 * reciprocity defects as TM_ERR_VALIDATION.
 * Outputs (device): d_tri32 int32[3T] (may equal d_tri when tri_bits == 32),
 * d_halfedge int32[3T], d_max_edge int8[T], d_seed uint8[T], d_trivertex int32[n]. */
int tm_label(tm_ctx *ctx, const double *d_xy, int64_t n_vertices, const void *d_tri, int tri_bits, int64_t T,
             int check, int32_t *d_tri32, int32_t *d_halfedge, int8_t *d_max_edge, uint8_t *d_seed,
             int32_t *d_trivertex, void *stream);

/* Recompute frontier bits and seeds from a caller max_edge (labeling.py:65-115
 * with a given max_edge); d_halfedge must hold packed words from tm_label. */
int tm_relabel(tm_ctx *ctx, int32_t *d_halfedge, const int8_t *d_max_edge, int64_t T, uint8_t *d_seed, void *stream);

/* neighbors[h] must equal twin[h] / 3 (or -1): TM_ERR_VALIDATION otherwise */
int tm_check_neighbors(tm_ctx *ctx, const int32_t *d_halfedge, const void *d_neighbors, int nb_bits, int64_t T,
                       void *stream);

/* expand packed words to the reference arrays (either output may be NULL) */
int tm_unpack_halfedges(tm_ctx *ctx, const int32_t *d_halfedge, int64_t T, int32_t *d_twin, uint8_t *d_frontier,
                        void *stream);
/* overwrite the frontier bits from a caller frontier array (bool/uint8 [3T]) */
int tm_pack_frontier(tm_ctx *ctx, int32_t *d_halfedge, const uint8_t *d_frontier, int64_t T, void *stream);

/* Traversal.  Capacities: cap_polys >= T and cap_slots >= 3T are REQUIRED
 * (TM_ERR_ARGUMENT otherwise; the output sizes are only known on the device,
 * #seeds <= T and #frontier half-edges <= 3T, and d_offsets needs cap_polys + 1
 * entries).  *n_polys / *n_slots are host outputs;
 * the call synchronizes `stream` before returning them. */
int tm_traverse(tm_ctx *ctx, const int32_t *d_tri32, const int32_t *d_halfedge, const uint8_t *d_seed, int64_t T,
                int64_t *d_offsets, int32_t *d_verts, int64_t cap_polys, int64_t cap_slots, int64_t *n_polys,
                int64_t *n_slots, void *stream);

/* Repair.  Mutates the frontier bits of d_halfedge exactly as repair_all
 * mutates labels.frontier.  Capacities cap_polys >= T and cap_slots >= 3T are
 * required (as for tm_traverse; the repaired output never exceeds them).  stats: host
 * int64[TM_NUM_STATS]. */
int tm_repair(tm_ctx *ctx, const int32_t *d_tri32, int32_t *d_halfedge, const int32_t *d_trivertex, int64_t T,
              const int64_t *d_offsets_in, const int32_t *d_verts_in, int64_t n_polys, int64_t *d_offsets_out,
              int32_t *d_verts_out, int64_t cap_polys, int64_t cap_slots, int64_t *n_polys_out, int64_t *n_slots_out,
              int64_t *stats, void *stream);

/* Whole path from HOST arrays in the reference dtypes (Triangulation.vertices
 * f64[2n], Triangulation.triangles i64[3T]); host->device copies, label,
 * traversal, repair and the device->host copy of the final CSR all happen
 * inside.  Output capacities T+1 / 3T always suffice.  Pinned host buffers
 * give full PCIe bandwidth. */
int tm_mesh_to_polygons_host(tm_ctx *ctx, const double *h_vertices, int64_t n_vertices, const int64_t *h_triangles,
                             int64_t T, int check, int64_t *h_offsets, int32_t *h_verts, int64_t cap_polys,
                             int64_t cap_slots, int64_t *n_polys, int64_t *n_slots, int64_t *stats);

/* Same pipeline on caller device buffers (no host copies). */
int tm_mesh_to_polygons(tm_ctx *ctx, const double *d_xy, int64_t n_vertices, const void *d_tri, int tri_bits,
                        int64_t T, int check, int64_t *d_offsets, int32_t *d_verts, int64_t cap_polys,
                        int64_t cap_slots, int64_t *n_polys, int64_t *n_slots, int64_t *stats, void *stream);

/* ---------------------------------------------------------------- around the path
 * Validation, polygon analytics and the canonical output form on the device
 * (paths relative to /root/reference/pkg/src/termesh). */

/* mesh_core.validate's trivertex rule (mesh_core.py:268-283): d_trivertex
 * int64[n]; TM_ERR_VALIDATION (kind TM_KIND_TRIVERTEX, first bad vertex) if an
 * entry is outside [-1, T), -1 for a referenced vertex, or a triangle that
 * does not contain the vertex. */
int tm_check_trivertex(tm_ctx *ctx, const void *d_tri, int tri_bits, int64_t T, const int64_t *d_trivertex,
                       int64_t n_vertices, void *stream);

/* Polygon-mesh analytics of traversal.py over a device CSR (vertex ids in
 * [0, n_vertices)): per-polygon tip flags (tip_flags, :112-124) and repeated-
 * vertex flags (repeated_vertex_flags, :127-137) into the optional uint8[P]
 * outputs, extra_vertex_visits (:140-147), the sorted distinct vertex ids
 * (unique_vertices, :150-153; optional int32[n_vertices] output) and their
 * count, and boundary_edge_count (:156-166).  n_vertices < 0: derived from
 * the largest id.  Synchronizes `stream`. */
int tm_polygon_stats(tm_ctx *ctx, const int64_t *d_offsets, const int32_t *d_verts, int64_t n_polys,
                     int64_t n_vertices, uint8_t *d_tip, uint8_t *d_repeated, int32_t *d_unique,
                     int64_t *extra_visits, int64_t *unique_vertices, int64_t *boundary_edges, void *stream);

/* enclosed_signed_areas (traversal.py:94-109): shoelace area per polygon in
 * numpy's summation order (np.add.reduceat, pairwise), d_area f64[P]. */
int tm_polygon_areas(tm_ctx *ctx, const int64_t *d_offsets, const int32_t *d_verts, int64_t n_polys,
                     const double *d_xy, double *d_area, void *stream);

/* oracle.canonicalize (oracle.py:124-141): every polygon rotated to its
 * lexicographically smallest rotation, polygons in Python tuple order.  Output
 * CSR d_offsets_out int64[P+1], d_verts_out int32[offsets[P]].  Counting sort
 * on the minimum vertex, then a lexicographic sort inside each bucket.
 * n_vertices < 0: derived from the largest id.  Synchronizes `stream`. */
int tm_canonicalize(tm_ctx *ctx, const int64_t *d_offsets, const int32_t *d_verts, int64_t n_polys,
                    int64_t n_vertices, int64_t *d_offsets_out, int32_t *d_verts_out, void *stream);

/* ---------------------------------------------------------------- GPU Delaunay (input generation)
 * Delaunay triangulation of n points inside box = {x0, y0, x1, y1}, which
 * must lie on the 2^-53 grid of [0, 1) (numpy uniform draws) for the exact
 * predicates (the reference uses Qhull,
 * io_formats.py:351-388).  Writes the CCW triangles whose smallest-index
 * vertex has a certified star (d_tri int32[3 * cap_tris]) and lists the points
 * whose star could not be certified locally (d_open int32[n]: the hull
 * region, triangulated by the caller).  *n_degenerate counts cocircular /
 * collinear ties (no unique triangulation). */
int tm_delaunay(tm_ctx *ctx, const double *d_xy, int64_t n, const double *box, int32_t *d_tri, int64_t cap_tris,
                int64_t *n_tris, int32_t *d_open, int64_t *n_open, int64_t *n_degenerate, void *stream);

/* ---------------------------------------------------------------- multi-GPU exchange
 * One NCCL communicator per rank (one process per GPU).  Rank 0 makes the
 * unique id (tm_comm_id_bytes() bytes), the host broadcasts it, every rank
 * calls tm_comm_init.  NCCL is bound at run time (libnccl.so.2).  The
 * seed-partitioned path exchanges each rank's (polygons, slots, pinch extra
 * visits, deferred items) with tm_comm_allgather and places its CSR at the
 * exclusive prefix (tm_shift_offsets). */
typedef struct tm_comm tm_comm;
int tm_comm_id_bytes(void);
int tm_comm_unique_id(void *id_out);
int tm_comm_init(tm_comm **out, int rank, int world, const void *id, int device);
/* d_recv[r * bytes_per_rank ...] = rank r's d_send (device buffers, on `stream`) */
int tm_comm_allgather(tm_comm *comm, const void *d_send, void *d_recv, size_t bytes_per_rank, void *stream);
void tm_comm_destroy(tm_comm *comm);
const char *tm_comm_last_error(void);

/* ---------------------------------------------------------------- host-side text I/O (no GPU)
 * Python repr(float) of x into out (io_formats.py:44-46); returns the length, -1 if cap is too small */
int tm_format_double(double x, char *out, size_t cap);
/* Triangle file readers (io_formats.py:48-158): kind 0 .node (f64[2*rows]),
 * 1 .ele / 2 .neigh (int64[3*rows], unnormalized), 3 .trivertex (int64[rows];
 * n_expected = vertex count).  Same comment / whitespace / header rules and
 * ParseError messages as the reference; tm_file_status returns 1 with
 * (line, message) on a parse error. */
typedef struct tm_file tm_file;
tm_file *tm_file_read(const char *path, int kind, int64_t n_expected);
int tm_file_status(const tm_file *f, int64_t *rows, int64_t *cols, int64_t *err_line, char *msg, size_t cap);
int tm_file_copy(const tm_file *f, void *dst);
void tm_file_close(tm_file *f);
/* write_polymesh (io_formats.py:251-262) of an already canonical CSR: header,
 * repr coordinates, polygon rows; byte-identical to the reference */
int tm_write_polymesh(const char *path, const double *xy, int64_t n_vertices, const int64_t *offsets,
                      const int32_t *verts, int64_t n_polys, char *err, size_t err_cap);
/* one file of write_triangulation (io_formats.py:213-248): which 0 .node (xy),
 * 1 .ele, 2 .neigh (rows3 int64[3*count]), 3 .trivertex (rows3 int64[count]) */
int tm_write_triangle_file(const char *path, int which, const double *xy, const int64_t *rows3, int64_t count,
                           char *err, size_t err_cap);

#ifdef __cplusplus
}
#endif
#endif
