// tm_internal.h -- launch wrappers shared between the kernel translation units
// and the C-ABI orchestration (tm_capi.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tmb {

struct DevStatus;

// tm_label.cu
size_t hash_bytes(int64_t n, int64_t T, int shrink = 0);  // bytes of the table at scale 2^-min(shrink, 0)
// counts kernels of this library launched (bench.py's gpu_launches)
void note_launch(int k);
// xy32 (nullable): scratch float2[n] for the fp32 LabelMax prefilter (not used with check)
void launch_label_a(const double* xy, int64_t n, const void* tri, int tri_is64, int64_t T, int check,
                    int32_t* tri32, int32_t* hw, int8_t* max_edge, uint8_t* seed, int32_t* tv, void* table,
                    DevStatus* st, cudaStream_t s, int shrink = 0, unsigned int* ovf = nullptr,
                    float* xy32 = nullptr, int one = 0);
void launch_xy32(const double* xy, int64_t n, float* xy32, cudaStream_t s);
// pass A split for copy overlap: prepare (table/trivertex init) once, then triangle ranges
// shrink = 1: half-size twin table (whole path; overflow sets *ovf, the host reruns at full size)
void launch_label_a_prepare(int64_t n, int64_t T, int32_t* tv, void* table, cudaStream_t s, int shrink = 0);
void launch_label_a_range(const double* xy, int64_t n, const void* tri, int tri_is64, int64_t T, int64_t t_begin,
                          int64_t t_end, int check, int32_t* tri32, int32_t* hw, int8_t* max_edge, uint8_t* seed,
                          int32_t* tv, void* table, DevStatus* st, cudaStream_t s, int shrink = 0,
                          unsigned int* ovf = nullptr, const float* xy32 = nullptr, int one = 0);
void launch_label_b(const int32_t* tri32, int64_t n, int64_t T, int32_t* hw, const int8_t* max_edge, uint8_t* seed,
                    int32_t* tv, void* table, int check, DevStatus* st, cudaStream_t s, int shrink = 0,
                    int one = 0);
// one = 1 (unchecked): single-pass labels -- pass A pairs every far edge in
// the table, pass B only scans it for border half-edges
void launch_relabel(const int8_t* max_edge, int64_t T, int32_t* hw, uint8_t* seed, cudaStream_t s);
// seed-partitioned labels (range-local twin table + boundary exchange)
size_t hash_bytes_range(int64_t n, int64_t T, int64_t keyT);
void launch_label_range(const double* xy, int64_t n, const void* tri, int tri_is64, int64_t T, int64_t b, int64_t e,
                        int32_t* tri32, int32_t* hw, int8_t* max_edge, uint8_t* seed, void* table, DevStatus* st,
                        unsigned int* ovf, cudaStream_t s);
void launch_tri32(const void* tri, int tri_is64, int64_t T, int32_t* tri32, cudaStream_t s);
void launch_boundary_extract(const int32_t* tri32, const int8_t* max_edge, const int32_t* hw, int64_t b, int64_t e,
                             unsigned long long* keys, int32_t* vals, unsigned long long* count, int64_t cap,
                             cudaStream_t s);
void launch_boundary_resolve(const unsigned long long* keys, const int32_t* vals, int64_t n_all, int64_t own0,
                             int64_t own1, int32_t* tab, int64_t tab_slots, int32_t* hw, uint8_t* seed,
                             cudaStream_t s);
void launch_check_neighbors(const int32_t* hw, const void* nb, int nb_is64, int64_t T, DevStatus* st, cudaStream_t s);
void launch_unpack(const int32_t* hw, int64_t T, int32_t* twin, uint8_t* fr, cudaStream_t s);
void launch_pack_frontier(int32_t* hw, int64_t T, const uint8_t* fr, cudaStream_t s);

// tm_scan.cu (device-count scans / compaction)
size_t scan_scratch_elems(int64_t n_cap);
void launch_scan_dev(const int64_t* in, int64_t* out, const int64_t* n_dev, int64_t n_cap, int64_t* tile_sums,
                     cudaStream_t s);
void launch_shift(int64_t* a, int64_t n, int64_t delta, cudaStream_t s);
// single-pass (decoupled look-back) exclusive scan of one or two arrays; in1/out1 may be null
size_t scan_lookback_bytes(int64_t n_cap);
// tot0 / tot1 (optional) receive out0[n] / out1[n]; csr_end (optional) gets csr_end[out0[n]] = out1[n]
void launch_scan_lookback(const int64_t* in0, const int64_t* in1, int64_t* out0, int64_t* out1,
                          const int64_t* n_dev, int64_t n_cap, void* scratch, cudaStream_t s, int64_t* tot0 = nullptr,
                          int64_t* tot1 = nullptr, int64_t* csr_end = nullptr);
void launch_gather_at(const int64_t* arr, const int64_t* idx, int64_t* dst, cudaStream_t s);
void launch_select_flags(const uint8_t* flag, int64_t n, int32_t* out, int64_t* n_out, int64_t* tile_sums,
                         cudaStream_t s, int64_t base_index = 0);

// tm_traverse.cu (Pp = device count, Pcap = host bound for the grid)
void launch_trav_start(const int32_t* hw, const int32_t* seeds, const int64_t* Pp, int64_t Pcap, int32_t* start,
                       int32_t* overflow, unsigned int* n_overflow, int32_t* queue, int32_t* stamp, uint32_t* bits,
                       DevStatus* st, cudaStream_t s);
// ruler record of half-edge h (a ruler): next ruler, run length (boundary steps to
// it), previous ruler -- one 16-byte record so each chain step is one sector
struct __align__(16) RulerRec {
  int32_t next, dist, prev, pad;
};
// rulers: starts of the selected seeds + sampled half-edges of triangles [t_begin, t_end)
void launch_ruler_walk(const int32_t* hw, uint32_t* bits, int64_t T, int64_t t_begin, int64_t t_end,
                       const int32_t* start, const int64_t* Pp, int64_t Pcap, RulerRec* R, DevStatus* st,
                       cudaStream_t s);
void launch_chain_count(const int32_t* seeds, const int32_t* start, const int64_t* Pp, int64_t Pcap, int64_t T,
                        const RulerRec* R, int64_t* len, int64_t* nrul,
                        int32_t* long_list, unsigned int* n_long, int4* cc, int64_t cc_cap, DevStatus* st,
                        cudaStream_t s);
void launch_chain_emit(const int32_t* start, const int64_t* Pp, int64_t Pcap, const RulerRec* R,
                       const int64_t* offsets, const int64_t* eoff,
                       int32_t* ent_r, int64_t* ent_base, int64_t ecap, const int4* cc, int64_t cc_cap, DevStatus* st,
                       cudaStream_t s);
void launch_ruler_write(const int32_t* tri, const int32_t* hw, const int64_t* n_entries, const int32_t* ent_r,
                        const int64_t* ent_base, const RulerRec* R, int64_t T, int64_t ecap, int32_t* verts,
                        int32_t* hv, cudaStream_t s);
// the runs of the listed (long) polygons only: entries eoff[i] .. eoff[i + 1]
void launch_ruler_write_list(const int32_t* tri, const int32_t* hw, const int32_t* list, const unsigned int* n_list,
                             const int64_t* eoff, const int32_t* ent_r, const int64_t* ent_base, const RulerRec* R,
                             int64_t T, int64_t Pcap, int32_t* verts, int32_t* hv, cudaStream_t s);

// tm_repair.cu
void launch_stamp(unsigned long long* slot, cudaStream_t s);  // debug timeline (globaltimer)
struct LongQueue {       // work items longer than kLongMin, longest class first
  int32_t* huge;
  int32_t* longq;
  unsigned int* n_huge;
  unsigned int* n_long;
  unsigned int* next;
  int32_t* parked;         // short items whose pinch pass waits for the global guard
  unsigned int* n_parked;
  int32_t* pinchq;         // short items with a pinch candidate left after the tip phase
  unsigned int* n_pinch;
  unsigned int* tip_next;  // work counter of k_repair_tips mode 0 (persistent warps)
  unsigned int* gm_next;   // work counter of k_repair_tips_seg's pool-region blocks
};
// polygons longer than this are classified by k_classify_long (one block each);
// on the whole path the traversal's chain pass lists them
constexpr int kClassifyShort = 48;

struct RepairArgs {
  const int32_t* tri;
  int32_t* hw;
  const int32_t* tv;     // a triangle incident to each polygon vertex (exact lowest iff tv_exact)
  int tv_exact;
  int64_t T;
  int32_t* pool;
  unsigned long long pool_cap;
  unsigned long long* pool_top;
  int32_t* undo;
  unsigned long long* undo_top;
  unsigned long long undo_cap;
  DevStatus* st;
  const int32_t* items;
  const unsigned int* n_items;
  const int64_t* off;
  const int32_t* v;
  int64_t* item_list;
  int32_t* item_n;
  int64_t* item_slots;
  int32_t* item_state;   // 0 todo, 1 done (shared-memory kernel), 2 resume, 3 warp kernel from scratch
  int32_t* item_depth;
  unsigned long long* stats;
  LongQueue q;
  unsigned long long* dbg;  // 64 timestamp slots (debug)
};
// tv[verts[k]] = hv[k] / 3 for every slot of the work items (any incident triangle)
void launch_tv_items(const int64_t* off, const int32_t* v, const int32_t* hv, const int32_t* items,
                     const unsigned int* n_items, int64_t Pcap, int32_t* tv, cudaStream_t s);
// hv (nullable): the traversal's slot half-edges -> tv[vertex] = an incident triangle for work items
void launch_classify(const int64_t* off, const int32_t* v, const int64_t* Pp, int64_t Pcap, int32_t* item_of,
                     int32_t* items, unsigned int* n_items, int32_t* long_list, unsigned int* n_long,
                     unsigned long long* stats, LongQueue q, const int32_t* hv, int32_t* tv, int which,
                     int32_t* item_state, int32_t* pool, unsigned long long* pool_top, unsigned long long pool_cap,
                     int32_t* item_depth, cudaStream_t s);  // item_state[k] = 0 for every item k created  // which: 0 all, 1 short polygons only, 2 the listed long ones only
void launch_repair_tips_long(const RepairArgs& a, cudaStream_t s);
// mode 0: items of length <= kLongMin; mode 1: long items handed back (state 2/3)
void launch_repair_tips(const RepairArgs& a, int mode, cudaStream_t s);
// mode 0: short items, beside the long-item kernel, under the extra visits known
// so far (a lower bound of the global guard; items reaching it are parked);
// mode 1: long items and parked ones, under the global guard
void launch_repair_pinch(const RepairArgs& a, int mode, cudaStream_t s);
void launch_out_counts(const int64_t* off, const int64_t* Pp, int64_t Pcap, const int32_t* item_of,
                       const int32_t* item_n, const int64_t* item_slots, int64_t* cnt, int64_t* slots,
                       const unsigned long long* stats, DevStatus* st, cudaStream_t s);
void launch_stitch(const int64_t* off, const int32_t* v, const int64_t* Pp, int64_t Pcap, const int32_t* item_of,
                   const int32_t* items, const unsigned int* n_items, const int64_t* item_list, const int32_t* item_n,
                   const int32_t* pool, const int64_t* pbase, const int64_t* sbase, int64_t* off_out, int32_t* v_out,
                   cudaStream_t s);
// the final CSR by units (runs of untouched polygons + the work item after each)
void launch_item_sort(const int32_t* item_of, const int64_t* Pp, int64_t Pcap, uint8_t* flag, int32_t* srt,
                      int64_t* n_srt, int64_t* tiles, cudaStream_t s);
void launch_unit_counts(const int64_t* off, const int64_t* Pp, int64_t Pcap, const int32_t* srt, const int64_t* n_srt,
                        const int32_t* item_of, const int32_t* item_n, const int64_t* item_slots, int64_t* cnt,
                        int64_t* slots, int64_t* n_units, const unsigned long long* stats, DevStatus* st,
                        cudaStream_t s);
void launch_stitch_units(const int64_t* off, const int32_t* v, const int64_t* Pp, const int32_t* srt,
                         const int64_t* n_srt, const int32_t* item_of, const int64_t* item_list, const int32_t* item_n,
                         const int32_t* pool, const int64_t* pbase, const int64_t* sbase, int64_t* off_out,
                         int32_t* v_out, cudaStream_t s);
void launch_finalize(const int64_t* Pp, const int64_t* pbase, const int64_t* sbase, int64_t* off_out,
                     int64_t* p_out, int64_t* f_out, cudaStream_t s);
void launch_undo(int32_t* hw, const int32_t* undo, const unsigned long long* undo_top, unsigned long long cap,
                 cudaStream_t s);

// tm_post.cu (validation, polygon analytics, canonical form)
void launch_check_trivertex(const void* tri, int tri_is64, int64_t T, const int64_t* tv, int64_t n, uint32_t* bits,
                            DevStatus* st, cudaStream_t s);
void launch_max_vertex(const int32_t* v, int64_t F, int* out, cudaStream_t s);
void launch_mark_vertices(const int32_t* v, int64_t F, int64_t n, uint8_t* flag, DevStatus* st, cudaStream_t s);
void launch_edge_set(const int64_t* off, int64_t P, const int32_t* v, unsigned long long* table, int64_t table_slots,
                     unsigned long long* count, cudaStream_t s);
void launch_poly_flags(const int64_t* off, int64_t P, const int32_t* v, uint8_t* tip, uint8_t* rep,
                       unsigned long long* extra, int32_t* long_list, unsigned int* n_long, int32_t* stamp,
                       cudaStream_t s);
void launch_poly_areas(const int64_t* off, int64_t P, const int32_t* v, const double* xy, double* area,
                       cudaStream_t s);
void launch_canon_rot(const int64_t* off, int64_t P, const int32_t* v, int64_t n, int32_t* rot, int32_t* bucket,
                      unsigned long long* hist, DevStatus* st, cudaStream_t s);
void launch_canon_sort(int64_t P, int64_t n, const int64_t* off, const int32_t* v, const int32_t* rot,
                       const int32_t* bucket, const int64_t* start, unsigned long long* cursor, int32_t* order,
                       cudaStream_t s);
void launch_canon_lengths(const int32_t* order, int64_t P, const int64_t* off, int64_t* len, cudaStream_t s);
void launch_canon_write(const int32_t* order, int64_t P, const int64_t* off, const int32_t* v, const int32_t* rot,
                        const int64_t* off_out, int32_t* v_out, cudaStream_t s);

// tm_delaunay.cu (GPU Delaunay input generation)
void launch_delaunay_cells(const double* xy, int64_t n, double x0, double y0, double x1, double y1, int G,
                           int32_t* cell, unsigned long long* hist, cudaStream_t s);
void launch_delaunay_scatter(const double* xy, int64_t n, int G, const int32_t* cell, const int64_t* start,
                             unsigned long long* cursor, int32_t* ids, double* sxy, cudaStream_t s);
void launch_delaunay_stars(const int64_t* start, const int32_t* ids, const double* sxy, int64_t n, double x0,
                           double y0, double x1, double y1, int G, int mode, int64_t* cnt, const int64_t* off,
                           int32_t* tri, int32_t* open_list, unsigned int* n_open, unsigned int* n_degenerate,
                           cudaStream_t s);

}  // namespace tmb
