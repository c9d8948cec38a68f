// tm_capi.cu -- extern "C" entry points (include/termesh_b200.h) and the host
// orchestration of the device phases.
//
// Every phase is *enqueued* without host round trips: element counts stay in
// device memory (a Counters block) and every kernel reads them from there, with
// host-known upper bounds (T, 3T) sizing the grids.  The whole mesh -> polygons
// path is therefore captured once as a CUDA graph and replayed; the host reads
// the counters (status, counts, repair stats) once at the end.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/termesh_b200.h"
#include "tm_common.cuh"
#include "tm_internal.h"

using namespace tmb;

namespace {

// Every (re)allocation of a library buffer bumps this generation: a captured
// graph and the "stamp buffer is all -1" fact are only valid for the
// generation they were made in (cudaFree + cudaMalloc may return the same address).
std::atomic<unsigned long long> g_alloc_gen{1};

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  unsigned long long gen = 0;  // g_alloc_gen value of the current allocation
  bool ensure(size_t want) {
    if (want <= bytes && p) return true;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    gen = g_alloc_gen.fetch_add(1) + 1;
    size_t b = want < 256 ? 256 : want;
    if (cudaMalloc(&p, b) != cudaSuccess) return false;
    bytes = b;
    return true;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// Device-side counters of one pipeline run (reset at the start of a run).
struct Counters {
  DevStatus st;
  int64_t n_seeds;     // P: polygons after traversal
  int64_t n_slots0;    // F: vertex slots after traversal
  int64_t n_entries;   // ruler entries
  int64_t p_in;        // repair input polygon count (tm_repair called with a host count)
  int64_t p_out;       // P': polygons after repair
  int64_t f_out;       // F': vertex slots after repair
  unsigned int n_overflow, n_items, n_long, n_pinch;
  unsigned int q_huge, q_long, q_next, n_parked;
  unsigned int tip_next, table_ovf, gm_next, pad3;
  unsigned long long pool_top, undo_top;
  // stats[0..7]: repair statistics (fill_stats); stats[8]: extra visits of the
  // other ranks (host-set before tm_resume_pinch); stats[9]: seed partition,
  // park items at the final local pinch guard (host-set in the reset image);
  // stats[10]: items parked there (deferred to tm_resume_pinch); stats[11]: local
  // guard cap (testing hook TERMESH_PINCH_GUARD_CAP, partitions only)
  unsigned long long stats[12];
  unsigned long long dbg[128];  // optional kernel timestamps / counters (tm_ctx_debug)
  // tm_polygon_stats / tm_canonicalize: extra visits, boundary edges, long-polygon
  // count, unique vertex count (int64), bucket count (int64)
  unsigned long long post_extra, post_edges;
  unsigned int post_nlong, post_pad;
  int64_t post_unique, post_nb;
  // tm_delaunay: cell count, point count, triangle total, open / degenerate stars
  int64_t dl_ncell, dl_n, dl_ntri;
  unsigned int dl_open, dl_degen;
  unsigned long long n_boundary;  // tm_label_range: boundary entries of the rank
  int64_t n_isrt, n_units;         // stitch: work items in polygon order, units (runs + items)
};

constexpr int kUploadChunks = 8;  // triangle upload chunks of tm_mesh_to_polygons_host
constexpr int kRetryTable = 100;  // internal: rerun the call with a twin table twice the size
constexpr int kMinShrink = -3;    // twin table at most 8x the full size

enum Seg {
  S_LABEL_A, S_LABEL_B, S_SEEDS, S_TRAV_START, S_TRAV_RULERS, S_TRAV_LEN, S_TRAV_SCAN, S_TRAV_WRITE,
  S_CLASSIFY, S_REPAIR_TIPS, S_REPAIR_PINCH, S_STITCH, S_NUM
};
const char* kSegNames[S_NUM] = {"label_a_tri_pass", "label_b_edges", "select_seeds", "trav_start", "trav_rulers",
                                "trav_chain", "trav_scan", "trav_write", "repair_classify", "repair_tips",
                                "repair_pinch", "repair_stitch"};

struct Prof {
  bool on = false;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
  std::vector<cudaEvent_t> free_ev;
  double ms[S_NUM] = {0};
  long long cnt[S_NUM] = {0};
};

std::atomic<long long> g_launches{0};

struct GraphKey {
  const void* xy = nullptr;
  const void* tri = nullptr;
  void* off = nullptr;
  void* v = nullptr;
  int64_t n = -1, T = -1, tb = 0, te = 0;
  int bits = 0, check = 0, ext = 0;
  unsigned long long pool_cap = 0;
  unsigned long long alloc_gen = 0;  // no library buffer reallocated since the capture
  bool operator==(const GraphKey& o) const {
    return xy == o.xy && tri == o.tri && off == o.off && v == o.v && n == o.n && T == o.T && tb == o.tb &&
           te == o.te && bits == o.bits && check == o.check && ext == o.ext && pool_cap == o.pool_cap &&
           alloc_gen == o.alloc_gen;
  }
};

}  // namespace

namespace tmb {
void note_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace tmb

struct tm_ctx {
  Prof prof;
  std::string err;
  int64_t defect_count[K_NUM] = {0};
  int64_t defect_first[K_NUM] = {0};
  double phase_ms[3] = {0, 0, 0};
  Buf counters;
  Counters* h_reset = nullptr;   // pinned, constant reset image
  Counters* h_result = nullptr;  // pinned, D2H target
  int64_t* h_pin = nullptr;      // pinned scratch (host counts for tm_repair)
  // label
  Buf slots, lbscan;
  // traversal
  Buf seeds, start, len, overflow, queue, stamp, tiles, nrul, eoff, rulers, startbits, ent_r, ent_base, ccache;
  int64_t cc_cap = 0;  // seeds whose short chains k_chain_count caches for k_chain_emit
  // repair
  Buf item_of, items, long_list, item_list, item_n, item_slots, item_state, item_depth, cnt, slotsz, pbase, sbase, pool,
      undo, hugeq, longq, parked, pinchq, iflag, isrt, itiles;
  // whole-path buffers
  Buf xy, tri, tri32, hw, max_edge, seed, tv, off0, v0, fin_off, fin_v, hw_snap, hv;
  // tm_post.cu scratch (validation, analytics, canonical form)
  Buf pbits, pflag, ptable, pstamp, ptip, prep, plong, prot, pbucket, porder, phist, pstart, pcursor, plen, ptiles;
  // tm_delaunay scratch
  Buf dcell, dhist, dstart, dcursor, dids, dsxy, dcnt, doff;
  // fp32 copy of the coordinates for the LabelMax prefilter: measured neutral to
  // slightly slower at 1M / 10M (the label pass is not bound by the coordinate
  // gathers), so off unless TERMESH_XY32=1
  Buf xy32;
  int use_xy32 = 0;
  unsigned long long pstamp_clean = 0;  // allocation generation of the all-INT_MAX stamp buffer
  cudaStream_t gstream = nullptr;
  cudaStream_t aux = nullptr;                            // long repair items run beside the short ones
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_cls = nullptr;
  // whole-path runs: the long polygons are written, classified and repaired on
  // ctx->aux right after the traversal's chain pass (enqueue_traverse)
  bool early_long = false;
  // whole path: half-size twin table (block-local matching leaves ~43% of the keys
  // to it); an overflow reruns the call at full size and keeps that for this ctx
  int table_shrink = 1;  // 2^-s buckets; lowered by one on every displacement overflow
  unsigned long long stamp_clean = 0;  // allocation generation of the stamp buffer known to be all -1
  int label_shrink = 0;  // what the label kernels of the current call use
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t graph = nullptr;
  GraphKey gkey;
  unsigned long long pool_cap = 0;
  int64_t ecap = 0;
  int use_graph = 1;
  int64_t part_begin = 0, part_end = -1;  // seed partition [begin, end) in triangles (-1: T)
  // whole-path runs: the traversal records each slot's boundary half-edge
  // (hv) and repair derives its fan starts from it instead of a trivertex
  int32_t* path_hv = nullptr;
  // host-array runs: counters reset and label pass A were enqueued by the
  // caller, chunk by chunk behind the triangle upload (copy/compute overlap)
  bool label_a_external = false;
  // host-array entry: pinned int32 staging of the triangles (host-side narrowing)
  int32_t* h_tri32 = nullptr;
  int64_t h_tri32_cap = 0;
  // measured: no gain at 10M (19.2 vs 19.4 ms e2e), +0.6 ms at 1M (thread start-up): the
  // host-side narrowing pass costs about what it saves on PCIe.  Off unless TERMESH_NARROW=1.
  bool host_narrow = false;
  // single-pass labels (tm_label.cu single_pass): -1 host-array entry only
  // (pass A overlaps the upload), 0 never, 1 every unchecked call (TERMESH_LABEL_ONE)
  int label_one = -1;
  // seed-partitioned labels: tri32 / hw / max_edge / seed of the whole mesh were
  // filled by tm_label_range + tm_label_resolve + the ranks' all-gather
  bool labels_external = false;
  Buf btab;  // boundary-entry resolution table
  cudaStream_t cstream = nullptr;
  cudaEvent_t chunk_ev[kUploadChunks] = {};
  long long graph_kernels = 0;  // kernels per graph replay (counted at capture)
  // tm_label: events around pass A (twin insert + LabelMax) and pass B (twin
  // lookup + LabelSeed/LabelFrontier), read by tm_ctx_label_ms
  bool label_timing = false;
  cudaEvent_t lev[3] = {nullptr, nullptr, nullptr};
  double label_ms[2] = {0, 0};
  // the last whole-path call, for tm_resume_pinch
  int64_t last_T = -1;
  bool last_host = false;
};

// host threads for a host-side pass over `work` elements
static int host_workers(int64_t work) {
  unsigned hc = std::thread::hardware_concurrency();
  int t = hc ? (int)hc : 1;
  if (t > 16) t = 16;
  const int64_t need = work / (1 << 20) + 1;
  return (int)(need < t ? need : t);
}

static int set_err(tm_ctx* c, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

static int cuda_fail(tm_ctx* c, cudaError_t e, const char* where) {
  return set_err(c, TM_ERR_CUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
}

#define CK(call)                                             \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call); \
  } while (0)

#define ENSURE(buf, bytes)                                                                                   \
  do {                                                                                                       \
    if (!ctx->buf.ensure(bytes))                                                                             \
      return set_err(ctx, TM_ERR_CUDA, "cudaMalloc of %zu bytes for %s failed", (size_t)(bytes), #buf);     \
  } while (0)

static Counters* dc_of(tm_ctx* ctx) { return ctx->counters.as<Counters>(); }

// ---------------------------------------------------------------- profiling
static cudaEvent_t prof_event(tm_ctx* ctx) {
  if (!ctx->prof.free_ev.empty()) {
    cudaEvent_t e = ctx->prof.free_ev.back();
    ctx->prof.free_ev.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct SegTimer {  // CUDA events on the launching stream around a kernel group
  tm_ctx* ctx;
  int seg;
  cudaStream_t s;
  cudaEvent_t b = nullptr;
  SegTimer(tm_ctx* c, int sg, cudaStream_t st) : ctx(c), seg(sg), s(st) {
    if (ctx->prof.on) {
      b = prof_event(ctx);
      cudaEventRecord(b, s);
    }
  }
  ~SegTimer() {
    if (b) {
      cudaEvent_t e = prof_event(ctx);
      cudaEventRecord(e, s);
      ctx->prof.pending.emplace_back(seg, b, e);
    }
  }
};

static void prof_flush(tm_ctx* ctx) {
  for (auto& t : ctx->prof.pending) {
    float ms = 0;
    cudaEventSynchronize(std::get<2>(t));
    cudaEventElapsedTime(&ms, std::get<1>(t), std::get<2>(t));
    ctx->prof.ms[std::get<0>(t)] += ms;
    ctx->prof.cnt[std::get<0>(t)] += 1;
    ctx->prof.free_ev.push_back(std::get<1>(t));
    ctx->prof.free_ev.push_back(std::get<2>(t));
  }
  ctx->prof.pending.clear();
}

// ---------------------------------------------------------------- counters
static int init_counters(tm_ctx* ctx) {
  if (!ctx->counters.ensure(sizeof(Counters))) return set_err(ctx, TM_ERR_CUDA, "cudaMalloc failed (counters)");
  if (!ctx->h_reset) {
    void* p = nullptr;
    if (cudaMallocHost(&p, 2 * sizeof(Counters) + 64) != cudaSuccess)
      return set_err(ctx, TM_ERR_CUDA, "cudaMallocHost failed");
    ctx->h_reset = static_cast<Counters*>(p);
    ctx->h_result = ctx->h_reset + 1;
    ctx->h_pin = reinterpret_cast<int64_t*>(ctx->h_result + 1);
    memset(ctx->h_reset, 0, sizeof(Counters));
    for (int k = 0; k < K_NUM; k++) ctx->h_reset->st.first[k] = ~0ull;
  }
  return TM_OK;
}

static int enqueue_reset(tm_ctx* ctx, cudaStream_t s) {
  CK(cudaMemcpyAsync(ctx->counters.p, ctx->h_reset, sizeof(Counters), cudaMemcpyHostToDevice, s));
  return TM_OK;
}

static int enqueue_readback(tm_ctx* ctx, cudaStream_t s) {
  CK(cudaMemcpyAsync(ctx->h_result, ctx->counters.p, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  return TM_OK;
}

static const char* kind_name(int k) {
  static const char* names[K_NUM] = {"index_range", "orientation", "degenerate", "duplicate", "reciprocity",
                                     "edge_count", "trivertex", "neighbors", "walk", "no_frontier",
                                     "no_converge", "split_law", "pool", "barrier", "no_internal", "structural"};
  return names[k];
}

// Device status -> the reference's error vocabulary.  Validation kinds (0..7)
// -> TM_ERR_VALIDATION; structural kinds -> TM_ERR_STRUCTURAL.
static int decode_status(tm_ctx* ctx, const Counters& h) {
  const DevStatus& st = h.st;
  bool any = false;
  for (int k = 0; k < K_NUM; k++) {
    ctx->defect_count[k] = st.count[k];
    ctx->defect_first[k] = st.count[k] ? (int64_t)st.first[k] : -1;
    any |= st.count[k] != 0;
  }
  if (!any) return TM_OK;
  std::string msg;
  bool validation = false;
  for (int k = 0; k <= K_NEIGHBORS; k++) {
    if (!st.count[k]) continue;
    validation = true;
    char b[160];
    snprintf(b, sizeof b, "%s%s[%lld]: %u defect(s)", msg.empty() ? "" : "; ", kind_name(k),
             (long long)st.first[k], st.count[k]);
    msg += b;
  }
  if (validation) return set_err(ctx, TM_ERR_VALIDATION, "invalid triangulation: %s", msg.c_str());
  for (int k = K_WALK; k < K_NUM; k++) {
    if (!st.count[k]) continue;
    long long f = (long long)st.first[k];
    switch (k) {
      case K_WALK:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[traversal] boundary walk from seed triangle %lld did not terminate", f);
      case K_NO_FRONTIER:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[traversal] no frontier edge reachable from triangle %lld", f);
      case K_NO_CONVERGE:
        return set_err(ctx, TM_ERR_STRUCTURAL,
                       "[reparation] tip removal did not converge (polygon %lld; initial repeated-vertex count %llu)",
                       f, h.stats[2]);
      case K_SPLIT_LAW:
        return set_err(ctx, TM_ERR_STRUCTURAL,
                       "[reparation] polygon %lld: split broke the length law |pa|+|pb| = |P|+2", f);
      case K_POOL:
        return set_err(ctx, TM_ERR_CAPACITY, "[reparation] repair scratch pool exhausted (polygon %lld)", f);
      case K_BARRIER:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[reparation] polygon %lld: barrier edge not found around tip vertex",
                       f);
      case K_NO_INTERNAL:
        return set_err(ctx, TM_ERR_STRUCTURAL,
                       "[reparation] polygon %lld: tip vertex has no internal edge to split on", f);
      default:
        return set_err(ctx, TM_ERR_STRUCTURAL, "structural failure at element %lld", f);
    }
  }
  return TM_OK;
}

// ---------------------------------------------------------------- buffers
static int prepare(tm_ctx* ctx, int64_t T, int64_t n = -1) {
  int rc = init_counters(ctx);
  if (rc) return rc;
  if (!ctx->aux) CK(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
  if (!ctx->ev_fork) CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  if (!ctx->ev_join) CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  if (!ctx->ev_cls) CK(cudaEventCreateWithFlags(&ctx->ev_cls, cudaEventDisableTiming));
  int64_t Tn = T > 0 ? T : 1;
  if (n >= 0) ENSURE(slots, hash_bytes(n, Tn, std::min(ctx->table_shrink, ctx->label_shrink)));
  if (n >= 0 && ctx->use_xy32) ENSURE(xy32, (n > 0 ? n : 1) * 2 * sizeof(float));
  ENSURE(seeds, Tn * sizeof(int32_t));
  ENSURE(start, Tn * sizeof(int32_t));
  ENSURE(len, (Tn + 1) * sizeof(int64_t));
  ENSURE(nrul, (Tn + 1) * sizeof(int64_t));
  ENSURE(eoff, (Tn + 1) * sizeof(int64_t));
  ENSURE(overflow, Tn * sizeof(int32_t));
  ENSURE(queue, Tn * sizeof(int32_t));
  ENSURE(stamp, Tn * sizeof(int32_t));
  if (ctx->stamp_clean != ctx->stamp.gen) {  // all -1 once per allocation; k_bfs_slow restores what it stamps
    CK(cudaMemset(ctx->stamp.p, 0xFF, ctx->stamp.bytes));
    CK(cudaDeviceSynchronize());
    ctx->stamp_clean = ctx->stamp.gen;
  }
  ENSURE(tiles, (scan_scratch_elems(3 * Tn) + 8) * sizeof(int64_t));
  ENSURE(lbscan, scan_lookback_bytes(Tn));
  ENSURE(rulers, (3 * Tn + 3) * sizeof(RulerRec));
  ENSURE(startbits, ((3 * Tn + 31) / 32) * sizeof(uint32_t));
  // ruler entries: seed starts + the 1/8 hash sample of half-edges (+ slack)
  ctx->ecap = Tn + (3 * Tn) / 8 + (3 * Tn) / 16 + 1024;
  ENSURE(ent_r, ctx->ecap * sizeof(int32_t));
  ENSURE(ent_base, ctx->ecap * sizeof(int64_t));
  ctx->cc_cap = Tn / 4 + 1024;  // seeds beyond it (never at Delaunay densities, P ~ 0.15 T) re-walk
  ENSURE(ccache, ctx->cc_cap * 2 * sizeof(int4));
  ENSURE(item_of, Tn * sizeof(int32_t));
  ENSURE(items, Tn * sizeof(int32_t));
  ENSURE(long_list, Tn * sizeof(int32_t));
  ENSURE(item_list, Tn * sizeof(int64_t));
  ENSURE(item_n, Tn * sizeof(int32_t));
  ENSURE(item_slots, Tn * sizeof(int64_t));
  ENSURE(item_state, Tn * sizeof(int32_t));
  ENSURE(item_depth, Tn * sizeof(int32_t));
  ENSURE(hugeq, Tn * sizeof(int32_t));
  ENSURE(parked, Tn * sizeof(int32_t));
  ENSURE(pinchq, Tn * sizeof(int32_t));
  ENSURE(longq, Tn * sizeof(int32_t));
  ENSURE(cnt, (Tn + 2) * sizeof(int64_t));  // per unit (<= items + 1) or per polygon, + the scan's end element
  ENSURE(slotsz, (Tn + 2) * sizeof(int64_t));
  ENSURE(pbase, (Tn + 2) * sizeof(int64_t));
  ENSURE(sbase, (Tn + 2) * sizeof(int64_t));
  ENSURE(iflag, Tn * sizeof(uint8_t));
  ENSURE(isrt, Tn * sizeof(int32_t));
  ENSURE(itiles, (scan_scratch_elems(Tn) + 8) * sizeof(int64_t));
  // item copies + pieces + per-warp arena slack
  unsigned long long want = 8ull * (unsigned long long)Tn + (1ull << 22);
  const char* forced = getenv("TERMESH_POOL_INIT");  // testing hook: start small, exercise the retry path
  if (forced && *forced) want = strtoull(forced, nullptr, 10);
  if (ctx->pool_cap < want) ctx->pool_cap = want;
  if (ctx->pool_cap >= (1ull << 32)) return set_err(ctx, TM_ERR_CAPACITY, "repair scratch pool exceeds 2^32 slots");
  ENSURE(pool, ctx->pool_cap * sizeof(int32_t));
  ENSURE(undo, ((unsigned long long)Tn + 1024) * sizeof(int32_t));
  return TM_OK;
}

// debug timeline (TERMESH_STAMPS=1): globaltimer when a stream reaches a point, in
// dbg[100 + k] (tm_ctx_debug; tools/trace_step.py).  Off: no launches.
static void stamp(tm_ctx* ctx, int k, cudaStream_t s) {
  static int on = -1;
  if (on < 0) on = getenv("TERMESH_STAMPS") != nullptr;
  if (on) launch_stamp(dc_of(ctx)->dbg + 100 + k, s);
}

// ---------------------------------------------------------------- enqueue (no host syncs)
static int label_one(const tm_ctx* ctx) {
  return ctx->label_one < 0 ? (ctx->label_a_external ? 1 : 0) : ctx->label_one;
}

static int enqueue_label(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T,
                         int check, int32_t* d_tri32, int32_t* d_hw, int8_t* d_me, uint8_t* d_seed, int32_t* d_tv,
                         cudaStream_t s) {
  Counters* dc = dc_of(ctx);
  // check = 1 sends every key to the table: never the half-size one
  const int shrink = check && ctx->label_shrink > 0 ? 0 : ctx->label_shrink;
  const bool lt = ctx->label_timing;  // phase API: device time of each pass (tm_ctx_label_ms)
  if (lt) CK(cudaEventRecord(ctx->lev[0], s));
  stamp(ctx, 0, s);
  if (!ctx->label_a_external) {
    SegTimer t_(ctx, S_LABEL_A, s);
    launch_label_a(d_xy, n, d_tri, tri_bits == 64, T, check, d_tri32, d_hw, d_me, d_seed, d_tv, ctx->slots.p,
                   &dc->st, s, shrink, &dc->table_ovf, ctx->use_xy32 ? ctx->xy32.as<float>() : nullptr,
                   label_one(ctx));
  }
  if (lt) CK(cudaEventRecord(ctx->lev[1], s));
  {
    SegTimer t_(ctx, S_LABEL_B, s);
    launch_label_b(tri_bits == 32 && d_tri32 == nullptr ? (const int32_t*)d_tri : d_tri32, n, T, d_hw, d_me, d_seed,
                   d_tv, ctx->slots.p, check, &dc->st, s, shrink, label_one(ctx));
  }
  if (lt) CK(cudaEventRecord(ctx->lev[2], s));
  stamp(ctx, 1, s);
  CK(cudaGetLastError());
  return TM_OK;
}

// the seed partition of this context clipped to [0, T]
static void part_range(const tm_ctx* ctx, int64_t T, int64_t* tb, int64_t* te) {
  int64_t b = ctx->part_begin, e = ctx->part_end < 0 ? T : ctx->part_end;
  if (b < 0) b = 0;
  if (b > T) b = T;
  if (e > T) e = T;
  if (e < b) e = b;
  *tb = b;
  *te = e;
}

static LongQueue long_queue(tm_ctx* ctx) {
  Counters* dc = dc_of(ctx);
  return LongQueue{ctx->hugeq.as<int32_t>(), ctx->longq.as<int32_t>(), &dc->q_huge,      &dc->q_long,
                   &dc->q_next,           ctx->parked.as<int32_t>(), &dc->n_parked, ctx->pinchq.as<int32_t>(),
                   &dc->n_pinch,          &dc->tip_next,         &dc->gm_next};
}

static RepairArgs repair_args(tm_ctx* ctx, const int32_t* d_tri32, int32_t* d_hw, const int32_t* d_tv, int64_t T,
                              const int64_t* d_off_in, const int32_t* d_v_in) {
  Counters* dc = dc_of(ctx);
  const int64_t Tn = T > 0 ? T : 1;
  const int tv_exact = ctx->path_hv == nullptr;
  return RepairArgs{d_tri32, d_hw, d_tv, tv_exact, T, ctx->pool.as<int32_t>(), ctx->pool_cap, &dc->pool_top,
                    ctx->undo.as<int32_t>(), &dc->undo_top, (unsigned long long)Tn + 1024, &dc->st,
                    ctx->items.as<int32_t>(), &dc->n_items, d_off_in, d_v_in, ctx->item_list.as<int64_t>(),
                    ctx->item_n.as<int32_t>(), ctx->item_slots.as<int64_t>(), ctx->item_state.as<int32_t>(),
                    ctx->item_depth.as<int32_t>(), dc->stats, long_queue(ctx), dc->dbg};
}

static int enqueue_traverse(tm_ctx* ctx, const int32_t* d_tri32, const int32_t* d_hw, const uint8_t* d_seed,
                            int64_t T, int64_t* d_off, int32_t* d_v, cudaStream_t s) {
  Counters* dc = dc_of(ctx);
  int64_t Tn = T > 0 ? T : 1;
  int64_t* tiles = ctx->tiles.as<int64_t>();
  int64_t tb = 0, te = 0;
  part_range(ctx, T, &tb, &te);
  {
    SegTimer t_(ctx, S_SEEDS, s);
    launch_select_flags(d_seed + tb, te - tb, ctx->seeds.as<int32_t>(), &dc->n_seeds, tiles, s, tb);
  }
  CK(cudaMemsetAsync(ctx->startbits.p, 0, ((3 * Tn + 31) / 32) * sizeof(uint32_t), s));
  {
    SegTimer t_(ctx, S_TRAV_START, s);
    launch_trav_start(d_hw, ctx->seeds.as<int32_t>(), &dc->n_seeds, Tn, ctx->start.as<int32_t>(),
                      ctx->overflow.as<int32_t>(), &dc->n_overflow, ctx->queue.as<int32_t>(),
                      ctx->stamp.as<int32_t>(), ctx->startbits.as<uint32_t>(), &dc->st, s);
  }
  {
    SegTimer t_(ctx, S_TRAV_RULERS, s);
    launch_ruler_walk(d_hw, ctx->startbits.as<uint32_t>(), T, tb, te, ctx->start.as<int32_t>(), &dc->n_seeds, Tn,
                      ctx->rulers.as<RulerRec>(), &dc->st, s);
  }
  {
    SegTimer t_(ctx, S_TRAV_LEN, s);
    launch_chain_count(ctx->seeds.as<int32_t>(), ctx->start.as<int32_t>(), &dc->n_seeds, Tn, T,
                       ctx->rulers.as<RulerRec>(),
                       ctx->len.as<int64_t>(), ctx->nrul.as<int64_t>(),
                       ctx->early_long ? ctx->long_list.as<int32_t>() : nullptr, &dc->n_long,
                       ctx->ccache.as<int4>(), ctx->cc_cap, &dc->st, s);
  }
  stamp(ctx, 2, s);
  {
    SegTimer t_(ctx, S_TRAV_SCAN, s);
    launch_scan_lookback(ctx->len.as<int64_t>(), ctx->nrul.as<int64_t>(), d_off, ctx->eoff.as<int64_t>(), &dc->n_seeds,
                         Tn, ctx->lbscan.p, s, &dc->n_slots0, &dc->n_entries);
  }
  stamp(ctx, 3, s);
  {
    SegTimer t_(ctx, S_TRAV_WRITE, s);
    launch_chain_emit(ctx->start.as<int32_t>(), &dc->n_seeds, Tn, ctx->rulers.as<RulerRec>(), d_off, ctx->eoff.as<int64_t>(), ctx->ent_r.as<int32_t>(), ctx->ent_base.as<int64_t>(),
                      ctx->ecap, ctx->ccache.as<int4>(), ctx->cc_cap, &dc->st, s);
    if (ctx->early_long) {
      // fork: the long polygons' runs -> their classification -> the long-item
      // repair kernel, on ctx->aux beside the rest of the traversal and the short items
      cudaStream_t a = ctx->aux;
      stamp(ctx, 4, s);
      CK(cudaEventRecord(ctx->ev_fork, s));
      CK(cudaStreamWaitEvent(a, ctx->ev_fork, 0));
      stamp(ctx, 11, a);
      launch_ruler_write_list(d_tri32, d_hw, ctx->long_list.as<int32_t>(), &dc->n_long, ctx->eoff.as<int64_t>(),
                              ctx->ent_r.as<int32_t>(), ctx->ent_base.as<int64_t>(), ctx->rulers.as<RulerRec>(), T, Tn,
                              d_v, ctx->path_hv, a);
      stamp(ctx, 12, a);
      launch_classify(d_off, d_v, &dc->n_seeds, Tn, ctx->item_of.as<int32_t>(), ctx->items.as<int32_t>(),
                      &dc->n_items, ctx->long_list.as<int32_t>(), &dc->n_long, dc->stats, long_queue(ctx),
                      ctx->path_hv, ctx->tv.as<int32_t>(), 2, ctx->item_state.as<int32_t>(), ctx->pool.as<int32_t>(),
                      &dc->pool_top, ctx->pool_cap, ctx->item_depth.as<int32_t>(), a);
      CK(cudaEventRecord(ctx->ev_cls, a));
      stamp(ctx, 13, a);
      {
        RepairArgs ra = repair_args(ctx, d_tri32, const_cast<int32_t*>(d_hw), ctx->tv.as<int32_t>(), T, d_off, d_v);
        launch_repair_tips_long(ra, a);
        stamp(ctx, 14, a);
        launch_repair_pinch(ra, 2, a);  // the finished long items' pinch pass, still beside the short items
      }
      stamp(ctx, 15, a);
      CK(cudaEventRecord(ctx->ev_join, a));
    }
    launch_ruler_write(d_tri32, d_hw, &dc->n_entries, ctx->ent_r.as<int32_t>(), ctx->ent_base.as<int64_t>(),
                       ctx->rulers.as<RulerRec>(), T, ctx->ecap, d_v, ctx->path_hv, s);
  }
  stamp(ctx, 5, s);
  CK(cudaGetLastError());
  return TM_OK;
}

// The final CSR from the input CSR and the repaired items.  Default: by units
// (runs of untouched polygons + the work item after each, tm_repair.cu); the
// item order is built here when `sort` (else enqueue_repair built it before
// waiting for the long items).
static void enqueue_stitch(tm_ctx* ctx, const int64_t* d_off_in, const int32_t* d_v_in, const int64_t* Pp, int64_t Tn,
                           int64_t* d_off_out, int32_t* d_v_out, bool sort, cudaStream_t s) {
  Counters* dc = dc_of(ctx);
#ifdef TM_OLD_STITCH  // A/B: per-polygon counts, scan and copy
  (void)sort;
  launch_out_counts(d_off_in, Pp, Tn, ctx->item_of.as<int32_t>(), ctx->item_n.as<int32_t>(),
                    ctx->item_slots.as<int64_t>(), ctx->cnt.as<int64_t>(), ctx->slotsz.as<int64_t>(), dc->stats,
                    &dc->st, s);
  launch_scan_lookback(ctx->cnt.as<int64_t>(), ctx->slotsz.as<int64_t>(), ctx->pbase.as<int64_t>(),
                       ctx->sbase.as<int64_t>(), Pp, Tn, ctx->lbscan.p, s, &dc->p_out, &dc->f_out, d_off_out);
  launch_stitch(d_off_in, d_v_in, Pp, Tn, ctx->item_of.as<int32_t>(), ctx->items.as<int32_t>(), &dc->n_items,
                ctx->item_list.as<int64_t>(), ctx->item_n.as<int32_t>(), ctx->pool.as<int32_t>(),
                ctx->pbase.as<int64_t>(), ctx->sbase.as<int64_t>(), d_off_out, d_v_out, s);
#else
  if (sort)
    launch_item_sort(ctx->item_of.as<int32_t>(), Pp, Tn, ctx->iflag.as<uint8_t>(), ctx->isrt.as<int32_t>(),
                     &dc->n_isrt, ctx->itiles.as<int64_t>(), s);
  launch_unit_counts(d_off_in, Pp, Tn, ctx->isrt.as<int32_t>(), &dc->n_isrt, ctx->item_of.as<int32_t>(),
                     ctx->item_n.as<int32_t>(), ctx->item_slots.as<int64_t>(), ctx->cnt.as<int64_t>(),
                     ctx->slotsz.as<int64_t>(), &dc->n_units, dc->stats, &dc->st, s);
  launch_scan_lookback(ctx->cnt.as<int64_t>(), ctx->slotsz.as<int64_t>(), ctx->pbase.as<int64_t>(),
                       ctx->sbase.as<int64_t>(), &dc->n_units, Tn, ctx->lbscan.p, s, &dc->p_out, &dc->f_out,
                       d_off_out);
  launch_stitch_units(d_off_in, d_v_in, Pp, ctx->isrt.as<int32_t>(), &dc->n_isrt, ctx->item_of.as<int32_t>(),
                      ctx->item_list.as<int64_t>(), ctx->item_n.as<int32_t>(), ctx->pool.as<int32_t>(),
                      ctx->pbase.as<int64_t>(), ctx->sbase.as<int64_t>(), d_off_out, d_v_out, s);
#endif
}

// Repair phase.  Pp: device polygon count of the input CSR.
static int enqueue_repair(tm_ctx* ctx, const int32_t* d_tri32, int32_t* d_hw, const int32_t* d_tv, int64_t T,
                          const int64_t* d_off_in, const int32_t* d_v_in, const int64_t* Pp, int64_t* d_off_out,
                          int32_t* d_v_out, cudaStream_t s) {
  Counters* dc = dc_of(ctx);
  int64_t Tn = T > 0 ? T : 1;
  LongQueue q = long_queue(ctx);
  const bool early = ctx->early_long;  // the long items already run on ctx->aux (enqueue_traverse)
  {
    SegTimer t_(ctx, S_CLASSIFY, s);
    launch_classify(d_off_in, d_v_in, Pp, Tn, ctx->item_of.as<int32_t>(), ctx->items.as<int32_t>(), &dc->n_items,
                    ctx->long_list.as<int32_t>(), &dc->n_long, dc->stats, q, ctx->path_hv,
                    const_cast<int32_t*>(d_tv), early ? 1 : 0, ctx->item_state.as<int32_t>(), ctx->pool.as<int32_t>(),
                    &dc->pool_top, ctx->pool_cap, ctx->item_depth.as<int32_t>(), s);
  }
  stamp(ctx, 6, s);
  if (early) CK(cudaStreamWaitEvent(s, ctx->ev_cls, 0));  // the item list is complete
  RepairArgs a = repair_args(ctx, d_tri32, d_hw, d_tv, T, d_off_in, d_v_in);
  {
    SegTimer t_(ctx, S_REPAIR_TIPS, s);
    // fork: the long items (one block each) on ctx->aux beside the short ones
    static int serial = -1;
    if (serial < 0) serial = getenv("TERMESH_SERIAL_REPAIR") != nullptr;  // debug: no fork
    if (!early) {
      cudaStream_t sl = serial ? s : ctx->aux;
      if (!serial) {
        CK(cudaEventRecord(ctx->ev_fork, s));
        CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
      }
      launch_repair_tips_long(a, sl);
      launch_repair_pinch(a, 2, sl);
      if (!serial) CK(cudaEventRecord(ctx->ev_join, ctx->aux));
    }
    stamp(ctx, 16, s);
    launch_repair_tips(a, 0, s);
    stamp(ctx, 7, s);
    {
      SegTimer t_(ctx, S_REPAIR_PINCH, s);
      launch_repair_pinch(a, 0, s);  // short items' pinch pass, still beside the long items
    }
    stamp(ctx, 17, s);
#ifndef TM_OLD_STITCH
    // the work items in polygon order for the stitch, while the long items still run
    launch_item_sort(ctx->item_of.as<int32_t>(), Pp, Tn, ctx->iflag.as<uint8_t>(), ctx->isrt.as<int32_t>(),
                     &dc->n_isrt, ctx->itiles.as<int64_t>(), s);
#endif
    if (early || !serial) CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
    stamp(ctx, 8, s);
    launch_repair_tips(a, 1, s);  // long items the shared-memory kernel handed back
  }
  {
    SegTimer t_(ctx, S_REPAIR_PINCH, s);
    launch_repair_pinch(a, 1, s);
  }
  stamp(ctx, 9, s);
  {
    SegTimer t_(ctx, S_STITCH, s);
    enqueue_stitch(ctx, d_off_in, d_v_in, Pp, Tn, d_off_out, d_v_out, false, s);
  }
  stamp(ctx, 10, s);
  CK(cudaGetLastError());
  return TM_OK;
}

// read back the counters (synchronizes s) and decode the status
static int finish(tm_ctx* ctx, cudaStream_t s, Counters* out) {
  int rc = enqueue_readback(ctx, s);
  if (rc) return rc;
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  *out = *ctx->h_result;
  return decode_status(ctx, *out);
}

static void fill_stats(const Counters& h, int64_t* stats) {
  if (!stats) return;
  stats[TM_STAT_ROUNDS] = h.stats[0] > 0 ? (int64_t)h.stats[0] : 1;
  stats[TM_STAT_SPLITS] = (int64_t)(h.stats[1] + h.stats[4]);
  stats[TM_STAT_INITIAL_TIPS] = (int64_t)h.stats[2];
  stats[TM_STAT_UNREPAIRED] = (int64_t)h.stats[3];
  stats[TM_STAT_NONSIMPLE] = (int64_t)h.stats[6];
  stats[TM_STAT_TIP_SPLITS] = (int64_t)h.stats[1];
  stats[TM_STAT_PINCH_SPLITS] = (int64_t)h.stats[4];
  stats[TM_STAT_WORK_ITEMS] = (int64_t)h.n_items;
  stats[TM_STAT_PINCH_EXTRA] = (int64_t)h.stats[5];
  stats[TM_STAT_PINCH_TRUNCATED] = (int64_t)h.stats[7];
  stats[TM_STAT_PINCH_DEFERRED] = (int64_t)h.stats[10];
}

// Pool overflow: restore the pre-repair frontier bits (restore()), grow the
// pool, and re-run the repair phase (outside any graph).
template <typename Restore>
static int retry_repair(tm_ctx* ctx, const int32_t* d_tri32, int32_t* d_hw, const int32_t* d_tv, int64_t T,
                        const int64_t* d_off_in, const int32_t* d_v_in, const int64_t* Pp, int64_t* d_off_out,
                        int32_t* d_v_out, cudaStream_t s, Counters* h, int rc, Restore restore) {
  for (int attempt = 0; attempt < 6 && rc == TM_ERR_CAPACITY && h->st.count[K_POOL]; attempt++) {
    Counters* dc = dc_of(ctx);
    int r = restore(s);
    if (r) return r;
    CK(cudaStreamSynchronize(s));
    ctx->pool_cap *= 4;
    if (ctx->pool_cap >= (1ull << 32)) return set_err(ctx, TM_ERR_CAPACITY, "repair pool exceeds 2^32 slots");
    ENSURE(pool, ctx->pool_cap * sizeof(int32_t));
    // reset the repair-side counters and the status; keep the traversal counts
    CK(cudaMemcpyAsync(&dc->st, &ctx->h_reset->st, sizeof(DevStatus), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(&dc->n_items, 0, 3 * sizeof(unsigned int), s));  // n_items, n_long, n_pinch
    CK(cudaMemsetAsync(&dc->q_huge, 0, 8 * sizeof(unsigned int), s));  // queues + tip_next
    CK(cudaMemsetAsync(&dc->pool_top, 0, 10 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(&dc->stats[10], 0, sizeof(unsigned long long), s));
    r = enqueue_repair(ctx, d_tri32, d_hw, d_tv, T, d_off_in, d_v_in, Pp, d_off_out, d_v_out, s);
    if (r) return r;
    rc = finish(ctx, s, h);
  }
  return rc;
}

extern "C" {

int tm_version(void) { return 2; }

int tm_ctx_create(tm_ctx** out) {
  if (!out) return TM_ERR_ARGUMENT;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TM_ERR_CUDA;
  *out = new tm_ctx();
  const char* g = getenv("TERMESH_NO_GRAPH");
  if (g && *g && *g != '0') (*out)->use_graph = 0;
  const char* nn = getenv("TERMESH_NARROW");  // A/B switch
  if (nn && *nn && *nn != '0') (*out)->host_narrow = true;
  const char* lo = getenv("TERMESH_LABEL_ONE");  // A/B switch / testing hook
  if (lo && *lo) (*out)->label_one = atoi(lo) ? 1 : 0;
  const char* x32 = getenv("TERMESH_XY32");  // A/B switch
  if (x32 && *x32 && *x32 != '0') (*out)->use_xy32 = 1;
  const char* ts = getenv("TERMESH_TABLE_SHRINK");  // testing hook: start with a 2^-s table (overflow/growth path)
  if (ts && *ts) (*out)->table_shrink = atoi(ts);
  return TM_OK;
}

void tm_ctx_destroy(tm_ctx* ctx) {
  if (!ctx) return;
  Buf* bufs[] = {&ctx->counters, &ctx->slots, &ctx->seeds, &ctx->start, &ctx->len, &ctx->overflow, &ctx->queue,
                 &ctx->stamp, &ctx->tiles, &ctx->nrul, &ctx->eoff, &ctx->rulers, &ctx->startbits,
                 &ctx->ent_r, &ctx->ent_base, &ctx->ccache, &ctx->item_of, &ctx->items, &ctx->long_list, &ctx->item_list,
                 &ctx->item_n, &ctx->item_slots, &ctx->item_state, &ctx->item_depth, &ctx->hugeq, &ctx->longq, &ctx->parked, &ctx->pinchq, &ctx->iflag, &ctx->isrt, &ctx->itiles, &ctx->cnt, &ctx->slotsz, &ctx->pbase, &ctx->sbase, &ctx->pool,
                 &ctx->undo, &ctx->xy, &ctx->tri, &ctx->tri32, &ctx->hw, &ctx->max_edge, &ctx->seed, &ctx->tv,
                 &ctx->off0, &ctx->v0, &ctx->fin_off, &ctx->fin_v, &ctx->hw_snap, &ctx->hv,
                 &ctx->lbscan, &ctx->pbits, &ctx->pflag, &ctx->ptable, &ctx->pstamp, &ctx->ptip, &ctx->prep,
                 &ctx->plong, &ctx->prot, &ctx->pbucket, &ctx->porder, &ctx->phist, &ctx->pstart, &ctx->pcursor,
                 &ctx->plen, &ctx->ptiles, &ctx->dcell, &ctx->dhist, &ctx->dstart, &ctx->dcursor, &ctx->dids,
                 &ctx->dsxy, &ctx->dcnt, &ctx->doff, &ctx->xy32, &ctx->btab};
  for (Buf* b : bufs) b->release();
  if (ctx->h_reset) cudaFreeHost(ctx->h_reset);
  if (ctx->h_tri32) cudaFreeHost(ctx->h_tri32);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_join, ctx->ev_cls, ctx->lev[0], ctx->lev[1], ctx->lev[2]})
    if (e) cudaEventDestroy(e);
  prof_flush(ctx);
  for (auto e : ctx->prof.free_ev) cudaEventDestroy(e);
  if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  for (auto e : ctx->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  delete ctx;
}

const char* tm_ctx_last_error(const tm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int tm_ctx_defects(const tm_ctx* ctx, int64_t* counts, int64_t* first) {
  if (!ctx) return TM_ERR_ARGUMENT;
  for (int k = 0; k < K_NUM; k++) {
    if (counts) counts[k] = ctx->defect_count[k];
    if (first) first[k] = ctx->defect_first[k];
  }
  return TM_OK;
}

int tm_ctx_set_profiling(tm_ctx* ctx, int on) {
  if (!ctx) return TM_ERR_ARGUMENT;
  ctx->prof.on = on != 0;
  return TM_OK;
}

int tm_ctx_segment_ms(tm_ctx* ctx, double* ms, int64_t* counts, int n, int reset) {
  if (!ctx) return TM_ERR_ARGUMENT;
  prof_flush(ctx);
  for (int k = 0; k < n && k < S_NUM; k++) {
    if (ms) ms[k] = ctx->prof.ms[k];
    if (counts) counts[k] = ctx->prof.cnt[k];
  }
  if (reset)
    for (int k = 0; k < S_NUM; k++) ctx->prof.ms[k] = 0, ctx->prof.cnt[k] = 0;
  return S_NUM;
}

const char* tm_segment_name(int k) { return (k >= 0 && k < S_NUM) ? kSegNames[k] : ""; }

int64_t tm_launch_count(void) { return g_launches.load(); }

// debug timestamps written by kernels into Counters.dbg during the last run
int tm_ctx_debug(const tm_ctx* ctx, uint64_t* out, int n) {
  if (!ctx || !ctx->h_result) return TM_ERR_ARGUMENT;
  for (int k = 0; k < n && k < 128; k++) out[k] = ctx->h_result->dbg[k];
  return TM_OK;
}

int tm_ctx_debug_copy(const tm_ctx* ctx, int which, void* dst, size_t bytes) {
  if (!ctx || !dst) return TM_ERR_ARGUMENT;
  const Buf* b = which == 0 ? &ctx->off0 : which == 1 ? &ctx->v0 : which == 2 ? &ctx->hw : which == 3 ? &ctx->hv
               : which == 4 ? &ctx->seed : nullptr;
  if (!b || !b->p) return TM_ERR_ARGUMENT;
  if (bytes > b->bytes) bytes = b->bytes;
  if (cudaMemcpy(dst, b->p, bytes, cudaMemcpyDeviceToDevice) != cudaSuccess) return TM_ERR_CUDA;
  return TM_OK;
}

int tm_ctx_set_partition(tm_ctx* ctx, int64_t t_begin, int64_t t_end) {
  if (!ctx) return TM_ERR_ARGUMENT;
  if (t_begin < 0 || (t_end >= 0 && t_end < t_begin)) return set_err(ctx, TM_ERR_ARGUMENT, "bad seed partition");
  ctx->part_begin = t_begin;
  ctx->part_end = t_end;
  return TM_OK;
}

int tm_shift_offsets(int64_t* d_offsets, int64_t n_polys, int64_t delta, void* stream) {
  if (n_polys < 0) return TM_ERR_ARGUMENT;
  if (delta != 0) launch_shift(d_offsets, n_polys, delta, (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

int tm_ctx_phase_ms(const tm_ctx* ctx, double* ms3) {
  if (!ctx || !ms3) return TM_ERR_ARGUMENT;
  for (int k = 0; k < 3; k++) ms3[k] = ctx->phase_ms[k];
  return TM_OK;
}

static int check_sizes(tm_ctx* ctx, int64_t n, int64_t T) {
  if (T < 0 || n < 0) return set_err(ctx, TM_ERR_ARGUMENT, "sizes must be non-negative");
  if (3 * T >= (int64_t)0x7FFFFFFF) return set_err(ctx, TM_ERR_ARGUMENT, "3T must fit in 31 bits");
  if (n >= (int64_t)0x7F7F7F7F) return set_err(ctx, TM_ERR_ARGUMENT, "vertex count must fit in 31 bits");
  return TM_OK;
}

int tm_label(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T, int check,
             int32_t* d_tri32, int32_t* d_hw, int8_t* d_max_edge, uint8_t* d_seed, int32_t* d_tv, void* stream) {
  if (!ctx) return TM_ERR_ARGUMENT;
  if (tri_bits != 32 && tri_bits != 64) return set_err(ctx, TM_ERR_ARGUMENT, "tri_bits must be 32 or 64");
  int rc = check_sizes(ctx, n, T);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  for (auto& e : ctx->lev)
    if (!e) CK(cudaEventCreate(&e));
  Counters h;
  // phase API: full-size twin table, twice the buckets after a displacement overflow
  for (ctx->label_shrink = std::min(0, ctx->table_shrink);; ctx->label_shrink--) {
    if ((rc = prepare(ctx, T, n)) || (rc = enqueue_reset(ctx, s))) return rc;
    ctx->label_timing = true;
    rc = enqueue_label(ctx, d_xy, n, d_tri, tri_bits, T, check, d_tri32, d_hw, d_max_edge, d_seed, d_tv, s);
    ctx->label_timing = false;
    if (rc) return rc;
    rc = finish(ctx, s, &h);
    if (!h.table_ovf) break;
    if (ctx->label_shrink <= kMinShrink)
      return set_err(ctx, TM_ERR_CAPACITY, "twin table displacement overflow at 8x size (degenerate keys?)");
  }
  for (int k = 0; k < 2; k++) {
    float ms = 0;
    ctx->label_ms[k] = cudaEventElapsedTime(&ms, ctx->lev[k], ctx->lev[k + 1]) == cudaSuccess ? ms : 0.0;
  }
  return rc;
}

int tm_ctx_label_ms(const tm_ctx* ctx, double* ms2) {
  if (!ctx || !ms2) return TM_ERR_ARGUMENT;
  ms2[0] = ctx->label_ms[0];
  ms2[1] = ctx->label_ms[1];
  return TM_OK;
}

int tm_relabel(tm_ctx* ctx, int32_t* d_hw, const int8_t* d_max_edge, int64_t T, uint8_t* d_seed, void* stream) {
  if (!ctx) return TM_ERR_ARGUMENT;
  launch_relabel(d_max_edge, T, d_hw, d_seed, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return TM_OK;
}

int tm_check_neighbors(tm_ctx* ctx, const int32_t* d_hw, const void* d_nb, int nb_bits, int64_t T, void* stream) {
  if (!ctx) return TM_ERR_ARGUMENT;
  if (nb_bits != 32 && nb_bits != 64) return set_err(ctx, TM_ERR_ARGUMENT, "nb_bits must be 32 or 64");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = init_counters(ctx);
  if (rc || (rc = enqueue_reset(ctx, s))) return rc;
  launch_check_neighbors(d_hw, d_nb, nb_bits == 64, T, &dc_of(ctx)->st, s);
  CK(cudaGetLastError());
  Counters h;
  return finish(ctx, s, &h);
}

int tm_unpack_halfedges(tm_ctx* ctx, const int32_t* d_hw, int64_t T, int32_t* d_twin, uint8_t* d_fr, void* stream) {
  if (!ctx) return TM_ERR_ARGUMENT;
  launch_unpack(d_hw, T, d_twin, d_fr, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return TM_OK;
}

int tm_pack_frontier(tm_ctx* ctx, int32_t* d_hw, const uint8_t* d_fr, int64_t T, void* stream) {
  if (!ctx) return TM_ERR_ARGUMENT;
  launch_pack_frontier(d_hw, T, d_fr, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return TM_OK;
}

int tm_traverse(tm_ctx* ctx, const int32_t* d_tri32, const int32_t* d_hw, const uint8_t* d_seed, int64_t T,
                int64_t* d_offsets, int32_t* d_verts, int64_t cap_polys, int64_t cap_slots, int64_t* n_polys,
                int64_t* n_slots, void* stream) {
  if (!ctx || !n_polys || !n_slots) return TM_ERR_ARGUMENT;
  if (cap_polys < T || cap_slots < 3 * T)
    return set_err(ctx, TM_ERR_ARGUMENT, "tm_traverse needs cap_polys >= T and cap_slots >= 3T");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = prepare(ctx, T);
  if (rc || (rc = enqueue_reset(ctx, s))) return rc;
  if ((rc = enqueue_traverse(ctx, d_tri32, d_hw, d_seed, T, d_offsets, d_verts, s))) return rc;
  Counters h;
  if ((rc = finish(ctx, s, &h))) return rc;
  *n_polys = h.n_seeds;
  *n_slots = h.n_slots0;
  return TM_OK;
}

int tm_repair(tm_ctx* ctx, const int32_t* d_tri32, int32_t* d_hw, const int32_t* d_tv, int64_t T,
              const int64_t* d_off_in, const int32_t* d_v_in, int64_t P, int64_t* d_off_out, int32_t* d_v_out,
              int64_t cap_polys, int64_t cap_slots, int64_t* n_polys_out, int64_t* n_slots_out, int64_t* stats,
              void* stream) {
  if (!ctx || !n_polys_out || !n_slots_out) return TM_ERR_ARGUMENT;
  if (cap_polys < T || cap_slots < 3 * T)
    return set_err(ctx, TM_ERR_ARGUMENT, "tm_repair needs cap_polys >= T and cap_slots >= 3T");
  if (P < 0 || P > (T > 0 ? T : 0)) return set_err(ctx, TM_ERR_ARGUMENT, "polygon count out of range");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = prepare(ctx, T);
  if (rc || (rc = enqueue_reset(ctx, s))) return rc;
  *ctx->h_pin = P;
  Counters* dc = dc_of(ctx);
  CK(cudaMemcpyAsync(&dc->p_in, ctx->h_pin, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  // caller-supplied frontier bits: keep a copy so a pool overflow can be rolled back
  ENSURE(hw_snap, 3 * (T > 0 ? T : 1) * sizeof(int32_t));
  CK(cudaMemcpyAsync(ctx->hw_snap.p, d_hw, 3 * T * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if ((rc = enqueue_repair(ctx, d_tri32, d_hw, d_tv, T, d_off_in, d_v_in, &dc->p_in, d_off_out, d_v_out, s)))
    return rc;
  Counters h;
  rc = finish(ctx, s, &h);
  if (rc == TM_ERR_CAPACITY)
    rc = retry_repair(ctx, d_tri32, d_hw, d_tv, T, d_off_in, d_v_in, &dc->p_in, d_off_out, d_v_out, s, &h, rc,
                      [&](cudaStream_t st) -> int {
                        CK(cudaMemcpyAsync(d_hw, ctx->hw_snap.p, 3 * T * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                           st));
                        return TM_OK;
                      });
  if (rc) return rc;
  *n_polys_out = h.p_out;
  *n_slots_out = h.f_out;
  fill_stats(h, stats);
  return TM_OK;
}

// Whole path on device buffers: one CUDA graph (captured on first use for a
// given set of pointers/sizes) on the context's stream, ordered after the
// caller's stream by events.  With profiling on, launches go to the caller's
// stream one by one so each kernel group can be timed.
// scratch and whole-path buffers for a mesh of n vertices / T triangles
static int path_buffers(tm_ctx* ctx, int64_t n, int64_t T) {
  int rc = check_sizes(ctx, n, T);
  if (rc || (rc = prepare(ctx, T, n))) return rc;
  int64_t Tn = T > 0 ? T : 1, nn = n > 0 ? n : 1;
  ENSURE(tri32, 3 * Tn * sizeof(int32_t));
  ENSURE(hw, 3 * Tn * sizeof(int32_t));
  ENSURE(max_edge, Tn);
  ENSURE(seed, Tn);
  ENSURE(tv, nn * sizeof(int32_t));
  ENSURE(off0, (Tn + 1) * sizeof(int64_t));
  ENSURE(v0, 3 * Tn * sizeof(int32_t));
  ENSURE(hv, 3 * Tn * sizeof(int32_t));
  return TM_OK;
}


static int run_device(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T,
                      int check, int64_t* d_off, int32_t* d_v, int64_t* n_polys, int64_t* n_slots, int64_t* stats,
                      cudaStream_t user) {
  int rc = path_buffers(ctx, n, T);
  if (rc) return rc;
  if (!ctx->gstream) CK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
  for (auto& e : ctx->ev)
    if (!e) CK(cudaEventCreate(&e));
  if (!ctx->ev_in) CK(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
  if (!ctx->ev_out) CK(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
  int32_t* tri32 = ctx->tri32.as<int32_t>();
  int32_t* hw = ctx->hw.as<int32_t>();
  int32_t* tv = ctx->tv.as<int32_t>();
  int64_t* off0 = ctx->off0.as<int64_t>();
  int32_t* v0 = ctx->v0.as<int32_t>();
  Counters* dc = dc_of(ctx);
  ctx->label_shrink = ctx->table_shrink;
  {
    // a seed partition parks the items its final LOCAL pinch guard would cut off
    // (the guard is global, reparation.py:322); tm_resume_pinch finishes them
    int64_t tb = 0, te = 0;
    part_range(ctx, T, &tb, &te);
    ctx->h_reset->stats[8] = 0;
    ctx->h_reset->stats[9] = (tb > 0 || te < T) ? 1 : 0;
    const char* cap = getenv("TERMESH_PINCH_GUARD_CAP");  // testing hook (partitions only)
    ctx->h_reset->stats[11] = (ctx->h_reset->stats[9] && cap && *cap) ? strtoull(cap, nullptr, 10) : 0;
  }
  ctx->last_T = -1;

  bool capturing = false;
  // external event nodes inside a capture, plain records otherwise
  auto rec = [&](cudaEvent_t e, cudaStream_t s) {
    return capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
  };
  // part 1: reset + labels; part 2: traversal + repair + readback; 3: both
  auto body = [&](cudaStream_t s, int part = 3) -> int {
    int r;
    if (part & 1) {
      if (!ctx->label_a_external && (r = enqueue_reset(ctx, s))) return r;
      CK(rec(ctx->ev[0], s));
      if (!ctx->labels_external &&
          (r = enqueue_label(ctx, d_xy, n, d_tri, tri_bits, T, check, tri32, hw, ctx->max_edge.as<int8_t>(),
                             ctx->seed.as<uint8_t>(), nullptr, s)))
        return r;
      CK(rec(ctx->ev[1], s));
    }
    if (!(part & 2)) return enqueue_readback(ctx, s);
    ctx->path_hv = ctx->hv.as<int32_t>();
    static int no_early = -1;
    if (no_early < 0) no_early = getenv("TERMESH_NO_EARLY") != nullptr;  // A/B switch
    ctx->early_long = !no_early;
    r = enqueue_traverse(ctx, tri32, hw, ctx->seed.as<uint8_t>(), T, off0, v0, s);
    if (r) { ctx->path_hv = nullptr; ctx->early_long = false; return r; }
    CK(rec(ctx->ev[2], s));
    r = enqueue_repair(ctx, tri32, hw, tv, T, off0, v0, &dc->n_seeds, d_off, d_v, s);
    ctx->path_hv = nullptr;
    ctx->early_long = false;
    if (r) return r;
    CK(rec(ctx->ev[3], s));
    return enqueue_readback(ctx, s);
  };

  cudaStream_t s = user;
  if (check) {
    // Validation first: a defective mesh (e.g. an out-of-range corner) must not
    // reach the traversal and repair kernels, which index by corner.  The label
    // passes run on their own, the status is decoded, then the rest follows.
    if ((rc = body(s, 1))) return rc;
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (ctx->h_result->table_ovf) return kRetryTable;  // (check mode uses the full table; defensive)
    if ((rc = decode_status(ctx, *ctx->h_result))) return rc;
    if ((rc = body(s, 2))) return rc;
  } else if (ctx->use_graph && !ctx->prof.on) {
    GraphKey key{d_xy, d_tri, d_off, d_v, n, T, 0, 0, tri_bits, check,
                 (ctx->label_a_external ? 1 : 0) | (ctx->labels_external ? 2 : 0), ctx->pool_cap,
                 g_alloc_gen.load()};
    part_range(ctx, T, &key.tb, &key.te);
    if (!ctx->graph || !(key == ctx->gkey)) {
      if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
      ctx->graph = nullptr;
      cudaGraph_t g = nullptr;
      long long k0 = g_launches.load();
      CK(cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal));
      capturing = true;
      int r = body(ctx->gstream);
      capturing = false;
      cudaError_t e = cudaStreamEndCapture(ctx->gstream, &g);
      ctx->graph_kernels = g_launches.load() - k0;
      g_launches.fetch_sub(ctx->graph_kernels);  // captured, not launched
      if (r) {
        if (g) cudaGraphDestroy(g);
        return r;
      }
      if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
      e = cudaGraphInstantiate(&ctx->graph, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
      ctx->gkey = key;
    }
    CK(cudaEventRecord(ctx->ev_in, user));
    CK(cudaStreamWaitEvent(ctx->gstream, ctx->ev_in, 0));
    CK(cudaGraphLaunch(ctx->graph, ctx->gstream));
    g_launches.fetch_add(ctx->graph_kernels);
    CK(cudaEventRecord(ctx->ev_out, ctx->gstream));
    CK(cudaStreamWaitEvent(user, ctx->ev_out, 0));
    s = ctx->gstream;
  } else {
    if ((rc = body(s))) return rc;
  }
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  Counters h = *ctx->h_result;
  if (h.table_ovf) {  // the half-size twin table overflowed: this call's labels are incomplete
    // rerun with twice the buckets (full size after the half-size table)
    ctx->table_shrink = std::min(ctx->table_shrink, ctx->label_shrink) - 1;
    if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
    ctx->graph = nullptr;
    if (ctx->table_shrink < kMinShrink)
      return set_err(ctx, TM_ERR_CAPACITY, "twin table displacement overflow at 8x size (degenerate keys?)");
    return kRetryTable;
  }
  rc = decode_status(ctx, h);
  if (rc == TM_ERR_CAPACITY) {
    // labels are ours: relabeling restores the pre-repair frontier exactly
    ctx->path_hv = ctx->hv.as<int32_t>();  // the traversal's slot half-edges are still in place
    rc = retry_repair(ctx, tri32, hw, tv, T, off0, v0, &dc->n_seeds, d_off, d_v, s, &h, rc,
                      [&](cudaStream_t st) -> int {
                        launch_relabel(ctx->max_edge.as<int8_t>(), T, hw, ctx->seed.as<uint8_t>(), st);
                        CK(cudaGetLastError());
                        return TM_OK;
                      });
    ctx->path_hv = nullptr;
    if (ctx->graph) cudaGraphExecDestroy(ctx->graph);  // pool size changed
    ctx->graph = nullptr;
  }
  if (rc) return rc;
  for (int k = 0; k < 3; k++) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ctx->ev[k], ctx->ev[k + 1]) == cudaSuccess) ctx->phase_ms[k] = ms;
  }
  *n_polys = h.p_out;
  *n_slots = h.f_out;
  fill_stats(h, stats);
  ctx->last_T = T;
  return TM_OK;
}

int tm_mesh_to_polygons(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T,
                        int check, int64_t* d_off, int32_t* d_v, int64_t cap_polys, int64_t cap_slots,
                        int64_t* n_polys, int64_t* n_slots, int64_t* stats, void* stream) {
  if (!ctx || !n_polys || !n_slots) return TM_ERR_ARGUMENT;
  if (tri_bits != 32 && tri_bits != 64) return set_err(ctx, TM_ERR_ARGUMENT, "tri_bits must be 32 or 64");
  if (cap_polys < T || cap_slots < 3 * T)
    return set_err(ctx, TM_ERR_ARGUMENT, "output capacities must be at least T polygons and 3T slots");
  int rc = run_device(ctx, d_xy, n, d_tri, tri_bits, T, check, d_off, d_v, n_polys, n_slots, stats,
                      (cudaStream_t)stream);
  while (rc == kRetryTable)  // displacement overflow: again with twice the buckets
    rc = run_device(ctx, d_xy, n, d_tri, tri_bits, T, check, d_off, d_v, n_polys, n_slots, stats,
                    (cudaStream_t)stream);
  ctx->last_host = false;
  return rc;
}

int tm_resume_pinch(tm_ctx* ctx, int64_t extra_total, int64_t* off_out, int32_t* v_out, int64_t cap_polys,
                    int64_t cap_slots, int64_t* n_polys, int64_t* n_slots, int64_t* stats, void* stream) {
  if (!ctx || !n_polys || !n_slots || !off_out || !v_out) return TM_ERR_ARGUMENT;
  if (ctx->last_T < 0) return set_err(ctx, TM_ERR_ARGUMENT, "tm_resume_pinch needs a preceding whole-path call");
  const int64_t T = ctx->last_T, Tn = T > 0 ? T : 1;
  const unsigned long long local = ctx->h_result->stats[5];
  if (extra_total < (int64_t)local)
    return set_err(ctx, TM_ERR_ARGUMENT, "global extra visits %lld below this rank's %llu", (long long)extra_total,
                   local);
  if (cap_polys < T || cap_slots < 3 * T)
    return set_err(ctx, TM_ERR_ARGUMENT, "output capacities must be at least T polygons and 3T slots");
  const bool host = ctx->last_host;
  cudaStream_t s = host ? ctx->gstream : (cudaStream_t)stream;
  Counters* dc = dc_of(ctx);
  int64_t* d_off = host ? ctx->fin_off.as<int64_t>() : off_out;
  int32_t* d_v = host ? ctx->fin_v.as<int32_t>() : v_out;
  const int64_t* off0 = ctx->off0.as<int64_t>();
  const int32_t* v0 = ctx->v0.as<int32_t>();
  *ctx->h_pin = extra_total - (int64_t)local;
  CK(cudaMemcpyAsync(&dc->stats[8], ctx->h_pin, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  ctx->path_hv = ctx->hv.as<int32_t>();
  RepairArgs a = repair_args(ctx, ctx->tri32.as<int32_t>(), ctx->hw.as<int32_t>(), ctx->tv.as<int32_t>(), T, off0,
                             v0);
  launch_repair_pinch(a, 3, s);
  ctx->path_hv = nullptr;
  enqueue_stitch(ctx, off0, v0, &dc->n_seeds, Tn, d_off, d_v, true, s);
  CK(cudaGetLastError());
  Counters h;
  int rc = finish(ctx, s, &h);
  if (rc) return rc;  // (a pool overflow here is not retried: the pinch pass allocates little)
  *n_polys = h.p_out;
  *n_slots = h.f_out;
  fill_stats(h, stats);
  if (host) {
    CK(cudaMemcpyAsync(off_out, d_off, (*n_polys + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v_out, d_v, *n_slots * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return TM_OK;
}

int tm_mesh_to_polygons_host(tm_ctx* ctx, const double* h_xy, int64_t n, const int64_t* h_tri, int64_t T, int check,
                             int64_t* h_off, int32_t* h_v, int64_t cap_polys, int64_t cap_slots, int64_t* n_polys,
                             int64_t* n_slots, int64_t* stats) {
  if (!ctx || !n_polys || !n_slots || (!h_xy && n) || (!h_tri && T)) return TM_ERR_ARGUMENT;
  int rc = check_sizes(ctx, n, T);
  if (rc) return rc;
  if (!ctx->gstream) CK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
  cudaStream_t s = ctx->gstream;
  int64_t Tn = T > 0 ? T : 1, nn = n > 0 ? n : 1;
  ENSURE(xy, 2 * nn * sizeof(double));
  ENSURE(tri, 3 * Tn * sizeof(int64_t));
  ENSURE(fin_off, (Tn + 1) * sizeof(int64_t));
  ENSURE(fin_v, 3 * Tn * sizeof(int32_t));
  if ((rc = path_buffers(ctx, n, T))) return rc;
  if (!ctx->cstream) CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  for (auto& e : ctx->chunk_ev)
    if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // Upload overlap: the vertices first (pass A gathers them at random), then
  // the triangles in chunks on a copy stream; label pass A runs on each chunk
  // as soon as it lands, so only the last chunk's pass A is exposed.  The
  // triangles are narrowed int64 -> int32 on the host first (host threads,
  // chunk k+1 while chunk k is in flight) into a pinned staging buffer: half
  // the PCIe bytes; an index outside [0, n) becomes -1, which the label pass
  // reports as index_range exactly like the int64 value.
  const bool narrow = ctx->host_narrow && T > 0;
  if (narrow && ctx->h_tri32_cap < 3 * Tn) {
    if (ctx->h_tri32) cudaFreeHost(ctx->h_tri32);
    ctx->h_tri32 = nullptr;
    ctx->h_tri32_cap = 0;
    CK(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_tri32), 3 * Tn * sizeof(int32_t)));
    ctx->h_tri32_cap = 3 * Tn;
  }
  CK(cudaMemcpyAsync(ctx->xy.p, h_xy, 2 * n * sizeof(double), cudaMemcpyHostToDevice, s));
  if ((rc = enqueue_reset(ctx, s))) return rc;
  const int shrink = check && ctx->table_shrink > 0 ? 0 : ctx->table_shrink;
  launch_label_a_prepare(n, T, nullptr, ctx->slots.p, s, shrink);
  float* xy32 = (ctx->use_xy32 && !check) ? ctx->xy32.as<float>() : nullptr;
  if (xy32) launch_xy32(ctx->xy.as<double>(), n, xy32, s);
  CK(cudaEventRecord(ctx->chunk_ev[0], s));
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->chunk_ev[0], 0));  // table reset before any chunk's pass A
  // host narrowing workers: worker w converts its slice of every chunk in
  // order and counts chunk k done; the main thread enqueues chunk k's copy as
  // soon as all workers have passed it
  std::vector<std::thread> workers;
  std::atomic<int> done[kUploadChunks];
  for (auto& d : done) d.store(0);
  const int nw = narrow ? host_workers(3 * T) : 0;
  int32_t* st32 = ctx->h_tri32;
  for (int w = 0; w < nw; w++)
    workers.emplace_back([&, w] {
      for (int k = 0; k < kUploadChunks; k++) {
        const int64_t a = 3 * (T * k / kUploadChunks), b = 3 * (T * (k + 1) / kUploadChunks);
        const int64_t x0 = a + (b - a) * w / nw, x1 = a + (b - a) * (w + 1) / nw;
        for (int64_t i = x0; i < x1; i++) {
          const int64_t x = h_tri[i];
          st32[i] = (x >= 0 && x < n) ? (int32_t)x : -1;
        }
        done[k].fetch_add(1, std::memory_order_release);
      }
    });
  int crc = TM_OK;
  for (int k = 0; k < kUploadChunks && crc == TM_OK; k++) {
    const int64_t t0 = T * k / kUploadChunks, t1 = T * (k + 1) / kUploadChunks;
    if (narrow) {
      while (done[k].load(std::memory_order_acquire) < nw) std::this_thread::yield();
      if (t1 > t0 && cudaMemcpyAsync(ctx->tri32.as<int32_t>() + 3 * t0, st32 + 3 * t0,
                                     3 * (t1 - t0) * sizeof(int32_t), cudaMemcpyHostToDevice,
                                     ctx->cstream) != cudaSuccess)
        crc = TM_ERR_CUDA;
    } else if (t1 > t0 && cudaMemcpyAsync(ctx->tri.as<int64_t>() + 3 * t0, h_tri + 3 * t0,
                                          3 * (t1 - t0) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                          ctx->cstream) != cudaSuccess) {
      crc = TM_ERR_CUDA;
    }
    if (crc) break;
    cudaEventRecord(ctx->chunk_ev[k], ctx->cstream);
    cudaStreamWaitEvent(s, ctx->chunk_ev[k], 0);
    if (narrow)
      launch_label_a_range(ctx->xy.as<double>(), n, ctx->tri32.p, 0, T, t0, t1, check, ctx->tri32.as<int32_t>(),
                           ctx->hw.as<int32_t>(), ctx->max_edge.as<int8_t>(), ctx->seed.as<uint8_t>(), nullptr,
                           ctx->slots.p, &dc_of(ctx)->st, s, shrink, &dc_of(ctx)->table_ovf, xy32, ctx->label_one != 0);
    else
      launch_label_a_range(ctx->xy.as<double>(), n, ctx->tri.p, 1, T, t0, t1, check, ctx->tri32.as<int32_t>(),
                           ctx->hw.as<int32_t>(), ctx->max_edge.as<int8_t>(), ctx->seed.as<uint8_t>(), nullptr,
                           ctx->slots.p, &dc_of(ctx)->st, s, shrink, &dc_of(ctx)->table_ovf, xy32, ctx->label_one != 0);
  }
  for (auto& t : workers) t.join();
  if (crc) return set_err(ctx, crc, "triangle upload failed");
  CK(cudaGetLastError());
  ctx->label_a_external = true;
  rc = run_device(ctx, ctx->xy.as<double>(), n, narrow ? ctx->tri32.p : ctx->tri.p, narrow ? 32 : 64, T, check,
                  ctx->fin_off.as<int64_t>(), ctx->fin_v.as<int32_t>(), n_polys, n_slots, stats, s);
  ctx->label_a_external = false;
  ctx->last_host = true;
  if (rc == kRetryTable)  // the half-size twin table overflowed: once more at full size
    return tm_mesh_to_polygons_host(ctx, h_xy, n, h_tri, T, check, h_off, h_v, cap_polys, cap_slots, n_polys,
                                    n_slots, stats);
  if (rc) return rc;
  if (*n_polys > cap_polys || *n_slots > cap_slots)
    return set_err(ctx, TM_ERR_CAPACITY, "host output capacity too small (%lld polygons, %lld slots needed)",
                   (long long)*n_polys, (long long)*n_slots);
  CK(cudaMemcpyAsync(h_off, ctx->fin_off.p, (*n_polys + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h_v, ctx->fin_v.p, *n_slots * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return TM_OK;
}

// n_vertices < 0: the largest vertex id of the CSR + 1 (one extra round trip)
static int resolve_vertex_count(tm_ctx* ctx, const int64_t* d_off, const int32_t* d_v, int64_t P, int64_t* n,
                                cudaStream_t s) {
  if (*n >= 0) return TM_OK;
  *n = 0;
  if (P <= 0) return TM_OK;
  CK(cudaMemcpyAsync(ctx->h_pin, d_off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t F = *ctx->h_pin;
  int* dmax = reinterpret_cast<int*>(&dc_of(ctx)->post_pad);
  launch_max_vertex(d_v, F, dmax, s);
  CK(cudaMemcpyAsync(ctx->h_pin, dmax, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *n = (int64_t)(*reinterpret_cast<int*>(ctx->h_pin)) + 1;
  return TM_OK;
}

// ---------------------------------------------------------------- validation / analytics / canonical form
// (tm_post.cu).  Each call enqueues on `stream`, reads the counters back and
// decodes the status like the phase functions.

int tm_check_trivertex(tm_ctx* ctx, const void* d_tri, int tri_bits, int64_t T, const int64_t* d_trivertex,
                       int64_t n, void* stream) {
  if (!ctx || (tri_bits != 32 && tri_bits != 64) || T < 0 || n < 0) return TM_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = init_counters(ctx);
  if (rc || (rc = enqueue_reset(ctx, s))) return rc;
  ENSURE(pbits, ((n + 31) / 32 + 1) * sizeof(uint32_t));
  launch_check_trivertex(d_tri, tri_bits == 64, T, d_trivertex, n, ctx->pbits.as<uint32_t>(), &dc_of(ctx)->st, s);
  CK(cudaGetLastError());
  Counters h;
  return finish(ctx, s, &h);
}

int tm_polygon_stats(tm_ctx* ctx, const int64_t* d_off, const int32_t* d_v, int64_t P, int64_t n_vertices,
                     uint8_t* d_tip, uint8_t* d_repeated, int32_t* d_unique, int64_t* extra_visits,
                     int64_t* unique_vertices, int64_t* boundary_edges, void* stream) {
  if (!ctx || P < 0) return TM_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = init_counters(ctx);
  if (rc || (rc = resolve_vertex_count(ctx, d_off, d_v, P, &n_vertices, s)) || (rc = enqueue_reset(ctx, s))) return rc;
  Counters* dc = dc_of(ctx);
  const int64_t Pn = P > 0 ? P : 1, nn = n_vertices > 0 ? n_vertices : 1;
  int64_t F = 0;
  if (P > 0) {
    CK(cudaMemcpyAsync(ctx->h_pin, d_off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    F = *ctx->h_pin;
  }
  ENSURE(ptip, Pn);
  ENSURE(prep, Pn);
  ENSURE(plong, Pn * sizeof(int32_t));
  ENSURE(pstamp, nn * sizeof(int32_t));
  if (ctx->pstamp_clean != ctx->pstamp.gen) {  // INT_MAX once per allocation; k_poly_flags_long restores it
    CK(cudaMemsetAsync(ctx->pstamp.p, 0x7F, ctx->pstamp.bytes, s));
    ctx->pstamp_clean = ctx->pstamp.gen;
  }
  ENSURE(pflag, nn);
  ENSURE(ptiles, (scan_scratch_elems(nn) + 8) * sizeof(int64_t));
  int64_t slots = 64;
  while (slots < 2 * F + 64) slots <<= 1;
  ENSURE(ptable, slots * sizeof(unsigned long long));
  uint8_t* tip = d_tip ? d_tip : ctx->ptip.as<uint8_t>();
  uint8_t* rep = d_repeated ? d_repeated : ctx->prep.as<uint8_t>();
  launch_poly_flags(d_off, P, d_v, tip, rep, &dc->post_extra, ctx->plong.as<int32_t>(), &dc->post_nlong,
                    ctx->pstamp.as<int32_t>(), s);
  launch_edge_set(d_off, P, d_v, ctx->ptable.as<unsigned long long>(), slots, &dc->post_edges, s);
  launch_mark_vertices(d_v, F, n_vertices, ctx->pflag.as<uint8_t>(), &dc->st, s);
  if (d_unique)
    launch_select_flags(ctx->pflag.as<uint8_t>(), n_vertices, d_unique, &dc->post_unique, ctx->ptiles.as<int64_t>(),
                        s, 0);
  else {
    ENSURE(porder, nn * sizeof(int32_t));
    launch_select_flags(ctx->pflag.as<uint8_t>(), n_vertices, ctx->porder.as<int32_t>(), &dc->post_unique,
                        ctx->ptiles.as<int64_t>(), s, 0);
  }
  CK(cudaGetLastError());
  Counters h;
  if ((rc = finish(ctx, s, &h))) return rc;
  if (extra_visits) *extra_visits = (int64_t)h.post_extra;
  if (unique_vertices) *unique_vertices = n_vertices > 0 ? h.post_unique : 0;
  if (boundary_edges) *boundary_edges = (int64_t)h.post_edges;
  return TM_OK;
}

int tm_polygon_areas(tm_ctx* ctx, const int64_t* d_off, const int32_t* d_v, int64_t P, const double* d_xy,
                     double* d_area, void* stream) {
  if (!ctx || P < 0) return TM_ERR_ARGUMENT;
  launch_poly_areas(d_off, P, d_v, d_xy, d_area, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return TM_OK;
}

int tm_canonicalize(tm_ctx* ctx, const int64_t* d_off, const int32_t* d_v, int64_t P, int64_t n_vertices,
                    int64_t* d_off_out, int32_t* d_v_out, void* stream) {
  if (!ctx || P < 0) return TM_ERR_ARGUMENT;
  if (n_vertices >= (int64_t)0x7FFFFFFF) return set_err(ctx, TM_ERR_ARGUMENT, "vertex ids must fit in 31 bits");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = init_counters(ctx);
  if (rc || (rc = resolve_vertex_count(ctx, d_off, d_v, P, &n_vertices, s)) || (rc = enqueue_reset(ctx, s))) return rc;
  Counters* dc = dc_of(ctx);
  const int64_t Pn = P > 0 ? P : 1, nb = n_vertices + 1;  // buckets: empty polygons, then one per minimum vertex
  ENSURE(prot, Pn * sizeof(int32_t));
  ENSURE(pbucket, Pn * sizeof(int32_t));
  ENSURE(porder, (Pn > nb ? Pn : nb) * sizeof(int32_t));
  ENSURE(phist, (nb + 2) * sizeof(int64_t));
  ENSURE(pstart, (nb + 2) * sizeof(int64_t));
  ENSURE(pcursor, (nb + 2) * sizeof(int64_t));
  ENSURE(plen, (Pn + 1) * sizeof(int64_t));
  ENSURE(lbscan, scan_lookback_bytes(Pn > nb ? Pn : nb));
  int64_t* hp = ctx->h_pin;
  hp[0] = nb;
  hp[1] = P;
  CK(cudaMemcpyAsync(&dc->post_nb, hp, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(&dc->p_in, hp + 1, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  unsigned long long* hist = ctx->phist.as<unsigned long long>();
  launch_canon_rot(d_off, P, d_v, n_vertices, ctx->prot.as<int32_t>(), ctx->pbucket.as<int32_t>(), hist, &dc->st, s);
  launch_scan_lookback(reinterpret_cast<const int64_t*>(hist), nullptr, ctx->pstart.as<int64_t>(), nullptr,
                       &dc->post_nb, nb, ctx->lbscan.p, s);
  launch_canon_sort(P, n_vertices, d_off, d_v, ctx->prot.as<int32_t>(), ctx->pbucket.as<int32_t>(),
                    ctx->pstart.as<int64_t>(), ctx->pcursor.as<unsigned long long>(), ctx->porder.as<int32_t>(), s);
  launch_canon_lengths(ctx->porder.as<int32_t>(), P, d_off, ctx->plen.as<int64_t>(), s);
  launch_scan_lookback(ctx->plen.as<int64_t>(), nullptr, d_off_out, nullptr, &dc->p_in, Pn, ctx->lbscan.p, s);
  launch_canon_write(ctx->porder.as<int32_t>(), P, d_off, d_v, ctx->prot.as<int32_t>(), d_off_out, d_v_out, s);
  CK(cudaGetLastError());
  Counters h;
  return finish(ctx, s, &h);
}

// ---------------------------------------------------------------- GPU Delaunay (tm_delaunay.cu)
int tm_delaunay(tm_ctx* ctx, const double* d_xy, int64_t n, const double* box, int32_t* d_tri, int64_t cap_tris,
                int64_t* n_tris, int32_t* d_open, int64_t* n_open, int64_t* n_degenerate, void* stream) {
  if (!ctx || !box || !n_tris || !n_open || n < 0 || n >= (int64_t)0x7FFFFFFF) return TM_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = init_counters(ctx);
  if (rc || (rc = enqueue_reset(ctx, s))) return rc;
  Counters* dc = dc_of(ctx);
  const double x0 = box[0], y0 = box[1], x1 = box[2], y1 = box[3];
  if (!(x1 > x0 && y1 > y0)) return set_err(ctx, TM_ERR_ARGUMENT, "empty box");
  int64_t G = 1;
  while ((G + 1) * (G + 1) * 2 <= n) G++;  // ~2 points per cell
  if (G > 46000) G = 46000;
  const int64_t nc = G * G, nn = n > 0 ? n : 1;
  ENSURE(dcell, nn * sizeof(int32_t));
  ENSURE(dhist, (nc + 2) * sizeof(int64_t));
  ENSURE(dstart, (nc + 2) * sizeof(int64_t));
  ENSURE(dcursor, (nc + 2) * sizeof(int64_t));
  ENSURE(dids, nn * sizeof(int32_t));
  ENSURE(dsxy, 2 * nn * sizeof(double));
  ENSURE(dcnt, (nn + 1) * sizeof(int64_t));
  ENSURE(doff, (nn + 1) * sizeof(int64_t));
  ENSURE(lbscan, scan_lookback_bytes(nc > nn ? nc : nn));
  int64_t* hp = ctx->h_pin;
  hp[0] = nc;
  hp[1] = n;
  CK(cudaMemcpyAsync(&dc->dl_ncell, hp, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  launch_delaunay_cells(d_xy, n, x0, y0, x1, y1, (int)G, ctx->dcell.as<int32_t>(),
                        ctx->dhist.as<unsigned long long>(), s);
  launch_scan_lookback(ctx->dhist.as<int64_t>(), nullptr, ctx->dstart.as<int64_t>(), nullptr, &dc->dl_ncell, nc,
                       ctx->lbscan.p, s);
  launch_delaunay_scatter(d_xy, n, (int)G, ctx->dcell.as<int32_t>(), ctx->dstart.as<int64_t>(),
                          ctx->dcursor.as<unsigned long long>(), ctx->dids.as<int32_t>(), ctx->dsxy.as<double>(), s);
  launch_delaunay_stars(ctx->dstart.as<int64_t>(), ctx->dids.as<int32_t>(), ctx->dsxy.as<double>(), n, x0, y0, x1, y1,
                        (int)G, 0, ctx->dcnt.as<int64_t>(), nullptr, nullptr, d_open, &dc->dl_open, &dc->dl_degen, s);
  launch_scan_lookback(ctx->dcnt.as<int64_t>(), nullptr, ctx->doff.as<int64_t>(), nullptr, &dc->dl_n, nn,
                       ctx->lbscan.p, s, &dc->dl_ntri);
  Counters h;
  if ((rc = finish(ctx, s, &h))) return rc;
  *n_tris = h.dl_ntri;
  *n_open = h.dl_open;
  if (n_degenerate) *n_degenerate = h.dl_degen;
  if (h.dl_ntri > cap_tris)
    return set_err(ctx, TM_ERR_CAPACITY, "triangle capacity %lld below %lld", (long long)cap_tris,
                   (long long)h.dl_ntri);
  launch_delaunay_stars(ctx->dstart.as<int64_t>(), ctx->dids.as<int32_t>(), ctx->dsxy.as<double>(), n, x0, y0, x1, y1,
                        (int)G, 1, ctx->dcnt.as<int64_t>(), ctx->doff.as<int64_t>(), d_tri, nullptr, nullptr, nullptr,
                        s);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return TM_OK;
}

// ---------------------------------------------------------------- seed-partitioned labels (multi-GPU)
int tm_label_range(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T,
                   int64_t t_begin, int64_t t_end, uint64_t* d_keys, int32_t* d_vals, int64_t cap,
                   int64_t* n_boundary, void* stream) {
  if (!ctx || !n_boundary || !d_keys || !d_vals || (tri_bits != 32 && tri_bits != 64)) return TM_ERR_ARGUMENT;
  if (t_begin < 0 || t_end > T || t_end < t_begin) return set_err(ctx, TM_ERR_ARGUMENT, "bad triangle range");
  int rc = path_buffers(ctx, n, T);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  ENSURE(slots, hash_bytes_range(n, T, t_end - t_begin));
  if ((rc = enqueue_reset(ctx, s))) return rc;
  Counters* dc = dc_of(ctx);
  int32_t* tri32 = ctx->tri32.as<int32_t>();
  launch_tri32(d_tri, tri_bits == 64, T, tri32, s);  // corners of the whole mesh (walks leave the range)
  launch_label_range(d_xy, n, d_tri, tri_bits == 64, T, t_begin, t_end, tri32, ctx->hw.as<int32_t>(),
                     ctx->max_edge.as<int8_t>(), ctx->seed.as<uint8_t>(), ctx->slots.p, &dc->st, &dc->table_ovf, s);
  launch_boundary_extract(tri32, ctx->max_edge.as<int8_t>(), ctx->hw.as<int32_t>(), t_begin, t_end,
                          reinterpret_cast<unsigned long long*>(d_keys), d_vals, &dc->n_boundary, cap, s);
  CK(cudaGetLastError());
  Counters h;
  if ((rc = finish(ctx, s, &h))) return rc;
  if (h.table_ovf) return set_err(ctx, TM_ERR_CAPACITY, "range twin table displacement overflow");
  *n_boundary = (int64_t)h.n_boundary;
  if (*n_boundary > cap)
    return set_err(ctx, TM_ERR_CAPACITY, "%lld boundary entries, capacity %lld", (long long)*n_boundary,
                   (long long)cap);
  return TM_OK;
}

int tm_ctx_label_buffers(tm_ctx* ctx, int32_t** tri32, int32_t** hw, int8_t** max_edge, uint8_t** seed) {
  if (!ctx) return TM_ERR_ARGUMENT;
  if (tri32) *tri32 = ctx->tri32.as<int32_t>();
  if (hw) *hw = ctx->hw.as<int32_t>();
  if (max_edge) *max_edge = ctx->max_edge.as<int8_t>();
  if (seed) *seed = ctx->seed.as<uint8_t>();
  return TM_OK;
}

int tm_ctx_copy_labels(tm_ctx* ctx, int to_ctx, int32_t* d_hw, uint8_t* d_seed, int8_t* d_max_edge, int64_t t_begin,
                       int64_t t_end, void* stream) {
  if (!ctx || t_begin < 0 || t_end < t_begin || !ctx->hw.p) return TM_ERR_ARGUMENT;
  if ((size_t)t_end * 3 * sizeof(int32_t) > ctx->hw.bytes) return set_err(ctx, TM_ERR_ARGUMENT, "range beyond T");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t m = t_end - t_begin;
  int32_t* hw = ctx->hw.as<int32_t>() + 3 * t_begin;
  uint8_t* sd = ctx->seed.as<uint8_t>() + t_begin;
  int8_t* me = ctx->max_edge.as<int8_t>() + t_begin;
  if (to_ctx) {
    if (d_hw) CK(cudaMemcpyAsync(hw, d_hw + 3 * t_begin, 3 * m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    if (d_seed) CK(cudaMemcpyAsync(sd, d_seed + t_begin, m, cudaMemcpyDeviceToDevice, s));
    if (d_max_edge) CK(cudaMemcpyAsync(me, d_max_edge + t_begin, m, cudaMemcpyDeviceToDevice, s));
  } else {
    if (d_hw) CK(cudaMemcpyAsync(d_hw + 3 * t_begin, hw, 3 * m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    if (d_seed) CK(cudaMemcpyAsync(d_seed + t_begin, sd, m, cudaMemcpyDeviceToDevice, s));
    if (d_max_edge) CK(cudaMemcpyAsync(d_max_edge + t_begin, me, m, cudaMemcpyDeviceToDevice, s));
  }
  return TM_OK;
}

int tm_label_resolve(tm_ctx* ctx, const uint64_t* d_keys_all, const int32_t* d_vals_all, int64_t n_all,
                     int64_t own_begin, int64_t own_count, void* stream) {
  if (!ctx || n_all < 0 || own_begin < 0 || own_count < 0 || own_begin + own_count > n_all) return TM_ERR_ARGUMENT;
  int64_t slots = 64;  // a table of this rank's entries only (k_boundary_insert / k_boundary_match)
  while (slots < 2 * own_count + 64) slots <<= 1;
  ENSURE(btab, slots * sizeof(int32_t));
  launch_boundary_resolve(reinterpret_cast<const unsigned long long*>(d_keys_all), d_vals_all, n_all, own_begin,
                          own_begin + own_count, ctx->btab.as<int32_t>(), slots, ctx->hw.as<int32_t>(),
                          ctx->seed.as<uint8_t>(), (cudaStream_t)stream);
  CK(cudaGetLastError());
  return TM_OK;
}

int tm_polygons_from_labels(tm_ctx* ctx, int64_t n, int64_t T, int64_t* d_off, int32_t* d_v, int64_t cap_polys,
                            int64_t cap_slots, int64_t* n_polys, int64_t* n_slots, int64_t* stats, void* stream) {
  if (!ctx || !n_polys || !n_slots) return TM_ERR_ARGUMENT;
  if (cap_polys < T || cap_slots < 3 * T)
    return set_err(ctx, TM_ERR_ARGUMENT, "output capacities must be at least T polygons and 3T slots");
  ctx->labels_external = true;
  int rc = run_device(ctx, nullptr, n, nullptr, 32, T, 0, d_off, d_v, n_polys, n_slots, stats, (cudaStream_t)stream);
  ctx->labels_external = false;
  ctx->last_host = false;
  return rc;
}

}  // extern "C"
