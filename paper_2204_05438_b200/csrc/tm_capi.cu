// tm_capi.cu -- extern "C" entry points (include/termesh_b200.h) and the host
// orchestration of the device phases: workspace management, status decoding
// into the reference's error vocabulary, and the whole-path drivers.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <tuple>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/termesh_b200.h"
#include "tm_common.cuh"
#include "tm_internal.h"

using namespace tmb;

namespace {

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  bool ensure(size_t want) {
    if (want <= bytes && p) return true;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
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

struct Counters {       // device scratch, zeroed per phase
  DevStatus st;
  int64_t n_seeds;
  unsigned int n_overflow;
  unsigned int n_items;
  unsigned int n_long;
  unsigned int pad;
  unsigned long long pool_top;
  unsigned long long undo_top;
  unsigned long long stats[8];
};

// timed segments (tm_ctx_segment_ms); names in kSegNames
enum Seg {
  S_LABEL_A, S_LABEL_B, S_SEEDS, S_TRAV_START, S_TRAV_RULERS, S_TRAV_LEN, S_TRAV_SCAN, S_TRAV_WRITE,
  S_CLASSIFY, S_REPAIR_TIPS, S_REPAIR_PINCH, S_STITCH, S_NUM
};
const char* kSegNames[S_NUM] = {"label_a_tri_pass", "label_b_edges", "select_seeds", "trav_start", "trav_rulers",
                                "trav_chain",
                                "trav_scan", "trav_write", "repair_classify", "repair_tips", "repair_pinch",
                                "repair_stitch"};

struct Prof {
  bool on = false;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
  std::vector<cudaEvent_t> free_ev;
  double ms[S_NUM] = {0};
  long long cnt[S_NUM] = {0};
};

std::atomic<long long> g_launches{0};

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
  Buf counters, pinned_counters;
  // label
  Buf slots;
  // traversal
  Buf seeds, start, len, overflow, queue, stamp, temp, nrul, eoff, rnext, rdist, startbits, ent_r, ent_base;
  // repair
  Buf item_of, items, long_list, item_list, item_n, item_slots, cnt, slotsz, pbase, sbase, pool, undo;
  // whole-path buffers
  Buf xy, tri, tri32, hw, max_edge, seed, tv, off0, v0, fin_off, fin_v;
  Buf h_pin_in, h_pin_out;
  cudaStream_t own_stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  unsigned long long pool_cap_hint = 0;
};

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

#define CK(call)                                                         \
  do {                                                                   \
    cudaError_t _e = (call);                                             \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call);             \
  } while (0)

#define ENSURE(buf, bytes)                                                        \
  do {                                                                            \
    if (!ctx->buf.ensure(bytes)) return set_err(ctx, TM_ERR_CUDA, "cudaMalloc of %zu bytes for %s failed", \
                                                (size_t)(bytes), #buf);           \
  } while (0)

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

// Segment timers: CUDA events recorded on the launching stream around the kernels.
struct SegTimer {
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

static Counters* dev_counters(tm_ctx* ctx) { return ctx->counters.as<Counters>(); }

static int reset_counters(tm_ctx* ctx, cudaStream_t s) {
  if (!ctx->counters.ensure(sizeof(Counters))) return set_err(ctx, TM_ERR_CUDA, "cudaMalloc failed (counters)");
  if (!ctx->pinned_counters.p) {
    void* p = nullptr;
    if (cudaMallocHost(&p, sizeof(Counters)) != cudaSuccess) return set_err(ctx, TM_ERR_CUDA, "cudaMallocHost failed");
    ctx->pinned_counters.p = p;
    ctx->pinned_counters.bytes = sizeof(Counters);
  }
  Counters h;
  memset(&h, 0, sizeof h);
  for (int k = 0; k < K_NUM; k++) h.st.first[k] = ~0ull;
  memcpy(ctx->pinned_counters.p, &h, sizeof h);
  CK(cudaMemcpyAsync(ctx->counters.p, ctx->pinned_counters.p, sizeof h, cudaMemcpyHostToDevice, s));
  return TM_OK;
}

// fetch the counters to host (synchronizes s)
static int read_counters(tm_ctx* ctx, cudaStream_t s, Counters* out) {
  CK(cudaMemcpyAsync(ctx->pinned_counters.p, ctx->counters.p, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  memcpy(out, ctx->pinned_counters.p, sizeof(Counters));
  return TM_OK;
}

static const char* kind_name(int k) {
  static const char* names[K_NUM] = {"index_range", "orientation", "degenerate", "duplicate", "reciprocity",
                                     "edge_count", "trivertex", "neighbors", "walk", "no_frontier",
                                     "no_converge", "split_law", "pool", "barrier", "no_internal", "structural"};
  return names[k];
}

// Decode device status.  Validation kinds (0..7) -> TM_ERR_VALIDATION,
// structural kinds -> TM_ERR_STRUCTURAL with the reference's message wording.
static int decode_status(tm_ctx* ctx, const DevStatus& st, const char* phase, const Counters* cn = nullptr) {
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
        return set_err(ctx, TM_ERR_STRUCTURAL, "[%s] boundary walk from seed triangle %lld did not terminate", phase, f);
      case K_NO_FRONTIER:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[%s] no frontier edge reachable from triangle %lld", phase, f);
      case K_NO_CONVERGE:
        return set_err(ctx, TM_ERR_STRUCTURAL,
                       "[%s] tip removal did not converge (polygon %lld; initial repeated-vertex count %llu)", phase,
                       f, cn ? cn->stats[2] : 0ull);
      case K_SPLIT_LAW:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[%s] polygon %lld: split broke the length law |pa|+|pb| = |P|+2",
                       phase, f);
      case K_POOL:
        return set_err(ctx, TM_ERR_CAPACITY, "[%s] repair scratch pool exhausted (polygon %lld)", phase, f);
      case K_BARRIER:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[%s] polygon %lld: barrier edge not found around tip vertex", phase, f);
      case K_NO_INTERNAL:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[%s] polygon %lld: tip vertex has no internal edge to split on", phase,
                       f);
      default:
        return set_err(ctx, TM_ERR_STRUCTURAL, "[%s] structural failure at element %lld", phase, f);
    }
  }
  return TM_OK;
}

extern "C" {

int tm_version(void) { return 1; }

int tm_ctx_create(tm_ctx** out) {
  if (!out) return TM_ERR_ARGUMENT;
  *out = new tm_ctx();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    delete *out;
    *out = nullptr;
    return TM_ERR_CUDA;
  }
  return TM_OK;
}

void tm_ctx_destroy(tm_ctx* ctx) {
  if (!ctx) return;
  Buf* bufs[] = {&ctx->counters, &ctx->slots, &ctx->seeds, &ctx->start, &ctx->len, &ctx->overflow, &ctx->queue,
                 &ctx->stamp, &ctx->temp, &ctx->nrul, &ctx->eoff, &ctx->rnext, &ctx->rdist, &ctx->startbits,
                 &ctx->ent_r, &ctx->ent_base, &ctx->item_of, &ctx->items, &ctx->long_list, &ctx->item_list,
                 &ctx->item_n, &ctx->item_slots, &ctx->cnt, &ctx->slotsz, &ctx->pbase, &ctx->sbase, &ctx->pool,
                 &ctx->undo, &ctx->xy, &ctx->tri, &ctx->tri32, &ctx->hw, &ctx->max_edge, &ctx->seed, &ctx->tv,
                 &ctx->off0, &ctx->v0, &ctx->fin_off, &ctx->fin_v};
  for (Buf* b : bufs) b->release();
  if (ctx->pinned_counters.p) cudaFreeHost(ctx->pinned_counters.p);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  prof_flush(ctx);
  for (auto e : ctx->prof.free_ev) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
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

int tm_ctx_phase_ms(const tm_ctx* ctx, double* ms3) {
  if (!ctx || !ms3) return TM_ERR_ARGUMENT;
  for (int k = 0; k < 3; k++) ms3[k] = ctx->phase_ms[k];
  return TM_OK;
}

int tm_label(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T, int check,
             int32_t* d_tri32, int32_t* d_hw, int8_t* d_max_edge, uint8_t* d_seed, int32_t* d_tv, void* stream) {
  if (!ctx) return TM_ERR_ARGUMENT;
  if ((tri_bits != 32 && tri_bits != 64) || T < 0 || n < 0)
    return set_err(ctx, TM_ERR_ARGUMENT, "tri_bits must be 32 or 64 and sizes non-negative");
  if (3 * T >= (int64_t)0x7FFFFFFF) return set_err(ctx, TM_ERR_ARGUMENT, "3T must fit in 31 bits");
  if (n >= (int64_t)0x7F7F7F7F) return set_err(ctx, TM_ERR_ARGUMENT, "vertex count must fit in 31 bits");
  cudaStream_t s = (cudaStream_t)stream;
  for (int k = 0; k < K_NUM; k++) ctx->defect_count[k] = 0, ctx->defect_first[k] = -1;
  int rc = reset_counters(ctx, s);
  if (rc) return rc;
  uint64_t cap = hash_capacity(T);
  ENSURE(slots, cap * sizeof(uint32_t));
  {
    SegTimer st_(ctx, S_LABEL_A, s);
    launch_label_a(d_xy, n, d_tri, tri_bits == 64, T, check, d_tri32, d_hw, d_max_edge, d_tv,
                   ctx->slots.as<uint32_t>(), cap, &dev_counters(ctx)->st, s);
  }
  {
    SegTimer st_(ctx, S_LABEL_B, s);
    launch_label_b(n, T, d_hw, d_max_edge, d_seed, d_tv, s);
  }
  CK(cudaGetLastError());
  Counters h;
  if ((rc = read_counters(ctx, s, &h))) return rc;
  return decode_status(ctx, h.st, "label");
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
  int rc = reset_counters(ctx, s);
  if (rc) return rc;
  launch_check_neighbors(d_hw, d_nb, nb_bits == 64, T, &dev_counters(ctx)->st, s);
  CK(cudaGetLastError());
  Counters h;
  if ((rc = read_counters(ctx, s, &h))) return rc;
  return decode_status(ctx, h.st, "validate");
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
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_counters(ctx, s);
  if (rc) return rc;
  Counters* dc = dev_counters(ctx);
  int64_t Tn = T > 0 ? T : 1;
  ENSURE(seeds, Tn * sizeof(int32_t));
  size_t tb = select_seeds_temp_bytes(Tn);
  size_t tb2 = scan_temp_bytes(Tn + 1);
  ENSURE(temp, (tb > tb2 ? tb : tb2) + 256);
  Counters h;
  int64_t P = 0;
  if (T > 0) {
    {
      SegTimer st_(ctx, S_SEEDS, s);
      launch_select_seeds(d_seed, T, ctx->seeds.as<int32_t>(), &dc->n_seeds, ctx->temp.p, ctx->temp.bytes, s);
    }
    CK(cudaGetLastError());
    if ((rc = read_counters(ctx, s, &h))) return rc;
    P = h.n_seeds;
  }
  if (P > cap_polys) return set_err(ctx, TM_ERR_CAPACITY, "polygon capacity %lld < %lld seeds", (long long)cap_polys, (long long)P);
  *n_polys = P;
  CK(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), s));
  if (P == 0) {
    *n_slots = 0;
    return TM_OK;
  }
  ENSURE(start, P * sizeof(int32_t));
  ENSURE(len, (P + 1) * sizeof(int64_t));
  ENSURE(nrul, (P + 1) * sizeof(int64_t));
  ENSURE(eoff, (P + 1) * sizeof(int64_t));
  ENSURE(overflow, P * sizeof(int32_t));
  ENSURE(queue, Tn * sizeof(int32_t));
  ENSURE(stamp, Tn * sizeof(int32_t));
  ENSURE(rnext, 3 * Tn * sizeof(int32_t));
  ENSURE(rdist, 3 * Tn * sizeof(int32_t));
  const int64_t nbits = (3 * Tn + 31) / 32;
  ENSURE(startbits, nbits * sizeof(uint32_t));
  // ruler entries: seed starts + the 1/8 hash sample of half-edges (+ slack)
  const int64_t ecap = P + (3 * Tn) / 8 + (3 * Tn) / 16 + 1024;
  ENSURE(ent_r, ecap * sizeof(int32_t));
  ENSURE(ent_base, ecap * sizeof(int64_t));
  CK(cudaMemsetAsync(ctx->stamp.p, 0xFF, Tn * sizeof(int32_t), s));
  CK(cudaMemsetAsync(ctx->startbits.p, 0, nbits * sizeof(uint32_t), s));
  {
    SegTimer st_(ctx, S_TRAV_START, s);
    launch_trav_start(d_hw, ctx->seeds.as<int32_t>(), P, ctx->start.as<int32_t>(), ctx->overflow.as<int32_t>(),
                      &dc->n_overflow, ctx->queue.as<int32_t>(), ctx->stamp.as<int32_t>(),
                      ctx->startbits.as<uint32_t>(), &dc->st, s);
  }
  {
    SegTimer st_(ctx, S_TRAV_RULERS, s);
    launch_ruler_walk(d_hw, ctx->startbits.as<uint32_t>(), T, ctx->rnext.as<int32_t>(), ctx->rdist.as<int32_t>(),
                      &dc->st, s);
  }
  CK(cudaMemsetAsync(ctx->len.as<int64_t>() + P, 0, sizeof(int64_t), s));
  CK(cudaMemsetAsync(ctx->nrul.as<int64_t>() + P, 0, sizeof(int64_t), s));
  {
    SegTimer st_(ctx, S_TRAV_LEN, s);
    launch_chain_count(ctx->seeds.as<int32_t>(), ctx->start.as<int32_t>(), P, T, ctx->rnext.as<int32_t>(),
                       ctx->rdist.as<int32_t>(), ctx->len.as<int64_t>(), ctx->nrul.as<int64_t>(), &dc->st, s);
  }
  {
    SegTimer st_(ctx, S_TRAV_SCAN, s);
    launch_scan(ctx->len.as<int64_t>(), d_offsets, P + 1, ctx->temp.p, ctx->temp.bytes, s);
    launch_scan(ctx->nrul.as<int64_t>(), ctx->eoff.as<int64_t>(), P + 1, ctx->temp.p, ctx->temp.bytes, s);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&dc->stats[0], d_offsets + P, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(&dc->stats[1], ctx->eoff.as<int64_t>() + P, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  if ((rc = read_counters(ctx, s, &h))) return rc;
  if ((rc = decode_status(ctx, h.st, "traversal"))) return rc;
  int64_t total = (int64_t)h.stats[0], n_ent = (int64_t)h.stats[1];
  if (total > cap_slots)
    return set_err(ctx, TM_ERR_STRUCTURAL, "[traversal] polygon storage capacity exceeded; labels are inconsistent");
  if (n_ent > ecap) return set_err(ctx, TM_ERR_CAPACITY, "[traversal] ruler entry capacity exceeded");
  {
    SegTimer st_(ctx, S_TRAV_WRITE, s);
    launch_chain_emit(ctx->start.as<int32_t>(), P, ctx->rnext.as<int32_t>(), ctx->rdist.as<int32_t>(), d_offsets,
                      ctx->eoff.as<int64_t>(), ctx->ent_r.as<int32_t>(), ctx->ent_base.as<int64_t>(), s);
    launch_ruler_write(d_tri32, d_hw, ctx->eoff.as<int64_t>() + P, ctx->ent_r.as<int32_t>(),
                       ctx->ent_base.as<int64_t>(), ctx->rdist.as<int32_t>(), T, d_verts, s);
  }
  CK(cudaGetLastError());
  *n_slots = total;
  return TM_OK;
}

int tm_repair(tm_ctx* ctx, const int32_t* d_tri32, int32_t* d_hw, const int32_t* d_tv, int64_t T,
              const int64_t* d_off_in, const int32_t* d_v_in, int64_t P, int64_t* d_off_out, int32_t* d_v_out,
              int64_t cap_polys, int64_t cap_slots, int64_t* n_polys_out, int64_t* n_slots_out, int64_t* stats,
              void* stream) {
  if (!ctx || !n_polys_out || !n_slots_out) return TM_ERR_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_counters(ctx, s);
  if (rc) return rc;
  Counters* dc = dev_counters(ctx);
  Counters h;
  int64_t Pn = P > 0 ? P : 1;
  if (stats)
    for (int k = 0; k < TM_NUM_STATS; k++) stats[k] = 0;
  if (P <= 0) {
    CK(cudaMemsetAsync(d_off_out, 0, sizeof(int64_t), s));
    CK(cudaStreamSynchronize(s));
    *n_polys_out = 0;
    *n_slots_out = 0;
    if (stats) stats[TM_STAT_ROUNDS] = 1;
    return TM_OK;
  }
  ENSURE(item_of, Pn * sizeof(int32_t));
  ENSURE(items, Pn * sizeof(int32_t));
  ENSURE(long_list, Pn * sizeof(int32_t));
  ENSURE(item_list, Pn * sizeof(int64_t));
  ENSURE(item_n, Pn * sizeof(int32_t));
  ENSURE(item_slots, Pn * sizeof(int64_t));
  {
    SegTimer st_(ctx, S_CLASSIFY, s);
    launch_classify(d_off_in, d_v_in, P, ctx->item_of.as<int32_t>(), ctx->items.as<int32_t>(), &dc->n_items,
                    ctx->long_list.as<int32_t>(), &dc->n_long, dc->stats, s);
  }
  CK(cudaGetLastError());
  int64_t in_slots = 0;
  CK(cudaMemcpyAsync(&dc->pool_top, d_off_in + P, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  if ((rc = read_counters(ctx, s, &h))) return rc;
  in_slots = (int64_t)h.pool_top;
  unsigned int n_items = h.n_items;
  unsigned long long pool_cap = ctx->pool_cap_hint;
  unsigned long long want = 4ull * (unsigned long long)in_slots + 64ull * n_items + (1ull << 20);
  if (pool_cap < want) pool_cap = want;
  unsigned long long undo_cap = (unsigned long long)T + 1024;
  ENSURE(undo, undo_cap * sizeof(int32_t));
  for (int attempt = 0;; attempt++) {
    if (pool_cap >= (1ull << 32)) return set_err(ctx, TM_ERR_CAPACITY, "[reparation] scratch pool exceeds 2^32 slots");
    ENSURE(pool, pool_cap * sizeof(int32_t));
    // reset repair-phase counters but keep classify results (stats[2], stats[6], n_items)
    CK(cudaMemsetAsync(&dc->pool_top, 0, sizeof(unsigned long long) * 2, s));
    CK(cudaMemsetAsync(&dc->stats[0], 0, sizeof(unsigned long long) * 2, s));
    CK(cudaMemsetAsync(&dc->stats[3], 0, sizeof(unsigned long long) * 3, s));
    RepairArgs a{d_tri32, d_hw, d_tv, T, ctx->pool.as<int32_t>(), pool_cap, &dc->pool_top, ctx->undo.as<int32_t>(),
                 &dc->undo_top, undo_cap, &dc->st, ctx->items.as<int32_t>(), &dc->n_items, d_off_in, d_v_in,
                 ctx->item_list.as<int64_t>(), ctx->item_n.as<int32_t>(), ctx->item_slots.as<int64_t>(), dc->stats};
    if (n_items > 0) {
      {
        SegTimer st_(ctx, S_REPAIR_TIPS, s);
        launch_repair_tips(a, s);
      }
      {
        SegTimer st_(ctx, S_REPAIR_PINCH, s);
        launch_repair_pinch(a, s);
      }
    }
    CK(cudaGetLastError());
    if ((rc = read_counters(ctx, s, &h))) return rc;
    if (h.st.count[K_POOL] && attempt < 6) {
      if (h.undo_top > undo_cap)
        return set_err(ctx, TM_ERR_CAPACITY, "[reparation] scratch pool and promotion log both overflowed");
      launch_undo(d_hw, ctx->undo.as<int32_t>(), &dc->undo_top, undo_cap, s);
      CK(cudaMemsetAsync(&dc->st, 0, sizeof(DevStatus), s));
      // DevStatus.first must be ~0: re-reset only the status block
      Counters z;
      memset(&z, 0, sizeof z);
      for (int k = 0; k < K_NUM; k++) z.st.first[k] = ~0ull;
      memcpy(ctx->pinned_counters.p, &z.st, sizeof z.st);
      CK(cudaMemcpyAsync(&dc->st, ctx->pinned_counters.p, sizeof z.st, cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));
      pool_cap *= 4;
      ctx->pool_cap_hint = pool_cap;
      continue;
    }
    if ((rc = decode_status(ctx, h.st, "reparation", &h))) return rc;
    break;
  }
  ENSURE(cnt, (Pn + 1) * sizeof(int64_t));
  ENSURE(slotsz, (Pn + 1) * sizeof(int64_t));
  ENSURE(pbase, (Pn + 1) * sizeof(int64_t));
  ENSURE(sbase, (Pn + 1) * sizeof(int64_t));
  size_t tb = scan_temp_bytes(Pn + 1);
  ENSURE(temp, tb + 256);
  SegTimer* stitch_timer = new SegTimer(ctx, S_STITCH, s);
  launch_out_counts(d_off_in, P, ctx->item_of.as<int32_t>(), ctx->item_n.as<int32_t>(),
                    ctx->item_slots.as<int64_t>(), ctx->cnt.as<int64_t>(), ctx->slotsz.as<int64_t>(), s);
  launch_scan(ctx->cnt.as<int64_t>(), ctx->pbase.as<int64_t>(), P + 1, ctx->temp.p, ctx->temp.bytes, s);
  launch_scan(ctx->slotsz.as<int64_t>(), ctx->sbase.as<int64_t>(), P + 1, ctx->temp.p, ctx->temp.bytes, s);
  CK(cudaGetLastError());
  int64_t tot[2];
  CK(cudaMemcpyAsync(&tot[0], ctx->pbase.as<int64_t>() + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&tot[1], ctx->sbase.as<int64_t>() + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (tot[0] > cap_polys || tot[1] > cap_slots) {
    delete stitch_timer;
    return set_err(ctx, TM_ERR_CAPACITY, "[reparation] output capacity (%lld polygons, %lld slots) < (%lld, %lld)",
                   (long long)cap_polys, (long long)cap_slots, (long long)tot[0], (long long)tot[1]);
  }
  launch_stitch(d_off_in, d_v_in, P, ctx->item_of.as<int32_t>(), ctx->item_list.as<int64_t>(),
                ctx->item_n.as<int32_t>(), ctx->pool.as<int32_t>(), ctx->pbase.as<int64_t>(),
                ctx->sbase.as<int64_t>(), d_off_out, d_v_out, s);
  delete stitch_timer;
  CK(cudaGetLastError());
  *n_polys_out = tot[0];
  *n_slots_out = tot[1];
  if (stats) {
    stats[TM_STAT_ROUNDS] = h.stats[0] > 0 ? (int64_t)h.stats[0] : 1;
    stats[TM_STAT_SPLITS] = (int64_t)(h.stats[1] + h.stats[4]);
    stats[TM_STAT_INITIAL_TIPS] = (int64_t)h.stats[2];
    stats[TM_STAT_UNREPAIRED] = (int64_t)h.stats[3];
    stats[TM_STAT_NONSIMPLE] = (int64_t)h.stats[6];
    stats[TM_STAT_TIP_SPLITS] = (int64_t)h.stats[1];
    stats[TM_STAT_PINCH_SPLITS] = (int64_t)h.stats[4];
    stats[TM_STAT_WORK_ITEMS] = (int64_t)h.n_items;
  }
  return TM_OK;
}

static int run_device(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T,
                      int check, int64_t* d_off, int32_t* d_v, int64_t cap_polys, int64_t cap_slots, int64_t* n_polys,
                      int64_t* n_slots, int64_t* stats, cudaStream_t s) {
  int64_t Tn = T > 0 ? T : 1, nn = n > 0 ? n : 1;
  ENSURE(tri32, 3 * Tn * sizeof(int32_t));
  ENSURE(hw, 3 * Tn * sizeof(int32_t));
  ENSURE(max_edge, Tn);
  ENSURE(seed, Tn);
  ENSURE(tv, nn * sizeof(int32_t));
  ENSURE(off0, (Tn + 1) * sizeof(int64_t));
  ENSURE(v0, 3 * Tn * sizeof(int32_t));
  for (auto& e : ctx->ev)
    if (!e) CK(cudaEventCreate(&e));
  CK(cudaEventRecord(ctx->ev[0], s));
  int rc = tm_label(ctx, d_xy, n, d_tri, tri_bits, T, check, ctx->tri32.as<int32_t>(), ctx->hw.as<int32_t>(),
                    ctx->max_edge.as<int8_t>(), ctx->seed.as<uint8_t>(), ctx->tv.as<int32_t>(), s);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev[1], s));
  int64_t P = 0, F = 0;
  rc = tm_traverse(ctx, ctx->tri32.as<int32_t>(), ctx->hw.as<int32_t>(), ctx->seed.as<uint8_t>(), T,
                   ctx->off0.as<int64_t>(), ctx->v0.as<int32_t>(), Tn, 3 * Tn, &P, &F, s);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev[2], s));
  rc = tm_repair(ctx, ctx->tri32.as<int32_t>(), ctx->hw.as<int32_t>(), ctx->tv.as<int32_t>(), T,
                 ctx->off0.as<int64_t>(), ctx->v0.as<int32_t>(), P, d_off, d_v, cap_polys, cap_slots, n_polys, n_slots,
                 stats, s);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev[3], s));
  CK(cudaEventSynchronize(ctx->ev[3]));
  for (int k = 0; k < 3; k++) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ctx->ev[k], ctx->ev[k + 1]));
    ctx->phase_ms[k] = ms;
  }
  return TM_OK;
}

int tm_mesh_to_polygons(tm_ctx* ctx, const double* d_xy, int64_t n, const void* d_tri, int tri_bits, int64_t T,
                        int check, int64_t* d_off, int32_t* d_v, int64_t cap_polys, int64_t cap_slots,
                        int64_t* n_polys, int64_t* n_slots, int64_t* stats, void* stream) {
  if (!ctx || !n_polys || !n_slots) return TM_ERR_ARGUMENT;
  return run_device(ctx, d_xy, n, d_tri, tri_bits, T, check, d_off, d_v, cap_polys, cap_slots, n_polys, n_slots,
                    stats, (cudaStream_t)stream);
}

int tm_mesh_to_polygons_host(tm_ctx* ctx, const double* h_xy, int64_t n, const int64_t* h_tri, int64_t T, int check,
                             int64_t* h_off, int32_t* h_v, int64_t cap_polys, int64_t cap_slots, int64_t* n_polys,
                             int64_t* n_slots, int64_t* stats) {
  if (!ctx || !n_polys || !n_slots || (!h_xy && n) || (!h_tri && T)) return TM_ERR_ARGUMENT;
  if (!ctx->own_stream) CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  cudaStream_t s = ctx->own_stream;
  int64_t Tn = T > 0 ? T : 1, nn = n > 0 ? n : 1;
  ENSURE(xy, 2 * nn * sizeof(double));
  ENSURE(tri, 3 * Tn * sizeof(int64_t));
  CK(cudaMemcpyAsync(ctx->xy.p, h_xy, 2 * n * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->tri.p, h_tri, 3 * T * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  // final CSR goes to device buffers sized by the bounds, then to host
  ENSURE(fin_off, (Tn + 1) * sizeof(int64_t));
  ENSURE(fin_v, 3 * Tn * sizeof(int32_t));
  Buf& out_off = ctx->fin_off;
  Buf& out_v = ctx->fin_v;
  int rc = run_device(ctx, ctx->xy.as<double>(), n, ctx->tri.p, 64, T, check, out_off.as<int64_t>(),
                      out_v.as<int32_t>(), Tn, 3 * Tn, n_polys, n_slots, stats, s);
  if (rc == TM_OK) {
    if (*n_polys + 1 > cap_polys + 1 || *n_slots > cap_slots) {
      rc = set_err(ctx, TM_ERR_CAPACITY, "host output capacity too small");
    } else {
      cudaError_t e1 = cudaMemcpyAsync(h_off, out_off.p, (*n_polys + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
      cudaError_t e2 = cudaMemcpyAsync(h_v, out_v.p, *n_slots * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaError_t e3 = cudaStreamSynchronize(s);
      if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) rc = cuda_fail(ctx, e3 != cudaSuccess ? e3 : (e1 != cudaSuccess ? e1 : e2), "D2H");
    }
  }
  return rc;
}

}  // extern "C"
