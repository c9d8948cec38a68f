/*
 * oracle.c -- CPU restatement of the reference `termesh` mesh -> polygons path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA path
 * in paper_2204_05438_b200/csrc and the CPU baseline ("kind": "port") timed by
 * bench.py.  Nothing in the product path links, loads or calls it.
 *
 * It restates, function by function, the algorithm of the Python reference
 * (/root/reference/pkg/src/termesh, cited as file:line below) on the
 * reference's own data layout:
 *     vertices  f64[2n]   (x0,y0,x1,y1,...)
 *     triangles i64[3T]   CCW, edge j opposite corner j
 *     neighbors i64[3T]   triangle across edge j, -1 = BORDER
 *     trivertex i64[n]    lowest incident triangle, -1 if isolated
 * and it uses the reference's adjacency (`neighbors`) -- NOT the twin build of
 * the CUDA path -- so agreement also checks the GPU half-edge construction.
 *
 * Repair follows the reference's *round* structure (reparation.py:343-377):
 * every round scans the whole mesh, splits each tipped polygon once, and a
 * final pinch pass runs rounds of trial splits.  The CUDA path uses a
 * per-polygon depth-first schedule instead; agreement between the two is the
 * evidence that the schedules are equivalent.
 *
 * Parity of this restatement is pinned against golden vectors produced by the
 * Python reference itself (tests/golden/make_golden.py, tests/test_oracle.py).
 *
 * Floating point: edge lengths are dx*dx + dy*dy with no FMA contraction
 * (compile with -ffp-contract=off), matching numpy's ((b-c)**2).sum(axis=1).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BORDER (-1)

enum { OR_OK = 0, OR_STRUCTURAL = 1, OR_VALUE = 2, OR_CAPACITY = 3, OR_NOMEM = 4 };

static __thread char g_err[512];

static int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
#include <stdarg.h>
static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char *or_last_error(void) { return g_err; }

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

typedef struct {
    const double *xy;
    const int64_t *tr;
    const int64_t *nb;
    const int64_t *tv;
    int64_t n, T;
    uint8_t *fr; /* frontier flags, mutated by repair */
} Mesh;

/* ---------------------------------------------------------------- algebra */
/* mesh_core.py:104-129: h = 3t+j; origin = corner (j+1)%3, target = (j+2)%3 */
static inline int64_t nxt(int64_t h) { return 3 * (h / 3) + (h % 3 + 1) % 3; }
static inline int64_t prv(int64_t h) { return 3 * (h / 3) + (h % 3 + 2) % 3; }
static inline int64_t org(const Mesh *m, int64_t h) { return m->tr[3 * (h / 3) + (h % 3 + 1) % 3]; }
static inline int64_t tgt(const Mesh *m, int64_t h) { return m->tr[3 * (h / 3) + (h % 3 + 2) % 3]; }

/* mesh_core.py:132-149: twin by endpoint match; *err set on a broken neighbor */
static int64_t twin_of(const Mesh *m, int64_t h, int *err) {
    int64_t n = m->nb[h];
    if (n == BORDER) return BORDER;
    int64_t o = org(m, h), g = tgt(m, h), base = 3 * n;
    for (int k = 0; k < 3; k++)
        if (m->tr[base + (k + 1) % 3] == g && m->tr[base + (k + 2) % 3] == o) return base + k;
    *err = fail(OR_STRUCTURAL,
                "triangle %lld is recorded as neighbor of half-edge %lld but shares no edge "
                "with endpoints (%lld, %lld)",
                (long long)n, (long long)h, (long long)o, (long long)g);
    return BORDER;
}

/* mesh_core.py:171-178: lowest incident triangle per vertex, -1 if none */
void or_compute_trivertex(const int64_t *tr, int64_t T, int64_t n, int64_t *out) {
    for (int64_t v = 0; v < n; v++) out[v] = -1;
    for (int64_t s = 3 * T - 1; s >= 0; s--) out[tr[s]] = s / 3;
}

/* ---------------------------------------------------------------- labels */
/* labeling.py:46-62 with numpy argmax semantics (first NaN, else first max) */
static inline int8_t argmax3(double l0, double l1, double l2) {
    double best = l0;
    int8_t m = 0;
    if (isnan(best)) return 0;
    if (!(l1 <= best)) { best = l1; m = 1; if (isnan(best)) return m; }
    if (!(l2 <= best)) { m = 2; }
    return m;
}

static inline double sqlen(const double *xy, int64_t p, int64_t q) {
    double dx = xy[2 * p] - xy[2 * q];
    double dy = xy[2 * p + 1] - xy[2 * q + 1];
    double a = dx * dx;
    double b = dy * dy;
    return a + b;
}

/* labeling.py:65-89 / 92-115: the back slot k is the FIRST slot of n pointing at t
 * (np.argmax over a boolean row), 0 when none does. */
static inline int back_slot(const int64_t *nb, int64_t n, int64_t t) {
    for (int k = 0; k < 3; k++)
        if (nb[3 * n + k] == t) return k;
    return 0;
}

int or_label(const double *xy, const int64_t *tr, const int64_t *nb, int64_t T, int nthreads,
             int8_t *max_edge, uint8_t *frontier, uint8_t *seed) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    /* label_max: labeling.py:52-59 (edge 0 joins corners 1,2; 1 joins 2,0; 2 joins 0,1) */
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; t++) {
        int64_t a = tr[3 * t], b = tr[3 * t + 1], c = tr[3 * t + 2];
        max_edge[t] = argmax3(sqlen(xy, b, c), sqlen(xy, c, a), sqlen(xy, a, b));
    }
    /* label_seeds: labeling.py:78-86 */
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; t++) {
        int64_t e = max_edge[t];
        int64_t n = nb[3 * t + e];
        if (n == BORDER) { seed[t] = 1; continue; }
        int k = back_slot(nb, n, t);
        seed[t] = (max_edge[n] == k) && (t < n);
    }
    /* label_frontiers: labeling.py:103-112 */
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; t++) {
        for (int j = 0; j < 3; j++) {
            int64_t n = nb[3 * t + j];
            if (n == BORDER) { frontier[3 * t + j] = 1; continue; }
            int own = max_edge[t] == j;
            int k = back_slot(nb, n, t);
            int other = max_edge[n] == k;
            frontier[3 * t + j] = !own && !other;
        }
    }
    return OR_OK;
}

/* --------------------------------------------------------------- int vector */
typedef struct { int64_t *d; int64_t n, cap; } Vec;
static int vpush(Vec *v, int64_t x) {
    if (v->n == v->cap) {
        int64_t nc = v->cap ? 2 * v->cap : 64;
        int64_t *nd = (int64_t *)realloc(v->d, (size_t)nc * sizeof *nd);
        if (!nd) return fail(OR_NOMEM, "out of host memory");
        v->d = nd; v->cap = nc;
    }
    v->d[v->n++] = x;
    return OR_OK;
}
static void vfree(Vec *v) { free(v->d); v->d = NULL; v->n = v->cap = 0; }

/* ------------------------------------------------------------ traversal */
/* traversal.py:172-192: smallest frontier slot of seed_t, else FIFO BFS across
 * non-frontier-or-not adjacency (every non-border neighbor is enqueued) */
static int64_t find_start_frontier(const Mesh *m, int64_t seed_t, int *err) {
    Vec q = {0};
    int64_t head = 0, res = -1;
    if ((*err = vpush(&q, seed_t))) return -1;
    while (head < q.n) {
        int64_t t = q.d[head++];
        for (int j = 0; j < 3; j++) {
            int64_t h = 3 * t + j;
            if (m->fr[h]) { res = h; goto done; }
            int64_t n = m->nb[h];
            if (n == BORDER) continue;
            int seen = 0;
            for (int64_t i = 0; i < q.n; i++)
                if (q.d[i] == n) { seen = 1; break; }
            if (!seen && (*err = vpush(&q, n))) goto done;
        }
    }
    *err = fail(OR_STRUCTURAL, "no frontier edge reachable from triangle %lld", (long long)seed_t);
done:
    vfree(&q);
    return res;
}

/* traversal.py:242-261 (_advance): rotation via the neighbor back-slot search */
static int64_t advance(const Mesh *m, int64_t h, int64_t limit) {
    int64_t c = nxt(h), spins = 0;
    while (!m->fr[c]) {
        int64_t n = m->nb[c];
        if (n < 0) return -1;
        int64_t t = c / 3;
        int k = m->nb[3 * n] == t ? 0 : (m->nb[3 * n + 1] == t ? 1 : 2);
        c = 3 * n + (k + 1) % 3;
        if (++spins > limit) return -1;
    }
    return c;
}

/* traversal.py:303-347 under SEQUENTIAL: ascending seed order, runs of
 * [origin(h0), origin(h1), ...].  Output as CSR (offsets[P+1], verts). */
int or_traverse(const int64_t *tr, const int64_t *nb, int64_t T, const uint8_t *frontier,
                const uint8_t *seed, int nthreads, int64_t *offsets, int64_t *verts,
                int64_t cap_polys, int64_t cap_slots, int64_t *n_polys) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    Mesh m = {NULL, tr, nb, NULL, 0, T, (uint8_t *)frontier};
    int64_t P = 0;
    for (int64_t t = 0; t < T; t++) P += seed[t] != 0;
    if (P > cap_polys) return fail(OR_CAPACITY, "polygon capacity %lld < %lld", (long long)cap_polys, (long long)P);
    int64_t *seeds = (int64_t *)malloc((size_t)(P ? P : 1) * sizeof(int64_t));
    int64_t *starts = (int64_t *)malloc((size_t)(P ? P : 1) * sizeof(int64_t));
    if (!seeds || !starts) { free(seeds); free(starts); return fail(OR_NOMEM, "out of host memory"); }
    for (int64_t t = 0, i = 0; t < T; t++)
        if (seed[t]) seeds[i++] = t;
    int64_t limit = 3 * T + 3;
    int rc = OR_OK;
    int64_t bad_seed = -1;
    /* traversal.py:323-335: start edges and walk lengths */
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < P; i++) {
        int64_t t = seeds[i], h0 = -1;
        for (int j = 0; j < 3; j++)
            if (frontier[3 * t + j]) { h0 = 3 * t + j; break; }
        if (h0 < 0) {
            int err = 0;
            h0 = find_start_frontier(&m, t, &err);
            if (err) {
#pragma omp critical
                { if (rc == OR_OK) rc = err; }
                continue;
            }
        }
        starts[i] = h0;
        int64_t len = 0, h = h0;
        for (;;) {
            if (++len > limit) { len = -1; break; }
            h = advance(&m, h, limit);
            if (h < 0) { len = -1; break; }
            if (h == h0) break;
        }
        offsets[i + 1] = len;
        if (len < 0) {
#pragma omp critical
            { if (bad_seed < 0 || t < bad_seed) bad_seed = t; }
        }
    }
    if (rc == OR_OK && bad_seed >= 0)
        rc = fail(OR_STRUCTURAL, "boundary walk from seed triangle %lld did not terminate", (long long)bad_seed);
    if (rc == OR_OK) {
        offsets[0] = 0;
        for (int64_t i = 0; i < P; i++) offsets[i + 1] += offsets[i];
        if (offsets[P] > cap_slots)
            rc = fail(OR_STRUCTURAL, "polygon storage capacity exceeded; labels are inconsistent");
    }
    if (rc == OR_OK) {
        /* traversal.py:284-300 (_walk_write) */
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t i = 0; i < P; i++) {
            int64_t w = offsets[i], h0 = starts[i], h = h0;
            for (;;) {
                verts[w++] = tr[3 * (h / 3) + (h % 3 + 1) % 3];
                h = advance(&m, h, limit);
                if (h == h0) break;
            }
        }
        *n_polys = P;
    }
    free(seeds);
    free(starts);
    return rc;
}

/* ---------------------------------------------------------- polygon lists */
typedef struct {
    Vec v;   /* vertex store */
    Vec off; /* polygon i = v[off[i] .. off[i+1]) ; off has count+1 entries */
} Polys;

static int polys_init(Polys *p) {
    memset(p, 0, sizeof *p);
    return vpush(&p->off, 0);
}
static void polys_free(Polys *p) { vfree(&p->v); vfree(&p->off); }
static int polys_add(Polys *p, const int64_t *s, int64_t len) {
    int rc;
    for (int64_t i = 0; i < len; i++)
        if ((rc = vpush(&p->v, s[i]))) return rc;
    return vpush(&p->off, p->v.n);
}
static inline int64_t pcount(const Polys *p) { return p->off.n - 1; }
static inline const int64_t *pget(const Polys *p, int64_t i, int64_t *len) {
    *len = p->off.d[i + 1] - p->off.d[i];
    return p->v.d + p->off.d[i];
}

/* traversal.py:112-124: any cyclic triple (a, b, a) */
static int has_tip(const int64_t *s, int64_t n) {
    for (int64_t pos = 0; pos < n; pos++)
        if (s[(pos - 1 + n) % n] == s[(pos + 1) % n]) return 1;
    return 0;
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* traversal.py:127-147: repeated-vertex count (len - distinct) */
static int64_t extra_visits(const int64_t *s, int64_t n, int64_t *scratch) {
    memcpy(scratch, s, (size_t)n * sizeof *s);
    qsort(scratch, (size_t)n, sizeof *scratch, cmp_i64);
    int64_t distinct = n ? 1 : 0;
    for (int64_t i = 1; i < n; i++) distinct += scratch[i] != scratch[i - 1];
    return n - distinct;
}

static int64_t max_len(const Polys *p) {
    int64_t mx = 0, l;
    for (int64_t i = 0; i < pcount(p); i++) { pget(p, i, &l); if (l > mx) mx = l; }
    return mx;
}

static int64_t mesh_extra_visits(const Polys *p) {
    int64_t mx = max_len(p), tot = 0, l;
    int64_t *scr = (int64_t *)malloc((size_t)(mx ? mx : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < pcount(p); i++) { const int64_t *s = pget(p, i, &l); tot += extra_visits(s, l, scr); }
    free(scr);
    return tot;
}

/* -------------------------------------------------------- repair helpers */
/* traversal.py:195-217 (next_frontier) with the endpoint-match twin */
static int64_t next_frontier(const Mesh *m, int64_t h, int *err) {
    if (!m->fr[h]) { *err = fail(OR_VALUE, "half-edge %lld is not a frontier edge", (long long)h); return -1; }
    int64_t c = nxt(h), spins = 0, limit = 3 * m->T;
    while (!m->fr[c]) {
        int64_t w = twin_of(m, c, err);
        if (*err) return -1;
        if (w == BORDER) {
            *err = fail(OR_STRUCTURAL, "rotation around vertex %lld crossed an unlabeled border edge", (long long)tgt(m, h));
            return -1;
        }
        c = nxt(w);
        if (++spins > limit) {
            *err = fail(OR_STRUCTURAL, "vertex %lld has no frontier edge", (long long)tgt(m, h));
            return -1;
        }
    }
    return c;
}

/* traversal.py:220-236 (poly_construction) into *out (cleared first) */
static int poly_construction(const Mesh *m, int64_t seed_t, Vec *out) {
    int err = 0;
    out->n = 0;
    int64_t h0 = find_start_frontier(m, seed_t, &err);
    if (err) return err;
    if ((err = vpush(out, org(m, h0)))) return err;
    int64_t h = next_frontier(m, h0, &err);
    if (err) return err;
    int64_t guard = 2 * 3 * m->T + 3;
    while (h != h0) {
        if ((err = vpush(out, org(m, h)))) return err;
        if (out->n > guard)
            return fail(OR_STRUCTURAL, "boundary walk from triangle %lld failed to close", (long long)seed_t);
        h = next_frontier(m, h, &err);
        if (err) return err;
    }
    return OR_OK;
}

/* reparation.py:82-88 */
static int64_t rot_ccw(const Mesh *m, int64_t h, int *err) { return twin_of(m, prv(h), err); }
static int64_t rot_cw(const Mesh *m, int64_t h, int *err) {
    int64_t w = twin_of(m, h, err);
    return w == BORDER ? BORDER : nxt(w);
}

/* reparation.py:91-115 (_fan_around) */
static int fan_around(const Mesh *m, int64_t v, int64_t g0, Vec *fan) {
    int err = 0;
    int64_t cap = 3 * m->T;
    fan->n = 0;
    if ((err = vpush(fan, g0))) return err;
    int64_t g = rot_ccw(m, g0, &err);
    if (err) return err;
    while (g != BORDER && g != g0) {
        if ((err = vpush(fan, g))) return err;
        if (fan->n > cap) return fail(OR_STRUCTURAL, "rotation around vertex %lld does not close", (long long)v);
        g = rot_ccw(m, g, &err);
        if (err) return err;
    }
    if (g == g0) return OR_OK;
    Vec back = {0};
    g = rot_cw(m, g0, &err);
    while (!err && g != BORDER) {
        if ((err = vpush(&back, g))) break;
        if (back.n > cap) { err = fail(OR_STRUCTURAL, "rotation around vertex %lld does not close", (long long)v); break; }
        g = rot_cw(m, g, &err);
    }
    for (int64_t i = back.n - 1; !err && i >= 0; i--) err = vpush(fan, back.d[i]);
    vfree(&back);
    return err;
}

/* reparation.py:74-79 and 118-124 (_halfedge_with_origin, _fan_at_vertex) */
static int fan_at_vertex(const Mesh *m, int64_t v, Vec *fan) {
    int64_t t0 = m->tv[v];
    if (t0 < 0) return fail(OR_STRUCTURAL, "vertex %lld has no incident triangle", (long long)v);
    for (int j = 0; j < 3; j++)
        if (org(m, 3 * t0 + j) == v) return fan_around(m, v, 3 * t0 + j, fan);
    return fail(OR_STRUCTURAL, "triangle %lld does not contain vertex %lld", (long long)t0, (long long)v);
}

/* reparation.py:59-71 (find_barrier_tip): first pos with s[pos-1] == s[pos+1] */
static int64_t find_barrier_tip(const int64_t *s, int64_t n) {
    for (int64_t pos = 0; pos < n; pos++)
        if (s[(pos - 1 + n) % n] == s[(pos + 1) % n]) return pos;
    return -1;
}

/* reparation.py:127-145 (middle_internal_edge) */
static int middle_internal_edge(const Mesh *m, int64_t v, int64_t barrier, int64_t *e_out) {
    Vec fan = {0};
    int rc = fan_at_vertex(m, v, &fan);
    if (rc) { vfree(&fan); return rc; }
    int64_t at = -1, k = 0;
    for (int64_t i = 0; i < fan.n; i++)
        if (tgt(m, fan.d[i]) == barrier && m->fr[fan.d[i]]) { at = i; break; }
    if (at < 0) {
        vfree(&fan);
        return fail(OR_STRUCTURAL, "barrier edge (%lld, %lld) not found around tip vertex %lld",
                    (long long)v, (long long)barrier, (long long)v);
    }
    for (int64_t i = 0; i < fan.n; i++) k += !m->fr[fan.d[i]];
    if (k == 0) { vfree(&fan); return fail(OR_STRUCTURAL, "tip vertex %lld has no internal edge to split on", (long long)v); }
    int64_t want = (k - 1) / 2, seen = 0;
    for (int64_t s = 0; s < fan.n; s++) {
        int64_t g = fan.d[(at + s) % fan.n];
        if (m->fr[g]) continue;
        if (seen++ == want) { *e_out = g; break; }
    }
    vfree(&fan);
    return OR_OK;
}

/* reparation.py:208-229 (_split_polygon).  Returns OR_OK with *ok=1 on a split,
 * *ok=0 after reverting a non-strict split that broke the length law. */
static int split_polygon(const Mesh *m, int64_t e, int64_t plen, int strict, int64_t pid,
                         Vec *pa, Vec *pb, int *ok) {
    int err = 0;
    int64_t w = twin_of(m, e, &err);
    if (err) return err;
    if (w == BORDER) return fail(OR_STRUCTURAL, "polygon %lld: promoted edge lies on the border", (long long)pid);
    m->fr[e] = 1;
    m->fr[w] = 1;
    if ((err = poly_construction(m, e / 3, pa))) return err;
    if ((err = poly_construction(m, w / 3, pb))) return err;
    if (pa->n + pb->n != plen + 2) {
        if (strict)
            return fail(OR_STRUCTURAL, "polygon %lld: split produced lengths %lld + %lld, expected %lld + 2",
                        (long long)pid, (long long)pa->n, (long long)pb->n, (long long)plen);
        m->fr[e] = 0;
        m->fr[w] = 0;
        *ok = 0;
        return OR_OK;
    }
    *ok = 1;
    return OR_OK;
}

/* reparation.py:148-166 (_wedge_internal_edges) */
static int wedge_internal_edges(const Mesh *m, const Vec *fan, int64_t v, int64_t out_vertex, Vec *out) {
    int64_t at = -1;
    out->n = 0;
    for (int64_t i = 0; i < fan->n; i++)
        if (tgt(m, fan->d[i]) == out_vertex && m->fr[fan->d[i]]) { at = i; break; }
    if (at < 0)
        return fail(OR_STRUCTURAL, "boundary edge (%lld, %lld) not found around vertex %lld",
                    (long long)v, (long long)out_vertex, (long long)v);
    for (int64_t step = 1; step < fan->n; step++) {
        int64_t g = fan->d[(at + step) % fan->n];
        if (m->fr[g]) break;
        int rc = vpush(out, g);
        if (rc) return rc;
    }
    return OR_OK;
}

/* reparation.py:169-205 (_pinch_candidates) driven by _pinch_pass's splitter
 * (reparation.py:326-332): first candidate whose trial split obeys the law wins. */
static int pinch_split(const Mesh *m, const int64_t *poly, int64_t n, int64_t pid, Vec *pa, Vec *pb, int *ok) {
    *ok = 0;
    int64_t v = -1, p1 = 0, p2 = 0;
    for (int64_t idx = 0; idx < n && v < 0; idx++)
        for (int64_t j = 0; j < idx; j++)
            if (poly[j] == poly[idx]) { v = poly[idx]; p1 = j; p2 = idx; break; }
    if (v < 0) return OR_OK;
    Vec fan = {0}, wedge = {0}, fx = {0};
    int rc = fan_at_vertex(m, v, &fan);
    int64_t poss[2] = {p2, p1};
    for (int q = 0; q < 2 && !rc && !*ok; q++) {
        int64_t pos = poss[q];
        rc = wedge_internal_edges(m, &fan, v, poly[(pos + 1) % n], &wedge);
        if (rc || wedge.n == 0) continue;
        int64_t mid = (wedge.n - 1) / 2;
        rc = split_polygon(m, wedge.d[mid], n, 0, pid, pa, pb, ok);
        for (int64_t i = 0; i < wedge.n && !rc && !*ok; i++) {
            if (i == mid) continue;
            rc = split_polygon(m, wedge.d[i], n, 0, pid, pa, pb, ok);
        }
    }
    for (int64_t idx = p1 + 1; idx < p2 && !rc && !*ok; idx++) {
        rc = fan_at_vertex(m, poly[idx], &fx);
        for (int64_t i = 0; i < fx.n && !rc && !*ok; i++) {
            if (m->fr[fx.d[i]]) continue;
            rc = split_polygon(m, fx.d[i], n, 0, pid, pa, pb, ok);
        }
    }
    vfree(&fan); vfree(&wedge); vfree(&fx);
    return rc;
}

static int has_repeat(const int64_t *s, int64_t n, int64_t *scratch) { return extra_visits(s, n, scratch) > 0; }

/* reparation.py:343-377 (repair_all) with the round structure of
 * repair_round (294-312), _execute_round (232-277) and _pinch_pass (315-340).
 * stats = {rounds, splits, initial_tips, unrepaired}. */
/* guard_extra >= 0 replaces the pinch guard's extra-visit count (a seed
 * partition runs under the GLOBAL guard: the extra visits summed over all
 * ranks' tip-phase outputs); stats[4] = this call's tip-phase extra visits. */
int or_repair(const int64_t *tr, const int64_t *nb, const int64_t *tv, int64_t T, int64_t nverts,
              uint8_t *frontier, const int64_t *off_in, const int64_t *v_in, int64_t P,
              int64_t *off_out, int64_t *v_out, int64_t cap_polys, int64_t cap_slots,
              int64_t *n_out, int64_t *stats, int64_t guard_extra) {
    Mesh m = {NULL, tr, nb, tv, nverts, T, frontier};
    Polys cur, nxtp;
    int rc = polys_init(&cur);
    for (int64_t i = 0; i < P && !rc; i++) rc = polys_add(&cur, v_in + off_in[i], off_in[i + 1] - off_in[i]);
    if (rc) { polys_free(&cur); return rc; }
    Vec pa = {0}, pb = {0};
    int64_t *scr = NULL, l;
    int64_t initial = mesh_extra_visits(&cur);
    int64_t max_rounds = initial + 1, rounds = 0, splits = 0;
    for (;;) {
        rounds++;
        if (rounds > max_rounds) {
            rc = fail(OR_STRUCTURAL, "tip removal did not converge after %lld rounds (initial repeated-vertex count %lld)",
                      (long long)(rounds - 1), (long long)initial);
            break;
        }
        if ((rc = polys_init(&nxtp))) break;
        for (int64_t i = 0; i < pcount(&cur) && !rc; i++) {
            const int64_t *s = pget(&cur, i, &l);
            if (!has_tip(s, l)) { rc = polys_add(&nxtp, s, l); continue; }
            int64_t pos = find_barrier_tip(s, l);
            int64_t e = -1;
            if ((rc = middle_internal_edge(&m, s[pos], s[(pos - 1 + l) % l], &e))) break;
            int ok = 0;
            if ((rc = split_polygon(&m, e, l, 1, i, &pa, &pb, &ok))) break;
            if ((rc = polys_add(&nxtp, pa.d, pa.n))) break;
            rc = polys_add(&nxtp, pb.d, pb.n);
            splits++;
        }
        polys_free(&cur);
        cur = nxtp;
        if (rc) break;
        int64_t tips = 0;
        for (int64_t i = 0; i < pcount(&cur); i++) { const int64_t *s = pget(&cur, i, &l); tips += has_tip(s, l); }
        if (tips == 0) break;
    }
    int64_t before = pcount(&cur), tip_extra = 0;
    if (!rc) {
        /* _pinch_pass: reparation.py:315-340 */
        tip_extra = mesh_extra_visits(&cur);
        int64_t guard = (guard_extra >= 0 ? guard_extra : tip_extra) + 1;
        scr = (int64_t *)malloc((size_t)(max_len(&cur) + 2 * guard + 8) * sizeof(int64_t) * 2);
        for (int64_t r = 0; r < guard && !rc; r++) {
            int64_t any = 0, rs = 0;
            free(scr);
            scr = (int64_t *)malloc((size_t)(max_len(&cur) + 8) * sizeof(int64_t));
            for (int64_t i = 0; i < pcount(&cur); i++) {
                const int64_t *s = pget(&cur, i, &l);
                if (has_repeat(s, l, scr) && !has_tip(s, l)) { any = 1; break; }
            }
            if (!any) break;
            if ((rc = polys_init(&nxtp))) break;
            for (int64_t i = 0; i < pcount(&cur) && !rc; i++) {
                const int64_t *s = pget(&cur, i, &l);
                if (!(has_repeat(s, l, scr) && !has_tip(s, l))) { rc = polys_add(&nxtp, s, l); continue; }
                int ok = 0;
                if ((rc = pinch_split(&m, s, l, i, &pa, &pb, &ok))) break;
                if (!ok) { rc = polys_add(&nxtp, s, l); continue; }
                if ((rc = polys_add(&nxtp, pa.d, pa.n))) break;
                rc = polys_add(&nxtp, pb.d, pb.n);
                rs++;
            }
            polys_free(&cur);
            cur = nxtp;
            if (rs == 0) break;
        }
    }
    if (!rc) {
        int64_t cnt = pcount(&cur), unrepaired = 0;
        if (cnt > cap_polys || cur.v.n > cap_slots) {
            rc = fail(OR_CAPACITY, "repair output capacity exceeded");
        } else {
            free(scr);
            scr = (int64_t *)malloc((size_t)(max_len(&cur) + 8) * sizeof(int64_t));
            for (int64_t i = 0; i <= cnt; i++) off_out[i] = cur.off.d[i];
            memcpy(v_out, cur.v.d, (size_t)cur.v.n * sizeof(int64_t));
            for (int64_t i = 0; i < cnt; i++) { const int64_t *s = pget(&cur, i, &l); unrepaired += has_repeat(s, l, scr); }
            *n_out = cnt;
            stats[0] = rounds;
            stats[1] = splits + (cnt - before);
            stats[2] = initial;
            stats[3] = unrepaired;
            stats[4] = tip_extra;
        }
    }
    free(scr);
    vfree(&pa);
    vfree(&pb);
    polys_free(&cur);
    return rc;
}

/* ------------------------------------------------------------ canonical */
/* oracle.py:124-141: min lexicographic rotation, then tuple-order sort */
typedef struct { const int64_t *s; int64_t n; } PRef;

static int cmp_poly(const void *a, const void *b) {
    const PRef *x = (const PRef *)a, *y = (const PRef *)b;
    int64_t k = x->n < y->n ? x->n : y->n;
    for (int64_t i = 0; i < k; i++)
        if (x->s[i] != y->s[i]) return x->s[i] < y->s[i] ? -1 : 1;
    return (x->n > y->n) - (x->n < y->n);
}

int or_canonicalize(const int64_t *off, const int64_t *v, int64_t P, int64_t *off_out, int64_t *v_out) {
    int64_t total = off[P];
    int64_t *rot = (int64_t *)malloc((size_t)(total ? total : 1) * sizeof(int64_t));
    PRef *refs = (PRef *)malloc((size_t)(P ? P : 1) * sizeof(PRef));
    if (!rot || !refs) { free(rot); free(refs); return fail(OR_NOMEM, "out of host memory"); }
    for (int64_t i = 0; i < P; i++) {
        const int64_t *s = v + off[i];
        int64_t n = off[i + 1] - off[i], best = -1, mn = INT64_MAX;
        for (int64_t k = 0; k < n; k++) if (s[k] < mn) mn = s[k];
        for (int64_t k = 0; k < n; k++) {
            if (s[k] != mn) continue;
            if (best < 0) { best = k; continue; }
            for (int64_t q = 0; q < n; q++) {
                int64_t a = s[(k + q) % n], b = s[(best + q) % n];
                if (a != b) { if (a < b) best = k; break; }
            }
        }
        for (int64_t q = 0; q < n; q++) rot[off[i] + q] = s[(best + q) % n];
        refs[i].s = rot + off[i];
        refs[i].n = n;
    }
    qsort(refs, (size_t)P, sizeof *refs, cmp_poly);
    int64_t w = 0;
    off_out[0] = 0;
    for (int64_t i = 0; i < P; i++) {
        memcpy(v_out + w, refs[i].s, (size_t)refs[i].n * sizeof(int64_t));
        w += refs[i].n;
        off_out[i + 1] = w;
    }
    free(rot);
    free(refs);
    return OR_OK;
}
