/*
 * p2m_oracle.c -- CPU ORACLE for the batched point-to-mesh query (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity checker, never the product.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product query path
 * (paper_2605_00429_b200/csrc/cuda) never links or calls anything here.
 *
 * What it restates (REF = /root/reference):
 *   - closest point on a triangle, squared distance: REF/proj/src/geom.cpp:31-70
 *     (Ericson Voronoi-region test; same operation order, no FMA -> bitwise equal d^2 / point)
 *   - minimal bounding sphere of a triangle:          REF/proj/src/geom.cpp:96-120
 *   - nearest_site (exact, ties -> lowest site id):    REF/SPEC.md:463-466, 482-487
 *   - DelaunayWalk nearest_site (greedy + tie flood):  REF/SPEC.md:476, 516
 *   - query_distance (pruned scan, d_min=+inf, strict): REF/SPEC.md:488-496, 513-515
 *   - batch_query (per-thread counters merged):        REF/SPEC.md:497-505, 518-519
 *   - brute_force_closest (lowest face id on ties):    REF/SPEC.md:536-544
 *
 * Parity pin: tests/test_oracle_pin.py checks every function here bit-for-bit against the
 * reference's own geom.cpp compiled from /root/reference into oracle/_ref (see Makefile),
 * against the SPEC known-answer tests, and against committed golden vectors in tests/golden/.
 *
 * When compiled with -DP2M_ORACLE_USE_REF the point-triangle kernel is the reference's own
 * p2mx::closest_on_triangle_sq (through oracle/ref_shim.cpp); that build is the "reference
 * CPU query path" timed by bench.py --impl reference.
 *
 * Build flags are pinned: -O2 -ffp-contract=off, no -march=native, so no
 * fused multiply-adds change the rounding relative to the reference's default build.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_EXPORT __attribute__((visibility("default")))

enum { SITE_MESH_VERTEX = 0, SITE_SENTINEL = 1, SITE_AUXILIARY = 2 };
enum { FLAG_FALLBACK = 1u, FLAG_OUT_OF_DOMAIN = 2u };
enum { PRUNE_OFF = 0, PRUNE_SAFE = 1, PRUNE_SPEC = 2 };

/* ------------------------------------------------------------------------------------------
 * Point-triangle closest point (restates REF/proj/src/geom.cpp:31-70).
 * Vector algebra follows REF/proj/include/p2mx/geom.hpp:17-41: a-b per component, dot as
 * (x*x + y*y) + z*z left to right, a + b*s per component.
 */
#ifdef P2M_ORACLE_USE_REF
void p2mref_closest_on_triangle_sq(const double *q, const double *a, const double *b,
                                   const double *c, double *d2, double *p);
#define CLOSEST p2mref_closest_on_triangle_sq
#else
#define CLOSEST orc_closest_on_triangle_sq
#endif

static inline double dot3(const double *u, const double *v) {
    return u[0] * v[0] + u[1] * v[1] + u[2] * v[2];
}
static inline void sub3(const double *u, const double *v, double *o) {
    o[0] = u[0] - v[0]; o[1] = u[1] - v[1]; o[2] = u[2] - v[2];
}
static inline double dist2_3(const double *u, const double *v) {
    double d[3]; sub3(u, v, d); return dot3(d, d);
}

ORC_EXPORT void orc_closest_on_triangle_sq(const double *q, const double *a, const double *b,
                                           const double *c, double *d2, double *p) {
    double ab[3], ac[3], aq[3];
    sub3(b, a, ab); sub3(c, a, ac); sub3(q, a, aq);
    const double d1 = dot3(ab, aq), d2v = dot3(ac, aq);
    if (d1 <= 0.0 && d2v <= 0.0) {                       /* vertex region A  (geom.cpp:34) */
        p[0] = a[0]; p[1] = a[1]; p[2] = a[2]; *d2 = dist2_3(q, a); return;
    }
    double bq[3]; sub3(q, b, bq);
    const double d3 = dot3(ab, bq), d4 = dot3(ac, bq);
    if (d3 >= 0.0 && d4 <= d3) {                         /* vertex region B  (geom.cpp:38) */
        p[0] = b[0]; p[1] = b[1]; p[2] = b[2]; *d2 = dist2_3(q, b); return;
    }
    const double vc = d1 * d4 - d3 * d2v;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {          /* edge AB          (geom.cpp:41-45) */
        const double v = d1 / (d1 - d3);
        p[0] = a[0] + ab[0] * v; p[1] = a[1] + ab[1] * v; p[2] = a[2] + ab[2] * v;
        *d2 = dist2_3(q, p); return;
    }
    double cq[3]; sub3(q, c, cq);
    const double d5 = dot3(ab, cq), d6 = dot3(ac, cq);
    if (d6 >= 0.0 && d5 <= d6) {                         /* vertex region C  (geom.cpp:49) */
        p[0] = c[0]; p[1] = c[1]; p[2] = c[2]; *d2 = dist2_3(q, c); return;
    }
    const double vb = d5 * d2v - d1 * d6;
    if (vb <= 0.0 && d2v >= 0.0 && d6 <= 0.0) {         /* edge AC          (geom.cpp:52-56) */
        const double w = d2v / (d2v - d6);
        p[0] = a[0] + ac[0] * w; p[1] = a[1] + ac[1] * w; p[2] = a[2] + ac[2] * w;
        *d2 = dist2_3(q, p); return;
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) { /* edge BC     (geom.cpp:59-63) */
        const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        double bc[3]; sub3(c, b, bc);
        p[0] = b[0] + bc[0] * w; p[1] = b[1] + bc[1] * w; p[2] = b[2] + bc[2] * w;
        *d2 = dist2_3(q, p); return;
    }
    /* face interior (geom.cpp:66-69): p = (a + ab*v) + ac*w */
    const double denom = 1.0 / (va + vb + vc);
    const double v = vb * denom, w = vc * denom;
    p[0] = (a[0] + ab[0] * v) + ac[0] * w;
    p[1] = (a[1] + ab[1] * v) + ac[1] * w;
    p[2] = (a[2] + ab[2] * v) + ac[2] * w;
    *d2 = dist2_3(q, p);
}

/* Minimal enclosing sphere (restates REF/proj/src/geom.cpp:96-120; degeneracy check omitted,
 * callers validate).  out = {cx, cy, cz, r}. */
ORC_EXPORT void orc_triangle_bounding_sphere(const double *t, double *out) {
    const double *A = t, *B = t + 3, *C = t + 6;
    const double *P = A, *Q = B, *R = C;
    const double ab = dist2_3(A, B), ac = dist2_3(A, C), bc = dist2_3(B, C);
    if (ac >= ab && ac >= bc) { Q = C; R = B; }
    else if (bc >= ab && bc >= ac) { P = B; Q = C; R = A; }
    double mid[3] = {(P[0] + Q[0]) * 0.5, (P[1] + Q[1]) * 0.5, (P[2] + Q[2]) * 0.5};
    const double rad2 = dist2_3(P, Q) * 0.25;
    if (dist2_3(R, mid) <= rad2) {
        out[0] = mid[0]; out[1] = mid[1]; out[2] = mid[2]; out[3] = sqrt(rad2); return;
    }
    double u[3], v[3]; sub3(B, A, u); sub3(C, A, v);
    const double uu = dot3(u, u), vv = dot3(v, v), uv = dot3(u, v);
    const double den = 2.0 * (uu * vv - uv * uv);
    const double s = (vv * (uu - uv)) / den;
    const double w = (uu * (vv - uv)) / den;
    double cen[3];
    for (int k = 0; k < 3; ++k) cen[k] = (A[k] + u[k] * s) + v[k] * w;
    double m = dist2_3(cen, A);
    double mb = dist2_3(cen, B), mc = dist2_3(cen, C);
    if (mb > m) m = mb;
    if (mc > m) m = mc;
    out[0] = cen[0]; out[1] = cen[1]; out[2] = cen[2]; out[3] = sqrt(m);
}

/* ------------------------------------------------------------------------------------------
 * Exact nearest site (REF/SPEC.md:473-487): left-balanced k-d tree over all sites, split on the
 * widest axis of each subset, implicit children 2k+1 / 2k+2.  The result is the lexicographic
 * minimum of (d^2, site id) -- independent of the tree -- because a subtree is skipped only
 * when the squared plane distance is STRICTLY larger than the best d^2 (equal-distance lower
 * ids are still visited).  The same tree definition is used by the device packer so the
 * "nodes visited" counter is comparable, but it is re-derived here from the raw site arrays.
 */
typedef struct {
    uint64_t n;
    uint32_t *node_site; /* site id per BFS node */
    uint8_t *node_dim;
    const double *xyz;   /* caller-owned site positions, 3 per site */
} orc_kdtree;

static uint64_t lb_left_size(uint64_t n) {
    if (n <= 1) return 0;
    int d = 63 - __builtin_clzll(n);           /* depth of the last level */
    uint64_t full = (1ull << d) - 1ull;        /* nodes on complete levels */
    uint64_t last = n - full;
    uint64_t half = 1ull << (d - 1);
    return (half - 1ull) + (last < half ? last : half);
}

static inline int key_less(const double *xyz, int dim, uint32_t a, uint32_t b) {
    double ka = xyz[3 * (uint64_t)a + dim], kb = xyz[3 * (uint64_t)b + dim];
    return ka < kb || (ka == kb && a < b);
}

/* deterministic quickselect: after it, idx[k] is the k-th smallest under (coord, id) and the
 * elements before / after it are the smaller / larger sets. */
static void select_kth(uint32_t *idx, uint64_t n, uint64_t k, const double *xyz, int dim) {
    uint64_t lo = 0, hi = n - 1;
    while (hi > lo) {
        uint64_t mid = lo + (hi - lo) / 2;
        /* median of three pivot */
        uint32_t a = idx[lo], b = idx[mid], c = idx[hi], piv;
        if (key_less(xyz, dim, a, b)) {
            if (key_less(xyz, dim, b, c)) piv = b; else if (key_less(xyz, dim, a, c)) piv = c; else piv = a;
        } else {
            if (key_less(xyz, dim, a, c)) piv = a; else if (key_less(xyz, dim, b, c)) piv = c; else piv = b;
        }
        uint64_t i = lo, j = hi;
        for (;;) {
            while (key_less(xyz, dim, idx[i], piv)) ++i;
            while (key_less(xyz, dim, piv, idx[j])) --j;
            if (i >= j) break;
            uint32_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
            ++i; --j;
        }
        /* now [lo, j] <= piv <= [j+1, hi] */
        if (k <= j) hi = j; else lo = j + 1;
    }
}

typedef struct { uint64_t lo, hi, node; } kd_task;

ORC_EXPORT orc_kdtree *orc_kdtree_build(const double *xyz, uint64_t n) {
    orc_kdtree *t = (orc_kdtree *)calloc(1, sizeof(orc_kdtree));
    if (!t) return NULL;
    t->n = n; t->xyz = xyz;
    t->node_site = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
    t->node_dim = (uint8_t *)malloc(n ? n : 1);
    uint32_t *idx = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
    kd_task *st = (kd_task *)malloc(sizeof(kd_task) * 128);
    if (!t->node_site || !t->node_dim || !idx || !st) { free(idx); free(st); return NULL; }
    for (uint64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
    int sp = 0;
    if (n) st[sp++] = (kd_task){0, n, 0};
    while (sp) {
        kd_task tk = st[--sp];
        uint64_t m = tk.hi - tk.lo;
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (uint64_t i = tk.lo; i < tk.hi; ++i)
            for (int k = 0; k < 3; ++k) {
                double v = xyz[3 * (uint64_t)idx[i] + k];
                if (v < lo[k]) lo[k] = v;
                if (v > hi[k]) hi[k] = v;
            }
        int dim = 0;
        double ext = hi[0] - lo[0];
        if (hi[1] - lo[1] > ext) { dim = 1; ext = hi[1] - lo[1]; }
        if (hi[2] - lo[2] > ext) { dim = 2; }
        uint64_t l = lb_left_size(m);
        select_kth(idx + tk.lo, m, l, xyz, dim);
        t->node_site[tk.node] = idx[tk.lo + l];
        t->node_dim[tk.node] = (uint8_t)dim;
        if (tk.hi > tk.lo + l + 1) st[sp++] = (kd_task){tk.lo + l + 1, tk.hi, 2 * tk.node + 2};
        if (l > 0) st[sp++] = (kd_task){tk.lo, tk.lo + l, 2 * tk.node + 1};
    }
    free(idx); free(st);
    return t;
}

ORC_EXPORT void orc_kdtree_free(orc_kdtree *t) {
    if (!t) return;
    free(t->node_site); free(t->node_dim); free(t);
}

/* export the BFS layout so tests can compare it with the device packer's tree */
ORC_EXPORT void orc_kdtree_layout(const orc_kdtree *t, uint32_t *node_site, uint8_t *node_dim) {
    memcpy(node_site, t->node_site, sizeof(uint32_t) * t->n);
    memcpy(node_dim, t->node_dim, t->n);
}

typedef struct { double d2; uint32_t id; uint64_t visited; } nn_state;

static void nn_rec(const orc_kdtree *t, uint64_t k, const double *q, nn_state *s) {
    if (k >= t->n) return;
    const uint32_t id = t->node_site[k];
    const double *p = t->xyz + 3 * (uint64_t)id;
    const double d2 = dist2_3(q, p);
    s->visited++;
    if (d2 < s->d2 || (d2 == s->d2 && id < s->id)) { s->d2 = d2; s->id = id; }
    const int dim = t->node_dim[k];
    const double diff = q[dim] - p[dim];
    const uint64_t close_c = diff > 0.0 ? 2 * k + 2 : 2 * k + 1;
    const uint64_t far_c = diff > 0.0 ? 2 * k + 1 : 2 * k + 2;
    nn_rec(t, close_c, q, s);
    if (diff * diff <= s->d2) nn_rec(t, far_c, q, s);
}

ORC_EXPORT uint32_t orc_nearest_site(const orc_kdtree *t, const double *q, double *d2_out,
                                     uint64_t *visited) {
    nn_state s = {INFINITY, UINT32_MAX, 0};
    nn_rec(t, 0, q, &s);
    if (d2_out) *d2_out = s.d2;
    if (visited) *visited = s.visited;
    return s.id;
}

/* linear-scan nearest site with the same tie rule ("linear-scan oracle") */
ORC_EXPORT uint32_t orc_nearest_site_brute(const double *xyz, uint64_t n, const double *q,
                                           double *d2_out) {
    double best = INFINITY; uint32_t id = UINT32_MAX;
    for (uint64_t i = 0; i < n; ++i) {
        double d2 = dist2_3(q, xyz + 3 * i);
        if (d2 < best) { best = d2; id = (uint32_t)i; }
    }
    if (d2_out) *d2_out = best;
    return id;
}

/* ------------------------------------------------------------------------------------------
 * DelaunayWalk nearest_site (REF/SPEC.md:476, 516): greedy descent on the Delaunay adjacency --
 * move to the neighbour with the smallest (d^2, id) while it beats the current site; on a
 * Delaunay graph the local minimum is the global nearest distance.  Equidistant sites need not be
 * adjacent to each other along an improving path (four cospherical sites around a Voronoi edge
 * form a cycle), so the walk then floods the tie set -- every site reachable through sites at
 * exactly the minimum d^2 -- and returns its lowest id (ties -> lowest site id, REF/SPEC.md:465).
 * steps (optional) counts the moves.  Restated for the strategy-neutrality check of
 * REF/SPEC.md:510; the device walk (p2m_traverse.cuh) follows the same definition.
 */
ORC_EXPORT uint32_t orc_walk_nearest(const double *xyz, const uint64_t *adj_off, const uint32_t *adj,
                                     uint64_t n_sites, const double *q, uint32_t start, double *d2_out,
                                     uint64_t *steps) {
    uint32_t v = start < n_sites ? start : 0;
    double dv = dist2_3(q, xyz + 3 * (uint64_t)v);
    uint64_t st = 0;
    for (;;) {
        uint32_t b = v;
        double bd = dv;
        for (uint64_t k = adj_off[v]; k < adj_off[v + 1]; ++k) {
            const uint32_t w = adj[k];
            const double d = dist2_3(q, xyz + 3 * (uint64_t)w);
            if (d < bd || (d == bd && w < b)) { b = w; bd = d; }
        }
        if (b == v) break;
        v = b; dv = bd; ++st;
    }
    /* tie flood */
    uint64_t cap = 64, n = 0, head = 0;
    uint32_t *set = (uint32_t *)malloc(cap * sizeof(uint32_t));
    uint32_t best = v;
    if (set) {
        set[n++] = v;
        while (head < n) {
            const uint32_t u = set[head++];
            for (uint64_t k = adj_off[u]; k < adj_off[u + 1]; ++k) {
                const uint32_t w = adj[k];
                if (dist2_3(q, xyz + 3 * (uint64_t)w) != dv) continue;
                int seen = 0;
                for (uint64_t i = 0; i < n; ++i) if (set[i] == w) { seen = 1; break; }
                if (seen) continue;
                if (n == cap) {
                    uint32_t *ns = (uint32_t *)realloc(set, 2 * cap * sizeof(uint32_t));
                    if (!ns) break;
                    set = ns; cap *= 2;
                }
                set[n++] = w;
                if (w < best) best = w;
            }
        }
        free(set);
    }
    if (d2_out) *d2_out = dv;
    if (steps) *steps += st;
    return best;
}

/* Batch walk with the SPEC's warm start: each thread's first query starts at site 0 and every
 * later query at the previous query's answer (REF/SPEC.md:516, per-thread state REF/SPEC.md:520). */
ORC_EXPORT void orc_batch_walk(const double *xyz, const uint64_t *adj_off, const uint32_t *adj,
                               uint64_t n_sites, const double *q, uint64_t n, int threads,
                               uint32_t *site, uint64_t *total_steps) {
    uint64_t ts = 0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads) reduction(+ : ts)
#endif
    {
        uint32_t prev = 0;
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t i = 0; i < (int64_t)n; ++i) {
            prev = orc_walk_nearest(xyz, adj_off, adj, n_sites, q + 3 * i, prev, NULL, &ts);
            site[i] = prev;
        }
    }
    (void)threads;
    if (total_steps) *total_steps = ts;
}

/* ------------------------------------------------------------------------------------------
 * brute_force_closest (REF/SPEC.md:536-544): linear scan, ties -> lowest face id.
 */
ORC_EXPORT uint32_t orc_brute_force_closest(const double *tri, uint64_t nf, const double *q,
                                            double *d2_out, double *p_out) {
    double best = INFINITY, bp[3] = {0, 0, 0}; uint32_t bf = UINT32_MAX;
    for (uint64_t f = 0; f < nf; ++f) {
        const double *t = tri + 9 * f;
        double d2, p[3];
        CLOSEST(q, t, t + 3, t + 6, &d2, p);
        if (d2 < best) { best = d2; bf = (uint32_t)f; bp[0] = p[0]; bp[1] = p[1]; bp[2] = p[2]; }
    }
    if (d2_out) *d2_out = best;
    if (p_out) { p_out[0] = bp[0]; p_out[1] = bp[1]; p_out[2] = bp[2]; }
    return bf;
}

/* brute_force_closest over a batch of queries (OpenMP over queries): the table-independent arbiter
 * of the acceptance check (REF/SPEC.md:508, 536-544, 665-667) on sampled queries. */
ORC_EXPORT void orc_batch_brute_force(const double *tri, uint64_t nf, const double *q, uint64_t n, int threads,
                                      double *d2_out, double *p_out, uint32_t *face_out) {
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(dynamic, 16)
    for (int64_t i = 0; i < (int64_t)n; ++i)
        face_out[i] = orc_brute_force_closest(tri, nf, q + 3 * i, d2_out + i, p_out + 3 * i);
}

/* ------------------------------------------------------------------------------------------
 * Engine context: the engine arrays are caller-owned (the same bytes the GPU consumes); the
 * oracle derives only its own k-d tree from the site positions.
 */
typedef struct {
    uint64_t n_sites, n_faces;
    const double *site_xyz;
    const uint8_t *site_kind;
    const double *tri;        /* 9 per face: a, b, c */
    const double *sphere;     /* 4 per face: cx, cy, cz, r */
    const uint64_t *list_off; /* n_sites + 1 */
    const uint32_t *list_faces;
    double dmin[3], dmax[3];
    double prune_eps;
    orc_kdtree *kd;
} orc_ctx;

typedef struct {
    uint64_t n_queries, candidates_visited, exact_evaluations, pruned, fallbacks, kd_nodes_visited;
} orc_counters;

/* prune_eps = 1e-9 * |D.max - D.min|, the same definition as the device engine
 * (paper_2605_00429_b200/csrc/cuda/p2m_engine.cu).  It only changes counters, never results. */
ORC_EXPORT orc_ctx *orc_ctx_create(uint64_t n_sites, const double *site_xyz, const uint8_t *site_kind,
                                   uint64_t n_faces, const double *tri, const double *sphere,
                                   const uint64_t *list_off, const uint32_t *list_faces,
                                   const double *domain6) {
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    if (!c) return NULL;
    c->n_sites = n_sites; c->n_faces = n_faces;
    c->site_xyz = site_xyz; c->site_kind = site_kind; c->tri = tri; c->sphere = sphere;
    c->list_off = list_off; c->list_faces = list_faces;
    for (int k = 0; k < 3; ++k) { c->dmin[k] = domain6[k]; c->dmax[k] = domain6[3 + k]; }
    c->prune_eps = 1e-9 * sqrt(dist2_3(c->dmax, c->dmin));
    c->kd = orc_kdtree_build(site_xyz, n_sites);
    if (!c->kd) { free(c); return NULL; }
    return c;
}

ORC_EXPORT void orc_ctx_free(orc_ctx *c) {
    if (!c) return;
    orc_kdtree_free(c->kd);
    free(c);
}

static inline int in_domain(const orc_ctx *c, const double *q) {
    return q[0] >= c->dmin[0] && q[0] <= c->dmax[0] && q[1] >= c->dmin[1] && q[1] <= c->dmax[1] &&
           q[2] >= c->dmin[2] && q[2] <= c->dmax[2];
}

/* query_distance.  Returns flags; writes d^2, point, face, site, counters.
 * prune modes:
 *   PRUNE_OFF  -- evaluate every candidate: the lexicographic argmin of (d^2, face id) over the
 *                 whole list (the list is ascending, so strict '<' keeps the lowest id on ties)
 *   PRUNE_SAFE -- skip a face only if |q-c|^2 > (r + d_min + eps)^2 (strict), which can never
 *                 skip a face that ties or beats d_min -> bit-identical to PRUNE_OFF
 *   PRUNE_SPEC -- the literal SPEC test "lb = |q-c| - r < d_min", kept to
 *                 demonstrate pruning neutrality in tests; not used for parity.
 */
static uint32_t query_one(const orc_ctx *c, const double *q, int prune, double *d2_out, double *p_out,
                          uint32_t *face_out, uint32_t *site_out, uint64_t *cnt /* C,E,nodes */) {
    uint64_t visited = 0;
    double sd2;
    const uint32_t s = orc_nearest_site(c->kd, q, &sd2, &visited);
    *site_out = s;
    cnt[2] = visited;
    uint32_t flags = 0;
    if (!in_domain(c, q)) flags |= FLAG_OUT_OF_DOMAIN;
    if (c->site_kind[s] == SITE_SENTINEL || (flags & FLAG_OUT_OF_DOMAIN)) {
        /* fallback: exact global minimum; the BVH result with lowest-face-id ties
         * equals the brute-force scan */
        flags |= FLAG_FALLBACK;
        *face_out = orc_brute_force_closest(c->tri, c->n_faces, q, d2_out, p_out);
        cnt[0] = 0; cnt[1] = 0;
        return flags;
    }
    const uint64_t beg = c->list_off[s], end = c->list_off[s + 1];
    double best = INFINITY, dmin = INFINITY;
    uint32_t bf = UINT32_MAX;
    uint64_t exact = 0;
    for (uint64_t j = beg; j < end; ++j) {
        const uint32_t f = c->list_faces[j];
        const double *sp = c->sphere + 4 * (uint64_t)f;
        if (prune == PRUNE_SAFE) {
            const double dc2 = dist2_3(q, sp);
            const double t = sp[3] + dmin + c->prune_eps;
            if (dc2 > t * t) continue;
        } else if (prune == PRUNE_SPEC) {
            const double lb = sqrt(dist2_3(q, sp)) - sp[3];
            if (!(lb < dmin)) continue;
        }
        const double *t = c->tri + 9 * (uint64_t)f;
        double d2, p[3];
        CLOSEST(q, t, t + 3, t + 6, &d2, p);
        ++exact;
        if (d2 < best) { best = d2; bf = f; dmin = sqrt(d2); }
    }
    cnt[0] = end - beg; cnt[1] = exact;
    *face_out = bf;
    *d2_out = best;
    if (bf != UINT32_MAX) {
        const double *t = c->tri + 9 * (uint64_t)bf;
        double d2;
        CLOSEST(q, t, t + 3, t + 6, &d2, p_out);
    } else {
        p_out[0] = p_out[1] = p_out[2] = NAN;
    }
    return flags;
}

/* batch_query: per-query results in input order.  per_query (optional) gets
 * 3 u64 per query: candidates_visited, exact_evaluations, kd nodes visited. */
ORC_EXPORT void orc_batch_query(const orc_ctx *c, const double *q, uint64_t n, int prune, int threads,
                                double *dist, double *closest, uint32_t *face, uint32_t *site,
                                uint32_t *flags, uint64_t *per_query, orc_counters *agg) {
    uint64_t tc = 0, te = 0, tf = 0, tn = 0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads) reduction(+ : tc, te, tf, tn)
#endif
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        double d2, p[3];
        uint32_t fo, so;
        uint64_t cnt[3];
        uint32_t fl = query_one(c, q + 3 * i, prune, &d2, p, &fo, &so, cnt);
        dist[i] = sqrt(d2);
        closest[3 * i] = p[0]; closest[3 * i + 1] = p[1]; closest[3 * i + 2] = p[2];
        face[i] = fo; site[i] = so;
        if (flags) flags[i] = fl;
        if (per_query) { per_query[3 * i] = cnt[0]; per_query[3 * i + 1] = cnt[1]; per_query[3 * i + 2] = cnt[2]; }
        tc += cnt[0]; te += cnt[1]; tn += cnt[2];
        if (fl & FLAG_FALLBACK) tf++;
    }
    (void)threads;
    if (agg) {
        agg->n_queries = n; agg->candidates_visited = tc; agg->exact_evaluations = te;
        agg->pruned = tc - te; agg->fallbacks = tf; agg->kd_nodes_visited = tn;
    }
}

ORC_EXPORT int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

ORC_EXPORT int orc_uses_reference_kernel(void) {
#ifdef P2M_ORACLE_USE_REF
    return 1;
#else
    return 0;
#endif
}
