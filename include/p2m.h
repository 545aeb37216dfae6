/*
 * p2m.h -- C ABI of the B200-native batched point-to-mesh query (P2M++ hot path).
 *
 * The reference (arxiv 2605.00429, REF=/root/reference) ships no FFI: its API surface is the
 * C++ namespace p2mx (REF/proj/include/p2mx/geom.hpp:9-145) plus the SPEC's build-then-query
 * engine ops (REF/SPEC.md:473-505) driven by cmd_build then cmd_query (REF/SPEC.md:598-612).
 * This header is the drop-in boundary for that path; every entry point cites the reference
 * interface it replaces.  Plain pointers and sizes only; no C++ exceptions or torch types cross
 * it.  All functions return P2M_OK (0) on success and a negative P2M_ERR_* on failure, with a
 * thread-local message in p2m_last_error().
 *
 * Two shared libraries implement it:
 *   libp2m_host.so  -- host C++ builder and synthetic mesh/query generators   (p2m_build*, p2m_mesh*, p2m_gen*)
 *   libp2m_cuda.so  -- device engine: CUDA sm_100a query kernels              (p2m_engine*, p2m_query*)
 * Conventions (REF/SPEC.md:99-100, 518-519, 611): the engine is immutable after build; queries
 * are pure and may be issued from several host threads; a query outside the domain D is never
 * an error, it is answered exactly and flagged per row.
 */
#ifndef P2M_H_
#define P2M_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2M_ABI_VERSION 2

/* ---- status codes (GeometryError REF/proj/include/p2mx/geom.hpp:88-91 -> P2M_ERR_GEOMETRY) ---- */
enum {
    P2M_OK = 0,
    P2M_ERR_INVALID = -1,   /* bad argument / null pointer / inconsistent sizes */
    P2M_ERR_CUDA = -2,      /* CUDA runtime failure or no usable device */
    P2M_ERR_NOT_BUILT = -3, /* "engine not built" (REF/SPEC.md:492) */
    P2M_ERR_GEOMETRY = -4,  /* degenerate input (REF/proj/src/geom.cpp:84,92,98) */
    P2M_ERR_OOM = -5,
    P2M_ERR_IO = -6,        /* EngineIndexFile magic/version/hash/truncation (REF/SPEC.md:640) */
    P2M_ERR_INTERNAL = -7
};

/* ---- site kinds (SiteSet, REF/SPEC.md:237-240) ---- */
enum { P2M_SITE_MESH_VERTEX = 0, P2M_SITE_SENTINEL = 1, P2M_SITE_AUXILIARY = 2 };

/* ---- per-query flags (QueryResult fallback flag, REF/SPEC.md:468,491,611) ---- */
enum {
    P2M_FLAG_FALLBACK = 1u,      /* answered by the exact BVH closest-point search, not a table */
    P2M_FLAG_OUT_OF_DOMAIN = 2u, /* q outside D (REF/SPEC.md:648) */
    P2M_FLAG_TABLE_MISS = 4u     /* the nearest site's list had no face within the distance bound
                                    |q - ref(site)| -- the table is not a superset of the faces that
                                    can be nearest in the site's cell (REF/SPEC.md:435 violated, e.g.
                                    a hand-filled p2m_engine_desc); the row is answered exactly by
                                    the BVH fallback and also carries P2M_FLAG_FALLBACK */
};

/* Thread-local description of the last failure on this thread ("" if none). */
const char *p2m_last_error(void);

/* =================================================================================================
 * Device engine (libp2m_cuda.so)
 * ================================================================================================= */

/* The engine as produced by the build phase (REF/SPEC.md:415-423 InterceptionIndex, 237-240
 * SiteSet, 118 per-face spheres, 588-591 EngineIndexFile fields).  All pointers are HOST
 * pointers, caller-owned, read only during p2m_engine_create. */
typedef struct p2m_engine_desc {
    uint64_t n_sites;
    const double *site_xyz;      /* 3 * n_sites, site positions (ids are array positions) */
    const uint8_t *site_kind;    /* n_sites, P2M_SITE_* */
    uint64_t n_faces;
    const double *tri_xyz;       /* 9 * n_faces: a.xyz, b.xyz, c.xyz (validated, non-degenerate) */
    const double *face_sphere;   /* 4 * n_faces: minimal bounding sphere c.xyz, r (geom.cpp:96-120) */
    const uint64_t *list_offsets;/* n_sites + 1: CSR offsets of the interception lists */
    const uint32_t *list_faces;  /* list_offsets[n_sites] face ids, ascending & unique per site */
    double domain_min[3];        /* query domain D (REF/SPEC.md:648: 10x mesh AABB) */
    double domain_max[3];
    const double *site_cell_box; /* optional (may be NULL): 6 * n_sites, AABB (min.xyz, max.xyz) of each
                                    site's Voronoi cell (NaN for sentinels).  Enables the exact grid
                                    cell-locate of nearest_site; without it the k-d tree is used. */
    const double *site_ref_xyz;  /* optional (may be NULL): 3 * n_sites, a point ON the mesh per site --
                                    auxiliary sites' projection proj(s, M) (REF/SPEC.md:238); ignored
                                    for mesh vertices (the vertex itself) and sentinels.  Seeds the
                                    grouped scan's d_min with the upper bound |q - ref| (result-neutral). */
    const uint64_t *adj_offsets; /* optional (may be NULL): n_sites + 1, CSR of the Delaunay adjacency */
    const uint32_t *adj_sites;   /* (sites whose Voronoi cells share a facet, symmetric, ascending);
                                    enables the DelaunayWalk nearest-site strategy (REF/SPEC.md:476) */
} p2m_engine_desc;

/* Aggregate counters (REF/SPEC.md:468, 500, 511). */
typedef struct p2m_counters {
    uint64_t n_queries;
    uint64_t candidates_visited; /* sum of nearest-site list lengths */
    uint64_t exact_evaluations;  /* point-triangle evaluations after sphere pruning */
    uint64_t pruned;             /* candidates_visited - exact_evaluations */
    uint64_t fallbacks;          /* rows answered by the BVH fallback */
    uint64_t kd_nodes_visited;   /* nearest-site candidates evaluated (k-d nodes or grid candidates) */
    uint64_t filter_passes;      /* grouped scan: candidates passing the first fp32 sphere test (diag.) */
    uint64_t warp_rare_iters;    /* grouped scan: warp-level rare-path iterations x 32 (diagnostic) */
    uint64_t structure_bytes;    /* grouped scan: bytes of the read-only structure the scan kernels load,
                                    each staged list chunk counted once per tile, each face record once
                                    per warp visit (the roofline's algorithmic bytes, with 64 B per row
                                    of q/row index in and results out) -- ABI v2 */
    uint64_t scan_tiles;         /* grouped scan: tiles scanned (CTA tiles + one-warp tiles) -- ABI v2 */
} p2m_counters;

typedef struct p2m_engine p2m_engine;

/* Upload an engine to n_devices GPUs (device_ids may be NULL -> 0..n-1).  The structure is packed
 * once on the host (k-d tree in BFS order, 128-byte face records, CSR), copied to the first device
 * and replicated to the others by a one-time peer copy.
 * Replaces: build_nns_index (REF/SPEC.md:473-481) + the engine hand-off of cmd_query
 * (REF/SPEC.md:607-612, 637-641). */
int p2m_engine_create(const p2m_engine_desc *desc, int n_devices, const int *device_ids,
                      p2m_engine **out);
void p2m_engine_destroy(p2m_engine *engine);

/* Device image of an engine (the EngineIndexFile loaded straight into the
 * device layout; REF/SPEC.md:588-591, 637-641).  save writes slot 0's packed layout -- k-d tree,
 * face records, fp32 records, spatially ordered lists with their group spheres, cell-locate grid,
 * fallback BVH, heavy-site flags, kernel parameters -- as "P2MD" v1 (little-endian, FNV-1a
 * checksum).  load validates every count, CSR and id range, then uploads it as is (no host desc,
 * no re-packing, no heavy-site estimate) and replicates it like p2m_engine_create.  Queries on a
 * loaded engine are bit-identical to the engine that was saved.  Errors: P2M_ERR_IO (open, magic,
 * version, truncation, checksum, invalid contents), P2M_ERR_CUDA. */
int p2m_engine_save(const p2m_engine *engine, const char *path);
int p2m_engine_load(const char *path, int n_devices, const int *device_ids, p2m_engine **out);

/* Number of devices the engine is replicated on, and the peer-replica timing of create. */
int p2m_engine_info(const p2m_engine *engine, int *n_devices, double *replicate_ms,
                    uint64_t *device_bytes);

/* batch_query (REF/SPEC.md:497-505) with query_distance semantics (REF/SPEC.md:488-496) per row.
 * HOST buffers: q_xyz (3n doubles, fp64 little-endian triples as cmd_query's --format bin,
 * REF/SPEC.md:609), outputs distance (n), closest_xyz (3n), face (n), site (n), flags (n, may be
 * NULL), counters (may be NULL).  Rows are sharded evenly over the engine's devices, one host
 * thread per device; synchronous. */
int p2m_query(p2m_engine *engine, const double *q_xyz, uint64_t n, double *distance,
              double *closest_xyz, uint32_t *face, uint32_t *site, uint32_t *flags,
              p2m_counters *counters);

/* Same on DEVICE-resident buffers of the engine's device `slot` (0..n_devices-1), enqueued on
 * `stream` (a cudaStream_t, NULL = legacy default); asynchronous unless counters != NULL.
 * This is the benchmarked hot path: Morton keys -> radix sort -> fused nearest-site descent +
 * pruned list scan -> results scattered to input order. */
int p2m_query_device(p2m_engine *engine, int slot, const double *d_q_xyz, uint64_t n,
                     double *d_distance, double *d_closest_xyz, uint32_t *d_face, uint32_t *d_site,
                     uint32_t *d_flags, void *stream, p2m_counters *counters);

/* nearest_site only (REF/SPEC.md:482-487), device buffers, for tests and the cell-locate split. */
int p2m_nearest_site_device(p2m_engine *engine, int slot, const double *d_q_xyz, uint64_t n,
                            uint32_t *d_site, void *stream);

/* Optional per-query counters for the last p2m_query_device on slot (3 x u64 per row in input
 * order: candidates, exact evaluations, kd nodes visited), for parity of counters. */
int p2m_query_device_counters(p2m_engine *engine, int slot, const double *d_q_xyz, uint64_t n,
                              uint64_t *d_per_query, void *stream);

/* Kernel-split timing (ms, CUDA events recorded on each call's own stream, no host sync):
 * ms[0] morton keys, [1] Morton sort, [2] nearest-site descent (or the whole fused query),
 * [3] regroup sort, [4] grouped list scan, [5] total -- mean over the p2m_query_device calls
 * recorded since p2m_set_profiling(e, 1) (up to 256), then the record is reset.  ms has 6 slots. */
int p2m_set_profiling(p2m_engine *engine, int enable);
int p2m_last_timings(p2m_engine *engine, int slot, float *ms);

/* Scan strategy (results are identical; counters too):
 *   P2M_SCAN_GROUPED (default) -- descend, regroup rows by nearest site, scan each site's list once
 *                                  per 256-row tile from shared memory
 *   P2M_SCAN_FUSED             -- one thread per row does descent + scan from global memory */
enum { P2M_SCAN_GROUPED = 0, P2M_SCAN_FUSED = 1 };
int p2m_set_scan_mode(p2m_engine *engine, int mode);

/* nearest_site strategy (REF/SPEC.md:473-481 NearestSiteIndex; all give the exact nearest site,
 * ties -> lowest id, so results never depend on it -- "strategy neutrality", REF/SPEC.md:510):
 *   P2M_NNS_GRID   (default) -- exact cell-locate grid over the Voronoi cell boxes, k-d tree
 *                               outside the grid box / when the engine has no cell boxes
 *   P2M_NNS_KDTREE           -- left-balanced k-d tree only
 *   P2M_NNS_WALK             -- greedy descent on the Delaunay adjacency (REF/SPEC.md:476, 516),
 *                               warm-started from a site listed in the query's grid cell (or site
 *                               0); needs desc.adj_offsets, else P2M_ERR_INVALID */
enum { P2M_NNS_GRID = 0, P2M_NNS_KDTREE = 1, P2M_NNS_WALK = 2 };
int p2m_set_nns_strategy(p2m_engine *engine, int strategy);

/* Number of kernels launched by one p2m_query_device call of n rows (for gpu_launches). */
int p2m_kernels_per_query(p2m_engine *engine, uint64_t n, int *launches);

/* =================================================================================================
 * Host builder (libp2m_host.so) -- preprocessing, produced once, reported not optimised
 * (REF/SPEC.md:112-456, cmd_build REF/SPEC.md:598-606)
 * ================================================================================================= */

typedef struct p2m_build_config {
    int augment;           /* --augment {on,off}; REF/SPEC.md:656 */
    double alpha;          /* tau = alpha * mean edge length; default 4.0 (REF/SPEC.md:367) */
    int k;                 /* density threshold; default 24 */
    double rho;            /* ring radius = rho * tau; default 0.75 */
    int max_rounds;        /* default 3 */
    double domain_scale;   /* D = AABB scaled about its centre; default 10.0 (REF/SPEC.md:648) */
    int n_threads;         /* 0 = all hardware threads */
    int strict_mesh;       /* --strict-mesh: degenerate faces are an error instead of removed */
    int aux_corner_union;  /* 1 (default): auxiliary table = union of B(u, |u-proj|) over the cell
                              corners -- the subset of the SPEC list that REF/SPEC.md:413 names, valid
                              by Theorem 1 about proj; 0: the literal single ball B(s, max_u |s-u| +
                              |u-proj|) of REF/SPEC.md:406-414 (whole-mesh lists for off-surface sites
                              whose cells reach the sentinels) */
} p2m_build_config;

typedef struct p2m_build_stats {
    uint64_t n_input_vertices, n_input_faces;
    uint64_t n_vertices, n_faces;       /* after validate_mesh (REF/SPEC.md:132-140) */
    uint64_t merged_vertices, removed_faces;
    uint64_t n_sites, n_aux_sites;
    int rounds_used;                    /* augmentation rounds that inserted sites */
    double mean_edge, tau;
    uint64_t list_entries;              /* total CSR entries */
    uint64_t list_max;                  /* Table 1 "Max" (REF/SPEC.md:424-432) */
    double list_avg;                    /* Table 1 "Avg" over non-sentinel sites */
    double t_voronoi_s, t_augment_s, t_tables_s, t_total_s; /* Table 3 split (REF/SPEC.md:593) */
    uint64_t cell_corners;              /* total Voronoi cell corners over real sites */
} p2m_build_stats;

typedef struct p2m_host_engine p2m_host_engine;

void p2m_build_config_default(p2m_build_config *cfg);

/* cmd_build minus file I/O: validate_mesh -> build_bvh -> make_bounded_site_set ->
 * augment_sites -> cell corners -> build_all_tables -> per-face spheres (REF/SPEC.md:598-606). */
int p2m_build(const double *vertices, uint64_t n_vertices, const uint32_t *faces, uint64_t n_faces,
              const p2m_build_config *cfg, p2m_host_engine **out);

/* build_all_tables as a job (REF/SPEC.md:397-423, ball enumeration REF/SPEC.md:192-200): site s's
 * list = every face f that meets one of its closed balls k -- a vertex of f within r2_k of c_k, or
 * closest_on_triangle_sq(c_k, f) <= r2_k -- found by walking the builder's BVH with the box test
 * box_sqdist(c_k) <= r2_k at every node from the root.  The set is fully determined by these
 * arrays, so any executor that evaluates the same fp64 tests gives the same tables. */
typedef struct p2m_table_job {
    uint64_t n_sites;
    const uint64_t *ball_off;   /* S+1 */
    const double *balls;        /* 4 per ball: centre xyz, r^2 */
    uint64_t n_faces;
    const double *tri;          /* 9 per face */
    uint64_t n_nodes;           /* BVH, depth-first: left child = node + 1 */
    const double *node_box;     /* 6 per node: lo xyz, hi xyz */
    const uint32_t *node_meta;  /* 3 per node: right child, first, count (count 0 = interior) */
    const uint32_t *perm;       /* leaf face order */
} p2m_table_job;
/* Fills off[0..S] and *lists (allocated with malloc, freed by the builder); each list ascending. */
typedef int (*p2m_table_fn)(void *ctx, const p2m_table_job *job, uint64_t *off, uint32_t **lists);
/* p2m_build with the table phase delegated to fn (NULL = the builder's own host threads). */
int p2m_build_with(const double *vertices, uint64_t n_vertices, const uint32_t *faces, uint64_t n_faces,
                   const p2m_build_config *cfg, p2m_table_fn fn, void *ctx, p2m_host_engine **out);
/* Delaunay adjacency of an arbitrary point set (no mesh): facet neighbours of the points' Voronoi
 * cells bounded by the builder's sentinels, symmetric, ascending, sentinels dropped -- the
 * DelaunayWalk graph (REF/SPEC.md:476) for queries inside 10x the points' AABB.  *off (n+1) and
 * *adj are malloc'd; release with p2m_free. */
int p2m_delaunay_adjacency(const double *xyz, uint64_t n, uint64_t **off, uint32_t **adj);

/* (libp2m_cuda.so) p2m_build with the table job run on GPU `device`: one
 * thread per ball walks a device copy of the same BVH, (site, face) hits are radix-sorted and
 * deduplicated into the CSR.  Tables are bit-identical to p2m_build's; t_tables_s is the GPU
 * phase including its copies. */
int p2m_build_device(const double *vertices, uint64_t n_vertices, const uint32_t *faces,
                     uint64_t n_faces, const p2m_build_config *cfg, int device, p2m_host_engine **out);
/* The table job alone on GPU `device` (fn-compatible: ctx points to the int device id). */
int p2m_table_job_device(void *ctx, const p2m_table_job *job, uint64_t *off, uint32_t **lists);
void p2m_host_engine_destroy(p2m_host_engine *h);

/* Pointers into the built engine (valid until destroy); feed straight into p2m_engine_create. */
int p2m_host_engine_desc(const p2m_host_engine *h, p2m_engine_desc *out);
int p2m_host_engine_stats(const p2m_host_engine *h, p2m_build_stats *out);
/* Validated mesh (face ids of all results refer to it). */
int p2m_host_engine_mesh(const p2m_host_engine *h, const double **vertices, uint64_t *n_vertices,
                         const uint32_t **faces, uint64_t *n_faces);
/* Auxiliary-site mesh projections (3 per site; NaN for non-auxiliary sites, REF/SPEC.md:238). */
int p2m_host_engine_site_refs(const p2m_host_engine *h, const double **ref_xyz);
/* Voronoi cell corners of a site (REF/SPEC.md:265-273), copied into out (3 per corner). */
int p2m_host_engine_cell_corners(const p2m_host_engine *h, uint64_t site, double *out,
                                 uint64_t capacity, uint64_t *n_corners);

/* bvh_closest_point (REF/SPEC.md:201-209) on the host BVH: exact, lowest face id on ties. */
int p2m_host_closest_point(const p2m_host_engine *h, const double *q, double *d2, double *p,
                           uint32_t *face);

/* EngineIndexFile "P2MX" (REF/SPEC.md:588-591, 637-641): lossless round trip of sites, tables,
 * config and D.  Load rebuilds the BVH and validates the mesh hash. */
int p2m_host_engine_save(const p2m_host_engine *h, const char *path);
int p2m_host_engine_load(const char *path, const double *vertices, uint64_t n_vertices,
                         const uint32_t *faces, uint64_t n_faces, p2m_host_engine **out);

/* ---- synthetic workloads (BASELINE.json configs 1..5) ---- */

/* Mesh of config cfg (1..5).  Arrays are allocated by the library; free with p2m_free. */
int p2m_mesh_config(int cfg, double **vertices, uint64_t *n_vertices, uint32_t **faces,
                    uint64_t *n_faces);
/* Unit-radius icosphere of the given subdivision level (tests). */
int p2m_mesh_icosphere(int level, double **vertices, uint64_t *n_vertices, uint32_t **faces,
                       uint64_t *n_faces);
/* Queries [first, first+count) of config cfg's deterministic query sequence on the given mesh. */
int p2m_gen_queries(int cfg, const double *vertices, uint64_t n_vertices, const uint32_t *faces,
                    uint64_t n_faces, uint64_t first, uint64_t count, double *out_xyz);
/* Seeded uniform points in a box (cmd_bench, REF/SPEC.md:613-616). */
int p2m_gen_uniform(uint64_t seed, const double *box_min, const double *box_max, uint64_t first,
                    uint64_t count, double *out_xyz);
void p2m_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* P2M_H_ */
