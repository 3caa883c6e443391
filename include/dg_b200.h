/* dg_b200.h -- C-ABI of the B200-native straightest-geodesic tracer (libdigeo_b200.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++/torch types. The host
 * C++ layer in include/digeo/ (same names and semantics as the reference's
 * proj/include/digeo/) is a thin shim over these entry points, and INTEGRATION.md shows
 * the binding a maintainer of the reference would add at each call site.
 *
 * Reference call sites replaced (paths relative to the reference tree):
 *   dg_mesh_derive        <- Mesh::build derived arrays        proj/src/mesh.cpp:34-130
 *   dg_mesh_create        <- (device mirror of) class Mesh     proj/include/digeo/mesh.hpp:40-83
 *   dg_trace_batch        <- trace_batch / trace_batch_serial  proj/src/tracer.cpp:596-610
 *                            (OpenMP loop at :600 over run_one :578 -> Kernel<S>::run :490)
 *   dg_trace_polylines    <- trace_batch with record_polyline  proj/src/tracer.cpp:84-89,596-603
 *   dg_transition         <- geodesic_step, transport_over_edge, transport_over_vertex,
 *                            boundary_continue                 proj/src/tracer.cpp:630-735
 *   dg_ep_jacobians       <- ep_jacobians (+ frames)           proj/src/diff.cpp:13-66
 *   dg_ep_backward        <- ep_jacobians + pullback_ambient   proj/src/diff.cpp:44-66,328-354
 *   dg_gfd_jacobians      <- gfd_batched_many / gfd_batched / gfd_jacobian_v/p
 *                                                              proj/src/diff.cpp:208-326
 *                            (pullback of g is fused into dg_ep_backward / dg_gfd_jacobians: pass g)
 *   dg_set_devices        <- the fork/join of trace_batch      proj/src/tracer.cpp:596-603
 *   dg_batch_*            <- the call pair trace_batch -> EP loop / gfd_batched_many of one
 *                            training step                        proj/src/gradcheck.cpp:70-89
 *
 * All functions return DG_OK (0) or a DG_ERR_* code, never throw and never abort;
 * dg_last_error() gives the message of the last failure on the calling thread.
 * Per-element failures of a batch are NOT errors of the call: they are reported in the
 * status / stall bytes of that element (reference: tracer.cpp:584-591).
 * There is no CPU fallback: every compute entry point fails with DG_ERR_NO_DEVICE when no
 * CUDA device is usable. dg_mesh_derive is host-only by design (it mirrors Mesh::build,
 * which is build-once host code in the reference too).
 */
#ifndef DG_B200_H
#define DG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_API __attribute__((visibility("default")))

typedef struct dg_mesh dg_mesh;

/* ---- return codes (mapped 1:1 to the reference's exception classes, geometry.hpp:187-200) */
enum {
  DG_OK = 0,
  DG_ERR_INVALID_ARGS = 1,         /* digeo::InvalidArgs */
  DG_ERR_CUDA = 2,                 /* CUDA runtime failure */
  DG_ERR_PARSE = 3,                /* digeo::ParseError (vertex index out of range) */
  DG_ERR_NON_MANIFOLD = 4,         /* digeo::NonManifoldError */
  DG_ERR_DEGENERATE_FACE = 5,      /* digeo::DegenerateFaceError */
  DG_ERR_DEGENERATE_DIRECTION = 6, /* digeo::DegenerateDirection */
  DG_ERR_GFD = 7,                  /* plain digeo::Error from diff.cpp:123,184 */
  DG_ERR_NO_DEVICE = 8,            /* no usable CUDA device: there is no CPU fallback */
  DG_ERR_NUMERICAL_STALL = 10,     /* digeo::NumericalStall (single-call wrappers) */
  DG_ERR_BOUNDARY_HIT = 11         /* digeo::BoundaryHit (transport_over_vertex) */
};

/* ---- per-element codes */
enum { DG_TERM_LENGTH_REACHED = 0, DG_TERM_BOUNDARY = 1, DG_TERM_MAX_STEPS = 2 };
enum { DG_STATUS_OK = 0, DG_STATUS_STALLED = 1 };
enum {
  DG_STALL_NONE = 0,
  DG_STALL_DEGENERATE_DIRECTION = 1, /* "degenerate direction in face"            tracer.cpp:183 */
  DG_STALL_NO_EXIT = 2,              /* "no positive exit parameter"              tracer.cpp:197 */
  DG_STALL_NORMAL_DIRECTION = 3,     /* "initial direction is normal to the anchor face" :474 */
  DG_STALL_FACE_RANGE = 4,           /* "trace: start face out of range"          tracer.cpp:459 */
  DG_STALL_BARY_RANGE = 5            /* "trace: start barycentric coordinates not in the simplex" :461 */
};
/* StepEvent, tracer.hpp:52 */
enum { DG_EVENT_ADVANCED = 0, DG_EVENT_CROSSED_EDGE = 1, DG_EVENT_CROSSED_VERTEX = 2,
       DG_EVENT_BOUNDARY_SLIDE = 3, DG_EVENT_BOUNDARY_STOP = 4 };

enum { DG_MEM_HOST = 0, DG_MEM_DEVICE = 1 };
enum { DG_SORT_AUTO = 0, DG_SORT_ON = 1, DG_SORT_OFF = 2 };
enum { DG_WALKER_AUTO = 0, DG_WALKER_GENERIC = 1, DG_WALKER_FAST_LOADS = 2, DG_WALKER_FAST_TMA = 3, DG_WALKER_FAST_COOP = 4 };
/* Arithmetic of the f64 tracer. The library is built without FMA contraction and the EXACT lane (the default, and
 * the parity anchor) follows the reference's operation order, so a trace that never takes a vertex branch (no libm
 * calls) is bit-identical to the reference CPU build; vertex branches agree to the last ulp of atan2/sin/cos.
 * DG_LANE_FAST is an opt-in TOLERANCE lane of the plain forward map (f64, crossing records, no payload / transport
 * matrix / polylines / hole avoidance; other requests run the exact lane): same decisions and tolerances as the exact
 * lane, cheaper arithmetic. It walks over HALF-SIZE crossing records (64 bytes: shared edge vector, third vertex of the
 * entered face, 1 / |edge|; built on the first request of the lane, + 192 B per face) with the fold in intrinsic form --
 * the unit direction lies in the plane of the face it leaves, so its transported image is e (d.e) + in_to sqrt(1 -
 * (d.e)^2) and the barycentric velocity in the entered face follows from the same numbers: no in_from, no Gram solve,
 * rsqrt instead of sqrt + divisions -- with reciprocal-multiply quotients, one reciprocal for the exit parameter and a
 * first-order renormalisation of the direction. Its bar is north_star's: identical face sequences on non-degenerate
 * queries, end points / directions within 1e-9 x bbox diagonal (measured: <= 1e-13), GFD Jacobians within 1e-5
 * relative -- not bit equality (c2 forward 3.61 -> 2.67 ms, c3 15.8 -> 11.2 ms per 1 M). With dg_diff_cfg.lane it applies to GFD's full-length re-traces (and the fused forward). */
enum { DG_LANE_DEFAULT = 0, DG_LANE_EXACT = 1, DG_LANE_FAST = 2 };

DG_API const char* dg_last_error(void);
DG_API const char* dg_version(void);
DG_API int dg_device_count(void);          /* 0 when no CUDA device / driver */
DG_API int dg_set_device(int ordinal);     /* device used by subsequently created meshes */
DG_API int dg_device_sm_count(void);
/* Multi-GPU (one box): the DEVICE SET used by subsequently created meshes. bit i of mask = CUDA device i; the
 * lowest set bit is the primary device. A mesh created under a set of G > 1 devices is uploaded to each of them,
 * and every batched entry point (dg_trace_batch, dg_ep_jacobians, dg_ep_backward, dg_gfd_jacobians[_with_base],
 * dg_batch_*) then fans a request of >= 16 384 x G elements (env DG_MULTI_MIN) out over the set: the request is cut
 * into G contiguous shards -- of equal expected work (requested length) for host pointers, of equal counts for
 * device pointers --, each shard runs on its device from its own host thread, and every result is written at the
 * request index of the caller's arrays. This is the reference's fork/join site (the OpenMP loop inside trace_batch,
 * tracer.cpp:596-603); results are bitwise independent of the set (acceptance.cpp:173-201). There is no exchange
 * step and no reduction: all jobs of a GFD sample stay on its device. DG_MEM_DEVICE pointers live on the primary
 * device; the other shards work on local copies moved by peer copies (NVLink P2P when the driver allows it).
 * dg_set_device(ordinal) goes back to a single device. dg_set_device_list takes the set as an ordered list and
 * lets an ordinal repeat (several copies on one GPU: the whole fan-out path on a one-GPU box, for tests). */
DG_API int dg_set_devices(uint64_t mask);
DG_API int dg_set_device_list(const int32_t* ordinals, int32_t count);

/* ---- mesh ------------------------------------------------------------------------------
 * dg_mesh_derive: host-side restatement of Mesh::build (mesh.cpp:34-130). Validates the
 * triangle soup and fills the derived arrays (any output pointer may be NULL):
 *   adj[3nf] (-1 = boundary; local edge k is opposite corner k), fnormal[3nf] unit,
 *   farea[nf], vangle[nv] total interior angle, varea[nv], vboundary[nv],
 *   csr_off[nv+1]/csr_list[3nf] vertex->faces in face order, mean edge length, total area.
 * err_index receives the offending face (or, for non-manifold edges, the smaller vertex). */
DG_API int dg_mesh_derive(const double* xyz, int32_t nv, const int32_t* tri, int32_t nf,
                          int32_t* adj, double* fnormal, double* farea, double* vangle,
                          double* varea, uint8_t* vboundary, int32_t* csr_off,
                          int32_t* csr_list, double* mean_edge, double* total_area,
                          int64_t* err_index);

/* Uploads an immutable mesh (host pointers) into the device SoA layout described in
 * DESIGN.md. All arrays are required and must come from dg_mesh_derive (or Mesh::build). */
DG_API int dg_mesh_create(const double* xyz, int32_t nv, const int32_t* tri, int32_t nf,
                          const int32_t* adj, const double* fnormal, const double* vangle,
                          const uint8_t* vboundary, const int32_t* csr_off,
                          const int32_t* csr_list, dg_mesh** out);
/* Same, with layout flags. The transport cache stores one 128-byte crossing record per directed
 * half-edge: the fold isometry of tracer.cpp:113-126 plus the two corner-0 edge vectors of the
 * entered face (computed on the device at upload by the same code the uncached walker runs, so
 * results are bit-identical). AUTO enables it while the records stay within 16 GB (about 40 M
 * faces): the fast walker gathers them with four 256-bit loads per lane up to 250 MB and with
 * cooperative 256-bit loads (four lanes per record, one request per line) beyond, where the
 * per-lane loads fall off a cliff; TMA tile::gather4 is the third, selectable gather
 * (dg_trace_cfg.walker). Env DG_TRANSPORT_CACHE=on|off overrides AUTO. */
enum { DG_MESH_TRANSPORT_AUTO = 0, DG_MESH_TRANSPORT_ON = 1, DG_MESH_TRANSPORT_OFF = 2 };
DG_API int dg_mesh_create_ex(const double* xyz, int32_t nv, const int32_t* tri, int32_t nf,
                             const int32_t* adj, const double* fnormal, const double* vangle,
                             const uint8_t* vboundary, const int32_t* csr_off,
                             const int32_t* csr_list, uint32_t flags, dg_mesh** out);
/* Memory the library keeps warm: its own stream-ordered pool per device for staging buffers (never the device's
 * default pool, which other frameworks of the process use), a resident batch behind large DG_MEM_HOST calls, the
 * small-batch blocks and the pinned polyline arrays of a mesh. dg_trim releases all of it (m may be NULL: only the
 * pool of the current device); everything is re-created on demand. */
DG_API int dg_trim(const dg_mesh* m);
DG_API int dg_mesh_has_transport_cache(const dg_mesh* m);
/* How the fast walker gathers this mesh's crossing records for a batch of lone traces
 * (DG_WALKER_AUTO): per-lane 256-bit loads (also: no records), TMA tile::gather4, or cooperative
 * 256-bit loads. dg_mesh_uses_tma_gather: 1 iff that is DG_GATHER_TMA. */
enum { DG_GATHER_LOADS = 0, DG_GATHER_TMA = 1, DG_GATHER_COOP = 2 };
DG_API int dg_mesh_gather_mode(const dg_mesh* m);
DG_API int dg_mesh_uses_tma_gather(const dg_mesh* m);

DG_API void dg_mesh_destroy(dg_mesh* m);
DG_API int32_t dg_mesh_face_count(const dg_mesh* m);
DG_API int32_t dg_mesh_vertex_count(const dg_mesh* m);
DG_API int64_t dg_mesh_device_bytes(const dg_mesh* m);
DG_API int dg_mesh_device(const dg_mesh* m);            /* the primary device */
DG_API int dg_mesh_device_count(const dg_mesh* m);      /* devices holding a copy of this mesh (>= 1) */

/* ---- forward tracing ------------------------------------------------------------------- */
typedef struct dg_trace_cfg {
  int32_t max_steps;             /* 0: 10*sqrt(F)+100 (tracer.cpp:543) */
  uint8_t hole_avoidance;
  uint8_t want_transport_matrix;
  uint8_t use_f32;               /* run the stepping arithmetic in single precision */
  uint8_t lane;                  /* DG_LANE_* */
  uint8_t memory;                /* DG_MEM_HOST: pointers are host memory, staged by the library
                                    DG_MEM_DEVICE: pointers are device memory on the mesh's GPU */
  uint8_t sort_by_face;          /* DG_SORT_*: schedule queries in start-face order (results stay at the request index,
                                    same bits). AUTO = on for batches >= 32 768 on meshes whose crossing records exceed
                                    the L2 (> 96 MB), where neighbouring starts share their fetches; off otherwise */
  uint8_t refill_min;            /* idle lanes a warp waits for before it steals work (0 = the walker's default:
                                    4 with a bounded wait for the fast walker, 1 for the general one) */
  uint8_t blocks_per_sm;         /* resident CTAs per SM of the persistent grid (0 = occupancy query) */
  uint8_t walker;                /* DG_WALKER_AUTO: the fast walker whenever the request is the plain f64
                                    forward map, gathering the crossing records with per-lane 256-bit loads
                                    up to 250 MB of records and with cooperative loads beyond;
                                    DG_WALKER_GENERIC: always the general state machine; DG_WALKER_FAST_LOADS /
                                    DG_WALKER_FAST_TMA / DG_WALKER_FAST_COOP: the fast walker with that gather. Same bits whatever
                                    the choice; selectable for cross-checks and measurements */
  uint8_t reserved[3];
  void* stream;                  /* cudaStream_t to launch on. DG_MEM_HOST: NULL = the mesh's private
                                    stream, the call returns when the results are in host memory.
                                    DG_MEM_DEVICE: NULL = the CUDA default stream; the call is
                                    asynchronous on that stream. */
} dg_trace_cfg;

typedef struct dg_trace_in {
  const int32_t* face;     /* [n]   start face */
  const double* bary;      /* [3n]  start barycentrics */
  const double* dir;       /* [3n]  ambient tangent vector; its norm is the requested length */
  const double* payload;   /* [3n] or NULL; an all-zero row means "no payload" (tracer.cpp:582) */
} dg_trace_in;

/* Every pointer may be NULL (that output is then skipped). */
typedef struct dg_trace_out {
  int32_t* face;        /* [n]  final face (-1 for a rejected start, as a default GeodesicTrace) */
  double* bary;         /* [3n] final barycentrics, renormalised as tracer.cpp:75-82 */
  double* dir;          /* [3n] final unit direction (0 for zero-length requests) */
  double* traced;       /* [n]  traced length */
  double* requested;    /* [n]  requested length */
  uint8_t* term;        /* [n]  DG_TERM_* */
  uint8_t* status;      /* [n]  DG_STATUS_* */
  uint8_t* stall;       /* [n]  DG_STALL_* */
  double* payload;      /* [3n] transported payload (rows of payload-free elements are 0) */
  double* transport;    /* [9n] row-major transport matrix (want_transport_matrix) */
  int32_t* npoints;     /* [n]  number of polyline points the trace emits */
  int32_t* crossings;   /* [n]  face-to-face transitions executed (edge crossings + fan faces) */
  uint64_t* total_crossings; /* [1] sum of crossings over the batch (overwritten) */
  /* polyline recording: pass offsets from an exclusive scan of npoints of a previous call */
  const int64_t* poly_offsets; /* [n]  first slot of trace i; recording is on iff non-NULL */
  int64_t poly_total;   /* number of slots in the three poly_* arrays (sum of npoints) */
  int32_t* poly_face;   /* [total] */
  double* poly_bary;    /* [3 total] */
  double* poly_seg;     /* [total] length of the segment ENDING at this point (0 at the start point) */
} dg_trace_out;

DG_API int dg_trace_batch(const dg_mesh* mesh, int64_t n, const dg_trace_in* in,
                          const dg_trace_cfg* cfg, dg_trace_out* out);
/* What a plain f64 forward request of n queries gets under cfg (NULL = defaults): *face_order = 1 when it is
 * scheduled in start-face order (dg_trace_cfg.sort_by_face resolved), *gather = the DG_GATHER_* of its launch.
 * Under start-face order that is the per-lane loads; on a mesh beyond 250 MB of records the request is queued on
 * the cooperative gather as well and the requested lengths, summed on the device, decide which of the two runs
 * (long traces: expected crossings x sqrt(faces) > 1e6 -- the cooperative one). For reports; same bits whatever
 * the plan. */
DG_API int dg_trace_plan(const dg_mesh* m, int64_t n, const dg_trace_cfg* cfg, int* face_order, int* gather);

/* trace_batch with the reference's DEFAULT TraceConfig, record_polyline = true (tracer.hpp:22), in ONE call: the
 * library records, sizes, compacts and copies on the device (capped first pass, device scan, compaction, a second pass
 * for the few traces that outgrew their slots) -- no host-side scan, no second call. out: as dg_trace_batch with the
 * poly_* fields NULL (npoints is filled when asked for). *poly receives the polylines in PINNED HOST arrays owned by
 * the mesh: offsets[n + 1] (exclusive scan of the point counts; offsets[n] = total), face[total], bary[3 total],
 * seg[total] (length of the segment ENDING at a point, 0 at a start point). They stay valid until the next
 * dg_trace_polylines call on this mesh or its destruction: copy what must live longer. Host pointers only
 * (cfg->memory = DG_MEM_HOST, cfg->stream = NULL); runs on the mesh's primary device. Same bits as the two-call
 * form (dg_trace_batch sized by npoints, then with poly_offsets). */
typedef struct dg_polylines {
  int64_t total;
  const int64_t* offsets;
  const int32_t* face;
  const double* bary;
  const double* seg;
} dg_polylines;
DG_API int dg_trace_polylines(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg,
                              dg_trace_out* out, dg_polylines* poly);

/* Registers per thread, resident CTAs per SM and CTA size of a tracer kernel variant.
 * full: bit 2 = the TMA-gather variant of the fast walker, bit 3 = its cooperative-loads variant,
 *       bit 4 = its sibling-schedule instantiation (6 CTAs per SM),
 *       bit 0 = payload / transport matrix / hole avoidance / polyline support compiled in,
 *       bit 1 = transport-cache variant. */
DG_API void dg_trace_kernel_info(int use_f32, int full, int* regs, int* blocks_per_sm,
                                 int* block_threads);

/* Single-transition operations on n independent states (host pointers).
 * which: 0 geodesic_step (uses remaining[], writes step_length/finished/event)
 *        1 transport_over_edge   2 transport_over_vertex   3 boundary_continue
 * rc[i] receives DG_OK or the DG_ERR_* the reference would have thrown for element i. */
DG_API int dg_transition(const dg_mesh* mesh, int which, int64_t n, const int32_t* face,
                         const double* bary, const double* v, const double* remaining,
                         int hole_avoidance, int32_t* out_face, double* out_bary, double* out_v,
                         double* step_length, uint8_t* finished, uint8_t* event, uint8_t* stall,
                         int32_t* rc);

/* ---- differentials --------------------------------------------------------------------- */
#define DG_FRAME_DOUBLES 33
/* frames block per sample: e_par, e_perp, normal (frame_in_v) | u_hat, v_hat, pinv_row0,
 * pinv_row1 (frame_in_p) | the same four for frame_out */

/* DG_MEM_DEVICE with the differentials: the pointers are device memory and the work runs on cfg->stream, but
 * dg_ep_jacobians, dg_ep_backward, dg_gfd_jacobians[_with_base] and dg_trace_gfd are HOST-SYNCHRONOUS: their
 * return code depends on an error word of the batch (first degenerate sample, failed base trace ...), so they wait
 * for cfg->stream before they return, and must not be called under stream capture. dg_gfd_pullback and
 * dg_trace_batch are asynchronous on the stream. */
typedef struct dg_diff_cfg {
  uint8_t memory;       /* DG_MEM_HOST / DG_MEM_DEVICE for all pointers of the call */
  uint8_t lane;         /* DG_LANE_*: arithmetic of GFD's full-length traces */
  uint8_t schedule;     /* GFD round 2: DG_GFD_SCHEDULE_AUTO = the full-length re-traces of a sample run as
                           sibling lanes of one warp and share every crossing-record fetch;
                           DG_GFD_SCHEDULE_PLAIN = job order; DG_GFD_SCHEDULE_FACE_ORDER = sibling groups handed
                           out in start-face order of their samples (what AUTO does for >= 32 768 samples on a
                           mesh whose crossing records exceed the L2). A schedule only: same bits either way. */
  uint8_t reserved[5];
  void* stream;
  int32_t max_steps;    /* GFD re-traces; 0 = default */
} dg_diff_cfg;
enum { DG_GFD_SCHEDULE_AUTO = 0, DG_GFD_SCHEDULE_PLAIN = 1, DG_GFD_SCHEDULE_FACE_ORDER = 2 };

/* Extrinsic-proxy Jacobians for n samples. rot[9n] = rotation_ep (row-major), frames
 * [DG_FRAME_DOUBLES n]; either may be NULL. Fails with DG_ERR_DEGENERATE_DIRECTION (and
 * *err_index = first offending sample) when |v| < 1e-12 or v is normal to its face. */
DG_API int dg_ep_jacobians(const dg_mesh* mesh, int64_t n, const int32_t* face,
                           const double* bary, const double* v, const int32_t* end_face,
                           const double* end_bary, const double* end_dir, const dg_diff_cfg* cfg,
                           double* rot, double* frames, int64_t* err_index);

/* Fused EP backward: grad_v[3n] = pullback_ambient(g, ep_jacobians(...)).grad_v; grad_p is
 * identically zero for EP and is only written when non-NULL. */
DG_API int dg_ep_backward(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v,
                          const int32_t* end_face, const double* end_dir, const double* g,
                          const dg_diff_cfg* cfg, double* grad_v, double* grad_p,
                          int64_t* err_index);

/* Geodesic finite differences for n samples in two batched trace rounds (+ a third for
 * one-sided fallbacks). jv/jp[4n] row-major 2x2 (a b c d), degraded[4n] = degraded_v[0..1],
 * degraded_p[0..1]; frames may be NULL. If g != NULL also writes grad_v/grad_p[3n]
 * (pullback_ambient). base_* (optional, may all be NULL) receive the base traces' end states.
 * Whole-call failures as in the reference: DG_ERR_DEGENERATE_DIRECTION (frames),
 * DG_ERR_GFD ("gfd: the base trace did not reach its requested length",
 * "gfd: start-point perturbation seeds failed to trace"). */
DG_API int dg_gfd_jacobians(const dg_mesh* mesh, int64_t n, const int32_t* face,
                            const double* bary, const double* v, double eps_v, double eps_p,
                            const double* g, const dg_diff_cfg* cfg, double* jv, double* jp,
                            uint8_t* degraded, double* frames, double* grad_v, double* grad_p,
                            int32_t* base_face, double* base_bary, double* base_dir,
                            int64_t* err_index);

/* The same with the base traces given -- the forward results (final face / barycentrics /
 * direction, termination and status bytes) of the same samples, as gfd_batched, gfd_jacobian_v and
 * gfd_jacobian_p take them (diff.hpp:63-73: the `trace` argument): only the four perturbed traces
 * per sample run. The caller guarantees the base traces were produced by dg_trace_batch on
 * (face, bary, v) in f64 with the step limit of cfg->max_steps; results are then bit-identical to
 * dg_gfd_jacobians. */
DG_API int dg_gfd_jacobians_with_base(const dg_mesh* mesh, int64_t n, const int32_t* face,
                                      const double* bary, const double* v, const int32_t* base_face,
                                      const double* base_bary, const double* base_dir,
                                      const uint8_t* base_term, const uint8_t* base_status,
                                      double eps_v, double eps_p, const double* g,
                                      const dg_diff_cfg* cfg, double* jv, double* jp,
                                      uint8_t* degraded, double* frames, double* grad_v,
                                      double* grad_p, int64_t* err_index);

/* Forward exp map AND GFD Jacobians of the same samples in ONE call. GFD's base trace of a sample is its forward
 * trace (diff.cpp:288-294: (p, v), no payload), and the Jacobians do not depend on the upstream gradient, so a
 * training step that will differentiate with GFD runs its forward here: the base traces ride in GFD's round 2 as the
 * FOURTH SIBLING of their sample's three full-length re-traces (the lanes of a group follow the same faces step for
 * step and share every crossing-record fetch), which costs less than half of a lone forward launch. *fwd receives the
 * forward results exactly as dg_trace_batch writes them (face, bary, dir, traced, requested, term, status, stall,
 * npoints, crossings, total_crossings; same bits; payload / transport / poly_* must be NULL), jv / jp / degraded /
 * frames as dg_gfd_jacobians. The backward of the step is then dg_gfd_pullback. When GFD fails as a whole
 * (DG_ERR_DEGENERATE_DIRECTION, DG_ERR_GFD ...) the forward results are still valid. */
DG_API int dg_trace_gfd(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v,
                        double eps_v, double eps_p, const dg_diff_cfg* cfg, dg_trace_out* fwd, double* jv, double* jp,
                        uint8_t* degraded, double* frames, int64_t* err_index);
/* pullback_ambient (diff.cpp:342-354) of upstream gradients g[3n] through GFD Jacobians that are already there
 * (jv, jp of dg_trace_gfd / dg_gfd_jacobians; end_face = the forward end faces): grad_v, grad_p [3n]. One light
 * kernel; DG_MEM_DEVICE: asynchronous on cfg->stream. Same bits as passing g to dg_gfd_jacobians. */
DG_API int dg_gfd_pullback(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v, const int32_t* end_face,
                           const double* jv, const double* jp, const double* g, const dg_diff_cfg* cfg, double* grad_v,
                           double* grad_p);

/* ---- resident batch (forward + backward on the same samples) --------------------------------
 * A training step runs trace_batch (tracer.hpp:94) and then the EP loop ep_jacobians +
 * pullback_ambient (gradcheck.cpp:76-89) or gfd_batched_many (gradcheck.cpp:74) on the SAME
 * samples. A dg_batch keeps the forward inputs and results of that step on the GPU between the
 * two calls, so the backward moves only the upstream gradient in and the gradients out. All
 * pointers are HOST pointers (pinned memory lets the copies overlap the kernels); the arithmetic
 * is that of dg_trace_batch / dg_ep_backward / dg_gfd_jacobians, bit for bit. A dg_batch is not
 * thread-safe (one per calling thread); it must be destroyed before its mesh. */
typedef struct dg_batch dg_batch;
DG_API int dg_batch_create(const dg_mesh* mesh, int64_t capacity, dg_batch** out);
DG_API void dg_batch_destroy(dg_batch* b);
DG_API int64_t dg_batch_size(const dg_batch* b);
/* Plain forward exp map (no payload / transport matrix / hole avoidance / polylines: those go
 * through dg_trace_batch). cfg->memory must be DG_MEM_HOST and cfg->stream NULL. From 2^18 queries in plain order
 * the call is streamed: one persistent walker runs while the queries arrive and the results leave, and the calling
 * thread spins on per-chunk completion flags to queue the copies back; below that, or in start-face
 * order, slices on separate streams. Same bits either way. */
DG_API int dg_batch_trace(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg,
                          dg_trace_out* out);
/* The forward of a step whose backward will be GFD: dg_trace_gfd on the resident batch (forward results out, the
 * Jacobians stay on the GPU). A following dg_batch_gfd with the same eps and step limit only pulls g back. A
 * whole-call GFD failure is reported by that dg_batch_gfd call, not here: the forward results are valid. */
DG_API int dg_batch_trace_gfd(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg, double eps_v,
                              double eps_p, dg_trace_out* out);
/* EP backward of the resident samples: g [3n] in, grad_v [3n] (and grad_p [3n], zero) out. */
DG_API int dg_batch_ep_backward(dg_batch* b, const double* g, double* grad_v, double* grad_p,
                                int64_t* err_index);
/* GFD Jacobians (+ pull-back when g is given) of the resident samples; outputs may be NULL. */
DG_API int dg_batch_gfd(dg_batch* b, double eps_v, double eps_p, const double* g, int32_t max_steps,
                        double* jv, double* jp, uint8_t* degraded, double* grad_v, double* grad_p,
                        int64_t* err_index);

#ifdef __cplusplus
}
#endif
#endif /* DG_B200_H */
