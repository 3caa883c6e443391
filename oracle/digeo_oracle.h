/* TEST INFRASTRUCTURE ONLY -- the CPU oracle. Never linked into, imported by or called from the
 * product (paper_2603_15780_b200/, include/); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may use it.
 *
 * Plain-C99 restatement of the reference's algorithm for the hot path (f64 lane):
 *   og_mesh_build        Mesh::build                 proj/src/mesh.cpp:34-130
 *   og_trace_batch       Kernel<double>::run / trace_batch   proj/src/tracer.cpp:44-603
 *   og_ep                ep_jacobians + pullback_ambient     proj/src/diff.cpp:13-66, 328-354
 *   og_gfd               gfd_batched_many                    proj/src/diff.cpp:116-326
 * Pinned against the reference's golden trace (proj/tests/golden/trace_square.json), the
 * Appendix-B known answers and fixtures generated from the unmodified reference
 * (tests/golden/, tests/test_oracle.py).
 */
#ifndef DIGEO_ORACLE_H
#define DIGEO_ORACLE_H
#include <stdint.h>

typedef struct og_mesh og_mesh;

/* error classes = the reference's exception types (geometry.hpp:187-200) */
enum { OG_OK = 0, OG_INVALID_ARGS = 1, OG_PARSE = 3, OG_NON_MANIFOLD = 4, OG_DEGENERATE_FACE = 5,
       OG_DEGENERATE_DIRECTION = 6, OG_ERROR = 7, OG_NUMERICAL_STALL = 10 };

og_mesh* og_mesh_build(const double* xyz, int nv, const int32_t* tri, int nf, int* err, char* msg, int msglen);
void og_mesh_free(og_mesh* m);
int og_mesh_nv(const og_mesh* m);
int og_mesh_nf(const og_mesh* m);
double og_mesh_mean_edge(const og_mesh* m);
/* any pointer may be NULL */
void og_mesh_get(const og_mesh* m, int32_t* adj, double* fnormal, double* farea, double* vangle, double* varea,
                 uint8_t* vboundary, int32_t* csr_off, int32_t* csr_list);

typedef struct og_cfg {
  int max_steps;       /* 0 = 10*sqrt(F)+100 */
  int hole_avoidance;
  int want_q;
  int threads;         /* OpenMP threads, 0 = default */
} og_cfg;

/* Outputs may be NULL. stall: 0 none, 1 degenerate direction, 2 no exit, 3 normal direction,
 * 4 face range, 5 bary range. Polyline recording is on iff poly_off != NULL (offsets from an
 * exclusive scan of npoints of a previous call; slot 0 of a trace holds segment length 0). */
void og_trace_batch(const og_mesh* m, int64_t n, const int32_t* face, const double* bary, const double* dir,
                    const double* payload, const og_cfg* cfg, int32_t* o_face, double* o_bary, double* o_dir,
                    double* o_traced, double* o_requested, uint8_t* o_term, uint8_t* o_status, uint8_t* o_stall,
                    double* o_payload, double* o_q, int32_t* o_npoints, const int64_t* poly_off,
                    int32_t* poly_face, double* poly_bary, double* poly_seg);

/* rot[9n], frames[33n], grad_v/grad_p[3n] may be NULL; g may be NULL. Returns an error class. */
int og_ep(const og_mesh* m, int64_t n, const int32_t* face, const double* v, const int32_t* end_face,
          const double* end_dir, const double* g, double* rot, double* frames, double* grad_v, double* grad_p,
          int64_t* err_index);

int og_gfd(const og_mesh* m, int64_t n, const int32_t* face, const double* bary, const double* v, double eps_v,
           double eps_p, const double* g, double* jv, double* jp, uint8_t* degraded, double* frames,
           double* grad_v, double* grad_p, int threads, char* msg, int msglen);

#endif
