// Launch interface between the C-ABI layer (dg_capi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dg_mesh_view.cuh"

namespace dg {

// One batch of trace jobs. All pointers are device pointers on the mesh's GPU; every output
// pointer may be null. Element i of the schedule is query perm[i] (or i when perm is null);
// results are always written at the query's own index.
struct TraceParams {
  // CUtensorMap of the crossing-record array ([3 nf] rows x 16 doubles, 128-byte swizzle) for the TMA
  // gather of the fast walker; opaque bytes here so that this header needs no driver API
  alignas(64) unsigned char he_map[128];
  MeshView mesh;
  int64_t n;
  const int32_t* face;
  const double* bary;
  const double* dir;
  const double* payload;  // null: no element has a payload
  const int32_t* perm;
  int32_t* o_face;
  double* o_bary;
  double* o_dir;
  double* o_traced;
  double* o_requested;
  uint8_t* o_term;
  uint8_t* o_status;
  uint8_t* o_stall;
  double* o_payload;
  double* o_transport;
  int32_t* o_npoints;
  int32_t* o_crossings;
  // o_traced / o_requested / o_stall / o_npoints / o_crossings and total_crossings cover the queries q >= aux_from
  // only, at index q - aux_from (0: every query). GFD's fused forward: the base traces are the last quarter of
  // round 2's jobs, and only they write the forward result record.
  int64_t aux_from;
  const int64_t* poly_offsets;  // non-null: record polylines, trace q from slot poly_offsets[q]
  int32_t poly_cap;             // > 0 (poly_offsets null): record polylines, trace q owns slots [q cap, (q + 1) cap);
                                // points beyond are counted in o_npoints but not written (dg_trace_polylines, pass 1)
  int32_t* poly_face;
  double* poly_bary;
  double* poly_seg;
  unsigned long long* queue_head;       // work-stealing cursor, zeroed before the launch
  unsigned long long* clear_word;       // optional: a word this launch zeroes (the cursor of the NEXT small-batch call)
  unsigned long long* total_crossings;  // optional: += sum of crossings of the batch
  int32_t max_steps;
  int32_t refill_min;  // refill a warp once this many lanes are idle (0 = the walker's default)
  // Sibling schedule (perm, if given, orders the GROUPS: stride entries): the first siblings * sibling_stride elements of the schedule are
  // groups of `siblings` queries {g, g + stride, ..., g + (siblings-1) stride}, handed to lanes of ONE warp
  // together. GFD's re-traces of one sample follow the same faces step for step, so the group gathers the
  // same crossing records at the same time: one HBM / L2 line serves all of them. 0 / 1 = plain order.
  int32_t siblings;
  int64_t sibling_stride;
  // 1 - 1e-10 (the vertex snap threshold, tracer.cpp:155) as a kernel parameter, set by launch_fast: the fast
  // step compares one weight of a pair against the literal and the other against this copy, because two
  // compares with the SAME constant get fused into fmax(a, b) >= c -- nine instructions instead of two
  double snap_hi;
  uint8_t hole_avoidance;
  uint8_t want_q;
  uint8_t he_map_ok;  // he_map is a valid tensor map of mesh.he
  uint8_t lane_fast;  // DG_LANE_FAST: plain forward requests over crossing records run the tolerance lane
  // Gate: the launch runs only if (*gate > gate_limit) == (gate_above != 0); null = runs. Two launches of one
  // request with complementary gates let a statistic computed on the device choose between two instantiations
  // without a host round trip (the gather of a batch in start-face order, dg_capi.cu).
  const double* gate;
  double gate_limit;
  uint8_t gate_above;
  // Streamed request (launch_trace_streamed; plain order only): the queries arrive and the results leave WHILE the
  // walker runs. The copy stream that uploads the queries chunk by chunk advances *stream_uploaded behind every
  // chunk; a warp takes work only below it. Every finished trace counts into its chunk (1 << stream_shift
  // queries), and the trace that completes a chunk raises the chunk's flag in mapped host memory -- the host
  // then copies that chunk's results back while the walker goes on.
  const unsigned long long* stream_uploaded;
  unsigned int* stream_done;    // [chunks] device
  unsigned int* stream_flags;   // [chunks] mapped pinned host memory
  unsigned int* stream_error;   // device: set when the wait for queries gave up (the copy stream failed)
  int32_t stream_shift;
};

struct LaunchShape {
  int sm_count;
  int blocks_per_sm;  // 0 = use the occupancy query
  int walker = 0;  // DG_WALKER_*: 0 auto, 1 general walker, 2 fast walker / 256-bit loads, 3 fast walker / TMA gather
};

// needs_full: any of payload / transport matrix / hole avoidance / polyline is requested.
cudaError_t launch_trace(const TraceParams& p, bool use_f32, bool needs_full, LaunchShape shape,
                         cudaStream_t stream);

// The streamed form of the plain f64 forward launch (TraceParams::stream_*). trace_streamable: whether launch_trace
// would run this request on the instantiation that has a streamed twin (crossing records, per-lane loads, exact
// lane, plain order).
bool trace_streamable(const TraceParams& p, bool use_f32, bool needs_full, LaunchShape shape);
cudaError_t launch_trace_streamed(const TraceParams& p, LaunchShape shape, cudaStream_t stream);

// Whether the fast walker gathers this mesh's crossing records through TMA (AUTO policy).
// gather of the crossing records for a lone-trace batch on this mesh: 0 per-lane loads, 1 TMA, 2 cooperative loads
int fast_walker_gather_mode(const MeshView& m, bool map_ok, bool face_order = false);

// Kernel attributes for reporting (registers, max resident blocks per SM).
void trace_kernel_info(bool use_f32, int variant, int* regs, int* blocks_per_sm, int* block_threads);

// ---- differentials (dg_diff_kernels.cu) ---------------------------------------------------

struct EpParams {
  MeshView mesh;
  int64_t n;
  const int32_t* face;      // start face
  const double* v;          // [3n]
  const int32_t* end_face;
  const double* end_dir;    // [3n]
  const double* g;          // [3n] upstream gradient (null for Jacobian-only)
  double* rot;              // [9n]  or null
  double* frames;           // [33n] or null
  double* grad_v;           // [3n]  or null
  double* grad_p;           // [3n]  or null
  unsigned long long* first_error;  // min index of a sample with a degenerate direction (init ~0ull)
};
cudaError_t launch_ep(const EpParams& p, cudaStream_t stream);

struct GfdBuffers {
  MeshView mesh;
  int64_t n;
  const int32_t* face;  // samples
  const double* bary;
  const double* v;
  double eps_v, eps_p;
  // round-1 job arrays (2n: seed_u | seed_v) and results
  int32_t* j1_face; double* j1_bary; double* j1_dir; double* j1_payload;
  int32_t* r1_face; double* r1_bary; double* r1_dir; double* r1_payload;
  uint8_t* r1_term; uint8_t* r1_status;
  // round-2 job arrays (4n: ret_u | ret_v | perp | par or base) and results
  int32_t* j2_face; double* j2_bary; double* j2_dir;
  int32_t* r2_face; double* r2_bary; uint8_t* r2_term; uint8_t* r2_status;
  // the base traces, indexed by sample: the caller's forward results, or slots [3n,4n) of round 2
  const int32_t* base_face; const double* base_bary; const double* base_dir;
  const uint8_t* base_term; const uint8_t* base_status;
  uint8_t base_in_round2;
  // the par jobs and their results, indexed by sample: slots [3n,4n) of round 2 with a known base,
  // arrays of their own otherwise
  int32_t* par_jface; double* par_jbary; double* par_jdir;
  const int32_t* par_face; const double* par_bary; const uint8_t* par_term; const uint8_t* par_status;
  // fallback rounds (4n slots, only flagged columns are live)
  int32_t* j3_face; double* j3_bary; double* j3_dir; double* j3_payload;
  int32_t* r3_face; double* r3_bary; double* r3_payload; uint8_t* r3_term; uint8_t* r3_status;
  int32_t* j4_face; double* j4_bary; double* j4_dir;
  int32_t* r4_face; double* r4_bary; uint8_t* r4_term; uint8_t* r4_status;
  // outputs
  double* jv; double* jp; uint8_t* degraded; double* frames;
  const double* g; double* grad_v; double* grad_p;
  // error words: [0] first degenerate-direction sample, [1] first base-not-reached sample,
  // [2] first seeds-failed sample, [3] number of samples needing the fallback rounds,
  // [4] first stalled fallback trace
  unsigned long long* err;
};
// pull-back of upstream gradients through resident GFD Jacobians (dg_gfd_pullback)
struct GfdPullback {
  MeshView mesh;
  int64_t n;
  const int32_t* face; const double* v; const int32_t* end_face;
  const double* jv; const double* jp; const double* g;
  double* grad_v; double* grad_p;
};
cudaError_t launch_gfd_pullback(const GfdPullback& b, cudaStream_t stream);
cudaError_t launch_gfd_round1_jobs(const GfdBuffers& b, cudaStream_t stream);
cudaError_t launch_gfd_round2_jobs(const GfdBuffers& b, cudaStream_t stream);
cudaError_t launch_gfd_par_jobs(const GfdBuffers& b, cudaStream_t stream);
cudaError_t launch_gfd_assemble(const GfdBuffers& b, cudaStream_t stream);
cudaError_t launch_gfd_fallback_jobs(const GfdBuffers& b, cudaStream_t stream);
cudaError_t launch_gfd_fallback_round2_jobs(const GfdBuffers& b, cudaStream_t stream);
cudaError_t launch_gfd_fallback_assemble(const GfdBuffers& b, cudaStream_t stream);

struct TransitionParams {
  MeshView mesh;
  int which;  // 0 geodesic_step, 1 transport_over_edge, 2 transport_over_vertex, 3 boundary_continue
  int64_t n;
  const int32_t* face; const double* bary; const double* v; const double* remaining;
  int hole_avoidance;
  int32_t* out_face; double* out_bary; double* out_v; double* step_length;
  uint8_t* finished; uint8_t* event; uint8_t* stall; int32_t* rc;
};
cudaError_t launch_transition(const TransitionParams& p, cudaStream_t stream);

// Builds the fat face records on the device from the indexed arrays.
cudaError_t launch_build_records(const double* xyz, const int32_t* tri, const int32_t* adj, int32_t nf,
                                 FaceRec* rec, cudaStream_t stream);

}  // namespace dg
