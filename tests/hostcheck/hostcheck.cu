// TEST INFRASTRUCTURE ONLY -- never linked into libdigeo_b200.so and never shipped.
//
// Compiles the device state machine (csrc/dg_tracer_core.cuh, a __host__ __device__ header) for
// the HOST so that the CPU-only test tier (`pytest -m "not gpu"`, no GPU in the build
// container) can check the kernel's control flow and arithmetic against the reference before
// any GPU time is spent. It is not a fallback: the product library has no host compute path
// and fails with DG_ERR_NO_DEVICE without a GPU.
#include <cstdint>
#include <vector>

#define DG_HOSTCHECK 1
#include "../../paper_2603_15780_b200/csrc/dg_fast_walk.cuh"
#include "../../paper_2603_15780_b200/csrc/dg_tracer_core.cuh"

using namespace dg;

#define HC_API extern "C" __attribute__((visibility("default")))

namespace {

struct HostMesh {
  std::vector<FaceRec> rec;
  std::vector<HalfEdgeRec> he;  // crossing records (built on demand by the same function the upload kernel runs)
  std::vector<HalfEdgeRec64> he64;  // the tolerance lane's half-size records (ditto)
  std::vector<double> fnormal, vangle;
  std::vector<int32_t> csr_off, csr_list;
  std::vector<uint8_t> vboundary;
  int32_t nf, nv;
  MeshView view(bool cached = false) const {
    MeshView v{rec.data(), cached ? he.data() : nullptr, fnormal.data(), vangle.data(), csr_off.data(),
               csr_list.data(), vboundary.data(), nf, nv};
    v.he64 = cached && !he64.empty() ? he64.data() : nullptr;
    return v;
  }
};

// The fast walker (csrc/dg_fast_walk.cuh) driven the way trace_fast_kernel drives a lane: lean
// start-up, fast steps, the generic paths for everything the fast step hands back.
template <bool kCached, int kPay, int kLane = 0>
void run_fast(const HostMesh& hm, const TraceParams& p) {
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t q = 0; q < p.n; ++q) {
    FastLane<kCached, kPay> L{};
    bool live = fast_init<kCached, kPay>(p, q, L);
    if (!live) {
      LaneState S;
      live = lane_init<kCached, kPay>(p, q, &S);
      lane_in<kCached, kPay>(p.mesh, S, L);
    }
    while (live) {
      StepSpill sp;
      const int action = fast_step<kCached, false, kPay, kLane>(p, L, sp);
      if (action == kActFast) continue;
      if (action == kActFinish) {
        fast_finish<kCached, kPay>(p, q, L, sp);
        break;
      }
      LaneState S;
      lane_out<kCached, kPay>(L, sp, S);
      live = lane_generic<kCached, kPay>(p, q, &S, action);
      lane_in<kCached, kPay>(p.mesh, S, L);
    }
  }
}

template <class S>
void run_batch(const HostMesh& hm, int64_t n, const int32_t* face, const double* bary, const double* dir,
               const double* payload, int max_steps, int hole, int want_q, int32_t* o_face, double* o_bary,
               double* o_dir, double* o_traced, double* o_requested, uint8_t* o_term, uint8_t* o_status,
               uint8_t* o_stall, double* o_payload, double* o_q, int32_t* o_npoints, int32_t* o_crossings,
               const int64_t* poly_off, int32_t* pf, double* pb, double* ps) {
  MeshView mv = hm.view();
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t q = 0; q < n; ++q) {
    Tracer<S, true> T(mv, max_steps, hole != 0);
    V3<double> b{bary[3 * q], bary[3 * q + 1], bary[3 * q + 2]};
    V3<double> v{dir[3 * q], dir[3 * q + 1], dir[3 * q + 2]};
    V3<double> pay{0, 0, 0};
    bool has_pay = false;
    if (payload) {
      pay = {payload[3 * q], payload[3 * q + 1], payload[3 * q + 2]};
      has_pay = norm2(pay) > 0.0;
    }
    if (poly_off) { T.sink.face = pf; T.sink.bary = pb; T.sink.seg = ps; T.sink.base = poly_off[q]; }
    bool live = T.initialise(face[q], b, v, pay, has_pay, want_q != 0);
    while (live) live = T.run_step();
    V3<double> wb = T.widened_bary();
    o_face[q] = T.face;
    o_bary[3 * q] = wb.x; o_bary[3 * q + 1] = wb.y; o_bary[3 * q + 2] = wb.z;
    V3<double> d = T.target > S(0) ? cast<double>(T.dir) : V3<double>{0, 0, 0};
    o_dir[3 * q] = d.x; o_dir[3 * q + 1] = d.y; o_dir[3 * q + 2] = d.z;
    o_traced[q] = T.traced; o_requested[q] = double(T.target);
    o_term[q] = T.term; o_status[q] = T.status; o_stall[q] = T.stall_code;
    V3<double> w = T.has_payload ? cast<double>(T.payload) : V3<double>{0, 0, 0};
    o_payload[3 * q] = w.x; o_payload[3 * q + 1] = w.y; o_payload[3 * q + 2] = w.z;
    double* o = o_q + 9 * q;
    if (T.want_q) {
      o[0] = T.q0.x; o[1] = T.q1.x; o[2] = T.q2.x; o[3] = T.q0.y; o[4] = T.q1.y; o[5] = T.q2.y;
      o[6] = T.q0.z; o[7] = T.q1.z; o[8] = T.q2.z;
    } else {
      for (int k = 0; k < 9; ++k) o[k] = 0;
    }
    o_npoints[q] = T.npoints; o_crossings[q] = T.crossings;
  }
}

}  // namespace

static int g_lane_fast = 0;

HC_API void* hc_mesh_create(const double* xyz, int32_t nv, const int32_t* tri, int32_t nf, const int32_t* adj,
                            const double* fnormal, const double* vangle, const uint8_t* vboundary,
                            const int32_t* csr_off, const int32_t* csr_list) {
  HostMesh* m = new HostMesh;
  m->nf = nf; m->nv = nv;
  m->rec.resize(nf);
  for (int f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      int v = tri[3 * f + k];
      m->rec[f].v[k] = v;
      m->rec[f].adj[k] = adj[3 * f + k];
      for (int c = 0; c < 3; ++c) m->rec[f].x[3 * k + c] = xyz[3 * v + c];
    }
  m->fnormal.assign(fnormal, fnormal + 3 * size_t(nf));
  m->vangle.assign(vangle, vangle + nv);
  m->vboundary.assign(vboundary, vboundary + nv);
  m->csr_off.assign(csr_off, csr_off + nv + 1);
  m->csr_list.assign(csr_list, csr_list + 3 * size_t(nf));
  return m;
}
HC_API void hc_mesh_free(void* h) { delete static_cast<HostMesh*>(h); }

HC_API void hc_trace_batch(void* h, int64_t n, const int32_t* face, const double* bary, const double* dir,
                           const double* payload, int max_steps, int hole, int want_q, int use_f32,
                           int32_t* o_face, double* o_bary, double* o_dir, double* o_traced, double* o_requested,
                           uint8_t* o_term, uint8_t* o_status, uint8_t* o_stall, double* o_payload, double* o_q,
                           int32_t* o_npoints, int32_t* o_crossings, const int64_t* poly_off, int32_t* pf,
                           double* pb, double* ps) {
  const HostMesh& hm = *static_cast<HostMesh*>(h);
  if (use_f32)
    run_batch<float>(hm, n, face, bary, dir, payload, max_steps, hole, want_q, o_face, o_bary, o_dir, o_traced,
                     o_requested, o_term, o_status, o_stall, o_payload, o_q, o_npoints, o_crossings, poly_off, pf, pb, ps);
  else
    run_batch<double>(hm, n, face, bary, dir, payload, max_steps, hole, want_q, o_face, o_bary, o_dir, o_traced,
                      o_requested, o_term, o_status, o_stall, o_payload, o_q, o_npoints, o_crossings, poly_off, pf, pb, ps);
}

// The fast walker on the host, with (cached = 1) or without crossing records. fast_steps (may be
// null) receives how many transitions the fast step committed, to prove it is the path under test.
HC_API void hc_trace_batch_fast(void* h, int64_t n, const int32_t* face, const double* bary, const double* dir,
                                const double* payload, double* o_payload, int hole, int want_q, double* o_q,
                                int max_steps, int cached, int32_t* o_face, double* o_bary, double* o_dir,
                                double* o_traced, double* o_requested, uint8_t* o_term, uint8_t* o_status,
                                uint8_t* o_stall, int32_t* o_npoints, int32_t* o_crossings, const int64_t* poly_off,
                                int32_t* pf, double* pb, double* ps) {
  HostMesh& hm = *static_cast<HostMesh*>(h);
  if (cached && hm.he.empty()) {
    hm.he.resize(3 * size_t(hm.nf));
    const MeshView mv = hm.view(false);
    for (int f = 0; f < hm.nf; ++f)
      for (int k = 0; k < 3; ++k) hm.he[3 * size_t(f) + k] = make_halfedge_rec(mv, f, k);
  }
  if (cached && g_lane_fast == 2 && hm.he64.empty()) {
    hm.he64.resize(3 * size_t(hm.nf));
    const MeshView mv = hm.view(false);
    for (int f = 0; f < hm.nf; ++f)
      for (int k = 0; k < 3; ++k) hm.he64[3 * size_t(f) + k] = make_halfedge_rec64(mv, f, k);
  }
  TraceParams p{};
  p.snap_hi = 1.0 - 1e-10;
  p.mesh = hm.view(cached != 0);
  p.n = n;
  p.face = face; p.bary = bary; p.dir = dir;
  p.o_face = o_face; p.o_bary = o_bary; p.o_dir = o_dir; p.o_traced = o_traced; p.o_requested = o_requested;
  p.o_term = o_term; p.o_status = o_status; p.o_stall = o_stall; p.o_npoints = o_npoints; p.o_crossings = o_crossings;
  p.max_steps = max_steps;
  p.payload = payload; p.o_payload = o_payload;
  p.hole_avoidance = uint8_t(hole != 0);
  p.poly_offsets = poly_off; p.poly_face = pf; p.poly_bary = pb; p.poly_seg = ps;
  p.want_q = uint8_t(want_q != 0); p.o_transport = o_q;
  if (want_q) { if (cached) run_fast<true, 2>(hm, p); else run_fast<false, 2>(hm, p); }
  else if (payload || hole || poly_off) { if (cached) run_fast<true, 1>(hm, p); else run_fast<false, 1>(hm, p); }
  else if (cached && g_lane_fast == 2) run_fast<true, 0, 2>(hm, p);   // DG_LANE_FAST over half-size records (intrinsic fold)
  else if (cached && g_lane_fast) run_fast<true, 0, 1>(hm, p);        // DG_LANE_FAST over the 128-byte records
  else { if (cached) run_fast<true, 0>(hm, p); else run_fast<false, 0>(hm, p); }
}

// 1 / 2: plain forward requests over crossing records run the tolerance lane (dg_trace_cfg.lane = DG_LANE_FAST) over
// the 128-byte records / over the half-size records
HC_API void hc_set_lane_fast(int on) { g_lane_fast = on; }

// signed_angle_nonneg (dg_math.cuh) for n triples (a, b, axis): out[i] = 1 when it holds.
HC_API void hc_signed_angle_nonneg(int64_t n, const double* a, const double* b, const double* axis, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    const dg::V3<double> A{a[3 * i], a[3 * i + 1], a[3 * i + 2]}, B{b[3 * i], b[3 * i + 1], b[3 * i + 2]},
        N{axis[3 * i], axis[3 * i + 1], axis[3 * i + 2]};
    out[i] = dg::signed_angle_nonneg(A, B, N) ? 1 : 0;
  }
}
