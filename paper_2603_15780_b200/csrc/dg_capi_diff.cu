// C-ABI entry points of the differentials and the single-transition operations.
#include "dg_capi_common.hpp"
#include <cstdlib>

using namespace dgapi;

namespace {

constexpr unsigned long long kNoError = ~0ull;

int check_common(const dg_mesh* mesh, int64_t n, const char* who) {
  if (!mesh) return fail(DG_ERR_INVALID_ARGS, "%s: missing mesh", who);
  if (n < 0 || n > 0x7fffffffLL / 4) return fail(DG_ERR_INVALID_ARGS, "%s: batch size out of range", who);
  return DG_OK;
}

// Runs one batch of trace jobs that already live on the device (GFD rounds).
// The forward result record the base traces of a fused forward + GFD call write (they are the jobs [from, n) of
// round 2): what dg_trace_batch reports beyond end face / barycentrics / direction / termination / status.
struct AuxOut {
  int64_t from = 0;
  double* traced = nullptr; double* requested = nullptr; uint8_t* stall = nullptr;
  int32_t* npoints = nullptr; int32_t* crossings = nullptr;
};

cudaError_t run_jobs(const dg_mesh* mesh, int64_t n, const int32_t* jf, const double* jb, const double* jd,
                     const double* jp, int32_t* rf, double* rb, double* rd, double* rp, uint8_t* rt, uint8_t* rs,
                     int max_steps, unsigned long long* total, cudaStream_t stream, unsigned long long* cursor,
                     int siblings = 0, int64_t sibling_stride = 0, const AuxOut* aux = nullptr, bool lane_fast = false,
                     const int32_t* sample_order = nullptr) {
  if (n <= 0) return cudaSuccess;
  dg::TraceParams p{};
  mesh->bind(p);
  p.n = n;
  p.face = jf; p.bary = jb; p.dir = jd; p.payload = jp;
  p.o_face = rf; p.o_bary = rb; p.o_dir = rd; p.o_payload = rp; p.o_term = rt; p.o_status = rs;
  p.max_steps = max_steps;
  p.refill_min = 0;  // the walker's own default
  p.siblings = siblings; p.sibling_stride = sibling_stride;
  p.perm = siblings > 1 ? sample_order : nullptr;   // with a sibling schedule: the order of the GROUPS (samples)
  p.lane_fast = lane_fast;   // (payload-carrying launches run the exact lane whatever this says)
  if (aux) {
    p.aux_from = aux->from;
    p.o_traced = aux->traced; p.o_requested = aux->requested; p.o_stall = aux->stall;
    p.o_npoints = aux->npoints; p.o_crossings = aux->crossings;
  }
  p.queue_head = cursor;   // zeroed by the caller (one word per launch of the call, from its own staging)
  p.total_crossings = total;
  return dg::launch_trace(p, false, jp != nullptr, dg::LaunchShape{mesh->sm_count, 0}, stream);
}

// DG_GFD_SIBLINGS=0 runs round 2 in plain order (the schedule is a hint: results do not depend on it)
int gfd_siblings() {
  static const int k = [] {
    const char* e = std::getenv("DG_GFD_SIBLINGS");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return k;
}

}  // namespace

extern "C" {

int dg_transition(const dg_mesh* mesh, int which, int64_t n, const int32_t* face, const double* bary,
                  const double* v, const double* remaining, int hole_avoidance, int32_t* out_face,
                  double* out_bary, double* out_v, double* step_length, uint8_t* finished, uint8_t* event,
                  uint8_t* stall, int32_t* rc) {
  if (int e = check_common(mesh, n, "dg_transition")) return e;
  if (which < 0 || which > 3) return fail(DG_ERR_INVALID_ARGS, "dg_transition: unknown operation %d", which);
  if (n == 0) return DG_OK;
  if (!face || !bary || !v || !out_face || !out_bary || !out_v || !rc || (which == 0 && !remaining))
    return fail(DG_ERR_INVALID_ARGS, "dg_transition: null argument");
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);
  cudaStream_t stream = mesh->stream;
  Stage st(stream, false);
  const size_t N = size_t(n);
  dg::TransitionParams p{};
  p.mesh = mesh->view();
  p.which = which;
  p.n = n;
  p.face = st.in(face, N); p.bary = st.in(bary, 3 * N); p.v = st.in(v, 3 * N);
  p.remaining = st.in(remaining, N);
  p.hole_avoidance = hole_avoidance;
  p.out_face = st.out(out_face, N); p.out_bary = st.out(out_bary, 3 * N); p.out_v = st.out(out_v, 3 * N);
  p.step_length = st.out(step_length, N); p.finished = st.out(finished, N); p.event = st.out(event, N);
  p.stall = st.out(stall, N); p.rc = st.out(rc, N);
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_transition staging");
  st.note(dg::launch_transition(p, stream));
  cudaError_t e = st.finish();
  if (e != cudaSuccess) return fail_cuda(e, "dg_transition");
  return DG_OK;
}

static int ep_common(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v,
                     const int32_t* end_face, const double* end_dir, const double* g, const dg_diff_cfg* cfg,
                     double* rot, double* frames, double* grad_v, double* grad_p, int64_t* err_index,
                     const char* who) {
  if (err_index) *err_index = -1;
  if (int e = check_common(mesh, n, who)) return e;
  if (n == 0) return DG_OK;
  if (!face || !v || !end_face || !end_dir) return fail(DG_ERR_INVALID_ARGS, "%s: null argument", who);
  dg_diff_cfg c{};
  if (cfg) c = *cfg;
  const bool device_mode = c.memory == DG_MEM_DEVICE;
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);
  cudaStream_t stream = (device_mode || c.stream) ? static_cast<cudaStream_t>(c.stream) : mesh->stream;
  Stage st(stream, device_mode);
  const size_t N = size_t(n);
  dg::EpParams p{};
  p.mesh = mesh->view();
  p.n = n;
  p.face = st.in(face, N); p.v = st.in(v, 3 * N);
  p.end_face = st.in(end_face, N); p.end_dir = st.in(end_dir, 3 * N);
  p.g = st.in(g, 3 * N);
  p.rot = st.out(rot, 9 * N); p.frames = st.out(frames, size_t(DG_FRAME_DOUBLES) * N);
  p.grad_v = st.out(grad_v, 3 * N); p.grad_p = st.out(grad_p, 3 * N);
  unsigned long long* err = st.scratch<unsigned long long>(1);
  if (st.error() != cudaSuccess || !err) return fail_cuda(st.error(), "ep staging");
  p.first_error = err;
  st.note(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), stream));
  st.note(dg::launch_ep(p, stream));
  unsigned long long h_err = kNoError;
  st.note(cudaMemcpyAsync(&h_err, err, sizeof h_err, cudaMemcpyDeviceToHost, stream));
  st.note(cudaStreamSynchronize(stream));  // the return code depends on the error word
  cudaError_t e = st.finish();
  if (e != cudaSuccess) return fail_cuda(e, who);
  return dgapi::ep_error_to_rc(h_err, who, err_index);
}

// A multi-GPU mesh: the samples are cut into one shard per device (host mode: equal expected work; device mode:
// equal counts, the caller's arrays on the primary device reach the other devices through peer copies).
static int ep_dispatch(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v,
                       const int32_t* end_face, const double* end_dir, const double* g, const dg_diff_cfg* cfg,
                       double* rot, double* frames, double* grad_v, double* grad_p, int64_t* err_index,
                       const char* who) {
  if (!mesh || !fan_out(mesh, n) || !face || !v || !end_face || !end_dir)
    return ep_common(mesh, n, face, v, end_face, end_dir, g, cfg, rot, frames, grad_v, grad_p, err_index, who);
  if (err_index) *err_index = -1;
  dg_diff_cfg c{};
  if (cfg) c = *cfg;
  const bool dev = c.memory == DG_MEM_DEVICE;
  const std::vector<Shard> shards = cut_shards(mesh, n, dev ? nullptr : v);
  cudaEvent_t ready = nullptr;
  if (dev) {
    DeviceGuard guard(mesh->device);
    DG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    DG_CUDA(cudaEventRecord(ready, static_cast<cudaStream_t>(c.stream)));
  }
  std::vector<int64_t> idx(shards.size(), -1);
  int failed = -1;
  const int rc = run_shards(shards, [&](const Shard& s, int k) {
    const size_t L = size_t(s.lo), M = size_t(s.n);
    auto at = [&](auto* p, size_t stride) { return p ? p + stride * L : p; };
    dg_diff_cfg sc = c;
    if (s.mesh == mesh || !dev) {
      if (s.mesh != mesh) sc.stream = nullptr;
      return ep_common(s.mesh, s.n, at(face, 1), at(v, 3), at(end_face, 1), at(end_dir, 3), at(g, 3), &sc, at(rot, 9),
                       at(frames, DG_FRAME_DOUBLES), at(grad_v, 3), at(grad_p, 3), &idx[size_t(k)], who);
    }
    DeviceGuard work(s.mesh->device);
    cudaStream_t ws = s.mesh->stream;
    PeerStage ps(mesh->device, s.mesh->device, ws);
    ps.note(cudaStreamWaitEvent(ws, ready, 0));
    sc.stream = ws;
    int r = ep_common(s.mesh, s.n, ps.in(at(face, 1), M), ps.in(at(v, 3), 3 * M), ps.in(at(end_face, 1), M),
                      ps.in(at(end_dir, 3), 3 * M), ps.in(at(g, 3), 3 * M), &sc, ps.out(at(rot, 9), 9 * M),
                      ps.out(at(frames, DG_FRAME_DOUBLES), size_t(DG_FRAME_DOUBLES) * M), ps.out(at(grad_v, 3), 3 * M),
                      ps.out(at(grad_p, 3), 3 * M), &idx[size_t(k)], who);
    ps.flush();
    ps.note(cudaStreamSynchronize(ws));   // these entry points return with the results in place (host-synchronous)
    if (r == DG_OK && ps.error() != cudaSuccess) r = fail_cuda(ps.error(), who);
    return r;
  }, &failed);
  if (ready) cudaEventDestroy(ready);
  if (rc != DG_OK && err_index && failed >= 0 && idx[size_t(failed)] >= 0) *err_index = idx[size_t(failed)] + shards[size_t(failed)].lo;
  return rc;
}

int dg_ep_jacobians(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v,
                    const int32_t* end_face, const double* end_bary, const double* end_dir,
                    const dg_diff_cfg* cfg, double* rot, double* frames, int64_t* err_index) {
  (void)bary; (void)end_bary;  // origins of the frames; they do not enter the arithmetic (diff.cpp:44-66)
  return ep_dispatch(mesh, n, face, v, end_face, end_dir, nullptr, cfg, rot, frames, nullptr, nullptr, err_index,
                   "dg_ep_jacobians");
}

int dg_ep_backward(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v, const int32_t* end_face,
                   const double* end_dir, const double* g, const dg_diff_cfg* cfg, double* grad_v, double* grad_p,
                   int64_t* err_index) {
  if (n > 0 && (!g || !grad_v)) return fail(DG_ERR_INVALID_ARGS, "dg_ep_backward: null argument");
  return ep_dispatch(mesh, n, face, v, end_face, end_dir, g, cfg, nullptr, nullptr, grad_v, grad_p, err_index,
                     "dg_ep_backward");
}

// GFD on a multi-GPU mesh: all seven jobs of a sample stay on the sample's device (round 2 depends only on that
// sample's round-1 results, diff.cpp:296-309), so the shards never exchange anything.
static int gfd_dispatch(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v,
                        double eps_v, double eps_p, const double* g, const dg_diff_cfg* cfg, double* jv, double* jp,
                        uint8_t* degraded, double* frames, double* grad_v, double* grad_p, int32_t* base_face,
                        double* base_bary, double* base_dir, int64_t* err_index, const GfdKnownBase* kb,
                        const dg_trace_out* fwd = nullptr) {
  if (!mesh || !fan_out(mesh, n) || !face || !bary || !v)
    return dgapi::gfd_jacobians_impl(mesh, n, face, bary, v, eps_v, eps_p, g, cfg, jv, jp, degraded, frames, grad_v, grad_p,
                                     base_face, base_bary, base_dir, err_index, kb, fwd);
  if (err_index) *err_index = -1;
  dg_diff_cfg c{};
  if (cfg) c = *cfg;
  const bool dev = c.memory == DG_MEM_DEVICE;
  const std::vector<Shard> shards = cut_shards(mesh, n, dev ? nullptr : v);
  cudaEvent_t ready = nullptr;
  if (dev) {
    DeviceGuard guard(mesh->device);
    DG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    DG_CUDA(cudaEventRecord(ready, static_cast<cudaStream_t>(c.stream)));
  }
  std::vector<int64_t> idx(shards.size(), -1);
  std::vector<int> rcs(shards.size(), DG_OK);
  std::vector<std::string> msgs(shards.size());
  std::vector<uint64_t> totals(shards.size(), 0);   // host mode: per-shard forward totals (fused forward)
  unsigned long long* dev_totals = nullptr;         // device mode: the same on the primary device
  if (fwd && fwd->total_crossings && dev) {
    DeviceGuard guard(mesh->device);
    DG_CUDA(cudaMalloc(reinterpret_cast<void**>(&dev_totals), shards.size() * sizeof(unsigned long long)));
    DG_CUDA(cudaMemsetAsync(dev_totals, 0, shards.size() * sizeof(unsigned long long), static_cast<cudaStream_t>(c.stream)));
  }
  run_shards(shards, [&](const Shard& s, int k) {
    const size_t L = size_t(s.lo), M = size_t(s.n);
    auto at = [&](auto* p, size_t stride) { return p ? p + stride * L : p; };
    dg_diff_cfg sc = c;
    int r;
    dg_trace_out sf{};
    if (fwd) {
      sf.face = at(fwd->face, 1); sf.bary = at(fwd->bary, 3); sf.dir = at(fwd->dir, 3); sf.traced = at(fwd->traced, 1);
      sf.requested = at(fwd->requested, 1); sf.term = at(fwd->term, 1); sf.status = at(fwd->status, 1);
      sf.stall = at(fwd->stall, 1); sf.npoints = at(fwd->npoints, 1); sf.crossings = at(fwd->crossings, 1);
      if (fwd->total_crossings) sf.total_crossings = dev ? reinterpret_cast<uint64_t*>(dev_totals + k) : &totals[size_t(k)];
    }
    if (s.mesh == mesh || !dev) {
      if (s.mesh != mesh) sc.stream = nullptr;
      GfdKnownBase skb{};
      if (kb) skb = GfdKnownBase{at(kb->face, 1), at(kb->bary, 3), at(kb->dir, 3), at(kb->term, 1), at(kb->status, 1)};
      r = dgapi::gfd_jacobians_impl(s.mesh, s.n, at(face, 1), at(bary, 3), at(v, 3), eps_v, eps_p, at(g, 3), &sc, at(jv, 4),
                                    at(jp, 4), at(degraded, 4), at(frames, DG_FRAME_DOUBLES), at(grad_v, 3), at(grad_p, 3),
                                    at(base_face, 1), at(base_bary, 3), at(base_dir, 3), &idx[size_t(k)], kb ? &skb : nullptr,
                                    fwd ? &sf : nullptr);
    } else {
      DeviceGuard work(s.mesh->device);
      cudaStream_t ws = s.mesh->stream;
      PeerStage ps(mesh->device, s.mesh->device, ws);
      ps.note(cudaStreamWaitEvent(ws, ready, 0));
      sc.stream = ws;
      GfdKnownBase skb{};
      if (kb) skb = GfdKnownBase{ps.in(at(kb->face, 1), M), ps.in(at(kb->bary, 3), 3 * M), ps.in(at(kb->dir, 3), 3 * M),
                                 ps.in(at(kb->term, 1), M), ps.in(at(kb->status, 1), M)};
      dg_trace_out lf{};
      if (fwd) {
        lf.face = ps.out(sf.face, M); lf.bary = ps.out(sf.bary, 3 * M); lf.dir = ps.out(sf.dir, 3 * M);
        lf.traced = ps.out(sf.traced, M); lf.requested = ps.out(sf.requested, M); lf.term = ps.out(sf.term, M);
        lf.status = ps.out(sf.status, M); lf.stall = ps.out(sf.stall, M); lf.npoints = ps.out(sf.npoints, M);
        lf.crossings = ps.out(sf.crossings, M); lf.total_crossings = ps.out(sf.total_crossings, 1);
      }
      r = dgapi::gfd_jacobians_impl(s.mesh, s.n, ps.in(at(face, 1), M), ps.in(at(bary, 3), 3 * M), ps.in(at(v, 3), 3 * M), eps_v,
                                    eps_p, ps.in(at(g, 3), 3 * M), &sc, ps.out(at(jv, 4), 4 * M), ps.out(at(jp, 4), 4 * M),
                                    ps.out(at(degraded, 4), 4 * M), ps.out(at(frames, DG_FRAME_DOUBLES), size_t(DG_FRAME_DOUBLES) * M),
                                    ps.out(at(grad_v, 3), 3 * M), ps.out(at(grad_p, 3), 3 * M), ps.out(at(base_face, 1), M),
                                    ps.out(at(base_bary, 3), 3 * M), ps.out(at(base_dir, 3), 3 * M), &idx[size_t(k)],
                                    kb ? &skb : nullptr, fwd ? &lf : nullptr);
      ps.flush();
      ps.note(cudaStreamSynchronize(ws));
      if (r == DG_OK && ps.error() != cudaSuccess) r = fail_cuda(ps.error(), "dg_gfd_jacobians peer copies");
    }
    rcs[size_t(k)] = r;
    if (r != DG_OK) msgs[size_t(k)] = last_error();
    return DG_OK;
  });
  if (ready) cudaEventDestroy(ready);
  if (fwd && fwd->total_crossings) {   // (every shard has synchronised its stream: these entry points are host-synchronous)
    uint64_t t = 0;
    if (dev) {
      DeviceGuard guard(mesh->device);
      cudaMemcpy(totals.data(), dev_totals, totals.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost);
      for (uint64_t x : totals) t += x;
      cudaMemcpy(fwd->total_crossings, &t, sizeof t, cudaMemcpyHostToDevice);
      cudaFree(dev_totals);
    } else {
      for (uint64_t x : totals) t += x;
      *fwd->total_crossings = t;
    }
  }
  // whole-call failures in the reference's order (diff.cpp:273-326): every sample's frames are built before any
  // trace runs, so a degenerate direction anywhere wins over a failed base trace; then request order
  int pick = -1;
  for (int k = 0; k < int(rcs.size()); ++k)
    if (rcs[size_t(k)] != DG_OK && (pick < 0 || (rcs[size_t(k)] == DG_ERR_DEGENERATE_DIRECTION && rcs[size_t(pick)] != DG_ERR_DEGENERATE_DIRECTION)))
      pick = k;
  if (pick < 0) return DG_OK;
  last_error() = msgs[size_t(pick)];
  if (err_index && idx[size_t(pick)] >= 0) *err_index = idx[size_t(pick)] + shards[size_t(pick)].lo;
  return rcs[size_t(pick)];
}

int dg_gfd_jacobians(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v,
                     double eps_v, double eps_p, const double* g, const dg_diff_cfg* cfg, double* jv, double* jp,
                     uint8_t* degraded, double* frames, double* grad_v, double* grad_p, int32_t* base_face,
                     double* base_bary, double* base_dir, int64_t* err_index) {
  return gfd_dispatch(mesh, n, face, bary, v, eps_v, eps_p, g, cfg, jv, jp, degraded, frames, grad_v, grad_p,
                      base_face, base_bary, base_dir, err_index, nullptr);
}

int dg_trace_gfd(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v, double eps_v,
                 double eps_p, const dg_diff_cfg* cfg, dg_trace_out* fwd, double* jv, double* jp, uint8_t* degraded,
                 double* frames, int64_t* err_index) {
  if (!fwd) return fail(DG_ERR_INVALID_ARGS, "dg_trace_gfd: null forward result block");
  if (fwd->payload || fwd->transport || fwd->poly_offsets)
    return fail(DG_ERR_INVALID_ARGS, "dg_trace_gfd: the plain forward map only (payload / transport matrix / polylines: dg_trace_batch)");
  return gfd_dispatch(mesh, n, face, bary, v, eps_v, eps_p, nullptr, cfg, jv, jp, degraded, frames, nullptr, nullptr, nullptr,
                      nullptr, nullptr, err_index, nullptr, fwd);
}

int dg_gfd_pullback(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v, const int32_t* end_face,
                    const double* jv, const double* jp, const double* g, const dg_diff_cfg* cfg, double* grad_v,
                    double* grad_p) {
  if (int e = check_common(mesh, n, "dg_gfd_pullback")) return e;
  if (n == 0) return DG_OK;
  if (!face || !v || !end_face || !jv || !jp || !g) return fail(DG_ERR_INVALID_ARGS, "dg_gfd_pullback: null argument");
  dg_diff_cfg c{};
  if (cfg) c = *cfg;
  const bool device_mode = c.memory == DG_MEM_DEVICE;
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);
  cudaStream_t stream = (device_mode || c.stream) ? static_cast<cudaStream_t>(c.stream) : mesh->stream;
  Stage st(stream, device_mode);
  const size_t N = size_t(n);
  dg::GfdPullback b{};
  b.mesh = mesh->view();
  b.n = n;
  b.face = st.in(face, N); b.v = st.in(v, 3 * N); b.end_face = st.in(end_face, N);
  b.jv = st.in(jv, 4 * N); b.jp = st.in(jp, 4 * N); b.g = st.in(g, 3 * N);
  b.grad_v = st.out(grad_v, 3 * N); b.grad_p = st.out(grad_p, 3 * N);
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_gfd_pullback staging");
  st.note(dg::launch_gfd_pullback(b, stream));
  cudaError_t e = st.finish();   // device mode: asynchronous on the caller's stream
  if (e != cudaSuccess) return fail_cuda(e, "dg_gfd_pullback");
  return DG_OK;
}

int dg_gfd_jacobians_with_base(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v,
                               const int32_t* base_face, const double* base_bary, const double* base_dir,
                               const uint8_t* base_term, const uint8_t* base_status, double eps_v, double eps_p,
                               const double* g, const dg_diff_cfg* cfg, double* jv, double* jp, uint8_t* degraded,
                               double* frames, double* grad_v, double* grad_p, int64_t* err_index) {
  if (n > 0 && (!base_face || !base_bary || !base_dir || !base_term || !base_status))
    return fail(DG_ERR_INVALID_ARGS, "dg_gfd_jacobians_with_base: null base trace array");
  const GfdKnownBase kb{base_face, base_bary, base_dir, base_term, base_status};
  return gfd_dispatch(mesh, n, face, bary, v, eps_v, eps_p, g, cfg, jv, jp, degraded, frames, grad_v, grad_p,
                      nullptr, nullptr, nullptr, err_index, &kb);
}

}  // extern "C"

cudaError_t dgapi::ep_backward_enqueue(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v,
                                       const int32_t* end_face, const double* end_dir, const double* g, double* grad_v,
                                       double* grad_p, unsigned long long* err_word, cudaStream_t stream) {
  dg::EpParams p{};
  p.mesh = mesh->view();
  p.n = n;
  p.face = face; p.v = v; p.end_face = end_face; p.end_dir = end_dir; p.g = g;
  p.grad_v = grad_v; p.grad_p = grad_p;
  p.first_error = err_word;
  cudaError_t e = cudaMemsetAsync(err_word, 0xff, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  return dg::launch_ep(p, stream);
}

int dgapi::ep_error_to_rc(unsigned long long word, const char* who, int64_t* err_index) {
  if (word == kEpNoError) return DG_OK;
  const int64_t idx = int64_t(word >> 2);
  if (err_index) *err_index = idx;
  switch (int(word & 3ull)) {
    case 0: return fail(DG_ERR_DEGENERATE_DIRECTION, "ep_jacobians: |v| too small");
    case 1: return fail(DG_ERR_DEGENERATE_DIRECTION, "direction is normal to the face");
    default: return fail(DG_ERR_INVALID_ARGS, "%s: face index out of range at sample %lld", who, (long long)idx);
  }
}

int dgapi::gfd_jacobians_impl(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v,
                              double eps_v, double eps_p, const double* g, const dg_diff_cfg* cfg, double* jv, double* jp,
                              uint8_t* degraded, double* frames, double* grad_v, double* grad_p, int32_t* base_face,
                              double* base_bary, double* base_dir, int64_t* err_index, const GfdKnownBase* known_base,
                              const dg_trace_out* fwd) {
  if (err_index) *err_index = -1;
  if (int e = check_common(mesh, n, "dg_gfd_jacobians")) return e;
  if (fwd && known_base) return fail(DG_ERR_INVALID_ARGS, "dg_trace_gfd: the forward traces are this call's own base traces");
  if (n == 0) return DG_OK;
  if (!face || !bary || !v) return fail(DG_ERR_INVALID_ARGS, "dg_gfd_jacobians: null argument");
  dg_diff_cfg c{};
  if (cfg) c = *cfg;
  const bool device_mode = c.memory == DG_MEM_DEVICE;
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);
  cudaStream_t stream = (device_mode || c.stream) ? static_cast<cudaStream_t>(c.stream) : mesh->stream;
  const int max_steps = c.max_steps > 0 ? c.max_steps : default_max_steps(mesh->nf);
  if (c.lane > DG_LANE_FAST) return fail(DG_ERR_INVALID_ARGS, "dg_gfd_jacobians: unknown arithmetic lane %d", int(c.lane));
  // DG_LANE_FAST: the full-length traces of round 2 (re-traces, and the base traces when they ride along) run the
  // tolerance lane -- all of them, so that the differences are taken between like and like. With a known base the
  // caller's forward traces must come from the same lane.
  const bool lane_fast = c.lane == DG_LANE_FAST;
  if (lane_fast) ensure_he64(mesh);

  Stage st(stream, device_mode);
  const size_t N = size_t(n);
  dg::GfdBuffers b{};
  b.mesh = mesh->view();
  b.n = n;
  b.face = st.in(face, N); b.bary = st.in(bary, 3 * N); b.v = st.in(v, 3 * N);
  b.eps_v = eps_v; b.eps_p = eps_p;
  b.g = st.in(g, 3 * N);
  b.jv = st.out(jv, 4 * N); b.jp = st.out(jp, 4 * N);
  b.degraded = degraded ? st.out(degraded, 4 * N) : st.scratch<uint8_t>(4 * N);
  b.frames = st.out(frames, size_t(DG_FRAME_DOUBLES) * N);
  b.grad_v = st.out(grad_v, 3 * N); b.grad_p = st.out(grad_p, 3 * N);
  // round 1 (seed_u | seed_v) and round 2 (ret_u | ret_v | perp | par or base) job and result arrays
  b.j1_face = st.scratch<int32_t>(2 * N); b.j1_bary = st.scratch<double>(6 * N);
  b.j1_dir = st.scratch<double>(6 * N); b.j1_payload = st.scratch<double>(6 * N);
  b.r1_face = st.scratch<int32_t>(2 * N); b.r1_bary = st.scratch<double>(6 * N);
  b.r1_dir = nullptr; b.r1_payload = st.scratch<double>(6 * N);   // a seed's end direction is not used, its payload is
  b.r1_term = st.scratch<uint8_t>(2 * N); b.r1_status = st.scratch<uint8_t>(2 * N);
  b.j2_face = st.scratch<int32_t>(4 * N); b.j2_bary = st.scratch<double>(12 * N); b.j2_dir = st.scratch<double>(12 * N);
  b.r2_face = st.scratch<int32_t>(4 * N); b.r2_bary = st.scratch<double>(12 * N);
  b.r2_term = st.scratch<uint8_t>(4 * N); b.r2_status = st.scratch<uint8_t>(4 * N);
  double* r2_dir = nullptr;
  int32_t* par_rface = nullptr; double* par_rbary = nullptr; uint8_t* par_rterm = nullptr; uint8_t* par_rstatus = nullptr;
  if (known_base) {
    // the base traces are the caller's forward results (read in place when they are on the device);
    // the par jobs ride in slots [3n,4n) of round 2
    b.base_in_round2 = 0;
    b.base_face = st.in(known_base->face, N); b.base_bary = st.in(known_base->bary, 3 * N);
    b.base_dir = st.in(known_base->dir, 3 * N);
    b.base_term = st.in(known_base->term, N); b.base_status = st.in(known_base->status, N);
    b.par_jface = b.j2_face + 3 * N; b.par_jbary = b.j2_bary + 9 * N; b.par_jdir = b.j2_dir + 9 * N;
    b.par_face = b.r2_face + 3 * N; b.par_bary = b.r2_bary + 9 * N;
    b.par_term = b.r2_term + 3 * N; b.par_status = b.r2_status + 3 * N;
  } else {
    // the base traces are the fourth sibling of round 2; the par jobs follow in a launch of their own
    // (job arrays: the seeds' slots [0,n) of round 1, free by then)
    b.base_in_round2 = 1;
    r2_dir = st.scratch<double>(12 * N);
    b.base_face = b.r2_face + 3 * N; b.base_bary = b.r2_bary + 9 * N; b.base_dir = r2_dir ? r2_dir + 9 * N : nullptr;
    b.base_term = b.r2_term + 3 * N; b.base_status = b.r2_status + 3 * N;
    b.par_jface = b.j1_face; b.par_jbary = b.j1_bary; b.par_jdir = b.j1_dir;
    par_rface = st.scratch<int32_t>(N); par_rbary = st.scratch<double>(3 * N);
    par_rterm = st.scratch<uint8_t>(N); par_rstatus = st.scratch<uint8_t>(N);
    b.par_face = par_rface; b.par_bary = par_rbary; b.par_term = par_rterm; b.par_status = par_rstatus;
  }
  b.err = st.scratch<unsigned long long>(8);
  unsigned long long* cursors = st.scratch<unsigned long long>(8);   // one work cursor per trace launch of this call
  if (cursors) st.note(cudaMemsetAsync(cursors, 0, 8 * sizeof(unsigned long long), stream));
  // fused forward (dg_trace_gfd): the base jobs [3n, 4n) of round 2 write the rest of the forward result record
  AuxOut aux;
  unsigned long long* fwd_total = nullptr;
  if (fwd) {
    aux.from = 3 * n;
    aux.traced = st.out(fwd->traced, N); aux.requested = st.out(fwd->requested, N); aux.stall = st.out(fwd->stall, N);
    aux.npoints = st.out(fwd->npoints, N); aux.crossings = st.out(fwd->crossings, N);
    if (fwd->total_crossings) fwd_total = st.scratch<unsigned long long>(1);
  }
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_gfd_jacobians staging");
  if (fwd_total) st.note(cudaMemsetAsync(fwd_total, 0, sizeof(unsigned long long), stream));

  unsigned long long h_err[8];
  for (auto& w : h_err) w = kNoError;
  h_err[3] = 0;
  st.note(cudaMemcpyAsync(b.err, h_err, sizeof h_err, cudaMemcpyHostToDevice, stream));

  // round 1: the two payload-carrying eps-length seeds of every sample
  st.note(dg::launch_gfd_round1_jobs(b, stream));
  st.note(run_jobs(mesh, 2 * n, b.j1_face, b.j1_bary, b.j1_dir, b.j1_payload, b.r1_face, b.r1_bary, b.r1_dir,
                   b.r1_payload, b.r1_term, b.r1_status, max_steps, nullptr, stream, cursors + 0));
  // round 2: the full-length jobs of every sample as one sibling group
  st.note(dg::launch_gfd_round2_jobs(b, stream));
  const int group = c.schedule == DG_GFD_SCHEDULE_PLAIN ? 0 : gfd_siblings();
  // On meshes beyond the L2 the sibling groups are handed out in start-face order of their samples, like lone
  // traces are (dg_trace_cfg.sort_by_face): samples that start side by side walk through the same neighbourhood
  // at the same time. A schedule only -- every job writes at its own index.
  const int32_t* order = nullptr;
  if (group && (c.schedule == DG_GFD_SCHEDULE_FACE_ORDER ||
                (beyond_l2(mesh) && n >= (int64_t(1) << 15) && !std::getenv("DG_GFD_PLAIN_SAMPLE_ORDER"))))
    order = start_face_order(mesh, n, b.face, b.bary, st, stream);
  if (known_base) {
    st.note(run_jobs(mesh, 4 * n, b.j2_face, b.j2_bary, b.j2_dir, nullptr, b.r2_face, b.r2_bary, nullptr, nullptr,
                     b.r2_term, b.r2_status, max_steps, nullptr, stream, cursors + 1, group ? 3 : 0, n, nullptr, lane_fast, order));
  } else {
    st.note(run_jobs(mesh, 4 * n, b.j2_face, b.j2_bary, b.j2_dir, nullptr, b.r2_face, b.r2_bary, r2_dir, nullptr,
                     b.r2_term, b.r2_status, max_steps, fwd_total, stream, cursors + 1, group ? 4 : 0, n, fwd ? &aux : nullptr, lane_fast, order));
    st.note(dg::launch_gfd_par_jobs(b, stream));
    st.note(run_jobs(mesh, n, b.par_jface, b.par_jbary, b.par_jdir, nullptr, par_rface, par_rbary, nullptr, nullptr,
                     par_rterm, par_rstatus, max_steps, nullptr, stream, cursors + 2));
  }
  st.note(dg::launch_gfd_assemble(b, stream));
  st.note(cudaMemcpyAsync(h_err, b.err, sizeof h_err, cudaMemcpyDeviceToHost, stream));
  st.note(cudaStreamSynchronize(stream));
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_gfd_jacobians");

  const bool hard_error = h_err[0] != kNoError || h_err[1] != kNoError || h_err[2] != kNoError;
  if (!hard_error && h_err[3] != 0) {
    // one-sided fallback for the columns whose + perturbation did not reach its length
    b.j3_face = st.scratch<int32_t>(4 * N); b.j3_bary = st.scratch<double>(12 * N);
    b.j3_dir = st.scratch<double>(12 * N); b.j3_payload = st.scratch<double>(12 * N);
    b.r3_face = st.scratch<int32_t>(4 * N); b.r3_bary = st.scratch<double>(12 * N);
    b.r3_payload = st.scratch<double>(12 * N);
    b.r3_term = st.scratch<uint8_t>(4 * N); b.r3_status = st.scratch<uint8_t>(4 * N);
    b.j4_face = st.scratch<int32_t>(2 * N); b.j4_bary = st.scratch<double>(6 * N); b.j4_dir = st.scratch<double>(6 * N);
    b.r4_face = st.scratch<int32_t>(2 * N); b.r4_bary = st.scratch<double>(6 * N);
    b.r4_term = st.scratch<uint8_t>(2 * N); b.r4_status = st.scratch<uint8_t>(2 * N);
    if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_gfd_jacobians fallback staging");
    st.note(dg::launch_gfd_fallback_jobs(b, stream));
    st.note(run_jobs(mesh, 4 * n, b.j3_face, b.j3_bary, b.j3_dir, b.j3_payload, b.r3_face, b.r3_bary, nullptr,
                     b.r3_payload, b.r3_term, b.r3_status, max_steps, nullptr, stream, cursors + 3));
    st.note(dg::launch_gfd_fallback_round2_jobs(b, stream));
    st.note(run_jobs(mesh, 2 * n, b.j4_face, b.j4_bary, b.j4_dir, nullptr, b.r4_face, b.r4_bary, nullptr, nullptr,
                     b.r4_term, b.r4_status, max_steps, nullptr, stream, cursors + 4));
    st.note(dg::launch_gfd_fallback_assemble(b, stream));
    st.note(cudaMemcpyAsync(h_err, b.err, sizeof h_err, cudaMemcpyDeviceToHost, stream));
    st.note(cudaStreamSynchronize(stream));
  }
  // base end states for callers that chain the forward result
  const cudaMemcpyKind kind = device_mode ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (base_face) st.note(cudaMemcpyAsync(base_face, b.base_face, N * sizeof(int32_t), kind, stream));
  if (base_bary) st.note(cudaMemcpyAsync(base_bary, b.base_bary, 3 * N * sizeof(double), kind, stream));
  if (base_dir) st.note(cudaMemcpyAsync(base_dir, b.base_dir, 3 * N * sizeof(double), kind, stream));
  if (fwd) {   // the forward results of the samples = the end states of the base traces
    if (fwd->face) st.note(cudaMemcpyAsync(fwd->face, b.base_face, N * sizeof(int32_t), kind, stream));
    if (fwd->bary) st.note(cudaMemcpyAsync(fwd->bary, b.base_bary, 3 * N * sizeof(double), kind, stream));
    if (fwd->dir) st.note(cudaMemcpyAsync(fwd->dir, b.base_dir, 3 * N * sizeof(double), kind, stream));
    if (fwd->term) st.note(cudaMemcpyAsync(fwd->term, b.base_term, N, kind, stream));
    if (fwd->status) st.note(cudaMemcpyAsync(fwd->status, b.base_status, N, kind, stream));
    if (fwd_total) st.note(cudaMemcpyAsync(fwd->total_crossings, fwd_total, sizeof(uint64_t), kind, stream));
  }
  cudaError_t e = st.finish();
  if (e != cudaSuccess) return fail_cuda(e, "dg_gfd_jacobians");

  if (h_err[0] != kNoError) {
    if (err_index) *err_index = int64_t(h_err[0]);
    return fail(DG_ERR_DEGENERATE_DIRECTION, "tangent frame needs a nonzero in-plane direction (sample %lld)",
                (long long)h_err[0]);
  }
  if (h_err[1] != kNoError) {
    if (err_index) *err_index = int64_t(h_err[1]);
    return fail(DG_ERR_GFD, "gfd: the base trace did not reach its requested length");
  }
  if (h_err[4] != kNoError && (h_err[2] == kNoError || h_err[4] <= h_err[2])) {
    if (err_index) *err_index = int64_t(h_err[4]);
    return fail(DG_ERR_NUMERICAL_STALL, "trace: a one-sided fallback trace stalled (sample %lld)", (long long)h_err[4]);
  }
  if (h_err[2] != kNoError) {
    if (err_index) *err_index = int64_t(h_err[2]);
    return fail(DG_ERR_GFD, "gfd: start-point perturbation seeds failed to trace");
  }
  return DG_OK;
}
