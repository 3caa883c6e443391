// Resident batch: the query batch of a training step (forward exp map, then EP or GFD backward)
// kept on the GPU between the two calls, so that the backward only moves the upstream gradient in
// and the gradients out. It replaces the call pair trace_batch (tracer.hpp:94) -> ep_jacobians +
// pullback_ambient loop / gfd_batched_many (gradcheck.cpp:70-89) when both run on the same
// samples. Host pointers in, host pointers out; the arithmetic is the device-mode path of
// dg_trace_batch / dg_ep_backward / dg_gfd_jacobians, so results are bit-identical to those calls.
#include <algorithm>

#include "dg_capi_common.hpp"
#include <vector>

using namespace dgapi;

struct dg_batch {
  const dg_mesh* mesh = nullptr;
  int device = 0;  // copy: dg_batch_destroy must not look at the mesh (it may already be gone)
  int64_t cap = 0, n = 0;
  bool traced = false;
  int32_t traced_max_steps = 0;   // effective step limit of the resident forward traces
  bool traced_f32 = false;
  static constexpr int kStreams = 8;
  cudaStream_t streams[kStreams] = {};
  // forward inputs and results
  int32_t *face = nullptr, *o_face = nullptr, *o_npoints = nullptr, *o_crossings = nullptr;
  double *bary = nullptr, *dir = nullptr, *o_bary = nullptr, *o_dir = nullptr, *o_traced = nullptr, *o_requested = nullptr;
  uint8_t *o_term = nullptr, *o_status = nullptr, *o_stall = nullptr;
  uint64_t* totals = nullptr;  // [kStreams] per-slice crossing counts / EP error words (device)
  uint64_t* words = nullptr;   // [kStreams] pinned host mirror (a pageable target would make the copy block)
  // streamed forward (batch_trace_streamed): upload cursor, per-chunk completion counts and error word on the device,
  // chunk flags and the cursor's values in pinned host memory
  static constexpr int kChunkShift = 14;   // smallest chunk (sizes the arrays); the request picks its own
  unsigned long long* up_word = nullptr;
  unsigned int* chunk_done = nullptr;      // [chunks + 1]: the last word is the error word
  unsigned int* chunk_flags = nullptr;     // pinned, mapped
  unsigned long long* up_table = nullptr;  // pinned: end index of every chunk
  unsigned long long* ctr = nullptr;       // device [2]: work cursor, crossing total
  cudaEvent_t ev_zero = nullptr;
  // backward
  double *g = nullptr, *grad_v = nullptr, *grad_p = nullptr, *jv = nullptr, *jp = nullptr;
  uint8_t* degraded = nullptr;
  // multi-GPU mesh: the resident request is cut into one shard per device; shard 0 lives in this batch, shard k in
  // subs[k - 1] on device k (created on demand). Empty `shards` = the whole request is resident here.
  std::vector<dgapi::Shard> shards;
  std::vector<dg_batch*> subs;
  int64_t n_total = 0;
  // dg_batch_trace_gfd: the GFD Jacobians of the resident samples are on the device already (jv, jp, degraded);
  // a whole-call GFD failure of that forward is kept for the backward call to report
  bool gfd_ready = false;
  double gfd_eps_v = 0, gfd_eps_p = 0;
  int32_t gfd_steps = 0;
  int gfd_rc = 0;
  int64_t gfd_err_index = -1;
  std::string gfd_msg;
};

namespace {

template <class T>
cudaError_t dev_alloc(T** p, size_t count) { return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)); }

cudaError_t ensure_backward(dg_batch* b) {
  if (b->g) return cudaSuccess;
  const size_t N = size_t(b->cap);
  cudaError_t e = dev_alloc(&b->g, 3 * N);
  if (e == cudaSuccess) e = dev_alloc(&b->grad_v, 3 * N);
  if (e == cudaSuccess) e = dev_alloc(&b->grad_p, 3 * N);
  return e;
}

int slices_for(int64_t n) {
  if (const char* env = getenv("DG_BATCH_SLICES")) return std::max(1, std::min(dg_batch::kStreams, atoi(env)));
  if (n >= (int64_t(1) << 18)) return 4;
  if (n >= (int64_t(1) << 16)) return 2;
  return 1;
}

// First element of slice s of the forward pipeline. The slices are weighted: a small first slice starts the
// walker early, and the last one is shorter than the one before it so that the device-to-host tail is short.
// Measured (scripts/slice_sweep.py, c2, 1 M geodesics, pinned buffers): 4 equal slices 4.89 ms, weights 1:3:3:1
// 4.77, 1:2:3:2 4.59, 1:2:4:3 **4.49**, five slices 1:3:3:3:1 4.56. DG_BATCH_SLICE_SHAPE="1,3,3,1" overrides.
int64_t trace_slice_begin(int64_t n, int s, int S) {
  static const std::vector<int> shape = [] {
    std::vector<int> w;
    if (const char* env = getenv("DG_BATCH_SLICE_SHAPE")) {
      for (const char* c = env; *c;) {
        w.push_back(std::max(1, atoi(c)));
        while (*c && *c != ',') ++c;
        if (*c == ',') ++c;
      }
    }
    return w;
  }();
  static const int kFour[4] = {1, 2, 4, 3};
  const int* w = int(shape.size()) == S ? shape.data() : (S == 4 && shape.empty() ? kFour : nullptr);
  if (!w) return n * s / S;
  int64_t total = 0, before = 0;
  for (int k = 0; k < S; ++k) { total += w[k]; if (k < s) before += w[k]; }
  return n * before / total;
}

}  // namespace

int dgapi::batch_create_one(const dg_mesh* mesh, int64_t capacity, dg_batch** out) {
  if (!out) return fail(DG_ERR_INVALID_ARGS, "dg_batch_create: null output handle");
  *out = nullptr;
  if (!mesh) return fail(DG_ERR_INVALID_ARGS, "dg_batch_create: missing mesh");
  if (capacity <= 0 || capacity > 0x7fffffffLL / 4) return fail(DG_ERR_INVALID_ARGS, "dg_batch_create: capacity out of range");
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);
  dg_batch* b = new dg_batch;
  b->mesh = mesh;
  b->device = mesh->device;
  b->cap = capacity;
  const size_t N = size_t(capacity);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  for (auto& s : b->streams) ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  ok(dev_alloc(&b->face, N)); ok(dev_alloc(&b->bary, 3 * N)); ok(dev_alloc(&b->dir, 3 * N));
  ok(dev_alloc(&b->o_face, N)); ok(dev_alloc(&b->o_bary, 3 * N)); ok(dev_alloc(&b->o_dir, 3 * N));
  ok(dev_alloc(&b->o_traced, N)); ok(dev_alloc(&b->o_requested, N));
  ok(dev_alloc(&b->o_term, N)); ok(dev_alloc(&b->o_status, N)); ok(dev_alloc(&b->o_stall, N));
  ok(dev_alloc(&b->o_npoints, N)); ok(dev_alloc(&b->o_crossings, N));
  ok(dev_alloc(&b->totals, size_t(dg_batch::kStreams)));
  ok(cudaMallocHost(reinterpret_cast<void**>(&b->words), dg_batch::kStreams * sizeof(uint64_t)));
  {
    const size_t chunks = (N >> dg_batch::kChunkShift) + 1;
    ok(dev_alloc(&b->up_word, 1)); ok(dev_alloc(&b->chunk_done, chunks + 1)); ok(dev_alloc(&b->ctr, 2));
    ok(cudaMallocHost(reinterpret_cast<void**>(&b->chunk_flags), chunks * sizeof(unsigned int)));
    ok(cudaMallocHost(reinterpret_cast<void**>(&b->up_table), chunks * sizeof(unsigned long long)));
    ok(cudaEventCreateWithFlags(&b->ev_zero, cudaEventDisableTiming));
  }
  // (the backward buffers g / grad_v / grad_p are allocated by the first backward call: a forward-only user --
  // the resident batch behind large DG_MEM_HOST dg_trace_batch calls -- never pays for them)
  if (e != cudaSuccess) {
    dg_batch_destroy(b);
    return fail_cuda(e, "dg_batch_create");
  }
  *out = b;
  return DG_OK;
}

extern "C" {

int dg_batch_create(const dg_mesh* mesh, int64_t capacity, dg_batch** out) { return batch_create_one(mesh, capacity, out); }

void dg_batch_destroy(dg_batch* b) {
  if (!b) return;
  for (dg_batch* sub : b->subs) dg_batch_destroy(sub);
  b->subs.clear();
  DeviceGuard guard(b->device);
  for (auto& s : b->streams) if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
  cudaFree(b->face); cudaFree(b->bary); cudaFree(b->dir); cudaFree(b->o_face); cudaFree(b->o_bary); cudaFree(b->o_dir);
  cudaFree(b->o_traced); cudaFree(b->o_requested); cudaFree(b->o_term); cudaFree(b->o_status); cudaFree(b->o_stall);
  cudaFree(b->o_npoints); cudaFree(b->o_crossings); cudaFree(b->totals);
  if (b->words) cudaFreeHost(b->words);
  cudaFree(b->up_word); cudaFree(b->chunk_done); cudaFree(b->ctr);
  if (b->chunk_flags) cudaFreeHost(b->chunk_flags);
  if (b->up_table) cudaFreeHost(b->up_table);
  if (b->ev_zero) cudaEventDestroy(b->ev_zero);
  cudaFree(b->g); cudaFree(b->grad_v); cudaFree(b->grad_p); cudaFree(b->jv); cudaFree(b->jp); cudaFree(b->degraded);
  delete b;
}

int64_t dg_batch_size(const dg_batch* b) { return b && b->traced ? (b->shards.empty() ? b->n : b->n_total) : 0; }

}  // extern "C"

// The streamed forward: ONE walker over the whole request while its queries arrive and its results leave.
//   copy-in stream   the queries in pieces (2^15, 2^15, 2^16, 2^17, then 2^18 each), the upload cursor advanced
//                    behind every piece;
//   walker stream    one persistent launch at full occupancy; a warp takes work only below the upload cursor, every
//                    finished trace is counted into its chunk of 32 768 and the one that completes a chunk raises
//                    the chunk's flag in mapped host memory (dg_fast_walk.cuh, kStream);
//   this thread      waits for the flags in order and queues the finished chunks' results on the copy-out stream.
// Against the sliced pipeline below (a walker per slice) nothing ramps up or drains between slices, the walker
// starts after 1.7 MB instead of a tenth of the request, and the device-to-host tail is what was still in flight
// when the queue ran dry instead of the last slice. c2, 1 M geodesics through pinned buffers: 4.06 ms against 4.48
// sliced (walker alone 3.61; the streamed walker 3.77: listing and counting the finished traces; ~0.06 ms until
// the first queries are there; ~0.2 ms of copies after the last trace). Plain order only: a schedule in start-face
// order finishes its traces all over the request. Same step code, same bits (tests/test_gpu_batch.py).
// DG_BATCH_STREAM=0 or DG_BATCH_SLICES=k selects the sliced pipeline.
static bool stream_enabled() {
  static const bool on = [] { const char* e = getenv("DG_BATCH_STREAM"); return !(e && e[0] == '0'); }();
  return on;
}
static int batch_trace_streamed(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c, dg_trace_out* out,
                                const dg::TraceParams& p_in, dg::LaunchShape shape) {
  // completion is counted per chunk of 32 768 traces (DG_BATCH_CHUNK_SHIFT); the copies are coarser where it costs
  // nothing: a copy call is ~4 us of this thread, and only the last chunks are on the critical path
  static const int sh = [] { const char* e = getenv("DG_BATCH_CHUNK_SHIFT"); return e ? std::max(int(dg_batch::kChunkShift), std::min(24, atoi(e))) : 15; }();
  const int64_t chunk = int64_t(1) << sh;
  const int K = int((n + chunk - 1) >> sh);
  cudaStream_t s_in = b->streams[0], s_walk = b->streams[1], s_out = b->streams[2];
  cudaError_t e = cudaSuccess;
  auto note = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  for (int k = 0; k < K; ++k) b->chunk_flags[k] = 0u;
  // queries [lo, hi) in, then the upload cursor to hi (its values live in pinned memory until the copy has run)
  int ups = 0;
  auto upload = [&](int64_t lo, int64_t hi) {
    const size_t L = size_t(lo), M = size_t(hi - lo);
    note(cudaMemcpyAsync(b->face + L, in->face + L, M * 4, cudaMemcpyHostToDevice, s_in));
    note(cudaMemcpyAsync(b->bary + 3 * L, in->bary + 3 * L, M * 24, cudaMemcpyHostToDevice, s_in));
    note(cudaMemcpyAsync(b->dir + 3 * L, in->dir + 3 * L, M * 24, cudaMemcpyHostToDevice, s_in));
    b->up_table[ups] = (unsigned long long)hi;
    note(cudaMemcpyAsync(b->up_word, b->up_table + ups, sizeof(unsigned long long), cudaMemcpyHostToDevice, s_in));
    ++ups;
  };
  note(cudaMemsetAsync(b->up_word, 0, sizeof(unsigned long long), s_in));
  note(cudaEventRecord(b->ev_zero, s_in));
  // Small first pieces start the walker early, the rest arrives in a few large ones (the link is ~4 x faster than
  // the walker consumes queries): 2^15, 2^15, 2^16, 2^17, then 2^18 queries each -- the resident lanes all have work
  // within ~0.1 ms. Every piece is queued BEFORE the walker is launched (~60 us of this thread): a launch that
  // blocks its thread until the kernel has ended -- any launch under a profiler or a sanitizer -- must not be
  // left waiting for queries this thread has yet to queue.
  const int64_t first = std::min<int64_t>(n, int64_t(1) << 15), piece = int64_t(1) << 18;
  upload(0, first);
  for (int64_t lo = first; lo < n;) { const int64_t len = std::min(piece, lo); upload(lo, std::min(n, lo + len)); lo += len; }
  dg::TraceParams p = p_in;
  p.queue_head = b->ctr;
  p.total_crossings = b->ctr + 1;
  p.stream_uploaded = b->up_word;
  p.stream_done = b->chunk_done;
  p.stream_error = b->chunk_done + K;
  p.stream_flags = b->chunk_flags;
  p.stream_shift = sh;
  note(cudaMemsetAsync(b->ctr, 0, 2 * sizeof(unsigned long long), s_walk));
  note(cudaMemsetAsync(b->chunk_done, 0, size_t(K + 1) * sizeof(unsigned int), s_walk));
  note(cudaStreamWaitEvent(s_walk, b->ev_zero, 0));
  note(dg::launch_trace_streamed(p, shape, s_walk));
  b->words[1] = 0;
  note(cudaMemcpyAsync(&b->words[0], b->ctr + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s_walk));
  note(cudaMemcpyAsync(&b->words[1], b->chunk_done + K, sizeof(unsigned int), cudaMemcpyDeviceToHost, s_walk));
  if (e == cudaSuccess) {
    const volatile unsigned int* flags = b->chunk_flags;
    bool walker_gone = false;
    // results out: four chunks per copy while the walker has most of its work ahead, chunk by chunk over the last 2^18
    const int fine_from = std::max(0, K - int((int64_t(1) << 18) >> sh));
    for (int k = 0; k < K;) {
      const int group = k < fine_from ? std::min(4, fine_from - k) : 1;
      for (int j = k; j < k + group; ++j)
        for (unsigned spins = 0; !flags[j] && !walker_gone; ++spins)
          if ((spins & 1023u) == 1023u && cudaStreamQuery(s_walk) != cudaErrorNotReady) walker_gone = true;   // ended (or failed) without the flag
      if (walker_gone) note(cudaStreamSynchronize(s_walk));   // (its writes are complete before anything is copied)
      const size_t L = size_t(k) << sh, M = size_t(std::min<int64_t>(chunk * group, n - int64_t(L)));
      auto back = [&](auto* host, const auto* dev, size_t stride) {
        if (host) note(cudaMemcpyAsync(host + stride * L, dev + stride * L, M * stride * sizeof(*host), cudaMemcpyDeviceToHost, s_out));
      };
      back(out->bary, b->o_bary, 3); back(out->dir, b->o_dir, 3); back(out->face, b->o_face, 1);
      back(out->traced, b->o_traced, 1); back(out->requested, b->o_requested, 1);
      back(out->term, b->o_term, 1); back(out->status, b->o_status, 1); back(out->stall, b->o_stall, 1);
      back(out->npoints, b->o_npoints, 1); back(out->crossings, b->o_crossings, 1);
      k += group;
    }
  }
  note(cudaStreamSynchronize(s_in));
  note(cudaStreamSynchronize(s_walk));
  note(cudaStreamSynchronize(s_out));
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_trace (streamed)");
  if (uint32_t(b->words[1]) != 0u) return fail(DG_ERR_CUDA, "dg_batch_trace: the walker gave up waiting for its queries");
  if (out->total_crossings) *out->total_crossings = b->words[0];
  b->traced = true;
  return DG_OK;
}

// Forward exp map of n host-resident queries. The request is cut into slices on separate streams:
// the H2D copy of slice i+1 and the D2H copy of slice i-1 overlap the walker of slice i.
int dgapi::batch_trace_one(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg, dg_trace_out* out) {
  if (!b) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace: missing batch");
  if (n < 0 || n > b->cap) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace: batch size exceeds the capacity");
  if (!in || !out) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace: null request or result block");
  if (n > 0 && (!in->face || !in->bary || !in->dir))
    return fail(DG_ERR_INVALID_ARGS, "trace_batch: starts and dirs differ in length");
  dg_trace_cfg c{};
  if (cfg) c = *cfg;
  if (in->payload || out->payload || out->transport || out->poly_offsets || c.want_transport_matrix || c.hole_avoidance)
    return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace: payload / transport matrix / hole avoidance / polylines go through dg_trace_batch");
  if (c.memory != DG_MEM_HOST || c.stream) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace: host pointers, library streams");
  DeviceGuard guard(b->mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", b->mesh->device);
  b->traced = false;
  b->gfd_ready = false;
  b->shards.clear();
  b->n = n;
  b->traced_max_steps = c.max_steps > 0 ? c.max_steps : default_max_steps(b->mesh->nf);
  b->traced_f32 = c.use_f32 != 0;
  if (n == 0) {
    if (out->total_crossings) *out->total_crossings = 0;
    b->traced = true;
    return DG_OK;
  }
  const int S = slices_for(n);
  if (S >= 4 && stream_enabled() && c.sort_by_face != DG_SORT_ON && !getenv("DG_BATCH_SLICES")) {
    // the streamed form, when this request would run in plain order on the instantiation that has one
    dg::TraceParams p{};
    b->mesh->bind(p);
    p.n = n;
    p.face = b->face; p.bary = b->bary; p.dir = b->dir;
    p.o_face = b->o_face; p.o_bary = b->o_bary; p.o_dir = b->o_dir; p.o_traced = b->o_traced; p.o_requested = b->o_requested;
    p.o_term = b->o_term; p.o_status = b->o_status; p.o_stall = b->o_stall;
    p.o_npoints = out->npoints ? b->o_npoints : nullptr;
    p.o_crossings = out->crossings ? b->o_crossings : nullptr;
    p.max_steps = b->traced_max_steps;
    p.refill_min = c.refill_min;
    p.lane_fast = c.lane == DG_LANE_FAST;
    const dg::LaunchShape shape{b->mesh->sm_count, int(c.blocks_per_sm), int(c.walker)};
    dg_trace_cfg probe = c;
    probe.memory = DG_MEM_DEVICE;
    int face_order = 0, gather = 0;
    if (dg_trace_plan(b->mesh, n, &probe, &face_order, &gather) == DG_OK && !face_order &&
        dg::trace_streamable(p, c.use_f32 != 0, false, shape))
      return batch_trace_streamed(b, n, in, c, out, p, shape);
  }
  cudaError_t e = cudaSuccess;
  auto note = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  int rc = DG_OK;
  for (int s = 0; s < S && rc == DG_OK; ++s) {
    const int64_t lo = trace_slice_begin(n, s, S), m = trace_slice_begin(n, s + 1, S) - lo;
    const size_t L = size_t(lo), M = size_t(m);
    cudaStream_t st = b->streams[s];
    note(cudaMemcpyAsync(b->face + L, in->face + L, M * 4, cudaMemcpyHostToDevice, st));
    note(cudaMemcpyAsync(b->bary + 3 * L, in->bary + 3 * L, M * 24, cudaMemcpyHostToDevice, st));
    note(cudaMemcpyAsync(b->dir + 3 * L, in->dir + 3 * L, M * 24, cudaMemcpyHostToDevice, st));
    dg_trace_in din{b->face + L, b->bary + 3 * L, b->dir + 3 * L, nullptr};
    dg_trace_out dout{};
    dout.face = b->o_face + L; dout.bary = b->o_bary + 3 * L; dout.dir = b->o_dir + 3 * L;
    dout.traced = b->o_traced + L; dout.requested = b->o_requested + L;
    dout.term = b->o_term + L; dout.status = b->o_status + L; dout.stall = b->o_stall + L;
    dout.npoints = out->npoints ? b->o_npoints + L : nullptr;
    dout.crossings = out->crossings ? b->o_crossings + L : nullptr;
    dout.total_crossings = b->totals + s;
    dg_trace_cfg dc = c;
    dc.memory = DG_MEM_DEVICE;
    dc.stream = st;
    // One resident CTA slot per SM is left to the neighbouring slice, so that its walker ramps up
    // while this one drains (measured, 1 M geodesics: 4 slices x 4 CTAs/SM 5.8 ms, x 3 CTAs/SM 5.1 ms).
    if (S > 1 && dc.blocks_per_sm == 0) dc.blocks_per_sm = 3;
    rc = trace_batch_one(b->mesh, m, &din, dc, &dout);
    if (rc != DG_OK) break;
    auto back = [&](auto* host, const auto* dev, size_t stride) {
      if (host) note(cudaMemcpyAsync(host + stride * L, dev + stride * L, M * stride * sizeof(*host), cudaMemcpyDeviceToHost, st));
    };
    back(out->face, b->o_face, 1); back(out->bary, b->o_bary, 3); back(out->dir, b->o_dir, 3);
    back(out->traced, b->o_traced, 1); back(out->requested, b->o_requested, 1);
    back(out->term, b->o_term, 1); back(out->status, b->o_status, 1); back(out->stall, b->o_stall, 1);
    back(out->npoints, b->o_npoints, 1); back(out->crossings, b->o_crossings, 1);
  }
  uint64_t totals[dg_batch::kStreams] = {};
  for (int s = 0; s < S; ++s) {
    if (rc == DG_OK && out->total_crossings)
      note(cudaMemcpyAsync(&totals[s], b->totals + s, sizeof(uint64_t), cudaMemcpyDeviceToHost, b->streams[s]));
    note(cudaStreamSynchronize(b->streams[s]));
  }
  if (rc != DG_OK) return rc;
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_trace");
  if (out->total_crossings) {
    uint64_t t = 0;
    for (int s = 0; s < S; ++s) t += totals[s];
    *out->total_crossings = t;
  }
  b->traced = true;
  return DG_OK;
}

// Forward of a GFD step (dg_trace_gfd on the resident arrays): inputs in, forward + Jacobians in one pass, forward
// results out; the Jacobians stay. One stream: the sibling launch is the step, there is nothing to pipeline against.
static int batch_trace_gfd_one(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg, double eps_v,
                               double eps_p, dg_trace_out* out) {
  if (!b) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace_gfd: missing batch");
  if (n < 0 || n > b->cap) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace_gfd: batch size exceeds the capacity");
  if (!in || !out) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace_gfd: null request or result block");
  if (n > 0 && (!in->face || !in->bary || !in->dir))
    return fail(DG_ERR_INVALID_ARGS, "trace_batch: starts and dirs differ in length");
  dg_trace_cfg c{};
  if (cfg) c = *cfg;
  if (in->payload || out->payload || out->transport || out->poly_offsets || c.want_transport_matrix || c.hole_avoidance || c.use_f32)
    return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace_gfd: the plain f64 forward map only");
  if (c.memory != DG_MEM_HOST || c.stream) return fail(DG_ERR_INVALID_ARGS, "dg_batch_trace_gfd: host pointers, library streams");
  DeviceGuard guard(b->mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", b->mesh->device);
  b->traced = false;
  b->gfd_ready = false;
  b->shards.clear();
  b->n = n;
  b->traced_max_steps = c.max_steps > 0 ? c.max_steps : default_max_steps(b->mesh->nf);
  b->traced_f32 = false;
  if (n == 0) {
    if (out->total_crossings) *out->total_crossings = 0;
    b->traced = true;
    return DG_OK;
  }
  const size_t N = size_t(n), C = size_t(b->cap);
  cudaError_t e = cudaSuccess;
  auto note = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  if (!b->jv) { note(dev_alloc(&b->jv, 4 * C)); note(dev_alloc(&b->jp, 4 * C)); note(dev_alloc(&b->degraded, 4 * C)); }
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_trace_gfd");
  cudaStream_t st = b->streams[0];
  note(cudaMemcpyAsync(b->face, in->face, N * 4, cudaMemcpyHostToDevice, st));
  note(cudaMemcpyAsync(b->bary, in->bary, N * 24, cudaMemcpyHostToDevice, st));
  note(cudaMemcpyAsync(b->dir, in->dir, N * 24, cudaMemcpyHostToDevice, st));
  dg_diff_cfg dc{};
  dc.memory = DG_MEM_DEVICE;
  dc.stream = st;
  dc.max_steps = c.max_steps;
  dc.lane = c.lane;
  dg_trace_out dout{};
  dout.face = b->o_face; dout.bary = b->o_bary; dout.dir = b->o_dir; dout.traced = b->o_traced; dout.requested = b->o_requested;
  dout.term = b->o_term; dout.status = b->o_status; dout.stall = b->o_stall;
  dout.npoints = out->npoints ? b->o_npoints : nullptr;
  dout.crossings = out->crossings ? b->o_crossings : nullptr;
  dout.total_crossings = out->total_crossings ? b->totals : nullptr;
  int64_t idx = -1;
  const int rc = gfd_jacobians_impl(b->mesh, n, b->face, b->bary, b->dir, eps_v, eps_p, nullptr, &dc, b->jv, b->jp, b->degraded,
                                    nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &idx, nullptr, &dout);
  if (rc == DG_ERR_CUDA || rc == DG_ERR_INVALID_ARGS || rc == DG_ERR_NO_DEVICE) return rc;
  b->gfd_rc = rc;   // a whole-call GFD failure: the forward results are valid, the backward call reports it
  b->gfd_err_index = idx;
  b->gfd_msg = rc != DG_OK ? last_error() : std::string();
  auto back = [&](auto* host, const auto* dev, size_t stride) {
    if (host) note(cudaMemcpyAsync(host, dev, N * stride * sizeof(*host), cudaMemcpyDeviceToHost, st));
  };
  back(out->face, b->o_face, 1); back(out->bary, b->o_bary, 3); back(out->dir, b->o_dir, 3);
  back(out->traced, b->o_traced, 1); back(out->requested, b->o_requested, 1);
  back(out->term, b->o_term, 1); back(out->status, b->o_status, 1); back(out->stall, b->o_stall, 1);
  back(out->npoints, b->o_npoints, 1); back(out->crossings, b->o_crossings, 1);
  if (out->total_crossings) note(cudaMemcpyAsync(&b->words[0], b->totals, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  note(cudaStreamSynchronize(st));
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_trace_gfd");
  if (out->total_crossings) *out->total_crossings = b->words[0];
  b->traced = true;
  b->gfd_ready = true;
  b->gfd_eps_v = eps_v; b->gfd_eps_p = eps_p; b->gfd_steps = b->traced_max_steps;
  return DG_OK;
}

// First sample of slice s of the EP backward: copy-bound both ways, so small end slices keep the lead-in (the first
// g in) and the tail (the last gradients out) short. DG_BATCH_EP_SHAPE="1,3,3,1" overrides.
static int64_t ep_slice_begin(int64_t n, int s, int S) {
  static const std::vector<int> shape = [] {
    std::vector<int> w;
    if (const char* env = getenv("DG_BATCH_EP_SHAPE"))
      for (const char* c = env; *c;) {
        w.push_back(std::max(1, atoi(c)));
        while (*c && *c != ',') ++c;
        if (*c == ',') ++c;
      }
    return w;
  }();
  static const int kFour[4] = {1, 3, 3, 1};   // 1 M samples, ms: equal 0.79, 1:3:3:1 0.73, 1:4:4:1 0.73, 1:2:4:2 0.79
  const int* w = int(shape.size()) == S ? shape.data() : (S == 4 && shape.empty() ? kFour : nullptr);
  if (!w) return n * s / S;
  int64_t total = 0, before = 0;
  for (int k = 0; k < S; ++k) { total += w[k]; if (k < s) before += w[k]; }
  return n * before / total;
}

// EP backward (diff.cpp:44-66, 328-354) on the resident samples: g in, grad_v (and grad_p) out.
static int batch_ep_backward_one(dg_batch* b, const double* g, double* grad_v, double* grad_p, int64_t* err_index) {
  if (err_index) *err_index = -1;
  if (!b || !b->traced) return fail(DG_ERR_INVALID_ARGS, "dg_batch_ep_backward: no traced batch is resident");
  const int64_t n = b->n;
  if (n == 0) return DG_OK;
  if (!g || !grad_v) return fail(DG_ERR_INVALID_ARGS, "dg_ep_backward: null argument");
  DeviceGuard guard(b->mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", b->mesh->device);
  const int S = slices_for(n);
  cudaError_t e = ensure_backward(b);
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_ep_backward");
  auto note = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  // per slice: g in, fused kernel, gradients out -- nothing waits on the host until every slice is queued
  // (totals[] doubles as the per-slice error words)
  uint64_t* words = b->words;
  for (int s = 0; s < S; ++s) {
    const size_t L = size_t(ep_slice_begin(n, s, S)), M = size_t(ep_slice_begin(n, s + 1, S)) - L;
    cudaStream_t st = b->streams[s];
    unsigned long long* word = reinterpret_cast<unsigned long long*>(b->totals + s);
    note(cudaMemcpyAsync(b->g + 3 * L, g + 3 * L, M * 24, cudaMemcpyHostToDevice, st));
    note(ep_backward_enqueue(b->mesh, int64_t(M), b->face + L, b->dir + 3 * L, b->o_face + L, b->o_dir + 3 * L,
                             b->g + 3 * L, b->grad_v + 3 * L, grad_p ? b->grad_p + 3 * L : nullptr, word, st));
    note(cudaMemcpyAsync(grad_v + 3 * L, b->grad_v + 3 * L, M * 24, cudaMemcpyDeviceToHost, st));
    if (grad_p) note(cudaMemcpyAsync(grad_p + 3 * L, b->grad_p + 3 * L, M * 24, cudaMemcpyDeviceToHost, st));
    note(cudaMemcpyAsync(&words[s], word, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  }
  for (int s = 0; s < S; ++s) note(cudaStreamSynchronize(b->streams[s]));
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_ep_backward");
  for (int s = 0; s < S; ++s) {  // the first failing sample in request order
    int64_t idx = -1;
    const int rc = ep_error_to_rc(words[s], "dg_batch_ep_backward", &idx);
    if (rc != DG_OK) {
      if (err_index) *err_index = idx + ep_slice_begin(n, s, S);
      return rc;
    }
  }
  return DG_OK;
}

// GFD backward (diff.cpp:273-326) on the resident samples.
static int batch_gfd_one(dg_batch* b, double eps_v, double eps_p, const double* g, int32_t max_steps, double* jv, double* jp,
                         uint8_t* degraded, double* grad_v, double* grad_p, int64_t* err_index) {
  if (err_index) *err_index = -1;
  if (!b || !b->traced) return fail(DG_ERR_INVALID_ARGS, "dg_batch_gfd: no traced batch is resident");
  const int64_t n = b->n;
  if (n == 0) return DG_OK;
  DeviceGuard guard(b->mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", b->mesh->device);
  const size_t N = size_t(n), C = size_t(b->cap);
  cudaError_t e = ensure_backward(b);
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_gfd");
  auto note = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  cudaStream_t st = b->streams[0];
  const int32_t want_steps = max_steps > 0 ? max_steps : default_max_steps(b->mesh->nf);
  if (b->gfd_ready && b->gfd_eps_v == eps_v && b->gfd_eps_p == eps_p && b->gfd_steps == want_steps) {
    // the forward of this step was dg_batch_trace_gfd: the Jacobians are resident, the backward is the pull-back
    if (b->gfd_rc != DG_OK) {
      if (err_index) *err_index = b->gfd_err_index;
      last_error() = b->gfd_msg;
      return b->gfd_rc;
    }
    // the Jacobians leave on a stream of their own while g arrives and the pull-back runs (the two copy directions
    // do not share an engine)
    cudaStream_t sj = b->streams[1];
    if (jv) note(cudaMemcpyAsync(jv, b->jv, N * 32, cudaMemcpyDeviceToHost, sj));
    if (jp) note(cudaMemcpyAsync(jp, b->jp, N * 32, cudaMemcpyDeviceToHost, sj));
    if (degraded) note(cudaMemcpyAsync(degraded, b->degraded, N * 4, cudaMemcpyDeviceToHost, sj));
    if (g) {
      note(cudaMemcpyAsync(b->g, g, N * 24, cudaMemcpyHostToDevice, st));
      dg::GfdPullback pb{};
      pb.mesh = b->mesh->view();
      pb.n = n;
      pb.face = b->face; pb.v = b->dir; pb.end_face = b->o_face; pb.jv = b->jv; pb.jp = b->jp; pb.g = b->g;
      pb.grad_v = grad_v ? b->grad_v : nullptr; pb.grad_p = grad_p ? b->grad_p : nullptr;
      note(dg::launch_gfd_pullback(pb, st));
      if (grad_v) note(cudaMemcpyAsync(grad_v, b->grad_v, N * 24, cudaMemcpyDeviceToHost, st));
      if (grad_p) note(cudaMemcpyAsync(grad_p, b->grad_p, N * 24, cudaMemcpyDeviceToHost, st));
    }
    note(cudaStreamSynchronize(st));
    note(cudaStreamSynchronize(sj));
    if (e != cudaSuccess) return fail_cuda(e, "dg_batch_gfd");
    return DG_OK;
  }
  if (!b->jv) { note(dev_alloc(&b->jv, 4 * C)); note(dev_alloc(&b->jp, 4 * C)); note(dev_alloc(&b->degraded, 4 * C)); }
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_gfd");
  if (g) note(cudaMemcpyAsync(b->g, g, N * 24, cudaMemcpyHostToDevice, st));
  dg_diff_cfg dc{};
  dc.memory = DG_MEM_DEVICE;
  dc.stream = st;
  dc.max_steps = max_steps;
  const bool pull = g != nullptr;
  // GFD's base trace of a sample IS its forward trace (diff.cpp:288-294: (p, v), no payload): when the
  // resident results were traced in f64 under the same step limit they are taken over, bit for bit,
  // and only the four perturbed traces per sample run
  const int32_t gfd_steps = max_steps > 0 ? max_steps : default_max_steps(b->mesh->nf);
  const GfdKnownBase kb{b->o_face, b->o_bary, b->o_dir, b->o_term, b->o_status};
  const bool reuse = !b->traced_f32 && b->traced_max_steps == gfd_steps && !getenv("DG_BATCH_GFD_RETRACE");
  int rc = gfd_jacobians_impl(b->mesh, n, b->face, b->bary, b->dir, eps_v, eps_p, pull ? b->g : nullptr, &dc, b->jv, b->jp,
                              b->degraded, nullptr, pull && grad_v ? b->grad_v : nullptr,
                              pull && grad_p ? b->grad_p : nullptr, nullptr, nullptr, nullptr, err_index, reuse ? &kb : nullptr);
  if (rc != DG_OK) return rc;
  if (jv) note(cudaMemcpyAsync(jv, b->jv, N * 32, cudaMemcpyDeviceToHost, st));
  if (jp) note(cudaMemcpyAsync(jp, b->jp, N * 32, cudaMemcpyDeviceToHost, st));
  if (degraded) note(cudaMemcpyAsync(degraded, b->degraded, N * 4, cudaMemcpyDeviceToHost, st));
  if (pull && grad_v) note(cudaMemcpyAsync(grad_v, b->grad_v, N * 24, cudaMemcpyDeviceToHost, st));
  if (pull && grad_p) note(cudaMemcpyAsync(grad_p, b->grad_p, N * 24, cudaMemcpyDeviceToHost, st));
  note(cudaStreamSynchronize(st));
  if (e != cudaSuccess) return fail_cuda(e, "dg_batch_gfd");
  return DG_OK;
}

// ---- dispatchers: a multi-GPU mesh fans the resident request out over its devices -------------------------------

static dg_batch* shard_batch(dg_batch* b, int k) { return k == 0 ? b : b->subs[size_t(k) - 1]; }

extern "C" {

}  // extern "C"

// the forward of a resident batch over the devices of a multi-GPU mesh; run_one runs a shard on its device's batch
template <class One>
static int batch_trace_dispatch(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg, dg_trace_out* out,
                                One run_one) {
  if (!b || !in || !out || n > b->cap || !fan_out(b->mesh, n) || !in->dir || (cfg && cfg->memory != DG_MEM_HOST))
    return run_one(b, n, in, cfg, out);
  const std::vector<Shard> shards = cut_shards(b->mesh, n, in->dir);
  const int S = int(shards.size());
  b->subs.resize(size_t(S) - 1, nullptr);
  for (int k = 1; k < S; ++k) {   // the other devices' resident batches, grown on demand
    dg_batch*& sub = b->subs[size_t(k) - 1];
    if (sub && sub->cap >= shards[size_t(k)].n) continue;
    if (sub) dg_batch_destroy(sub);
    sub = nullptr;
    const int64_t cap = std::max<int64_t>(1, shards[size_t(k)].n + shards[size_t(k)].n / 8);
    if (int rc = batch_create_one(shards[size_t(k)].mesh, cap, &sub)) return rc;
  }
  std::vector<uint64_t> totals(size_t(S), 0);
  const size_t one = 1;
  int rc = run_shards(shards, [&](const Shard& s, int k) {
    const size_t L = size_t(s.lo);
    auto at = [&](auto* p, size_t stride) { return p ? p + stride * L : p; };
    dg_trace_in sin{in->face + L, in->bary + 3 * L, in->dir + 3 * L, nullptr};
    dg_trace_out so = *out;
    so.face = at(out->face, one); so.bary = at(out->bary, 3); so.dir = at(out->dir, 3);
    so.traced = at(out->traced, one); so.requested = at(out->requested, one);
    so.term = at(out->term, one); so.status = at(out->status, one); so.stall = at(out->stall, one);
    so.npoints = at(out->npoints, one); so.crossings = at(out->crossings, one);
    so.total_crossings = out->total_crossings ? &totals[size_t(k)] : nullptr;
    return run_one(shard_batch(b, k), s.n, &sin, cfg, &so);
  });
  if (rc != DG_OK) { b->traced = false; return rc; }
  if (out->total_crossings) {
    uint64_t t = 0;
    for (uint64_t v : totals) t += v;
    *out->total_crossings = t;
  }
  b->shards = shards;
  b->n_total = n;
  b->traced = true;
  return DG_OK;
}

extern "C" {

int dg_batch_trace(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg, dg_trace_out* out) {
  return batch_trace_dispatch(b, n, in, cfg, out, [](dg_batch* sb, int64_t m, const dg_trace_in* i, const dg_trace_cfg* c,
                                                     dg_trace_out* o) { return batch_trace_one(sb, m, i, c, o); });
}

int dg_batch_trace_gfd(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg, double eps_v, double eps_p,
                       dg_trace_out* out) {
  return batch_trace_dispatch(b, n, in, cfg, out, [=](dg_batch* sb, int64_t m, const dg_trace_in* i, const dg_trace_cfg* c,
                                                      dg_trace_out* o) { return batch_trace_gfd_one(sb, m, i, c, eps_v, eps_p, o); });
}

int dg_batch_ep_backward(dg_batch* b, const double* g, double* grad_v, double* grad_p, int64_t* err_index) {
  if (!b || b->shards.empty() || !b->traced) return batch_ep_backward_one(b, g, grad_v, grad_p, err_index);
  if (err_index) *err_index = -1;
  if (!g || !grad_v) return fail(DG_ERR_INVALID_ARGS, "dg_ep_backward: null argument");
  std::vector<int64_t> idx(b->shards.size(), -1);
  int failed = -1;
  int rc = run_shards(b->shards, [&](const Shard& s, int k) {
    const size_t L = size_t(s.lo);
    return batch_ep_backward_one(shard_batch(b, k), g + 3 * L, grad_v + 3 * L, grad_p ? grad_p + 3 * L : nullptr, &idx[size_t(k)]);
  }, &failed);
  if (rc != DG_OK && err_index && failed >= 0 && idx[size_t(failed)] >= 0) *err_index = idx[size_t(failed)] + b->shards[size_t(failed)].lo;
  return rc;
}

int dg_batch_gfd(dg_batch* b, double eps_v, double eps_p, const double* g, int32_t max_steps, double* jv, double* jp,
                 uint8_t* degraded, double* grad_v, double* grad_p, int64_t* err_index) {
  if (!b || b->shards.empty() || !b->traced)
    return batch_gfd_one(b, eps_v, eps_p, g, max_steps, jv, jp, degraded, grad_v, grad_p, err_index);
  if (err_index) *err_index = -1;
  std::vector<int64_t> idx(b->shards.size(), -1);
  std::vector<int> rcs(b->shards.size(), DG_OK);
  std::vector<std::string> msgs(b->shards.size());
  run_shards(b->shards, [&](const Shard& s, int k) {
    const size_t L = size_t(s.lo);
    auto at = [&](auto* p, size_t stride) { return p ? p + stride * L : p; };
    rcs[size_t(k)] = batch_gfd_one(shard_batch(b, k), eps_v, eps_p, at(g, 3), max_steps, at(jv, 4), at(jp, 4), at(degraded, 4),
                                   at(grad_v, 3), at(grad_p, 3), &idx[size_t(k)]);
    if (rcs[size_t(k)] != DG_OK) msgs[size_t(k)] = last_error();
    return DG_OK;
  });
  // whole-call failures in the reference's order (diff.cpp:273-326): the frames of every sample are built before
  // any trace runs, so a degenerate direction anywhere wins over a failed base trace; then request order
  int pick = -1;
  for (int k = 0; k < int(rcs.size()); ++k)
    if (rcs[size_t(k)] != DG_OK && (pick < 0 || (rcs[size_t(k)] == DG_ERR_DEGENERATE_DIRECTION && rcs[size_t(pick)] != DG_ERR_DEGENERATE_DIRECTION)))
      pick = k;
  if (pick < 0) return DG_OK;
  last_error() = msgs[size_t(pick)];
  if (err_index && idx[size_t(pick)] >= 0) *err_index = idx[size_t(pick)] + b->shards[size_t(pick)].lo;
  return rcs[size_t(pick)];
}

}  // extern "C"
