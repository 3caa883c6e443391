// dg_trace_polylines: trace_batch with the reference's DEFAULT configuration, record_polyline = true
// (tracer.hpp:22: every advance / slide pushes one polyline point, tracer.cpp:84-89), in ONE call.
//
// A polyline's length is only known once the trace has run. Instead of two full calls with a host-side scan in
// between (count, then fill), the call makes one device-side pipeline of it:
//   pass 1   the walker records every trace into a slot of `cap` points of its own (cap = the step limit + 2 while
//            n x cap fits the slot budget -- always, for the batches of the reference's benchmark sweep up to 10^4 --
//            else the budget / n) and counts all its points;
//   scan     exclusive sum of the counts on the device -> poly offsets + total (the one word the host waits for);
//   compact  slots -> the contiguous per-trace polylines of GeodesicTrace::points / segment_lengths; traces that
//            needed more than `cap` points are listed;
//   pass 2   only the listed traces run again, writing straight into their compacted ranges;
//   copy     everything goes back in one stream-ordered sweep into pinned host arrays owned by the mesh.
// The arithmetic is the walker's, so every bit equals the two-call form.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "dg_capi_common.hpp"

using namespace dgapi;

namespace {

__global__ void poly_finish_scan_kernel(const int32_t* npoints, int64_t* offsets, int64_t n) {
  // offsets[0..n) hold the exclusive sum; close it with the total
  offsets[n] = offsets[n - 1] + npoints[n - 1];
}

// One warp per trace: slot -> compacted range; a trace that outgrew its slot is appended to `redo`.
__global__ void poly_compact_kernel(const int32_t* __restrict__ npoints, const int64_t* __restrict__ offsets, int64_t n,
                                    int32_t cap, const int32_t* __restrict__ s_face, const double* __restrict__ s_bary,
                                    const double* __restrict__ s_seg, int32_t* __restrict__ c_face,
                                    double* __restrict__ c_bary, double* __restrict__ c_seg, int32_t* redo,
                                    unsigned long long* redo_count) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (q >= n) return;
  const int32_t np = npoints[q];
  if (np > cap) {
    if (lane == 0) redo[atomicAdd(redo_count, 1ull)] = int32_t(q);
    return;
  }
  const int64_t src = q * int64_t(cap), dst = offsets[q];
  for (int32_t j = lane; j < np; j += 32) {
    c_face[dst + j] = s_face[src + j];
    c_seg[dst + j] = s_seg[src + j];
  }
  for (int32_t j = lane; j < 3 * np; j += 32) c_bary[3 * dst + j] = s_bary[3 * src + j];
}

// Small batches, one block: exclusive scan of the point counts (offsets[n] = total T), then slot -> packed
// polylines at `packed`, whose layout depends on T (PackedPoints): face | seg | bary. n <= kSmallMax.
constexpr int kSmallMax = 2048;
__global__ void __launch_bounds__(1024) poly_scan_compact_small_kernel(const int32_t* __restrict__ npoints, int64_t* offsets, int n,
                                                                       int32_t cap, const int32_t* __restrict__ s_face,
                                                                       const double* __restrict__ s_bary,
                                                                       const double* __restrict__ s_seg, char* packed,
                                                                       unsigned long long* overflow,
                                                                       unsigned long long* words_out) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int per = (n + 1023) / 1024, lo = min(n, t * per), hi = min(n, lo + per);
  int64_t sum = 0;
  for (int q = lo; q < hi; ++q) sum += npoints[q];
  part[t] = sum;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {   // inclusive scan of the per-thread sums
    const int64_t v = t >= d ? part[t - d] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - sum;
  for (int q = lo; q < hi; ++q) { offsets[q] = run; run += npoints[q]; }
  const int64_t T = part[1023];
  if (t == 0) offsets[n] = T;
  __syncthreads();
  const size_t seg_off = (4 * size_t(T) + 7) & ~size_t(7);
  int32_t* c_face = reinterpret_cast<int32_t*>(packed);
  double* c_seg = reinterpret_cast<double*>(packed + seg_off);
  double* c_bary = c_seg + T;
  const int warp = t >> 5, lane = t & 31;
  for (int q = warp; q < n; q += 32) {
    const int32_t np = npoints[q];
    if (np > cap) { if (lane == 0) atomicAdd(overflow, 1ull); continue; }
    const int64_t src = int64_t(q) * cap, dst = offsets[q];
    for (int32_t j = lane; j < np; j += 32) { c_face[dst + j] = s_face[src + j]; c_seg[dst + j] = s_seg[src + j]; }
    for (int32_t j = lane; j < 3 * np; j += 32) c_bary[3 * dst + j] = s_bary[3 * src + j];
  }
  if (words_out) {   // mapped call: the work counters {queue head, total crossings, overflow count} go to the host block too
    __syncthreads();
    if (t == 0) { words_out[0] = overflow[-2]; words_out[1] = overflow[-1]; words_out[2] = overflow[0]; }
  }
}

// Most points a trace can record: the start point, then one per step (advance, tracer.cpp:202,212) -- two with hole
// avoidance, where a step that reaches a boundary edge pushes its advance AND the slide that follows it
// (cross_edge -> slide_from_edge -> slide_along, tracer.cpp:371-405).
int64_t most_points(int32_t max_steps, bool hole_avoidance) { return (hole_avoidance ? 2 : 1) * int64_t(max_steps) + 2; }

size_t slot_budget() {
  const char* e = getenv("DG_POLY_SLOT_BUDGET");   // points of slot space of pass 1 (36 B each)
  return e ? size_t(std::max<long long>(1024, atoll(e))) : (size_t(8) << 20);
}

}  // namespace

struct dg_poly_store {   // what a mesh keeps between dg_trace_polylines calls
  int64_t* offsets = nullptr; size_t offsets_cap = 0;   // pinned host, large path
  char* points = nullptr; size_t points_bytes = 0;      // pinned host: the packed polylines [face | seg | bary] of T points
  uint64_t* words = nullptr;                            // pinned host [2]: total, redo count
  // small batches: one pinned block + one device block hold the whole request (no allocation, one copy each way)
  char* small_host = nullptr; char* small_dev = nullptr; size_t small_host_bytes = 0, small_dev_bytes = 0;
};

// Packed polylines of T points: face[T] (4 T bytes, padded to 8) | seg[T] | bary[3 T]. One block, one copy.
struct PackedPoints {
  size_t seg_off, bary_off, bytes;
  explicit PackedPoints(size_t T) : seg_off((4 * T + 7) & ~size_t(7)), bary_off(seg_off + 8 * T), bytes(bary_off + 24 * T) {}
};

void dgapi::poly_store_free(dg_poly_store* s) {
  if (!s) return;
  cudaFreeHost(s->offsets); cudaFreeHost(s->points); cudaFreeHost(s->words); cudaFreeHost(s->small_host);
  cudaFree(s->small_dev);
  delete s;
}

// n <= kSmallMax with slots that cover the step limit: the whole request lives in one pinned block and one device
// block the mesh keeps (inputs, results, offsets, counters), so a call is one copy in, the walker, one fused
// scan + compaction block, one copy of the results out, one copy of the packed polylines out.
static int trace_polylines_small(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c,
                                 dg_trace_out* out, dg_polylines* poly, dg_poly_store& ps, int32_t max_steps, int32_t cap) {
  const size_t N = size_t(n), slots = N * size_t(cap);
  struct Field { const void* src; void* dst; size_t bytes; size_t off; };
  auto up8 = [](size_t x) { return (x + 7) & ~size_t(7); };
  Field fin[4] = {{in->face, nullptr, 4 * N, 0}, {in->bary, nullptr, 24 * N, 0}, {in->dir, nullptr, 24 * N, 0},
                  {in->payload, nullptr, in->payload ? 24 * N : 0, 0}};
  Field fout[13] = {{nullptr, out->face, out->face ? 4 * N : 0, 0}, {nullptr, out->bary, out->bary ? 24 * N : 0, 0},
                    {nullptr, out->dir, out->dir ? 24 * N : 0, 0}, {nullptr, out->traced, out->traced ? 8 * N : 0, 0},
                    {nullptr, out->requested, out->requested ? 8 * N : 0, 0}, {nullptr, out->payload, out->payload ? 24 * N : 0, 0},
                    {nullptr, out->transport, out->transport ? 72 * N : 0, 0}, {nullptr, out->npoints, 4 * N, 0},
                    {nullptr, out->crossings, out->crossings ? 4 * N : 0, 0}, {nullptr, out->term, out->term ? N : 0, 0},
                    {nullptr, out->status, out->status ? N : 0, 0}, {nullptr, out->stall, out->stall ? N : 0, 0},
                    {nullptr, nullptr, 8 * (N + 1), 0}};   // [12] = poly offsets
  size_t in_bytes = 32;   // 4 words: queue head, total crossings, overflow count, spare
  for (auto& f : fin) { f.off = in_bytes; in_bytes += up8(f.bytes); }
  size_t io_bytes = in_bytes;
  const size_t out_begin = io_bytes;
  for (auto& f : fout) { f.off = io_bytes; io_bytes += up8(f.bytes); }
  const size_t slot_off = io_bytes, packed_off = slot_off + up8(4 * slots) + 32 * slots;
  const size_t dev_bytes = packed_off + PackedPoints(slots).bytes;
  if (ps.small_host_bytes < io_bytes) {
    cudaFreeHost(ps.small_host); ps.small_host = nullptr; ps.small_host_bytes = 0;
    DG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ps.small_host), std::max<size_t>(2 * io_bytes, size_t(1) << 16)));
    ps.small_host_bytes = std::max<size_t>(2 * io_bytes, size_t(1) << 16);
  }
  if (ps.small_dev_bytes < dev_bytes) {
    cudaFree(ps.small_dev); ps.small_dev = nullptr; ps.small_dev_bytes = 0;
    DG_CUDA(cudaMalloc(reinterpret_cast<void**>(&ps.small_dev), dev_bytes + dev_bytes / 2));
    ps.small_dev_bytes = dev_bytes + dev_bytes / 2;
  }
  char* hp = ps.small_host;
  char* dp = ps.small_dev;
  // The smallest batches skip every copy (as dg_trace_batch does up to 256 queries): the pinned blocks are mapped
  // into the device's address space, the walker reads its queries from and writes its results to the host block,
  // the scan + compaction block writes the offsets and the packed polylines straight into the host arrays; only
  // the work counters and the slots live in device memory (the second launch hands the counters to the host block).
  // One memset, two launches, one synchronisation.
  const bool mapped = n <= 256 && slots <= (size_t(1) << 18);
  if (mapped && ps.points_bytes < PackedPoints(slots).bytes) {
    cudaFreeHost(ps.points); ps.points = nullptr; ps.points_bytes = 0;
    const size_t want = std::max<size_t>(PackedPoints(slots).bytes, size_t(1) << 16);
    DG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ps.points), want));
    ps.points_bytes = want;
  }
  std::memset(hp, 0, 32);
  for (auto& f : fin) if (f.bytes) std::memcpy(hp + f.off, f.src, f.bytes);
  cudaStream_t stream = mesh->stream;
  if (mapped) DG_CUDA(cudaMemsetAsync(dp, 0, 32, stream));
  else DG_CUDA(cudaMemcpyAsync(dp, hp, in_bytes, cudaMemcpyHostToDevice, stream));
  char* io = mapped ? hp : dp;   // where the walker finds the request and leaves the results

  dg::TraceParams p{};
  mesh->bind(p);
  p.n = n;
  auto din = [&](int i) { return fin[i].bytes ? io + fin[i].off : nullptr; };
  auto dout = [&](int i) { return fout[i].bytes ? io + fout[i].off : nullptr; };
  p.face = reinterpret_cast<const int32_t*>(din(0)); p.bary = reinterpret_cast<const double*>(din(1));
  p.dir = reinterpret_cast<const double*>(din(2)); p.payload = reinterpret_cast<const double*>(din(3));
  p.o_face = reinterpret_cast<int32_t*>(dout(0)); p.o_bary = reinterpret_cast<double*>(dout(1));
  p.o_dir = reinterpret_cast<double*>(dout(2)); p.o_traced = reinterpret_cast<double*>(dout(3));
  p.o_requested = reinterpret_cast<double*>(dout(4)); p.o_payload = reinterpret_cast<double*>(dout(5));
  p.o_transport = reinterpret_cast<double*>(dout(6)); p.o_npoints = reinterpret_cast<int32_t*>(dout(7));
  p.o_crossings = reinterpret_cast<int32_t*>(dout(8)); p.o_term = reinterpret_cast<uint8_t*>(dout(9));
  p.o_status = reinterpret_cast<uint8_t*>(dout(10)); p.o_stall = reinterpret_cast<uint8_t*>(dout(11));
  int64_t* d_off = reinterpret_cast<int64_t*>(dout(12));
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(dp);
  p.queue_head = ctr;
  p.total_crossings = out->total_crossings ? ctr + 1 : nullptr;
  p.poly_cap = cap;
  p.poly_face = reinterpret_cast<int32_t*>(dp + slot_off);
  p.poly_seg = reinterpret_cast<double*>(dp + slot_off + up8(4 * slots));
  p.poly_bary = p.poly_seg + slots;
  p.max_steps = max_steps;
  p.refill_min = c.refill_min;
  p.hole_avoidance = c.hole_avoidance;
  p.want_q = c.want_transport_matrix;
  DG_CUDA(dg::launch_trace(p, c.use_f32 != 0, true, dg::LaunchShape{mesh->sm_count, int(c.blocks_per_sm), int(c.walker)}, stream));
  poly_scan_compact_small_kernel<<<1, 1024, 0, stream>>>(p.o_npoints, d_off, int(n), cap, p.poly_face, p.poly_bary, p.poly_seg,
                                                         mapped ? ps.points : dp + packed_off, ctr + 2,
                                                         mapped ? reinterpret_cast<unsigned long long*>(hp) : nullptr);
  DG_CUDA(cudaGetLastError());
  if (!mapped) DG_CUDA(cudaMemcpyAsync(hp, dp, 32, cudaMemcpyDeviceToHost, stream));
  if (!mapped) DG_CUDA(cudaMemcpyAsync(hp + out_begin, dp + out_begin, io_bytes - out_begin, cudaMemcpyDeviceToHost, stream));
  DG_CUDA(cudaStreamSynchronize(stream));
  const int64_t* h_off = reinterpret_cast<const int64_t*>(hp + fout[12].off);
  const size_t T = size_t(h_off[N]);
  uint64_t words[4];
  std::memcpy(words, hp, 32);
  if (words[2] != 0) return fail(DG_ERR_CUDA, "dg_trace_polylines: a trace recorded more points than its step limit allows");
  const PackedPoints pk(T);
  if (ps.points_bytes < pk.bytes) {
    cudaFreeHost(ps.points); ps.points = nullptr; ps.points_bytes = 0;
    const size_t want = std::max<size_t>(pk.bytes + pk.bytes / 2, size_t(1) << 16);
    DG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ps.points), want));
    ps.points_bytes = want;
  }
  if (T && !mapped) {
    DG_CUDA(cudaMemcpyAsync(ps.points, dp + packed_off, pk.bytes, cudaMemcpyDeviceToHost, stream));
    DG_CUDA(cudaStreamSynchronize(stream));
  }
  for (int i = 0; i < 12; ++i)
    if (fout[i].bytes && fout[i].dst) std::memcpy(fout[i].dst, hp + fout[i].off, fout[i].bytes);
  if (out->total_crossings) *out->total_crossings = words[1];
  poly->total = int64_t(T);
  poly->offsets = h_off;
  poly->face = reinterpret_cast<const int32_t*>(ps.points);
  poly->seg = reinterpret_cast<const double*>(ps.points + pk.seg_off);
  poly->bary = reinterpret_cast<const double*>(ps.points + pk.bary_off);
  return DG_OK;
}

extern "C" int dg_trace_polylines(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg,
                                  dg_trace_out* out, dg_polylines* poly) {
  if (!mesh) return fail(DG_ERR_INVALID_ARGS, "trace_batch: missing mesh");
  if (n < 0 || n > 0x7fffffffLL) return fail(DG_ERR_INVALID_ARGS, "trace_batch: batch size out of range");
  if (!in || !out || !poly) return fail(DG_ERR_INVALID_ARGS, "trace_batch: null request or result block");
  if (n > 0 && (!in->face || !in->bary || !in->dir))
    return fail(DG_ERR_INVALID_ARGS, "trace_batch: starts and dirs differ in length");
  dg_trace_cfg c{};
  if (cfg) c = *cfg;
  if (c.memory != DG_MEM_HOST || c.stream) return fail(DG_ERR_INVALID_ARGS, "dg_trace_polylines: host pointers, library stream");
  if (c.lane > DG_LANE_FAST) return fail(DG_ERR_INVALID_ARGS, "trace_batch: unknown arithmetic lane %d", int(c.lane));
  if (out->poly_offsets || out->poly_face || out->poly_bary || out->poly_seg)
    return fail(DG_ERR_INVALID_ARGS, "dg_trace_polylines: the polylines come back in *poly, not in out->poly_*");
  *poly = dg_polylines{};
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);

  std::lock_guard<std::mutex> lock(mesh->poly_mu);
  if (!mesh->poly) mesh->poly = new dg_poly_store;
  dg_poly_store& ps = *mesh->poly;
  auto grow_host = [&](auto** p, size_t count) {
    cudaFreeHost(*p);
    *p = nullptr;
    return cudaMallocHost(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(**p));
  };
  if (!ps.words) DG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ps.words), 2 * sizeof(uint64_t)));
  const size_t N = size_t(n);
  {
    const int32_t steps = c.max_steps > 0 ? c.max_steps : default_max_steps(mesh->nf);
    const int64_t full = most_points(steps, c.hole_avoidance != 0);
    if (n > 0 && n <= kSmallMax && full <= 0x7fffffff && N * size_t(full) <= slot_budget())
      return trace_polylines_small(mesh, n, in, c, out, poly, ps, steps, int32_t(full));
  }
  if (ps.offsets_cap < N + 1) {
    const size_t cap = std::max<size_t>(2 * (N + 1), 1024);
    ps.offsets_cap = 0;
    DG_CUDA(grow_host(&ps.offsets, cap));
    ps.offsets_cap = cap;
  }
  if (n == 0) {
    ps.offsets[0] = 0;
    if (out->total_crossings) *out->total_crossings = 0;
    poly->offsets = ps.offsets;
    return DG_OK;
  }

  cudaStream_t stream = mesh->stream;
  Stage st(stream, false);
  const int32_t max_steps = c.max_steps > 0 ? c.max_steps : default_max_steps(mesh->nf);
  const int64_t full_cap = most_points(max_steps, c.hole_avoidance != 0);
  const int32_t cap = int32_t(std::max<int64_t>(8, std::min<int64_t>(full_cap, int64_t(slot_budget() / N))));
  const size_t slots = N * size_t(cap);

  dg::TraceParams p{};
  mesh->bind(p);
  p.n = n;
  p.face = st.in(in->face, N); p.bary = st.in(in->bary, 3 * N); p.dir = st.in(in->dir, 3 * N);
  p.payload = st.in(in->payload, 3 * N);
  p.o_face = st.out(out->face, N); p.o_bary = st.out(out->bary, 3 * N); p.o_dir = st.out(out->dir, 3 * N);
  p.o_traced = st.out(out->traced, N); p.o_requested = st.out(out->requested, N);
  p.o_term = st.out(out->term, N); p.o_status = st.out(out->status, N); p.o_stall = st.out(out->stall, N);
  p.o_payload = st.out(out->payload, 3 * N); p.o_transport = st.out(out->transport, 9 * N);
  p.o_crossings = st.out(out->crossings, N);
  int32_t* d_np = out->npoints ? st.out(out->npoints, N) : st.scratch<int32_t>(N);
  p.o_npoints = d_np;
  p.poly_cap = cap;
  p.poly_face = st.scratch<int32_t>(slots); p.poly_bary = st.scratch<double>(3 * slots); p.poly_seg = st.scratch<double>(slots);
  p.max_steps = max_steps;
  p.refill_min = c.refill_min;
  p.hole_avoidance = c.hole_avoidance;
  p.want_q = c.want_transport_matrix;
  unsigned long long* ctr = st.scratch<unsigned long long>(4);   // queue head, total crossings, redo count, queue head of pass 2
  int64_t* d_off = st.scratch<int64_t>(N + 1);
  if (st.error() != cudaSuccess || !ctr || !d_off) return fail_cuda(st.error(), "dg_trace_polylines staging");
  p.queue_head = ctr;
  p.total_crossings = out->total_crossings ? ctr + 1 : nullptr;
  st.note(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), stream));
  const dg::LaunchShape shape{mesh->sm_count, int(c.blocks_per_sm), int(c.walker)};
  st.note(dg::launch_trace(p, c.use_f32 != 0, true, shape, stream));

  size_t tmp_bytes = 0;
  st.note(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_np, d_off, int(n), stream));
  void* tmp = st.scratch<char>(tmp_bytes);
  if (!tmp) return fail_cuda(st.error(), "dg_trace_polylines scan staging");
  st.note(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, d_np, d_off, int(n), stream));
  poly_finish_scan_kernel<<<1, 1, 0, stream>>>(d_np, d_off, n);
  // Slots that cover the step limit (small batches): no trace can outgrow its slot, the total is at most the slot
  // space, so the compaction is queued right behind the scan and the host waits once for {total, redo count}.
  // Otherwise the total sizes the compacted arrays first.
  const bool roomy = cap == full_cap;
  size_t T = slots;
  if (!roomy) {
    st.note(cudaMemcpyAsync(&ps.words[0], d_off + N, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    st.note(cudaStreamSynchronize(stream));
    if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_trace_polylines pass 1");
    T = size_t(ps.words[0]);
  }
  // the compacted polylines as one packed block [face | seg | bary]; laid out for the largest total this pass
  // can produce (the layout of the copy back is fixed below, once the total is on the host)
  char* packed = st.scratch<char>(PackedPoints(T).bytes);
  int32_t* c_face = reinterpret_cast<int32_t*>(packed);
  double* c_seg = packed ? reinterpret_cast<double*>(packed + PackedPoints(T).seg_off) : nullptr;
  double* c_bary = packed ? reinterpret_cast<double*>(packed + PackedPoints(T).bary_off) : nullptr;
  const PackedPoints dev_layout(T);
  int32_t* redo = st.scratch<int32_t>(N);
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_trace_polylines compaction staging");
  {
    const unsigned threads = 256;
    const unsigned blocks = unsigned((N * 32 + threads - 1) / threads);
    poly_compact_kernel<<<blocks, threads, 0, stream>>>(d_np, d_off, n, cap, p.poly_face, p.poly_bary, p.poly_seg, c_face, c_bary,
                                                        c_seg, redo, ctr + 2);
    st.note(cudaGetLastError());
  }
  st.note(cudaMemcpyAsync(&ps.words[0], d_off + N, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  st.note(cudaMemcpyAsync(&ps.words[1], ctr + 2, sizeof(uint64_t), cudaMemcpyDeviceToHost, stream));
  st.note(cudaStreamSynchronize(stream));
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_trace_polylines compaction");
  T = size_t(ps.words[0]);
  const int64_t again = int64_t(ps.words[1]);
  if (again > 0 && roomy) return fail(DG_ERR_CUDA, "dg_trace_polylines: a trace recorded more points than its step limit allows");
  if (again > 0) {   // pass 2: the traces that outgrew their slots, straight into their compacted ranges
    dg::TraceParams r = p;
    r.n = again;
    r.perm = redo;
    r.poly_cap = 0;
    r.poly_offsets = d_off;
    r.poly_face = c_face; r.poly_bary = c_bary; r.poly_seg = c_seg;
    r.queue_head = ctr + 3;
    r.total_crossings = nullptr;   // counted in pass 1
    st.note(dg::launch_trace(r, c.use_f32 != 0, true, shape, stream));
  }
  const PackedPoints host_layout(T);   // T: the real total by now
  if (ps.points_bytes < host_layout.bytes) {
    cudaFreeHost(ps.points); ps.points = nullptr; ps.points_bytes = 0;
    const size_t want = std::max<size_t>(host_layout.bytes + host_layout.bytes / 2, size_t(1) << 16);
    DG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ps.points), want));
    ps.points_bytes = want;
  }
  st.note(cudaMemcpyAsync(ps.offsets, d_off, (N + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  if (T) {   // (three ranges of the device layout, which was fixed before the total was known in the roomy case)
    st.note(cudaMemcpyAsync(ps.points, c_face, T * sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    st.note(cudaMemcpyAsync(ps.points + host_layout.seg_off, c_seg, T * sizeof(double), cudaMemcpyDeviceToHost, stream));
    st.note(cudaMemcpyAsync(ps.points + host_layout.bary_off, c_bary, 3 * T * sizeof(double), cudaMemcpyDeviceToHost, stream));
  }
  if (out->total_crossings)
    st.note(cudaMemcpyAsync(out->total_crossings, ctr + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, stream));
  cudaError_t e = st.finish();
  if (e != cudaSuccess) return fail_cuda(e, "dg_trace_polylines");
  poly->total = int64_t(T);
  poly->offsets = ps.offsets;
  poly->face = reinterpret_cast<const int32_t*>(ps.points);
  poly->seg = reinterpret_cast<const double*>(ps.points + host_layout.seg_off);
  poly->bary = reinterpret_cast<const double*>(ps.points + host_layout.bary_off);
  return DG_OK;
}
