// Shared plumbing of the C-ABI translation units: the mesh handle, error reporting, device
// guard and the host<->device staging helper used by DG_MEM_HOST calls.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <functional>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/dg_b200.h"
#include "dg_kernels.cuh"

struct dg_batch;
struct dg_poly_store;

struct dg_mesh {
  int device = 0;
  int sm_count = 0;
  int32_t nf = 0, nv = 0;
  dg::FaceRec* rec = nullptr;
  dg::HalfEdgeRec* he = nullptr;  // transport cache (null when off)
  alignas(64) unsigned char he_map[128] = {};  // CUtensorMap over `he` for the TMA gather (valid iff he_map_ok)
  bool he_map_ok = false;
  double* fnormal = nullptr;
  double* cangle = nullptr;   // per-corner interior angles (dg_mesh_view.cuh), built on the device at upload
  double* vangle = nullptr;
  int32_t* csr_off = nullptr;
  int32_t* csr_list = nullptr;
  uint8_t* vboundary = nullptr;
  int64_t bytes = 0;
  double mean_edge = 0.0;   // mean length of a face's edges (the length scale of the schedule's trace-length estimate)
  cudaStream_t stream = nullptr;
  // small-batch path: one pinned host block + one device block, reused across calls
  mutable std::mutex small_mu;
  mutable void* small_pin = nullptr;
  mutable void* small_dev = nullptr;
  mutable size_t small_cap = 0;
  mutable unsigned small_calls = 0;      // parity picks the work cursor of a mapped small-batch call
  mutable bool small_cursors_clean = false;
  // large plain host-mode batches run through a resident batch (dg_capi_batch.cu) owned by the mesh
  mutable std::mutex host_batch_mu;
  mutable struct dg_batch* host_batch = nullptr;
  mutable int64_t host_batch_cap = 0;
  // one-call polyline recording (dg_capi_poly.cu): pinned host arrays handed to the caller, reused across calls
  mutable std::mutex poly_mu;
  mutable dg_poly_store* poly = nullptr;
  // multi-GPU (dg_set_devices): copies of this mesh on the other devices of the set. Large requests are cut into
  // contiguous shards of equal expected work, one per device, and run concurrently (dg_capi_multi.cu); results land
  // at the request index. A replica has no replicas of its own.
  std::vector<dg_mesh*> replicas;

  // the tolerance lane's half-size crossing records (dg_mesh_view.cuh), built by the first DG_LANE_FAST request
  mutable dg::HalfEdgeRec64* he64 = nullptr;
  mutable std::mutex he64_mu;
  mutable bool he64_tried = false;
  dg::MeshView view() const {
    dg::MeshView v{rec, he, fnormal, vangle, csr_off, csr_list, vboundary, nf, nv};
    v.he64 = he64;
    v.cangle = cangle;
    return v;
  }
  // the same mesh without the transport cache (f32 lane: its transports are float arithmetic)
  dg::MeshView view_uncached() const {
    return dg::MeshView{rec, nullptr, fnormal, vangle, csr_off, csr_list, vboundary, nf, nv};
  }
  // binds the mesh (and the tensor map of its crossing records) into a trace request
  void bind(dg::TraceParams& p) const {
    p.mesh = view();
    for (int i = 0; i < 128; ++i) p.he_map[i] = he_map[i];
    p.he_map_ok = he_map_ok ? 1 : 0;
  }
};

namespace dgapi {

std::string& last_error();
int fail(int code, const char* fmt, ...);
int fail_cuda(cudaError_t e, const char* where);

#define DG_CUDA(expr)                                          \
  do {                                                         \
    cudaError_t e__ = (expr);                                  \
    if (e__ != cudaSuccess) return dgapi::fail_cuda(e__, #expr); \
  } while (0)

// The library's OWN stream-ordered memory pool of a device (staging buffers, GFD scratch, peer copies): freed
// blocks stay cached in it between calls (release threshold = keep everything), and the process-wide default pool
// of the device -- which other frameworks in the process allocate from -- is never touched. dg_trim() empties it.
cudaMemPool_t staging_pool(int device);
// cudaMallocAsync from that pool (the current device's)
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t stream);

// Makes the mesh's device current for the scope of a call.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; }
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// Stream-ordered staging of host arrays. in(): device copy of a host array; out(): device
// buffer whose contents are copied back by finish(). With device_mode the user pointers are
// passed through untouched.
class Stage {
 public:
  Stage(cudaStream_t s, bool device_mode) : stream_(s), device_mode_(device_mode) {}
  ~Stage() { release(); }

  template <class T>
  const T* in(const T* user, size_t count) {
    if (!user || device_mode_ || count == 0) return user;
    void* d = alloc(count * sizeof(T));
    if (!d) return nullptr;
    note(cudaMemcpyAsync(d, user, count * sizeof(T), cudaMemcpyHostToDevice, stream_));
    return static_cast<const T*>(d);
  }
  template <class T>
  T* out(T* user, size_t count) {
    if (!user || device_mode_ || count == 0) return user;
    void* d = alloc(count * sizeof(T));
    if (!d) return nullptr;
    backs_.push_back({d, user, count * sizeof(T)});
    return static_cast<T*>(d);
  }
  // scratch that is never copied back (both modes)
  template <class T>
  T* scratch(size_t count) { return static_cast<T*>(alloc(count * sizeof(T))); }

  // Copies the outputs back and waits (host mode); in device mode only frees scratch.
  cudaError_t finish() {
    flush_async();
    if (!device_mode_) note(cudaStreamSynchronize(stream_));
    return err_;
  }
  // Enqueues the copies back and the frees without waiting (the caller synchronises the stream).
  void flush_async() {
    for (auto& b : backs_) note(cudaMemcpyAsync(b.host, b.dev, b.bytes, cudaMemcpyDeviceToHost, stream_));
    backs_.clear();
    release();
  }
  cudaError_t error() const { return err_; }
  void note(cudaError_t e) { if (err_ == cudaSuccess && e != cudaSuccess) err_ = e; }

 private:
  struct Back { void* dev; void* host; size_t bytes; };
  void* alloc(size_t bytes) {
    void* d = nullptr;
    cudaError_t e = pool_alloc(&d, bytes ? bytes : 1, stream_);
    if (e != cudaSuccess) { note(e); return nullptr; }
    allocs_.push_back(d);
    return d;
  }
  void release() {
    for (void* d : allocs_) cudaFreeAsync(d, stream_);
    allocs_.clear();
  }
  cudaStream_t stream_;
  bool device_mode_;
  cudaError_t err_ = cudaSuccess;
  std::vector<void*> allocs_;
  std::vector<Back> backs_;
};

// Base traces GFD takes over instead of re-tracing them (n entries, same memory space as the other
// pointers of the call): the forward results of the same samples under the same step limit.
struct GfdKnownBase {
  const int32_t* face; const double* bary; const double* dir; const uint8_t* term; const uint8_t* status;
};
int gfd_jacobians_impl(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, const double* v,
                       double eps_v, double eps_p, const double* g, const dg_diff_cfg* cfg, double* jv, double* jp,
                       uint8_t* degraded, double* frames, double* grad_v, double* grad_p, int32_t* base_face,
                       double* base_bary, double* base_dir, int64_t* err_index, const GfdKnownBase* known_base,
                       const dg_trace_out* fwd = nullptr);

// EP backward on device-resident arrays without a host round trip: *err_word (device) receives
// kEpNoError or (sample index << 2 | reason), decoded by ep_error_to_rc after the stream is synced.
constexpr unsigned long long kEpNoError = ~0ull;
cudaError_t ep_backward_enqueue(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* v,
                                const int32_t* end_face, const double* end_dir, const double* g, double* grad_v,
                                double* grad_p, unsigned long long* err_word, cudaStream_t stream);
int ep_error_to_rc(unsigned long long word, const char* who, int64_t* err_index);

// ---- multi-GPU fan-out (dg_capi_multi.cu) ---------------------------------------------------------------
// The reference's fork/join site is the OpenMP loop inside trace_batch (tracer.cpp:596-603); here the same call
// fans one request out over the devices of the mesh's set. A shard is a contiguous slice [lo, lo + n) of the
// request handled by one device's copy of the mesh.
struct Shard { const dg_mesh* mesh; int64_t lo, n; };
// true when a request of n elements on this mesh is to be cut (the mesh has replicas and n is large enough)
bool fan_out(const dg_mesh* mesh, int64_t n);
// Cuts [0, n) into one shard per device. host_dirs (3n doubles in HOST memory, or null): the requested lengths
// are the weights, so shards have equal expected work (sampled every 64th query; cuts are multiples of 64);
// null: equal counts.
std::vector<Shard> cut_shards(const dg_mesh* mesh, int64_t n, const double* host_dirs);
// Runs fn(shard, index) for every shard, shard 0 on the calling thread and the others on one host thread each;
// returns DG_OK or the rc of the failing shard that comes first in request order (its message becomes the calling
// thread's dg_last_error(); *first_failed receives its index).
int run_shards(const std::vector<Shard>& shards, const std::function<int(const Shard&, int)>& fn, int* first_failed = nullptr);

// Device-mode requests on a multi-GPU mesh: the caller's arrays live on the primary device; a shard that runs on
// another device works on stream-ordered local copies, moved with peer copies (NVLink P2P when enabled) -- in()
// copies a slice over, out() hands out a local buffer that flush() copies back into the caller's array.
class PeerStage {
 public:
  PeerStage(int home_dev, int work_dev, cudaStream_t work_stream) : home_(home_dev), work_(work_dev), stream_(work_stream) {}
  ~PeerStage() { release(); }
  template <class T>
  const T* in(const T* home_ptr, size_t count) {
    if (!home_ptr || count == 0) return home_ptr;
    void* d = alloc(count * sizeof(T));
    if (d) note(cudaMemcpyPeerAsync(d, work_, home_ptr, home_, count * sizeof(T), stream_));
    return static_cast<const T*>(d);
  }
  template <class T>
  T* out(T* home_ptr, size_t count) {
    if (!home_ptr || count == 0) return home_ptr;
    void* d = alloc(count * sizeof(T));
    if (d) backs_.push_back({d, home_ptr, count * sizeof(T)});
    return static_cast<T*>(d);
  }
  void flush() {
    for (auto& b : backs_) note(cudaMemcpyPeerAsync(b.home, home_, b.local, work_, b.bytes, stream_));
    backs_.clear();
    release();
  }
  cudaError_t error() const { return err_; }
  void note(cudaError_t e) { if (err_ == cudaSuccess && e != cudaSuccess) err_ = e; }

 private:
  struct Back { void* local; void* home; size_t bytes; };
  void* alloc(size_t bytes) {
    void* d = nullptr;
    cudaError_t e = pool_alloc(&d, bytes ? bytes : 1, stream_);
    if (e != cudaSuccess) { note(e); return nullptr; }
    allocs_.push_back(d);
    return d;
  }
  void release() {
    for (void* d : allocs_) cudaFreeAsync(d, stream_);
    allocs_.clear();
  }
  int home_, work_;
  cudaStream_t stream_;
  cudaError_t err_ = cudaSuccess;
  std::vector<void*> allocs_;
  std::vector<Back> backs_;
};

// Start-face scheduling (dg_capi.cu): whether the mesh's crossing records exceed what the L2 holds, and the
// permutation that lists n device-resident queries in start-face order (null: staging failed, run in plain order).
bool beyond_l2(const dg_mesh* mesh);
// length_sum (optional, device, zeroed by the caller): receives the sum of the requested lengths |dir| of every
// 64th query -- what decides the gather of a long-trace batch (enqueue_trace).
const int32_t* start_face_order(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, Stage& st,
                                cudaStream_t stream, const double* dir = nullptr, double* length_sum = nullptr);

void poly_store_free(dg_poly_store* s);
// Builds the half-size records of the tolerance lane on first use (no-op afterwards; quietly leaves he64 null when
// the mesh has no crossing records or the memory is not there: the lane then runs over the 128-byte records).
void ensure_he64(const dg_mesh* mesh);
// one-device forms of the resident batch (the dg_batch_* entry points dispatch over the devices of a multi-GPU mesh)
int trace_batch_one(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c, dg_trace_out* out);
int batch_create_one(const dg_mesh* mesh, int64_t capacity, dg_batch** out);
int batch_trace_one(dg_batch* b, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg, dg_trace_out* out);

inline int default_max_steps(int32_t nf) {  // tracer.cpp:543-545
  return int(10.0 * std::sqrt(double(nf))) + 100;
}

}  // namespace dgapi
