// Multi-GPU fan-out behind the C-ABI: one request, the devices of the mesh's set (dg_set_devices), results at
// the request index. Replaces the reference's fork/join inside trace_batch (tracer.cpp:596-603, OpenMP
// `parallel for` over the geodesics): the mesh is replicated, the request is cut into contiguous shards of
// equal expected work, every shard runs on its device from its own host thread, and nothing is exchanged --
// there is no reduction on this path. All 7 jobs of a GFD sample stay on the sample's device.
// Results are bitwise independent of the number of devices (acceptance.cpp:173-201): a trace's arithmetic does
// not depend on the schedule, and a shard's outputs are written at its own offsets of the caller's arrays.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <thread>

#include "dg_capi_common.hpp"

namespace dgapi {

cudaMemPool_t staging_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    unsigned long long keep = ~0ull;   // a DG_MEM_HOST call must not pay for physical allocation every time
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[device] = pool;
  }
  return pools[device];
}

cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = staging_pool(dev);
  if (!pool) return cudaMallocAsync(p, bytes, stream);   // (pool creation failed: the default pool, untouched)
  return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

bool fan_out(const dg_mesh* mesh, int64_t n) {
  if (!mesh || mesh->replicas.empty()) return false;
  static const int64_t min_per_device = [] {
    const char* e = getenv("DG_MULTI_MIN");   // smallest shard worth a second device (launch + thread hand-off)
    return e ? std::max<int64_t>(1, atoll(e)) : int64_t(16384);
  }();
  return n >= min_per_device * int64_t(mesh->replicas.size() + 1);
}

std::vector<Shard> cut_shards(const dg_mesh* mesh, int64_t n, const double* host_dirs) {
  const int G = int(mesh->replicas.size()) + 1;
  auto device_mesh = [&](int g) { return g == 0 ? mesh : mesh->replicas[size_t(g) - 1]; };
  std::vector<int64_t> cut(size_t(G) + 1, n);
  cut[0] = 0;
  constexpr int64_t kStride = 64;
  const int64_t blocks = n / kStride;
  bool weighted = false;
  if (host_dirs && blocks >= G) {
    // expected work of block j = requested length of its first query (a 1-in-64 sample of the request)
    std::vector<double> acc(size_t(blocks) + 1, 0.0);
    for (int64_t j = 0; j < blocks; ++j) {
      const double* d = host_dirs + 3 * (j * kStride);
      const double w = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
      acc[size_t(j) + 1] = acc[size_t(j)] + (std::isfinite(w) && w > 0 ? w : 0.0);
    }
    const double total = acc[size_t(blocks)];
    if (total > 0 && std::isfinite(total)) {
      weighted = true;
      for (int g = 1; g < G; ++g) {
        const double target = total * double(g) / double(G);
        const int64_t j = std::lower_bound(acc.begin(), acc.end(), target) - acc.begin();
        cut[size_t(g)] = std::min<int64_t>(n, std::max<int64_t>(cut[size_t(g) - 1], j * kStride));
      }
    }
  }
  if (!weighted)
    for (int g = 1; g < G; ++g) cut[size_t(g)] = n * g / G;
  std::vector<Shard> shards;
  for (int g = 0; g < G; ++g) shards.push_back({device_mesh(g), cut[size_t(g)], cut[size_t(g) + 1] - cut[size_t(g)]});
  return shards;
}

int run_shards(const std::vector<Shard>& shards, const std::function<int(const Shard&, int)>& fn, int* first_failed) {
  const int S = int(shards.size());
  std::vector<int> rc(size_t(S), DG_OK);
  std::vector<std::string> msg(static_cast<size_t>(S));
  auto work = [&](int k) {
    rc[size_t(k)] = shards[size_t(k)].n > 0 ? fn(shards[size_t(k)], k) : DG_OK;
    if (rc[size_t(k)] != DG_OK) msg[size_t(k)] = last_error();   // last_error() is thread-local
  };
  std::vector<std::thread> threads;
  for (int k = 1; k < S; ++k) threads.emplace_back(work, k);
  work(0);
  for (auto& t : threads) t.join();
  if (first_failed) *first_failed = -1;
  for (int k = 0; k < S; ++k)
    if (rc[size_t(k)] != DG_OK) {
      last_error() = msg[size_t(k)];
      if (first_failed) *first_failed = k;
      return rc[size_t(k)];
    }
  return DG_OK;
}

}  // namespace dgapi
