// C-ABI entry points: devices, mesh store and forward tracing (include/dg_b200.h).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cuda.h>

#include "dg_capi_common.hpp"
#include "dg_fast_walk.cuh"
#include "dg_tracer_core.cuh"

namespace dgapi {

std::string& last_error() {
  thread_local std::string s;
  return s;
}
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}
int fail_cuda(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear the sticky-free error state
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    return fail(DG_ERR_NO_DEVICE, "no usable CUDA device (%s): there is no CPU fallback", cudaGetErrorString(e));
  return fail(DG_ERR_CUDA, "CUDA error %s at %s", cudaGetErrorString(e), where);
}

}  // namespace dgapi

using namespace dgapi;

namespace {

thread_local int g_device = 0;
// device set of meshes created afterwards (dg_set_devices); empty = the single device g_device. An ordinal may
// repeat (dg_set_device_list): two copies on one GPU exercise the whole fan-out path on a one-GPU box.
thread_local std::vector<int> g_devices;

__global__ void sum_totals_kernel(const unsigned long long* parts, int count, unsigned long long* total) {
  unsigned long long s = 0;
  for (int i = 0; i < count; ++i) s += parts[i];
  *total = s;
}

__global__ void build_records_kernel(const double* __restrict__ xyz, const int32_t* __restrict__ tri,
                                     const int32_t* __restrict__ adj, int32_t nf, dg::FaceRec* rec) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  dg::FaceRec r;
  for (int k = 0; k < 3; ++k) {
    int v = tri[3 * f + k];
    r.v[k] = v;
    r.adj[k] = adj[3 * f + k];
    r.x[3 * k + 0] = xyz[3 * size_t(v) + 0];
    r.x[3 * k + 1] = xyz[3 * size_t(v) + 1];
    r.x[3 * k + 2] = xyz[3 * size_t(v) + 2];
  }
  rec[f] = r;
}

// Transport cache: one thread per directed half-edge runs the reference's make_edge_transport
// (tracer.cpp:113-126) through the very functions the uncached walker uses, so cached and
// uncached traces are bit-identical.
__global__ void build_halfedges_kernel(const dg::MeshView m, dg::HalfEdgeRec* he) {
  using namespace dg;
  const int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (s >= 3 * int64_t(m.nf)) return;
  const int f = int(s / 3), k = int(s % 3);
  const HalfEdgeRec r = make_halfedge_rec(m, f, k);
  he[s] = r;
}

// Interior angle of every face corner, through the function the fan walk calls per fan face (dg_tracer_core.cuh).
__global__ void build_corner_angles_kernel(const dg::MeshView m, double* cangle) {
  using namespace dg;
  const int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (s >= 3 * int64_t(m.nf)) return;
  const int f = int(s / 3), k = int(s % 3);
  const Face<double> c = load_face<double>(m, f);
  const V3<double> x0 = c.pos(k);
  cangle[s] = angle_between(c.pos(k == 2 ? 0 : k + 1) - x0, c.pos(k == 0 ? 2 : k - 1) - x0);
}

__global__ void build_halfedges64_kernel(const dg::MeshView m, dg::HalfEdgeRec64* he) {
  const int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (s >= 3 * int64_t(m.nf)) return;
  he[s] = dg::make_halfedge_rec64(m, int(s / 3), int(s % 3));
}

// Tensor map of the crossing records for the TMA tile::gather4 fetch of the fast walker: a 2-D
// f64 tensor [3 nf rows][16 doubles], box = one row, 128-byte swizzle. The driver entry point is
// taken through the runtime so that the library does not link libcuda.
bool encode_record_map(const dg::HalfEdgeRec* he, size_t rows, unsigned char* out128) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap is 128 bytes");
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  CUtensorMap map;
  const cuuint64_t dims[2] = {16, cuuint64_t(rows)}, strides[1] = {sizeof(dg::HalfEdgeRec)};
  const cuuint32_t box[2] = {16, 1}, estr[2] = {1, 1};
  const CUresult r = reinterpret_cast<EncodeFn>(fn)(
      &map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<dg::HalfEdgeRec*>(he), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  memcpy(out128, &map, 128);
  return true;
}

// Scheduling key of query i and its own index: start face, plus one bit above the face bits for starts that
// snap_bary will put ON A VERTEX (tracer.cpp:148-161). Such traces begin in the vertex branch -- and, aimed along an
// edge, stay in it vertex after vertex (config 5) --, which runs through the general state machine; a warp that
// mixes them with plain edge-crossing traces executes both paths one after the other (c5, 1 M geodesics: 853 ms
// mixed, 506 ms with the two kinds in warps of their own). A schedule only: results stay at the request index.
__global__ void sort_keys_kernel(const int32_t* __restrict__ face, const double* __restrict__ bary, int64_t n, int32_t nf,
                                 int bits, int32_t* keys, int32_t* index, const double* __restrict__ dir, double* length_sum) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  if (length_sum && (i & 63) == 0) {   // requested length of every 64th query (finite ones)
    const double x = dir[3 * i], y = dir[3 * i + 1], z = dir[3 * i + 2], len = sqrt(x * x + y * y + z * z);
    if (len < 1e300) atomicAdd(length_sum, len);
  }
  const int32_t f = face[i];
  const double b0 = bary[3 * i], b1 = bary[3 * i + 1], b2 = bary[3 * i + 2];
  const double hi = 1.0 - 1e-10;
  const bool vertex = b0 >= hi || b1 >= hi || b2 >= hi;
  keys[i] = (f >= 0 && f < nf ? f : 0) | (vertex ? (int32_t(1) << bits) : 0);
  index[i] = int32_t(i);
}

}  // namespace

// dg_trace_cfg.sort_by_face resolved for a request of n queries
static bool schedules_by_face(const dg_mesh* mesh, int64_t n, const dg_trace_cfg& c, bool record) {
  const bool big_mesh = beyond_l2(mesh);
  return c.sort_by_face == DG_SORT_ON || (c.sort_by_face == DG_SORT_AUTO && big_mesh && n >= (int64_t(1) << 15) && !record);
}

// The permutation that lists n device-resident queries in start-face order (vertex starts last), in staging of
// the call; null when the staging could not be had (the request then runs in plain order).
const int32_t* dgapi::start_face_order(const dg_mesh* mesh, int64_t n, const int32_t* face, const double* bary, Stage& st,
                                       cudaStream_t stream, const double* dir, double* length_sum) {
  const size_t N = size_t(n);
  int32_t* keys_in = st.scratch<int32_t>(N);
  int32_t* keys_out = st.scratch<int32_t>(N);
  int32_t* iota = st.scratch<int32_t>(N);
  int32_t* perm = st.scratch<int32_t>(N);
  if (!keys_in || !keys_out || !iota || !perm) return nullptr;
  int bits = 1;
  while ((int64_t(1) << bits) < int64_t(mesh->nf) && bits < 30) ++bits;
  sort_keys_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(face, bary, n, mesh->nf, bits, keys_in, iota, dir,
                                                                  dir ? length_sum : nullptr);
  size_t tmp_bytes = 0;
  st.note(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys_out, iota, perm, int(n), 0, bits + 1, stream));
  void* tmp = st.scratch<char>(tmp_bytes);
  if (!tmp) return nullptr;
  st.note(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, iota, perm, int(n), 0, bits + 1, stream));
  return perm;
}
bool dgapi::beyond_l2(const dg_mesh* mesh) {
  return mesh->he && size_t(3) * size_t(mesh->nf) * sizeof(dg::HalfEdgeRec) > (size_t(96) << 20);
}

void dgapi::ensure_he64(const dg_mesh* m) {
  if (!m || !m->he) return;
  std::lock_guard<std::mutex> lock(m->he64_mu);
  if (m->he64_tried) return;
  m->he64_tried = true;
  const size_t bytes = size_t(3) * size_t(m->nf) * sizeof(dg::HalfEdgeRec64);
  if (bytes > (size_t(8) << 30)) return;
  DeviceGuard guard(m->device);
  dg::HalfEdgeRec64* p = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&p), bytes) != cudaSuccess) { cudaGetLastError(); return; }
  build_halfedges64_kernel<<<unsigned((size_t(3) * size_t(m->nf) + 127) / 128), 128, 0, m->stream>>>(m->view_uncached(), p);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(m->stream) != cudaSuccess) { cudaGetLastError(); cudaFree(p); return; }
  m->he64 = p;
}

namespace dg {
cudaError_t launch_build_records(const double* xyz, const int32_t* tri, const int32_t* adj, int32_t nf,
                                 FaceRec* rec, cudaStream_t stream) {
  if (nf <= 0) return cudaSuccess;
  build_records_kernel<<<(nf + 255) / 256, 256, 0, stream>>>(xyz, tri, adj, nf, rec);
  return cudaGetLastError();
}
}  // namespace dg

extern "C" {

const char* dg_last_error(void) { return last_error().c_str(); }
const char* dg_version(void) { return "digeo-b200 0.1 (sm_100a)"; }

int dg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int dg_set_device(int ordinal) {
  int n = dg_device_count();
  if (n == 0) return fail(DG_ERR_NO_DEVICE, "no usable CUDA device: there is no CPU fallback");
  if (ordinal < 0 || ordinal >= n) return fail(DG_ERR_INVALID_ARGS, "dg_set_device: ordinal %d out of range [0,%d)", ordinal, n);
  g_device = ordinal;
  g_devices.clear();
  return DG_OK;
}

int dg_set_device_list(const int32_t* ordinals, int32_t count) {
  const int n = dg_device_count();
  if (n == 0) return fail(DG_ERR_NO_DEVICE, "no usable CUDA device: there is no CPU fallback");
  if (!ordinals || count < 1 || count > 64) return fail(DG_ERR_INVALID_ARGS, "dg_set_device_list: 1..64 ordinals expected");
  for (int i = 0; i < count; ++i)
    if (ordinals[i] < 0 || ordinals[i] >= n)
      return fail(DG_ERR_INVALID_ARGS, "dg_set_device_list: ordinal %d out of range [0,%d)", int(ordinals[i]), n);
  g_device = ordinals[0];
  g_devices.assign(ordinals, ordinals + count);
  if (count == 1) g_devices.clear();
  return DG_OK;
}

int dg_set_devices(uint64_t mask) {
  int32_t list[64];
  int count = 0;
  for (int d = 0; d < 64; ++d)
    if (mask >> d & 1) list[count++] = d;
  if (count == 0) return fail(DG_ERR_INVALID_ARGS, "dg_set_devices: empty device mask");
  return dg_set_device_list(list, count);
}

int dg_mesh_device_count(const dg_mesh* m) { return m ? int(m->replicas.size()) + 1 : 0; }

int dg_device_sm_count(void) {
  if (dg_device_count() == 0) return 0;
  int sm = 0;
  if (cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, g_device) != cudaSuccess) return 0;
  return sm;
}

// ------------------------------------------------------------------------------------ mesh

// Host restatement of Mesh::build (proj/src/mesh.cpp:34-130). The reference matches edges
// through a std::map keyed by sorted vertex pairs; here the 3F half-edges are sorted by the
// same key, which visits the edges in the map's order (so the mean edge length is summed in
// the same order) in O(F log F) without node allocations.
int dg_mesh_derive(const double* xyz, int32_t nv, const int32_t* tri, int32_t nf, int32_t* adj,
                   double* fnormal, double* farea, double* vangle, double* varea, uint8_t* vboundary,
                   int32_t* csr_off, int32_t* csr_list, double* mean_edge, double* total_area,
                   int64_t* err_index) {
  if (err_index) *err_index = -1;
  if (nv < 0 || nf < 0 || (nv > 0 && !xyz) || (nf > 0 && !tri))
    return fail(DG_ERR_INVALID_ARGS, "dg_mesh_derive: null or negative-size input");
  using V = dg::V3<double>;
  auto P = [&](int v) { return V{xyz[3 * size_t(v)], xyz[3 * size_t(v) + 1], xyz[3 * size_t(v) + 2]}; };

  for (int f = 0; f < nf; ++f) {  // mesh.cpp:41-49
    const int32_t* c = tri + 3 * size_t(f);
    for (int k = 0; k < 3; ++k)
      if (c[k] < 0 || c[k] >= nv) {
        if (err_index) *err_index = f;
        return fail(DG_ERR_PARSE, "face %d references vertex out of range", f);
      }
    if (c[0] == c[1] || c[1] == c[2] || c[0] == c[2]) {
      if (err_index) *err_index = f;
      return fail(DG_ERR_DEGENERATE_FACE, "face %d has repeated vertices", f);
    }
  }

  std::vector<double> area_store;
  if (!farea && varea) { area_store.resize(nf); farea = area_store.data(); }
  double area_sum = 0;
  for (int f = 0; f < nf; ++f) {  // mesh.cpp:55-68
    const int32_t* c = tri + 3 * size_t(f);
    V e1 = P(c[1]) - P(c[0]);
    V e2 = P(c[2]) - P(c[0]);
    V n = dg::cross(e1, e2);
    double a2 = dg::norm(n);
    double longest2 = std::max({dg::norm2(e1), dg::norm2(e2), dg::norm2(P(c[2]) - P(c[1]))});
    if (a2 <= 1e-14 * longest2 || longest2 == 0.0) {
      if (err_index) *err_index = f;
      return fail(DG_ERR_DEGENERATE_FACE, "face %d has zero area", f);
    }
    if (fnormal) {
      V u = n / a2;
      fnormal[3 * size_t(f)] = u.x; fnormal[3 * size_t(f) + 1] = u.y; fnormal[3 * size_t(f) + 2] = u.z;
    }
    double a = 0.5 * a2;
    if (farea) farea[f] = a;
    area_sum += a;
  }
  if (total_area) *total_area = area_sum;

  // adjacency, mesh.cpp:71-90
  struct HalfEdge { uint64_t key; int32_t slot; };  // slot = 3 f + k (scan order of the reference)
  std::vector<HalfEdge> he(size_t(3) * nf);
  for (int f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      int a = tri[3 * size_t(f) + (k + 1) % 3], b = tri[3 * size_t(f) + (k + 2) % 3];
      uint64_t lo = uint64_t(std::min(a, b)), hi = uint64_t(std::max(a, b));
      he[3 * size_t(f) + k] = {(lo << 32) | hi, int32_t(3 * f + k)};
    }
  std::sort(he.begin(), he.end(), [](const HalfEdge& x, const HalfEdge& y) {
    return x.key != y.key ? x.key < y.key : x.slot < y.slot;
  });
  if (adj) std::fill(adj, adj + size_t(3) * nf, -1);
  if (vboundary) std::fill(vboundary, vboundary + nv, uint8_t(0));
  int64_t bad_slot = -1;
  uint64_t bad_key = 0;
  double edge_len_sum = 0;
  int64_t edge_count = 0;
  for (size_t i = 0; i < he.size();) {
    size_t j = i;
    while (j < he.size() && he[j].key == he[i].key) ++j;
    const int a = int(he[i].key >> 32), b = int(he[i].key & 0xffffffffu);
    if (j - i >= 3) {  // the reference throws when it meets the third incidence in scan order
      if (bad_slot < 0 || he[i + 2].slot < bad_slot) { bad_slot = he[i + 2].slot; bad_key = he[i].key; }
    } else if (j - i == 2) {
      if (adj) { adj[he[i].slot] = he[i + 1].slot / 3; adj[he[i + 1].slot] = he[i].slot / 3; }
    } else if (vboundary) {
      vboundary[a] = 1; vboundary[b] = 1;
    }
    edge_len_sum += dg::norm(P(a) - P(b));  // mesh.cpp:96, map order
    ++edge_count;
    i = j;
  }
  if (bad_slot >= 0) {
    if (err_index) *err_index = int64_t(bad_key >> 32);
    return fail(DG_ERR_NON_MANIFOLD, "edge (%d,%d) incident to 3+ faces", int(bad_key >> 32), int(bad_key & 0xffffffffu));
  }
  if (mean_edge) *mean_edge = edge_count ? edge_len_sum / double(edge_count) : 0.0;

  // total angles and vertex areas, mesh.cpp:106-115
  if (vangle) std::fill(vangle, vangle + nv, 0.0);
  if (varea) std::fill(varea, varea + nv, 0.0);
  if (vangle || varea)
    for (int f = 0; f < nf; ++f) {
      const int32_t* c = tri + 3 * size_t(f);
      for (int k = 0; k < 3; ++k) {
        if (vangle) {
          V apex = P(c[k]);
          vangle[c[k]] += dg::angle_between(P(c[(k + 1) % 3]) - apex, P(c[(k + 2) % 3]) - apex);
        }
        if (varea) varea[c[k]] += farea[f] / 3.0;
      }
    }

  // vertex -> faces CSR, mesh.cpp:118-127
  if (csr_off) {
    std::fill(csr_off, csr_off + nv + 1, 0);
    for (int f = 0; f < nf; ++f)
      for (int k = 0; k < 3; ++k) csr_off[tri[3 * size_t(f) + k] + 1]++;
    for (int v = 0; v < nv; ++v) csr_off[v + 1] += csr_off[v];
    if (csr_list) {
      std::vector<int32_t> cursor(csr_off, csr_off + nv);
      for (int f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) csr_list[cursor[tri[3 * size_t(f) + k]]++] = f;
    }
  }
  return DG_OK;
}

int dg_mesh_create(const double* xyz, int32_t nv, const int32_t* tri, int32_t nf, const int32_t* adj,
                   const double* fnormal, const double* vangle, const uint8_t* vboundary,
                   const int32_t* csr_off, const int32_t* csr_list, dg_mesh** out) {
  return dg_mesh_create_ex(xyz, nv, tri, nf, adj, fnormal, vangle, vboundary, csr_off, csr_list,
                           DG_MESH_TRANSPORT_AUTO, out);
}

int dg_mesh_create_ex(const double* xyz, int32_t nv, const int32_t* tri, int32_t nf, const int32_t* adj,
                      const double* fnormal, const double* vangle, const uint8_t* vboundary,
                      const int32_t* csr_off, const int32_t* csr_list, uint32_t flags, dg_mesh** out) {
  if (!out) return fail(DG_ERR_INVALID_ARGS, "dg_mesh_create: null output handle");
  *out = nullptr;
  if (nv <= 0 || nf <= 0 || !xyz || !tri || !adj || !fnormal || !vangle || !vboundary || !csr_off || !csr_list)
    return fail(DG_ERR_INVALID_ARGS, "dg_mesh_create: every mesh array is required (use dg_mesh_derive)");
  if (dg_device_count() == 0) return fail(DG_ERR_NO_DEVICE, "no usable CUDA device: there is no CPU fallback");
  DeviceGuard guard(g_device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", g_device);

  dg_mesh* m = new dg_mesh;
  m->device = g_device;
  m->nf = nf;
  m->nv = nv;
  {   // mean length of a face's edges: the length scale of the schedule's estimate of a trace's crossings
    double sum = 0.0;
    for (int32_t f = 0; f < nf; ++f)
      for (int k = 0; k < 3; ++k) {
        const double* a = xyz + 3 * size_t(tri[3 * size_t(f) + size_t(k)]);
        const double* b = xyz + 3 * size_t(tri[3 * size_t(f) + size_t((k + 1) % 3)]);
        sum += std::sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]) + (a[2] - b[2]) * (a[2] - b[2]));
      }
    m->mean_edge = sum / (3.0 * double(nf));
  }
  auto cleanup = [&](int rc) { dg_mesh_destroy(m); return rc; };
  cudaError_t e;
#define DG_TRY(expr) if ((e = (expr)) != cudaSuccess) return cleanup(fail_cuda(e, #expr))
  DG_TRY(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, g_device));
  DG_TRY(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
  const size_t F = size_t(nf), Vn = size_t(nv);
  DG_TRY(cudaMalloc(&m->rec, F * sizeof(dg::FaceRec)));
  DG_TRY(cudaMalloc(&m->fnormal, 3 * F * sizeof(double)));
  DG_TRY(cudaMalloc(&m->cangle, 3 * F * sizeof(double)));
  DG_TRY(cudaMalloc(&m->vangle, Vn * sizeof(double)));
  DG_TRY(cudaMalloc(&m->csr_off, (Vn + 1) * sizeof(int32_t)));
  DG_TRY(cudaMalloc(&m->csr_list, 3 * F * sizeof(int32_t)));
  DG_TRY(cudaMalloc(&m->vboundary, Vn));
  m->bytes = int64_t(F * sizeof(dg::FaceRec) + 3 * F * 8 + 3 * F * 8 + Vn * 8 + (Vn + 1) * 4 + 3 * F * 4 + Vn);
  // Transport cache policy (384 B per face on top of the 96 B face record).
  bool cache = (flags & 3u) == DG_MESH_TRANSPORT_ON;
  if ((flags & 3u) == DG_MESH_TRANSPORT_AUTO) {
    const char* env = getenv("DG_TRANSPORT_CACHE");
    if (env && (!strcmp(env, "on") || !strcmp(env, "1"))) {
      cache = true;
    } else if (env && (!strcmp(env, "off") || !strcmp(env, "0"))) {
      cache = false;
    } else {
      // Measured (profiles/tuning_r1.md, scripts/sweep_cache_policy.py): the walker over crossing
      // records beats the one over face records at every mesh size once the records are gathered
      // one request per record beyond 250 MB (cooperative loads or TMA; gather_mode, dg_trace_kernel.cu),
      // so AUTO only guards capacity.
      cache = 3 * F * sizeof(dg::HalfEdgeRec) <= (size_t(16) << 30);
    }
  }
  if (cache) {
    DG_TRY(cudaMalloc(&m->he, 3 * F * sizeof(dg::HalfEdgeRec)));
    m->bytes += int64_t(3 * F * sizeof(dg::HalfEdgeRec));
  }

  // indexed arrays are only needed to assemble the records
  double* d_xyz = nullptr;
  int32_t *d_tri = nullptr, *d_adj = nullptr;
  DG_TRY(pool_alloc(reinterpret_cast<void**>(&d_xyz), 3 * Vn * sizeof(double), m->stream));
  DG_TRY(pool_alloc(reinterpret_cast<void**>(&d_tri), 3 * F * sizeof(int32_t), m->stream));
  DG_TRY(pool_alloc(reinterpret_cast<void**>(&d_adj), 3 * F * sizeof(int32_t), m->stream));
  DG_TRY(cudaMemcpyAsync(d_xyz, xyz, 3 * Vn * sizeof(double), cudaMemcpyHostToDevice, m->stream));
  DG_TRY(cudaMemcpyAsync(d_tri, tri, 3 * F * sizeof(int32_t), cudaMemcpyHostToDevice, m->stream));
  DG_TRY(cudaMemcpyAsync(d_adj, adj, 3 * F * sizeof(int32_t), cudaMemcpyHostToDevice, m->stream));
  DG_TRY(dg::launch_build_records(d_xyz, d_tri, d_adj, nf, m->rec, m->stream));
  build_corner_angles_kernel<<<unsigned((3 * F + 127) / 128), 128, 0, m->stream>>>(m->view_uncached(), m->cangle);
  DG_TRY(cudaGetLastError());
  if (const char* env = getenv("DG_CORNER_ANGLES"))   // =0: the fan walk computes its angles (A/B measurements; same bits)
    if (env[0] == '0') { cudaStreamSynchronize(m->stream); cudaFree(m->cangle); m->cangle = nullptr; m->bytes -= int64_t(3 * F * 8); }
  if (m->he) {
    build_halfedges_kernel<<<unsigned((3 * F + 127) / 128), 128, 0, m->stream>>>(m->view_uncached(), m->he);
    DG_TRY(cudaGetLastError());
    m->he_map_ok = encode_record_map(m->he, 3 * F, m->he_map);
  }
  DG_TRY(cudaMemcpyAsync(m->fnormal, fnormal, 3 * F * sizeof(double), cudaMemcpyHostToDevice, m->stream));
  DG_TRY(cudaMemcpyAsync(m->vangle, vangle, Vn * sizeof(double), cudaMemcpyHostToDevice, m->stream));
  DG_TRY(cudaMemcpyAsync(m->csr_off, csr_off, (Vn + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, m->stream));
  DG_TRY(cudaMemcpyAsync(m->csr_list, csr_list, 3 * F * sizeof(int32_t), cudaMemcpyHostToDevice, m->stream));
  DG_TRY(cudaMemcpyAsync(m->vboundary, vboundary, Vn, cudaMemcpyHostToDevice, m->stream));
  DG_TRY(cudaFreeAsync(d_xyz, m->stream));
  DG_TRY(cudaFreeAsync(d_tri, m->stream));
  DG_TRY(cudaFreeAsync(d_adj, m->stream));
  DG_TRY(cudaStreamSynchronize(m->stream));
#undef DG_TRY
  // multi-GPU: one copy of the mesh per further device of the set (one host-to-device upload each)
  if (g_devices.size() > 1) {
    const std::vector<int> set = g_devices;
    const int primary = g_device;
    int rc = DG_OK;
    for (size_t i = 1; i < set.size() && rc == DG_OK; ++i) {
      g_devices.clear();
      g_device = set[i];
      dg_mesh* copy = nullptr;
      rc = dg_mesh_create_ex(xyz, nv, tri, nf, adj, fnormal, vangle, vboundary, csr_off, csr_list, flags, &copy);
      if (rc == DG_OK) {
        m->replicas.push_back(copy);
        if (copy->device != m->device) {   // NVLink P2P for the peer copies of device-mode requests; failure = staged copies
          int can = 0;
          if (cudaDeviceCanAccessPeer(&can, m->device, copy->device) == cudaSuccess && can) {
            { DeviceGuard a(m->device); cudaDeviceEnablePeerAccess(copy->device, 0); }
            { DeviceGuard b(copy->device); cudaDeviceEnablePeerAccess(m->device, 0); }
            cudaGetLastError();   // "already enabled" is fine
          }
        }
      }
    }
    g_device = primary;
    g_devices = set;
    if (rc != DG_OK) { dg_mesh_destroy(m); return rc; }
  }
  *out = m;
  return DG_OK;
}

void dg_mesh_destroy(dg_mesh* m) {
  if (!m) return;
  for (dg_mesh* copy : m->replicas) dg_mesh_destroy(copy);
  m->replicas.clear();
  DeviceGuard guard(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  if (m->host_batch) dg_batch_destroy(m->host_batch);
  poly_store_free(m->poly);
  if (m->small_pin) cudaFreeHost(m->small_pin);
  cudaFree(m->small_dev);
  cudaFree(m->he64);
  cudaFree(m->rec); cudaFree(m->he); cudaFree(m->fnormal); cudaFree(m->cangle); cudaFree(m->vangle); cudaFree(m->csr_off);
  cudaFree(m->csr_list); cudaFree(m->vboundary);
  if (m->stream) cudaStreamDestroy(m->stream);
  delete m;
}

// Releases what the library keeps warm between calls: the mesh's hidden buffers (the resident batch behind large
// DG_MEM_HOST calls, the small-batch blocks, the pinned polyline arrays; m may be NULL) and the cached blocks of the
// library's staging pool on the mesh's device (or the current device). They are re-created on demand.
int dg_trim(const dg_mesh* m) {
  int device = g_device;
  if (m) {
    device = m->device;
    DeviceGuard guard(m->device);
    cudaStreamSynchronize(m->stream);
    {
      std::lock_guard<std::mutex> lock(m->host_batch_mu);
      if (m->host_batch) dg_batch_destroy(m->host_batch);
      m->host_batch = nullptr;
      m->host_batch_cap = 0;
    }
    {
      std::lock_guard<std::mutex> lock(m->small_mu);
      if (m->small_pin) cudaFreeHost(m->small_pin);
      cudaFree(m->small_dev);
      m->small_pin = m->small_dev = nullptr;
      m->small_cap = 0;
      m->small_cursors_clean = false;
    }
    {
      std::lock_guard<std::mutex> lock(m->poly_mu);
      poly_store_free(m->poly);
      m->poly = nullptr;
    }
    for (const dg_mesh* copy : m->replicas) dg_trim(copy);
  }
  if (dg_device_count() == 0) return DG_OK;
  if (cudaMemPool_t pool = staging_pool(device)) cudaMemPoolTrimTo(pool, 0);
  return DG_OK;
}

int dg_mesh_has_transport_cache(const dg_mesh* m) { return m && m->he ? 1 : 0; }
int dg_mesh_gather_mode(const dg_mesh* m) { return m ? dg::fast_walker_gather_mode(m->view(), m->he_map_ok) : 0; }
// The decisions a plain f64 forward request of n queries gets under cfg (NULL = defaults): *face_order = 1 when
// it is scheduled in start-face order, *gather = DG_GATHER_* of its crossing-record fetch.
int dg_trace_plan(const dg_mesh* m, int64_t n, const dg_trace_cfg* cfg, int* face_order, int* gather) {
  if (!m) return fail(DG_ERR_INVALID_ARGS, "dg_trace_plan: missing mesh");
  dg_trace_cfg c{};
  if (cfg) c = *cfg;
  const bool sort = schedules_by_face(m, n, c, false) && !(c.memory == DG_MEM_HOST && !c.stream && n <= 8192 && c.sort_by_face != DG_SORT_ON);
  if (face_order) *face_order = sort ? 1 : 0;
  if (gather) *gather = dg::fast_walker_gather_mode(m->view(), m->he_map_ok, sort);
  return DG_OK;
}
int dg_mesh_uses_tma_gather(const dg_mesh* m) { return dg_mesh_gather_mode(m) == DG_GATHER_TMA ? 1 : 0; }
int32_t dg_mesh_face_count(const dg_mesh* m) { return m ? m->nf : 0; }
int32_t dg_mesh_vertex_count(const dg_mesh* m) { return m ? m->nv : 0; }
int64_t dg_mesh_device_bytes(const dg_mesh* m) { return m ? m->bytes : 0; }
int dg_mesh_device(const dg_mesh* m) { return m ? m->device : -1; }

// ------------------------------------------------------------------------- forward tracing

// Small host-mode batches (the opt.cpp:298-323 use: ~50 seeds per call) are launch-latency bound:
// instead of one allocation + one copy per array, all inputs are packed into ONE pinned block
// (one H2D), all outputs into one device block (one D2H); both blocks are kept per mesh.
#ifndef DG_SMALL_MAPPED_MAX_DEFAULT
#define DG_SMALL_MAPPED_MAX_DEFAULT 256
#endif
static int trace_small(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c,
                       const dg_trace_out* out) {
  const size_t N = size_t(n);
  struct Field { const void* src; void* dst; size_t bytes; size_t off; };
  Field fin[4] = {{in->face, nullptr, 4 * N, 0}, {in->bary, nullptr, 24 * N, 0}, {in->dir, nullptr, 24 * N, 0},
                  {in->payload, nullptr, in->payload ? 24 * N : 0, 0}};
  Field fout[13] = {{nullptr, out->face, out->face ? 4 * N : 0, 0},
                    {nullptr, out->bary, out->bary ? 24 * N : 0, 0},
                    {nullptr, out->dir, out->dir ? 24 * N : 0, 0},
                    {nullptr, out->traced, out->traced ? 8 * N : 0, 0},
                    {nullptr, out->requested, out->requested ? 8 * N : 0, 0},
                    {nullptr, out->payload, out->payload ? 24 * N : 0, 0},
                    {nullptr, out->transport, out->transport ? 72 * N : 0, 0},
                    {nullptr, out->npoints, out->npoints ? 4 * N : 0, 0},
                    // (a mapped call sums the batch total on the host from this array: it is written whenever the total is asked for)
                    {nullptr, out->crossings, (out->crossings || out->total_crossings) ? 4 * N : 0, 0},
                    {nullptr, out->term, out->term ? N : 0, 0},
                    {nullptr, out->status, out->status ? N : 0, 0},
                    {nullptr, out->stall, out->stall ? N : 0, 0},
                    {nullptr, out->total_crossings, out->total_crossings ? size_t(8) : 0, 0}};
  auto up8 = [](size_t x) { return (x + 7) & ~size_t(7); };
  size_t in_bytes = 16, total = 0;  // the first 16 bytes of the block are the work counters
  for (auto& f : fin) { f.off = in_bytes; in_bytes += up8(f.bytes); }
  total = in_bytes;
  const size_t out_begin = total;
  for (auto& f : fout) { f.off = total; total += up8(f.bytes); }

  std::lock_guard<std::mutex> lock(mesh->small_mu);
  if (mesh->small_cap < total) {
    if (mesh->small_pin) cudaFreeHost(mesh->small_pin);
    if (mesh->small_dev) cudaFree(mesh->small_dev);
    mesh->small_pin = mesh->small_dev = nullptr;
    mesh->small_cap = 0;
    const size_t cap = std::max<size_t>(total * 2, size_t(1) << 16);
    DG_CUDA(cudaMallocHost(&mesh->small_pin, cap));
    DG_CUDA(cudaMalloc(&mesh->small_dev, cap));
    mesh->small_cap = cap;
    mesh->small_cursors_clean = false;
  }
  char* hp = static_cast<char*>(mesh->small_pin);
  char* dp = static_cast<char*>(mesh->small_dev);
  // The smallest batches skip both copies: the pinned block is mapped into the device's address space (unified
  // addressing), the kernel reads its queries from it and writes its results into it over PCIe, and only the 16
  // bytes of work cursors live in device memory (atomics). Measured (tests/cpp/bench_small_batch.cpp, us per call
  // with the transport matrix, copies -> mapped): 1 seed 40.7 -> 30.8, 50 seeds 70.3 -> 65.4, 1 000 seeds 112.7 -> 111.7,
  // 8 000 seeds 524 -> 596: mapped up to 256 queries. DG_SMALL_MAPPED_MAX overrides the limit.
  static const int64_t mapped_max = [] {
    const char* e = getenv("DG_SMALL_MAPPED_MAX");
    return e ? int64_t(atoll(e)) : int64_t(DG_SMALL_MAPPED_MAX_DEFAULT);
  }();
  const bool mapped = n <= mapped_max;
  std::memset(hp, 0, 16);
  for (auto& f : fin) if (f.bytes) std::memcpy(hp + f.off, f.src, f.bytes);
  cudaStream_t stream = mesh->stream;
  // Mapped calls alternate between two work cursors in device memory; every launch zeroes the one the NEXT call
  // uses (TraceParams::clear_word), so a call is one kernel launch and one synchronisation -- no memset, no copy.
  // Anything that may have left the cursors dirty (first use, reallocation, a copied call, an error) resets both.
  unsigned long long* cursors = reinterpret_cast<unsigned long long*>(dp);
  const unsigned turn = mesh->small_calls++ & 1u;
  if (mapped) {
    if (!mesh->small_cursors_clean) DG_CUDA(cudaMemsetAsync(dp, 0, 16, stream));
    mesh->small_cursors_clean = false;   // set again once this call has completed
  } else {
    mesh->small_cursors_clean = false;
    DG_CUDA(cudaMemcpyAsync(dp, hp, in_bytes, cudaMemcpyHostToDevice, stream));
  }

  if (c.lane == DG_LANE_FAST) ensure_he64(mesh);
  dg::TraceParams p{};
  mesh->bind(p);
  p.n = n;
  char* base = mapped ? hp : dp;
  auto din = [&](int i) { return fin[i].bytes ? base + fin[i].off : nullptr; };
  auto dout = [&](int i) { return fout[i].bytes ? base + fout[i].off : nullptr; };
  p.face = reinterpret_cast<const int32_t*>(din(0));
  p.bary = reinterpret_cast<const double*>(din(1));
  p.dir = reinterpret_cast<const double*>(din(2));
  p.payload = reinterpret_cast<const double*>(din(3));
  p.o_face = reinterpret_cast<int32_t*>(dout(0));
  p.o_bary = reinterpret_cast<double*>(dout(1));
  p.o_dir = reinterpret_cast<double*>(dout(2));
  p.o_traced = reinterpret_cast<double*>(dout(3));
  p.o_requested = reinterpret_cast<double*>(dout(4));
  p.o_payload = reinterpret_cast<double*>(dout(5));
  p.o_transport = reinterpret_cast<double*>(dout(6));
  p.o_npoints = reinterpret_cast<int32_t*>(dout(7));
  p.o_crossings = reinterpret_cast<int32_t*>(dout(8));
  p.o_term = reinterpret_cast<uint8_t*>(dout(9));
  p.o_status = reinterpret_cast<uint8_t*>(dout(10));
  p.o_stall = reinterpret_cast<uint8_t*>(dout(11));
  p.queue_head = mapped ? cursors + turn : cursors;
  p.clear_word = mapped ? cursors + (turn ^ 1u) : nullptr;
  // mapped: the sum of the batch is taken on the host from the per-query counts
  p.total_crossings = (fout[12].bytes && !mapped) ? reinterpret_cast<unsigned long long*>(dp + fout[12].off) : nullptr;
  p.max_steps = c.max_steps > 0 ? c.max_steps : default_max_steps(mesh->nf);
  p.refill_min = 0;
  p.hole_avoidance = c.hole_avoidance;
  p.want_q = c.want_transport_matrix;
  p.lane_fast = c.lane == DG_LANE_FAST;
  if (p.total_crossings && !mapped) DG_CUDA(cudaMemsetAsync(p.total_crossings, 0, 8, stream));
  const bool needs_full = in->payload || c.want_transport_matrix || c.hole_avoidance || out->payload || out->transport;
  DG_CUDA(dg::launch_trace(p, c.use_f32 != 0, needs_full, dg::LaunchShape{mesh->sm_count, int(c.blocks_per_sm), int(c.walker)}, stream));
  if (!mapped && total > out_begin)
    DG_CUDA(cudaMemcpyAsync(hp + out_begin, dp + out_begin, total - out_begin, cudaMemcpyDeviceToHost, stream));
  DG_CUDA(cudaStreamSynchronize(stream));
  if (mapped) {
    mesh->small_cursors_clean = true;
    if (fout[12].bytes) {
      uint64_t sum = 0;
      const int32_t* cr = reinterpret_cast<const int32_t*>(hp + fout[8].off);
      for (size_t i = 0; i < N; ++i) sum += uint64_t(cr[i]);
      std::memcpy(hp + fout[12].off, &sum, 8);
    }
  }
  for (auto& f : fout) if (f.bytes && f.dst) std::memcpy(f.dst, hp + f.off, f.bytes);
  return DG_OK;
}

// Enqueues a trace request on `stream` (staging through `st`).
static int enqueue_trace(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c,
                         const dg_trace_out* out, bool record, cudaStream_t stream, Stage& st, uint64_t* total_dst) {
  const bool device_mode = c.memory == DG_MEM_DEVICE;
  const size_t N = size_t(n);
  auto at = [](auto* ptr, size_t) { return ptr; };
  if (c.lane == DG_LANE_FAST) ensure_he64(mesh);
  dg::TraceParams p{};
  mesh->bind(p);
  p.n = n;
  p.face = st.in(at(in->face, 1), N);
  p.bary = st.in(at(in->bary, 3), 3 * N);
  p.dir = st.in(at(in->dir, 3), 3 * N);
  p.payload = st.in(at(in->payload, 3), 3 * N);
  p.o_face = st.out(at(out->face, 1), N);
  p.o_bary = st.out(at(out->bary, 3), 3 * N);
  p.o_dir = st.out(at(out->dir, 3), 3 * N);
  p.o_traced = st.out(at(out->traced, 1), N);
  p.o_requested = st.out(at(out->requested, 1), N);
  p.o_term = st.out(at(out->term, 1), N);
  p.o_status = st.out(at(out->status, 1), N);
  p.o_stall = st.out(at(out->stall, 1), N);
  p.o_payload = st.out(at(out->payload, 3), 3 * N);
  p.o_transport = st.out(at(out->transport, 9), 9 * N);
  p.o_npoints = st.out(at(out->npoints, 1), N);
  p.o_crossings = st.out(at(out->crossings, 1), N);
  if (record) {
    const size_t T = size_t(out->poly_total);
    p.poly_offsets = st.in(out->poly_offsets, N);
    p.poly_face = st.out(out->poly_face, T);
    p.poly_bary = st.out(out->poly_bary, 3 * T);
    p.poly_seg = st.out(out->poly_seg, T);
  }
  p.max_steps = c.max_steps > 0 ? c.max_steps : default_max_steps(mesh->nf);
  p.refill_min = c.refill_min;  // 0 = the walker's own default
  p.hole_avoidance = c.hole_avoidance;
  p.want_q = c.want_transport_matrix;
  p.lane_fast = c.lane == DG_LANE_FAST;

  // the work cursor and the crossing total of THIS call, stream-ordered like the rest of its staging
  unsigned long long* ctr = st.scratch<unsigned long long>(3);   // [2]: sum of sampled requested lengths (a double)
  if (!ctr) return fail_cuda(st.error(), "dg_trace_batch staging");
  p.queue_head = ctr;
  p.total_crossings = total_dst ? ctr + 1 : nullptr;
  st.note(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), stream));

  // Schedule in start-face order (results stay at the request index). AUTO: on for large batches on meshes whose
  // crossing records do not fit the L2 -- traces that start side by side walk through the same neighbourhood at the
  // same time, so the in-flight set is a travelling wavefront instead of the whole mesh and more of its records are
  // L2 hits (c3, 1 M-face torus, 384 MB of records: forward 17.9 -> 16.5 ms per 1 M, 179 -> 160 ms per 10 M;
  // c2, L2-resident: +-1 %, stays off). The face order of the mesh is the caller's: a locality-preserving
  // numbering (grid, Morton, Hilbert) is what makes neighbours in the queue neighbours on the surface.
  const bool sort = schedules_by_face(mesh, n, c, record);
  double* length_sum = reinterpret_cast<double*>(ctr + 2);
  if (sort) p.perm = start_face_order(mesh, n, p.face, p.bary, st, stream, p.dir, length_sum);
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_trace_batch staging");

  const bool needs_full = in->payload || c.want_transport_matrix || c.hole_avoidance || record ||
                          out->payload || out->transport;
  dg::LaunchShape shape{mesh->sm_count, int(c.blocks_per_sm), int(c.walker)};
  // Start-face order keeps the per-lane loads ahead only while the records the resident lanes walk over stay within
  // reach of the L2; beyond that every lane's four sector requests go to HBM on their own and the cooperative gather
  // (one line request per record) is 1.5-2.8 x faster. Consecutive entries of the order start in a band across the
  // mesh, and a trace of L crossings carries the band L / 2 cells further: the footprint of the wavefront grows as
  // L sqrt(F) faces, whatever the size of the batch. Measured on tori of 1 M / 2.25 M / 4 M faces with 0.5 M - 10 M
  // traces (scripts/dev/gather_crossover.py, per-lane / cooperative, ms): 1 M faces, 500 k traces of 520 crossings
  // 5.9 / 6.3, 1 045 crossings 12.5 / 12.4, 1 570 32.3 / 18.4, 5 220 (config 5's random half) 122 / 62; 2.25 M faces,
  // 4 M traces of 510 crossings 42.5 / 47.4, 1 020 203 / 92; 4 M faces, 10 M traces of 680 crossings 312 / 162 -- the
  // two tie at L sqrt(F) = 1e6 in every case. L is known only on the device (the requested lengths), so the sort's
  // key pass sums the length of every 64th query, both instantiations are queued with complementary gates on that
  // sum, and the one whose side of the limit it falls on runs (the other returns at once): no host round trip, the
  // call stays asynchronous. (About 2.5 crossings per mean edge length travelled.)
  const bool two_gathers = sort && p.perm && !needs_full && !c.use_f32 && c.walker == DG_WALKER_AUTO && mesh->mean_edge > 0.0 &&
                           dg::fast_walker_gather_mode(mesh->view(), mesh->he_map_ok, false) == 2 &&
                           dg::fast_walker_gather_mode(mesh->view(), mesh->he_map_ok, true) == 0 && !getenv("DG_FAST_GATHER");
  if (two_gathers) {
    dg::LaunchShape loads = shape, coop = shape;
    loads.walker = DG_WALKER_FAST_LOADS;
    coop.walker = DG_WALKER_FAST_COOP;
    dg::TraceParams q = p;
    q.mesh.he64 = nullptr;   // (the tolerance lane has no cooperative gather of its half-size records: its
                             // instantiation over the 128-byte records takes that road)
    const double samples = double((n + 63) / 64), tie_crossings = 1e6 / std::sqrt(double(mesh->nf));
    p.gate = q.gate = length_sum;
    p.gate_limit = q.gate_limit = samples * tie_crossings * mesh->mean_edge / 2.5;
    p.gate_above = 0;
    q.gate_above = 1;
    st.note(dg::launch_trace(p, false, false, loads, stream));
    st.note(dg::launch_trace(q, false, false, coop, stream));
  } else {
    st.note(dg::launch_trace(p, c.use_f32 != 0, needs_full, shape, stream));
  }
  if (total_dst) {
    st.note(cudaMemcpyAsync(total_dst, ctr + 1, sizeof(uint64_t),
                            device_mode ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, stream));
  }
  if (st.error() != cudaSuccess) return fail_cuda(st.error(), "dg_trace_batch launch");
  return DG_OK;
}

// One device: the request runs on `mesh` (a primary without fan-out, or one device's copy).
}  // extern "C"

int dgapi::trace_batch_one(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c, dg_trace_out* out) {
  const bool device_mode = c.memory == DG_MEM_DEVICE;
  const bool record = out->poly_offsets != nullptr;
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);
  // device mode: the caller's stream, NULL = the CUDA default stream (ordering with the caller's
  // own work is the caller's contract); host mode: the mesh's private stream unless one is given
  cudaStream_t stream = (device_mode || c.stream) ? static_cast<cudaStream_t>(c.stream) : mesh->stream;
  if (n == 0) {
    if (out->total_crossings) {
      if (device_mode) DG_CUDA(cudaMemsetAsync(out->total_crossings, 0, sizeof(uint64_t), stream));
      else *out->total_crossings = 0;
    }
    return DG_OK;
  }

  if (!device_mode && !c.stream && !record && c.sort_by_face != DG_SORT_ON && n <= 8192) return trace_small(mesh, n, in, c, out);

  // Host mode, large plain batch: the copy/compute pipeline of the resident batch (slices on
  // separate streams: the H2D copy of slice i+1 and the D2H copy of slice i-1 overlap the walker
  // of slice i) over device buffers the mesh keeps between calls. Measured on B200, 1 M geodesics
  // x 207 crossings, walker 4.0 ms: single stream 6.4 ms, pipeline 5.1 ms (stream-ordered
  // allocations per slice serialise the streams and give 6.3-6.8 ms, which is why the buffers persist).
  const bool plain = !in->payload && !out->payload && !out->transport && !c.want_transport_matrix && !c.hole_avoidance;
  if (!device_mode && !c.stream && !record && plain && n >= (int64_t(1) << 16)) {
    std::lock_guard<std::mutex> lock(mesh->host_batch_mu);
    if (!mesh->host_batch || mesh->host_batch_cap < n) {
      if (mesh->host_batch) dg_batch_destroy(mesh->host_batch);
      mesh->host_batch = nullptr;
      mesh->host_batch_cap = 0;
      int rc = dgapi::batch_create_one(mesh, n, &mesh->host_batch);
      if (rc != DG_OK) return rc;
      mesh->host_batch_cap = n;
    }
    return dgapi::batch_trace_one(mesh->host_batch, n, in, &c, out);
  }

  Stage st(stream, device_mode);
  int rc = enqueue_trace(mesh, n, in, c, out, record, stream, st, out->total_crossings);
  if (rc != DG_OK) return rc;
  cudaError_t e = st.finish();
  if (e != cudaSuccess) return fail_cuda(e, "dg_trace_batch");
  return DG_OK;
}

extern "C" {

// Shard [lo, lo + m) of a request: the same pointers, offset.
static void shard_io(const dg_trace_in* in, const dg_trace_out* out, int64_t lo, dg_trace_in* sin, dg_trace_out* so) {
  const size_t L = size_t(lo);
  auto at = [&](auto* p, size_t stride) { return p ? p + stride * L : p; };
  *sin = dg_trace_in{at(in->face, 1), at(in->bary, 3), at(in->dir, 3), at(in->payload, 3)};
  *so = dg_trace_out{};
  so->face = at(out->face, 1); so->bary = at(out->bary, 3); so->dir = at(out->dir, 3);
  so->traced = at(out->traced, 1); so->requested = at(out->requested, 1);
  so->term = at(out->term, 1); so->status = at(out->status, 1); so->stall = at(out->stall, 1);
  so->payload = at(out->payload, 3); so->transport = at(out->transport, 9);
  so->npoints = at(out->npoints, 1); so->crossings = at(out->crossings, 1);
}

// Host-mode request on a multi-GPU mesh: contiguous shards of equal expected work, one host thread per device,
// every shard the one-device path on its own slice of the caller's arrays (results at the request index).
static int trace_batch_multi_host(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c,
                                  dg_trace_out* out) {
  const bool record = out->poly_offsets != nullptr;
  const std::vector<Shard> shards = cut_shards(mesh, n, in->dir);
  std::vector<uint64_t> totals(shards.size(), 0);
  std::vector<std::vector<int64_t>> rel(shards.size());   // polyline offsets relative to the shard's first slot
  int rc = run_shards(shards, [&](const Shard& s, int k) {
    dg_trace_in sin;
    dg_trace_out so;
    shard_io(in, out, s.lo, &sin, &so);
    so.total_crossings = out->total_crossings ? &totals[size_t(k)] : nullptr;
    if (record) {
      const int64_t first = out->poly_offsets[s.lo];
      const int64_t end = s.lo + s.n < n ? out->poly_offsets[s.lo + s.n] : out->poly_total;
      auto& r = rel[size_t(k)];
      r.resize(size_t(s.n));
      for (int64_t i = 0; i < s.n; ++i) r[size_t(i)] = out->poly_offsets[s.lo + i] - first;
      so.poly_offsets = r.data();
      so.poly_total = end - first;
      so.poly_face = out->poly_face + first; so.poly_bary = out->poly_bary + 3 * first; so.poly_seg = out->poly_seg + first;
    }
    dg_trace_cfg sc = c;
    if (s.mesh != mesh) sc.stream = nullptr;   // a caller's stream belongs to the primary device
    return trace_batch_one(s.mesh, s.n, &sin, sc, &so);
  });
  if (rc != DG_OK) return rc;
  if (out->total_crossings) {
    uint64_t t = 0;
    for (uint64_t v : totals) t += v;
    *out->total_crossings = t;
  }
  return DG_OK;
}

// Device-mode request on a multi-GPU mesh: the caller's arrays live on the PRIMARY device and the call stays
// asynchronous on the caller's stream. Shard 0 runs in place; every other shard runs on its device's stream after
// an event of the caller's stream, on local copies moved by peer copies (PeerStage), and the caller's stream waits
// for the event that follows its copy back. Equal-count shards (the weights are not on the host).
static int trace_batch_multi_device(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg& c,
                                    dg_trace_out* out) {
  const std::vector<Shard> shards = cut_shards(mesh, n, nullptr);
  const int S = int(shards.size());
  cudaStream_t home = static_cast<cudaStream_t>(c.stream);
  DeviceGuard guard(mesh->device);
  if (!guard.ok) return fail(DG_ERR_CUDA, "cannot select device %d", mesh->device);
  cudaEvent_t ready = nullptr;
  DG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  unsigned long long* parts = nullptr;
  if (out->total_crossings) {
    DG_CUDA(pool_alloc(reinterpret_cast<void**>(&parts), size_t(S) * sizeof(unsigned long long), home));
    DG_CUDA(cudaMemsetAsync(parts, 0, size_t(S) * sizeof(unsigned long long), home));
  }
  DG_CUDA(cudaEventRecord(ready, home));
  int rc = DG_OK;
  std::vector<cudaEvent_t> joins;
  for (int k = 0; k < S && rc == DG_OK; ++k) {
    const Shard& s = shards[size_t(k)];
    if (s.n == 0) continue;
    dg_trace_in sin;
    dg_trace_out so;
    shard_io(in, out, s.lo, &sin, &so);
    so.total_crossings = parts ? reinterpret_cast<uint64_t*>(parts + k) : nullptr;
    if (s.mesh == mesh) {
      rc = trace_batch_one(mesh, s.n, &sin, c, &so);
      continue;
    }
    DeviceGuard work(s.mesh->device);
    cudaStream_t ws = s.mesh->stream;
    const size_t M = size_t(s.n);
    PeerStage ps(mesh->device, s.mesh->device, ws);
    ps.note(cudaStreamWaitEvent(ws, ready, 0));
    dg_trace_in lin{ps.in(sin.face, M), ps.in(sin.bary, 3 * M), ps.in(sin.dir, 3 * M), ps.in(sin.payload, 3 * M)};
    dg_trace_out lo{};
    lo.face = ps.out(so.face, M); lo.bary = ps.out(so.bary, 3 * M); lo.dir = ps.out(so.dir, 3 * M);
    lo.traced = ps.out(so.traced, M); lo.requested = ps.out(so.requested, M);
    lo.term = ps.out(so.term, M); lo.status = ps.out(so.status, M); lo.stall = ps.out(so.stall, M);
    lo.payload = ps.out(so.payload, 3 * M); lo.transport = ps.out(so.transport, 9 * M);
    lo.npoints = ps.out(so.npoints, M); lo.crossings = ps.out(so.crossings, M);
    lo.total_crossings = ps.out(so.total_crossings, 1);
    if (ps.error() != cudaSuccess) { rc = fail_cuda(ps.error(), "dg_trace_batch peer staging"); break; }
    dg_trace_cfg wc = c;
    wc.stream = ws;
    rc = trace_batch_one(s.mesh, s.n, &lin, wc, &lo);
    ps.flush();
    cudaEvent_t done = nullptr;
    ps.note(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    if (done) {
      ps.note(cudaEventRecord(done, ws));
      joins.push_back(done);   // the caller's stream waits for it below, with the primary device current again
    }
    if (rc == DG_OK && ps.error() != cudaSuccess) rc = fail_cuda(ps.error(), "dg_trace_batch peer copies");
  }
  for (cudaEvent_t done : joins) {
    if (cudaStreamWaitEvent(home, done, 0) != cudaSuccess && rc == DG_OK) rc = fail(DG_ERR_CUDA, "dg_trace_batch: joining the shards");
    cudaEventDestroy(done);   // released once the recorded work has completed
  }
  cudaEventDestroy(ready);
  if (parts) {
    if (rc == DG_OK) {
      sum_totals_kernel<<<1, 1, 0, home>>>(parts, S, reinterpret_cast<unsigned long long*>(out->total_crossings));
      if (cudaGetLastError() != cudaSuccess) rc = fail(DG_ERR_CUDA, "dg_trace_batch: total of the shards");
    }
    cudaFreeAsync(parts, home);
  }
  return rc;
}

int dg_trace_batch(const dg_mesh* mesh, int64_t n, const dg_trace_in* in, const dg_trace_cfg* cfg,
                   dg_trace_out* out) {
  // whole-call contract violations, tracer.cpp:566-576
  if (!mesh) return fail(DG_ERR_INVALID_ARGS, "trace_batch: missing mesh");
  if (n < 0 || n > 0x7fffffffLL) return fail(DG_ERR_INVALID_ARGS, "trace_batch: batch size out of range");
  if (!in || !out) return fail(DG_ERR_INVALID_ARGS, "trace_batch: null request or result block");
  if (n > 0 && (!in->face || !in->bary || !in->dir))
    return fail(DG_ERR_INVALID_ARGS, "trace_batch: starts and dirs differ in length");
  dg_trace_cfg c{};
  if (cfg) c = *cfg;
  if (c.lane > DG_LANE_FAST) return fail(DG_ERR_INVALID_ARGS, "trace_batch: unknown arithmetic lane %d", int(c.lane));
  const bool record = out->poly_offsets != nullptr;
  if (record && (!out->poly_face || !out->poly_bary || !out->poly_seg || out->poly_total < 0))
    return fail(DG_ERR_INVALID_ARGS, "trace_batch: polyline recording needs poly_face/poly_bary/poly_seg and poly_total");
  // the reference's fork/join site (tracer.cpp:596-603): one request over the devices of the mesh's set
  if (fan_out(mesh, n)) {
    if (c.memory != DG_MEM_DEVICE) return trace_batch_multi_host(mesh, n, in, c, out);
    if (!record) return trace_batch_multi_device(mesh, n, in, c, out);   // (device-resident polyline offsets: one device)
  }
  return trace_batch_one(mesh, n, in, c, out);
}

void dg_trace_kernel_info(int use_f32, int full, int* regs, int* blocks_per_sm, int* block_threads) {
  if (regs) *regs = 0;
  if (blocks_per_sm) *blocks_per_sm = 0;
  if (block_threads) *block_threads = 0;
  if (dg_device_count() == 0) return;
  DeviceGuard guard(g_device);
  dg::trace_kernel_info(use_f32 != 0, full, regs, blocks_per_sm, block_threads);
}

}  // extern "C"
