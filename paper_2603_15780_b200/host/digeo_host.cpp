// Host shim: the reference's C++ operator interface (include/digeo_b200/digeo.hpp) over the
// C-ABI of libdigeo_b200.so. Packs the reference's AoS request types into SoA arrays, calls the
// GPU entry points and unpacks into the reference's result types; maps DG_ERR_* codes and
// per-element stall codes back to the reference's exception classes and message strings.
#include "digeo_b200/digeo.hpp"

#include <algorithm>
#include <limits>
#include <mutex>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <thread>

#include "dg_b200.h"

namespace digeo {

// ------------------------------------------------------------------------------ errors
namespace {

[[noreturn]] void raise(int code) {
  const std::string msg = dg_last_error();
  switch (code) {
    case DG_ERR_INVALID_ARGS: throw InvalidArgs(msg);
    case DG_ERR_PARSE: throw ParseError(msg);
    case DG_ERR_NON_MANIFOLD: throw NonManifoldError(msg);
    case DG_ERR_DEGENERATE_FACE: throw DegenerateFaceError(msg);
    case DG_ERR_DEGENERATE_DIRECTION: throw DegenerateDirection(msg);
    case DG_ERR_GFD: throw Error(msg);
    case DG_ERR_NUMERICAL_STALL: throw NumericalStall(msg);
    case DG_ERR_BOUNDARY_HIT: throw BoundaryHit(msg);
    default: throw DeviceError(msg);
  }
}
void check(int rc) { if (rc != DG_OK) raise(rc); }

const char* stall_message(uint8_t code) {  // tracer.cpp:183,197,474,459,461
  switch (code) {
    case DG_STALL_DEGENERATE_DIRECTION: return "degenerate direction in face";
    case DG_STALL_NO_EXIT: return "no positive exit parameter";
    case DG_STALL_NORMAL_DIRECTION: return "initial direction is normal to the anchor face";
    case DG_STALL_FACE_RANGE: return "trace: start face out of range";
    case DG_STALL_BARY_RANGE: return "trace: start barycentric coordinates not in the simplex";
    default: return "";
  }
}

void put3(std::vector<double>& a, size_t i, const Vec3d& v) { a[3 * i] = v.x; a[3 * i + 1] = v.y; a[3 * i + 2] = v.z; }

// Marshalling between the reference's per-element objects (GeodesicTrace with its vectors of points: 280 bytes plus
// heap per element) and the SoA of the C-ABI is host work the GPU call does not hide; for large batches it runs on
// the host's cores (100 000 traces with polylines: 83 -> the time of the slowest chunk). body(lo, hi) per chunk.
template <class Body>
void parallel_chunks(size_t n, const Body& body) {
  const size_t kMin = 4096;
  size_t workers = std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()), (n + kMin - 1) / kMin);
  if (const char* cap = std::getenv("DIGEO_WORKERS")) workers = std::min<size_t>(workers, std::max(1, std::atoi(cap)));
  if (workers <= 1) { body(size_t(0), n); return; }
  std::vector<std::thread> pool;
  const size_t chunk = (n + workers - 1) / workers;
  for (size_t w = 1; w < workers; ++w) pool.emplace_back([&, w] { body(std::min(n, w * chunk), std::min(n, (w + 1) * chunk)); });
  body(size_t(0), std::min(n, chunk));
  for (auto& t : pool) t.join();
}
Vec3d get3(const double* a, size_t i) { return {a[3 * i], a[3 * i + 1], a[3 * i + 2]}; }

}  // namespace

// ------------------------------------------------------------------------------ Mat3
Mat3 Mat3::operator*(const Mat3& o) const {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += (*this)(i, k) * o(k, j);
      r(i, j) = s;
    }
  return r;
}
Mat3 Mat3::transposed() const {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = (*this)(j, i);
  return r;
}
double Mat3::det() const {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) + m[2] * (m[3] * m[7] - m[4] * m[6]);
}

// ------------------------------------------------------------------------------ mesh
class DeviceMesh {
 public:
  explicit DeviceMesh(dg_mesh* h) : h_(h) {}
  ~DeviceMesh() { dg_mesh_destroy(h_); }
  DeviceMesh(const DeviceMesh&) = delete;
  DeviceMesh& operator=(const DeviceMesh&) = delete;
  const dg_mesh* handle() const { return h_; }
  // serialises polyline-recording calls on this mesh: their polylines live in arrays the mesh hands out until
  // its next recording call (dg_trace_polylines), and trace_batch must stay re-entrant
  std::mutex& polyline_mutex() const { return poly_mu_; }

 private:
  dg_mesh* h_;
  mutable std::mutex poly_mu_;
};

namespace {
struct FlatMesh {
  std::vector<double> xyz;
  std::vector<int32_t> tri;
};
FlatMesh flatten(const std::vector<Vec3d>& v, const std::vector<std::array<int, 3>>& f) {
  FlatMesh m;
  m.xyz.resize(3 * v.size());
  m.tri.resize(3 * f.size());
  for (size_t i = 0; i < v.size(); ++i) { m.xyz[3 * i] = v[i].x; m.xyz[3 * i + 1] = v[i].y; m.xyz[3 * i + 2] = v[i].z; }
  for (size_t i = 0; i < f.size(); ++i) for (int k = 0; k < 3; ++k) m.tri[3 * i + k] = f[i][k];
  return m;
}
}  // namespace

Mesh Mesh::build(std::vector<Vec3d> vertices, std::vector<std::array<int, 3>> faces) {
  Mesh m;
  m.vertices = std::move(vertices);
  m.faces = std::move(faces);
  const int nv = m.vertex_count(), nf = m.face_count();
  FlatMesh flat = flatten(m.vertices, m.faces);
  std::vector<int32_t> adj(3 * size_t(nf)), off(size_t(nv) + 1), lst(3 * size_t(nf));
  std::vector<double> fn(3 * size_t(nf)), va(nv), ar(nv);
  std::vector<uint8_t> vb(nv);
  m.face_areas.resize(nf);
  int64_t bad = -1;
  check(dg_mesh_derive(flat.xyz.data(), nv, flat.tri.data(), nf, adj.data(), fn.data(), m.face_areas.data(), va.data(),
                       ar.data(), vb.data(), off.data(), lst.data(), &m.mean_edge_length_, &m.total_area_, &bad));
  m.face_adjacency.resize(nf);
  m.face_normals.resize(nf);
  for (int f = 0; f < nf; ++f) {
    m.face_adjacency[f] = {adj[3 * f], adj[3 * f + 1], adj[3 * f + 2]};
    m.face_normals[f] = get3(fn.data(), f);
  }
  m.vertex_total_angle = std::move(va);
  m.vertex_area = std::move(ar);
  m.vertex_on_boundary.assign(vb.begin(), vb.end());
  m.vertex_face_offsets_.assign(off.begin(), off.end());
  m.vertex_face_list_.assign(lst.begin(), lst.end());
  return m;
}

int Mesh::neighbor_across(int f, int a, int b) const {
  for (int k = 0; k < 3; ++k) {
    const int u = faces[f][(k + 1) % 3], v = faces[f][(k + 2) % 3];
    if ((u == a && v == b) || (u == b && v == a)) return face_adjacency[f][k];
  }
  return -1;
}
std::span<const int> Mesh::vertex_faces(int v) const {
  return {vertex_face_list_.data() + vertex_face_offsets_[v], vertex_face_list_.data() + vertex_face_offsets_[v + 1]};
}

void Mesh::set_device(int ordinal) { check(dg_set_device(ordinal)); }
void Mesh::set_devices(std::uint64_t mask) { check(dg_set_devices(mask)); }
void Mesh::set_device_list(const std::vector<int>& ordinals) {
  std::vector<int32_t> list(ordinals.begin(), ordinals.end());
  check(dg_set_device_list(list.data(), int32_t(list.size())));
}

const DeviceMesh& Mesh::device() const {
  if (!device_) {
    const int nv = vertex_count(), nf = face_count();
    FlatMesh flat = flatten(vertices, faces);
    std::vector<int32_t> adj(3 * size_t(nf));
    std::vector<double> fn(3 * size_t(nf));
    std::vector<uint8_t> vb(nv);
    for (int f = 0; f < nf; ++f)
      for (int k = 0; k < 3; ++k) {
        adj[3 * f + k] = face_adjacency[f][k];
        fn[3 * f + k] = face_normals[f][k];
      }
    for (int v = 0; v < nv; ++v) vb[v] = vertex_on_boundary[v] ? 1 : 0;
    std::vector<int32_t> off(vertex_face_offsets_.begin(), vertex_face_offsets_.end());
    std::vector<int32_t> lst(vertex_face_list_.begin(), vertex_face_list_.end());
    dg_mesh* h = nullptr;
    check(dg_mesh_create(flat.xyz.data(), nv, flat.tri.data(), nf, adj.data(), fn.data(), vertex_total_angle.data(),
                         vb.data(), off.data(), lst.data(), &h));
    device_ = std::make_shared<DeviceMesh>(h);
  }
  return *device_;
}

Mesh load_obj(std::istream& in) {
  std::vector<Vec3d> verts;
  std::vector<std::array<int, 3>> faces;
  std::string line;
  int lineno = 0;
  const auto where = [&] { return "line " + std::to_string(lineno) + ": "; };
  while (std::getline(in, line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      Vec3d p;
      if (!(ls >> p.x >> p.y >> p.z)) throw ParseError(where() + "malformed vertex");
      verts.push_back(p);
    } else if (tag == "f") {
      std::vector<int> poly;
      std::string tok;
      while (ls >> tok) {  // "v", "v/vt", "v//vn", "v/vt/vn"; negative = relative
        int idx = 0;
        try {
          idx = std::stoi(tok.substr(0, tok.find('/')));
        } catch (const std::exception&) {
          throw ParseError(where() + "bad face index '" + tok + "'");
        }
        if (idx < 0) idx += int(verts.size()) + 1;
        if (idx < 1 || idx > int(verts.size())) throw ParseError(where() + "face index out of range");
        poly.push_back(idx - 1);
      }
      if (poly.size() < 3) throw ParseError(where() + "face with <3 vertices");
      for (size_t i = 1; i + 1 < poly.size(); ++i) faces.push_back({poly[0], poly[i], poly[i + 1]});  // fan split
    }
  }
  if (verts.empty() || faces.empty()) throw ParseError("OBJ contains no triangles");
  return Mesh::build(std::move(verts), std::move(faces));
}
Mesh load_obj_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IOError("cannot open '" + path + "'");
  return load_obj(in);
}
void write_obj(const Mesh& m, std::ostream& out) {
  out.precision(17);
  for (const auto& v : m.vertices) out << "v " << v.x << " " << v.y << " " << v.z << "\n";
  for (const auto& f : m.faces) out << "f " << f[0] + 1 << " " << f[1] + 1 << " " << f[2] + 1 << "\n";
}
void write_obj_file(const Mesh& m, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IOError("cannot open '" + path + "' for writing");
  write_obj(m, out);
}
Mesh concat_meshes(const Mesh& a, const Mesh& b) {
  std::vector<Vec3d> v = a.vertices;
  v.insert(v.end(), b.vertices.begin(), b.vertices.end());
  std::vector<std::array<int, 3>> f = a.faces;
  const int shift = a.vertex_count();
  for (const auto& t : b.faces) f.push_back({t[0] + shift, t[1] + shift, t[2] + shift});
  return Mesh::build(std::move(v), std::move(f));
}
Vec3d embed(const SurfacePoint& p, const Mesh& m) {
  const auto& c = m.faces[p.face];
  return m.vertices[c[0]] * p.bary[0] + m.vertices[c[1]] * p.bary[1] + m.vertices[c[2]] * p.bary[2];
}
PointClassification classify(const SurfacePoint& p, double tol) {
  int hi = 0, lo = 0;
  for (int i = 1; i < 3; ++i) {
    if (p.bary[i] > p.bary[hi]) hi = i;
    if (p.bary[i] < p.bary[lo]) lo = i;
  }
  if (p.bary[hi] >= 1.0 - tol) return {PointClass::Vertex, hi};
  if (p.bary[lo] <= tol) return {PointClass::Edge, lo};
  return {PointClass::Interior, -1};
}
bool bary_valid(const Vec3d& b, double tol) {
  if (std::abs(b[0] + b[1] + b[2] - 1.0) > tol) return false;
  for (int i = 0; i < 3; ++i)
    if (b[i] < -tol || b[i] > 1.0 + tol) return false;
  return true;
}
double total_angle(int vertex, const Mesh& m) { return m.vertex_total_angle[vertex]; }

// mesh.cpp:233-261: barycentrics of the point of face f closest to q -- the in-plane coefficients when they lie in
// the simplex, else the nearest of the three clamped edge projections (edge k is opposite corner k; first minimum wins).
Vec3d project_to_face(const Mesh& m, int f, const Vec3d& q) {
  const auto& c = m.faces[f];
  const Vec3d corner[3] = {m.vertices[c[0]], m.vertices[c[1]], m.vertices[c[2]]};
  const auto coef = plane_coefficients(corner[1] - corner[0], corner[2] - corner[0], q - corner[0]);
  if (coef[0] >= 0 && coef[1] >= 0 && coef[0] + coef[1] <= 1.0) return {1.0 - coef[0] - coef[1], coef[0], coef[1]};
  Vec3d nearest{1, 0, 0};
  double nearest_d2 = std::numeric_limits<double>::infinity();
  for (int k = 0; k < 3; ++k) {
    const int i = (k + 1) % 3, j = (k + 2) % 3;
    const Vec3d along = corner[j] - corner[i];
    const double t = std::clamp(dot(q - corner[i], along) / norm2(along), 0.0, 1.0);
    const double d2 = norm2(q - (corner[i] + along * t));
    if (d2 < nearest_d2) {
      nearest_d2 = d2;
      nearest = Vec3d{0, 0, 0};
      nearest[i] = 1.0 - t;
      nearest[j] = t;
    }
  }
  return nearest;
}

// ------------------------------------------------------------------------------ tracing
int default_max_steps(const Mesh& m) { return int(10.0 * std::sqrt(double(m.face_count()))) + 100; }

int resolve_workers(int requested) {  // kept for source compatibility (tracer.cpp:547-555)
  if (requested > 0) return requested;
  int base = int(std::max(1u, std::thread::hardware_concurrency()));
  if (const char* env = std::getenv("DIGEO_WORKERS")) {
    const int cap = std::atoi(env);
    if (cap > 0) base = std::min(base, cap);
  }
  return std::max(1, base);
}

namespace {

dg_trace_cfg to_cfg(const TraceConfig& c) {
  dg_trace_cfg k{};
  k.max_steps = c.max_steps;
  k.hole_avoidance = c.hole_avoidance;
  k.want_transport_matrix = c.want_transport_matrix;
  k.use_f32 = c.use_f32;
  k.memory = DG_MEM_HOST;
  return k;
}

// Runs a batch given as SoA and materialises the reference's result objects.
std::vector<GeodesicTrace> run_batch(const Mesh& m, const std::vector<int32_t>& face, const std::vector<double>& bary,
                                     const std::vector<double>& dir, const std::vector<double>& payload,
                                     const TraceConfig& cfg) {
  const size_t n = face.size();
  std::vector<GeodesicTrace> out(n);
  if (n == 0) return out;
  const dg_mesh* h = m.device().handle();
  std::vector<int32_t> of(n), np(n);
  std::vector<double> ob(3 * n), od(3 * n), tr(n), rq(n), pay, q;
  std::vector<uint8_t> term(n), status(n), stall(n);
  const bool any_payload = !payload.empty();
  if (any_payload) pay.resize(3 * n);
  if (cfg.want_transport_matrix) q.resize(9 * n);
  dg_trace_cfg k = to_cfg(cfg);
  dg_trace_in in{face.data(), bary.data(), dir.data(), any_payload ? payload.data() : nullptr};
  dg_trace_out o{};
  o.face = of.data(); o.bary = ob.data(); o.dir = od.data(); o.traced = tr.data(); o.requested = rq.data();
  o.term = term.data(); o.status = status.data(); o.stall = stall.data();
  o.payload = any_payload ? pay.data() : nullptr;
  o.transport = cfg.want_transport_matrix ? q.data() : nullptr;
  o.npoints = np.data();
  // record_polyline (the reference's default): one call -- the device sizes, compacts and copies the polylines
  // (dg_trace_polylines); they are read straight out of the mesh's pinned arrays below
  dg_polylines pl{};
  std::unique_lock<std::mutex> poly_lock(m.device().polyline_mutex(), std::defer_lock);
  if (cfg.record_polyline) poly_lock.lock();
  if (cfg.record_polyline) check(dg_trace_polylines(h, int64_t(n), &in, &k, &o, &pl));
  else check(dg_trace_batch(h, int64_t(n), &in, &k, &o));
  const int64_t* off = pl.offsets;
  const int32_t* pf = pl.face;
  const double *pb = pl.bary, *ps = pl.seg;
  parallel_chunks(n, [&](size_t lo, size_t hi) {
  for (size_t i = lo; i < hi; ++i) {
    GeodesicTrace& t = out[i];
    t.final_point = SurfacePoint{of[i], get3(ob.data(), i)};
    t.final_dir = get3(od.data(), i);
    t.traced_length = tr[i];
    t.requested_length = rq[i];
    t.terminated_by = TraceTermination(term[i]);
    t.status = TraceStatus(status[i]);
    if (status[i]) t.error = stall_message(stall[i]);
    const bool rejected = stall[i] == DG_STALL_FACE_RANGE || stall[i] == DG_STALL_BARY_RANGE;
    if (!rejected) {  // a rejected start is a default-constructed slot (tracer.cpp:586-591)
      const bool has_payload = any_payload && (payload[3 * i] * payload[3 * i] + payload[3 * i + 1] * payload[3 * i + 1] +
                                               payload[3 * i + 2] * payload[3 * i + 2]) > 0;
      if (has_payload) t.transported_payload = get3(pay.data(), i);
      if (cfg.want_transport_matrix) {
        Mat3 mm;
        std::copy(q.begin() + 9 * i, q.begin() + 9 * i + 9, mm.m.begin());
        t.transport_matrix = mm;
      }
    }
    if (cfg.record_polyline && np[i] > 0) {
      t.points.resize(np[i]);
      t.segment_lengths.resize(np[i] - 1);
      for (int j = 0; j < np[i]; ++j) {
        const size_t s = size_t(off[i]) + j;
        t.points[j] = SurfacePoint{pf[s], get3(pb, s)};
        if (j > 0) t.segment_lengths[j - 1] = ps[s];
      }
    }
  }
  });
  return out;
}

}  // namespace

GeodesicTrace trace(const Mesh& m, const SurfacePoint& p, const TangentVector& v, const TraceConfig& cfg) {
  // single-call contract: rejected starts throw InvalidArgs, stalls throw NumericalStall (tracer.cpp:557-562)
  if (p.face < 0 || p.face >= m.face_count()) throw InvalidArgs("trace: start face out of range");
  if (!bary_valid(p.bary, 1e-6)) throw InvalidArgs("trace: start barycentric coordinates not in the simplex");
  std::vector<double> pay;
  if (cfg.transport_payload) pay = {cfg.transport_payload->x, cfg.transport_payload->y, cfg.transport_payload->z};
  auto r = run_batch(m, {p.face}, {p.bary.x, p.bary.y, p.bary.z}, {v.dir.x, v.dir.y, v.dir.z}, pay, cfg);
  GeodesicTrace t = std::move(r[0]);
  // the reference attaches a payload whenever one was configured, even a zero one
  if (cfg.transport_payload && !t.transported_payload) t.transported_payload = Vec3d{0, 0, 0};
  if (t.status == TraceStatus::Stalled) throw NumericalStall("trace: " + t.error);
  return t;
}

std::vector<GeodesicTrace> trace_batch(const BatchRequest& req, int /*workers*/) {
  if (!req.mesh) throw InvalidArgs("trace_batch: missing mesh");
  if (req.starts.size() != req.dirs.size()) throw InvalidArgs("trace_batch: starts and dirs differ in length");
  if (!req.payloads.empty() && req.payloads.size() != req.starts.size())
    throw InvalidArgs("trace_batch: payloads must be empty or match the batch size");
  const size_t n = req.starts.size();
  std::vector<int32_t> face(n);
  std::vector<double> bary(3 * n), dir(3 * n), pay(req.payloads.empty() ? 0 : 3 * n);
  parallel_chunks(n, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      face[i] = req.starts[i].face;
      put3(bary, i, req.starts[i].bary);
      put3(dir, i, req.dirs[i].dir);  // dirs[i].anchor is ignored, as in the reference (tracer.cpp:585)
      if (!pay.empty()) put3(pay, i, req.payloads[i]);
    }
  });
  TraceConfig cfg = req.config;
  cfg.transport_payload.reset();
  return run_batch(*req.mesh, face, bary, dir, pay, cfg);
}
std::vector<GeodesicTrace> trace_batch_serial(const BatchRequest& req) { return trace_batch(req, 1); }

bool traces_bit_equal(const GeodesicTrace& a, const GeodesicTrace& b) {
  return a.points == b.points && a.segment_lengths == b.segment_lengths && a.final_point == b.final_point &&
         a.final_dir == b.final_dir && a.traced_length == b.traced_length && a.terminated_by == b.terminated_by &&
         a.status == b.status && a.transported_payload.has_value() == b.transported_payload.has_value() &&
         (!a.transported_payload || *a.transported_payload == *b.transported_payload);
}

TraceSoA trace_batch_soa(const Mesh& m, std::span<const int32_t> face, std::span<const double> bary,
                         std::span<const double> dir, std::span<const double> payload, const TraceConfig& cfg) {
  const size_t n = face.size();
  if (bary.size() != 3 * n || dir.size() != 3 * n) throw InvalidArgs("trace_batch: starts and dirs differ in length");
  if (!payload.empty() && payload.size() != 3 * n) throw InvalidArgs("trace_batch: payloads must be empty or match the batch size");
  TraceSoA r;
  r.face.resize(n); r.bary.resize(3 * n); r.dir.resize(3 * n); r.traced.resize(n); r.requested.resize(n);
  r.term.resize(n); r.status.resize(n); r.stall.resize(n); r.crossings.resize(n);
  if (!payload.empty()) r.payload.resize(3 * n);
  if (cfg.want_transport_matrix) r.transport.resize(9 * n);
  dg_trace_cfg k = to_cfg(cfg);
  dg_trace_in in{face.data(), bary.data(), dir.data(), payload.empty() ? nullptr : payload.data()};
  dg_trace_out o{};
  o.face = r.face.data(); o.bary = r.bary.data(); o.dir = r.dir.data(); o.traced = r.traced.data();
  o.requested = r.requested.data(); o.term = r.term.data(); o.status = r.status.data(); o.stall = r.stall.data();
  o.payload = r.payload.empty() ? nullptr : r.payload.data();
  o.transport = r.transport.empty() ? nullptr : r.transport.data();
  o.crossings = r.crossings.data(); o.total_crossings = &r.total_crossings;
  check(dg_trace_batch(m.device().handle(), int64_t(n), &in, &k, &o));
  return r;
}

// resident batch ------------------------------------------------------------------------
ResidentBatch::ResidentBatch(const Mesh& m, size_t capacity) {
  check(dg_batch_create(m.device().handle(), int64_t(capacity), &h_));
}
ResidentBatch::~ResidentBatch() { dg_batch_destroy(h_); }
size_t ResidentBatch::size() const { return size_t(dg_batch_size(h_)); }

TraceSoA ResidentBatch::trace(std::span<const int32_t> face, std::span<const double> bary, std::span<const double> dir,
                              const TraceConfig& cfg, const GfdConfig* gfd_follows) {
  const size_t n = face.size();
  if (bary.size() != 3 * n || dir.size() != 3 * n) throw InvalidArgs("trace_batch: starts and dirs differ in length");
  TraceSoA r;
  r.face.resize(n); r.bary.resize(3 * n); r.dir.resize(3 * n); r.traced.resize(n); r.requested.resize(n);
  r.term.resize(n); r.status.resize(n); r.stall.resize(n); r.crossings.resize(n);
  dg_trace_cfg k = to_cfg(cfg);
  dg_trace_in in{face.data(), bary.data(), dir.data(), nullptr};
  dg_trace_out o{};
  o.face = r.face.data(); o.bary = r.bary.data(); o.dir = r.dir.data(); o.traced = r.traced.data();
  o.requested = r.requested.data(); o.term = r.term.data(); o.status = r.status.data(); o.stall = r.stall.data();
  o.crossings = r.crossings.data(); o.total_crossings = &r.total_crossings;
  // gfd_follows: the backward of this step will be GFD -- the forward traces ride in GFD's round 2 as the fourth
  // sibling of their sample's re-traces, the Jacobians stay on the GPU and gfd() only pulls g back (dg_batch_trace_gfd)
  if (gfd_follows) check(dg_batch_trace_gfd(h_, int64_t(n), &in, &k, gfd_follows->eps_v, gfd_follows->eps_p, &o));
  else check(dg_batch_trace(h_, int64_t(n), &in, &k, &o));
  return r;
}

std::vector<double> ResidentBatch::ep_backward(std::span<const double> g) {
  const size_t n = size();
  if (g.size() != 3 * n) throw InvalidArgs("ep_backward: one upstream gradient per resident sample");
  std::vector<double> grad_v(3 * n);
  check(dg_batch_ep_backward(h_, g.data(), grad_v.data(), nullptr, nullptr));
  return grad_v;
}

ResidentBatch::Gfd ResidentBatch::gfd(const GfdConfig& cfg, std::span<const double> g) {
  const size_t n = size();
  if (!g.empty() && g.size() != 3 * n) throw InvalidArgs("gfd: one upstream gradient per resident sample");
  Gfd r;
  r.jv.resize(4 * n); r.jp.resize(4 * n); r.degraded.resize(4 * n);
  if (!g.empty()) { r.grad_v.resize(3 * n); r.grad_p.resize(3 * n); }
  check(dg_batch_gfd(h_, cfg.eps_v, cfg.eps_p, g.empty() ? nullptr : g.data(), 0, r.jv.data(), r.jp.data(),
                     r.degraded.data(), g.empty() ? nullptr : r.grad_v.data(), g.empty() ? nullptr : r.grad_p.data(),
                     nullptr));
  return r;
}

// single transitions --------------------------------------------------------------------
namespace {
struct Transition {
  int32_t face = -1;
  double bary[3]{}, v[3]{}, step = 0;
  uint8_t finished = 0, event = 0, stall = 0;
  int32_t rc = 0;
};
Transition transition(const Mesh& m, int which, int f, const Vec3d& b, const Vec3d& v, double remaining, bool hole) {
  Transition t;
  const int32_t face = f;
  const double bb[3] = {b.x, b.y, b.z}, vv[3] = {v.x, v.y, v.z};
  check(dg_transition(m.device().handle(), which, 1, &face, bb, vv, &remaining, hole, &t.face, t.bary, t.v, &t.step,
                      &t.finished, &t.event, &t.stall, &t.rc));
  return t;
}
}  // namespace

StepResult geodesic_step(const Mesh& m, const SurfacePoint& p, const Vec3d& v_unit, double remaining, const TraceConfig& cfg) {
  if (p.face < 0 || p.face >= m.face_count()) throw InvalidArgs("geodesic_step: face out of range");
  Transition t = transition(m, 0, p.face, p.bary, v_unit, remaining, cfg.hole_avoidance);
  if (t.rc == DG_ERR_NUMERICAL_STALL) throw NumericalStall(std::string("geodesic_step: ") + stall_message(t.stall));
  StepResult r;
  r.point = SurfacePoint{t.face, {t.bary[0], t.bary[1], t.bary[2]}};
  r.dir = {t.v[0], t.v[1], t.v[2]};
  r.step_length = t.step;
  r.finished = t.finished != 0;
  r.event = StepEvent(t.event);
  return r;
}
std::pair<SurfacePoint, Vec3d> transport_over_edge(const Mesh& m, int f, const Vec3d& b, const Vec3d& v) {
  if (f < 0 || f >= m.face_count()) throw InvalidArgs("transport_over_edge: face out of range");
  const auto cls = classify({f, b});
  if (cls.kind != PointClass::Edge) throw InvalidArgs("transport_over_edge: point is not on an edge");
  if (m.face_adjacency[f][cls.local] < 0) throw InvalidArgs("transport_over_edge: edge is on the boundary");
  Transition t = transition(m, 1, f, b, v, 0, false);
  return {SurfacePoint{t.face, {t.bary[0], t.bary[1], t.bary[2]}}, {t.v[0], t.v[1], t.v[2]}};
}
std::pair<SurfacePoint, Vec3d> transport_over_vertex(const Mesh& m, int f, const Vec3d& b, const Vec3d& v) {
  if (f < 0 || f >= m.face_count()) throw InvalidArgs("transport_over_vertex: face out of range");
  if (classify({f, b}).kind != PointClass::Vertex) throw InvalidArgs("transport_over_vertex: point is not at a vertex");
  Transition t = transition(m, 2, f, b, v, 0, false);
  if (t.rc == DG_ERR_BOUNDARY_HIT) throw BoundaryHit("transport_over_vertex: fan ends at the boundary");
  return {SurfacePoint{t.face, {t.bary[0], t.bary[1], t.bary[2]}}, {t.v[0], t.v[1], t.v[2]}};
}
std::pair<SurfacePoint, Vec3d> boundary_continue(const Mesh& m, const SurfacePoint& p, const Vec3d& v) {
  if (p.face < 0 || p.face >= m.face_count()) throw InvalidArgs("boundary_continue: face out of range");
  const auto cls = classify(p);
  if (cls.kind == PointClass::Vertex) {
    if (!m.vertex_on_boundary[m.faces[p.face][cls.local]]) throw InvalidArgs("boundary_continue: vertex is not on the boundary");
  } else if (cls.kind == PointClass::Edge) {
    if (m.face_adjacency[p.face][cls.local] >= 0) throw InvalidArgs("boundary_continue: edge is not on the boundary");
  } else {
    throw InvalidArgs("boundary_continue: point is not on the boundary");
  }
  Transition t = transition(m, 3, p.face, p.bary, v, 0, true);
  return {SurfacePoint{t.face, {t.bary[0], t.bary[1], t.bary[2]}}, {t.v[0], t.v[1], t.v[2]}};
}

// ------------------------------------------------------------------------------ differentials
GfdConfig default_gfd_config(const Mesh& m) {
  const double eps = 1e-4 * m.mean_edge_length();
  return {eps, eps};
}

namespace {

struct SampleSoA {
  std::vector<int32_t> face;
  std::vector<double> bary, v;
  explicit SampleSoA(const std::vector<GfdSample>& s) : face(s.size()), bary(3 * s.size()), v(3 * s.size()) {
    for (size_t i = 0; i < s.size(); ++i) { face[i] = s[i].p.face; put3(bary, i, s[i].p.bary); put3(v, i, s[i].v); }
  }
};

void unpack_frames(const double* f, JacobianPair& j, const SurfacePoint& p, const SurfacePoint& end) {
  j.frame_in_v = {p, get3(f, 0), get3(f, 1), get3(f, 2)};
  j.frame_in_p = {p, get3(f, 3), get3(f, 4), get3(f, 5), get3(f, 6)};
  j.frame_out = {end, get3(f, 7), get3(f, 8), get3(f, 9), get3(f, 10)};
}

}  // namespace

std::vector<JacobianPair> ep_jacobians_batch(const Mesh& m, const std::vector<GfdSample>& samples,
                                             const std::vector<GeodesicTrace>& traces) {
  const size_t n = samples.size();
  if (traces.size() != n) throw InvalidArgs("ep_jacobians_batch: samples and traces differ in length");
  std::vector<JacobianPair> out(n);
  if (n == 0) return out;
  SampleSoA s(samples);
  std::vector<int32_t> ef(n);
  std::vector<double> eb(3 * n), ed(3 * n), rot(9 * n), frames(size_t(DG_FRAME_DOUBLES) * n);
  for (size_t i = 0; i < n; ++i) {
    ef[i] = traces[i].final_point.face;
    put3(eb, i, traces[i].final_point.bary);
    put3(ed, i, traces[i].final_dir);
  }
  int64_t bad = -1;
  check(dg_ep_jacobians(m.device().handle(), int64_t(n), s.face.data(), s.bary.data(), s.v.data(), ef.data(), eb.data(),
                        ed.data(), nullptr, rot.data(), frames.data(), &bad));
  for (size_t i = 0; i < n; ++i) {
    unpack_frames(frames.data() + size_t(DG_FRAME_DOUBLES) * i, out[i], samples[i].p, traces[i].final_point);
    Mat3 r;
    std::copy(rot.begin() + 9 * i, rot.begin() + 9 * i + 9, r.m.begin());
    out[i].rotation_ep = r;
  }
  return out;
}

JacobianPair ep_jacobians(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace) {
  return ep_jacobians_batch(m, {GfdSample{p, v}}, {trace})[0];
}

std::vector<Vec3d> ep_backward_batch(const Mesh& m, const std::vector<GfdSample>& samples,
                                     const std::vector<GeodesicTrace>& traces, const std::vector<Vec3d>& g) {
  const size_t n = samples.size();
  if (traces.size() != n || g.size() != n) throw InvalidArgs("ep_backward_batch: argument lengths differ");
  std::vector<Vec3d> out(n);
  if (n == 0) return out;
  SampleSoA s(samples);
  std::vector<int32_t> ef(n);
  std::vector<double> ed(3 * n), gg(3 * n), gv(3 * n);
  for (size_t i = 0; i < n; ++i) { ef[i] = traces[i].final_point.face; put3(ed, i, traces[i].final_dir); put3(gg, i, g[i]); }
  int64_t bad = -1;
  check(dg_ep_backward(m.device().handle(), int64_t(n), s.face.data(), s.v.data(), ef.data(), ed.data(), gg.data(), nullptr,
                       gv.data(), nullptr, &bad));
  for (size_t i = 0; i < n; ++i) out[i] = get3(gv.data(), i);
  return out;
}

TangentFrame make_tangent_frame(const Mesh& m, const SurfacePoint& p, const Vec3d& v) {
  // frames come out of the same device code that the Jacobian kernels use
  if (norm(v) < 1e-12) throw DegenerateDirection("tangent frame needs a nonzero direction");
  GeodesicTrace t;
  t.final_point = p;
  t.final_dir = v;
  return ep_jacobians(m, p, v, t).frame_in_v;
}
BaryFrame make_bary_frame(const Mesh& m, const SurfacePoint& p) {
  // any in-plane direction will do for the frame_in_p block: use the first face edge
  const auto& c = m.faces[p.face];
  const Vec3d e = m.vertices[c[1]] - m.vertices[c[0]];
  GeodesicTrace t;
  t.final_point = p;
  t.final_dir = e;
  return ep_jacobians(m, p, e, t).frame_in_p;
}

std::vector<JacobianPair> gfd_batched_many(const Mesh& m, const std::vector<GfdSample>& samples, const GfdConfig& cfg,
                                           int /*workers*/) {
  const size_t n = samples.size();
  std::vector<JacobianPair> out(n);
  if (n == 0) return out;
  SampleSoA s(samples);
  std::vector<double> jv(4 * n), jp(4 * n), frames(size_t(DG_FRAME_DOUBLES) * n), bb(3 * n);
  std::vector<uint8_t> deg(4 * n);
  std::vector<int32_t> bf(n);
  int64_t bad = -1;
  check(dg_gfd_jacobians(m.device().handle(), int64_t(n), s.face.data(), s.bary.data(), s.v.data(), cfg.eps_v, cfg.eps_p,
                         nullptr, nullptr, jv.data(), jp.data(), deg.data(), frames.data(), nullptr, nullptr, bf.data(),
                         bb.data(), nullptr, &bad));
  for (size_t i = 0; i < n; ++i) {
    JacobianPair& j = out[i];
    unpack_frames(frames.data() + size_t(DG_FRAME_DOUBLES) * i, j, samples[i].p, SurfacePoint{bf[i], get3(bb.data(), i)});
    j.j_v = {jv[4 * i], jv[4 * i + 1], jv[4 * i + 2], jv[4 * i + 3]};
    j.j_p = {jp[4 * i], jp[4 * i + 1], jp[4 * i + 2], jp[4 * i + 3]};
    j.degraded_v = {deg[4 * i] != 0, deg[4 * i + 1] != 0};
    j.degraded_p = {deg[4 * i + 2] != 0, deg[4 * i + 3] != 0};
  }
  return out;
}

namespace {
void require_base(const GeodesicTrace& base) {  // diff.cpp:121-124
  if (base.status != TraceStatus::Ok || base.terminated_by != TraceTermination::LengthReached)
    throw Error("gfd: the base trace did not reach its requested length");
}
}  // namespace

JacobianPair gfd_batched(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace,
                         const GfdConfig& cfg, int workers) {
  require_base(trace);
  return gfd_batched_many(m, {GfdSample{p, v}}, cfg, workers)[0];
}
Mat2 gfd_jacobian_v(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace, const GfdConfig& cfg) {
  return gfd_batched(m, p, v, trace, cfg, 0).j_v;
}
Mat2 gfd_jacobian_p(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace, const GfdConfig& cfg) {
  return gfd_batched(m, p, v, trace, cfg, 0).j_p;
}

std::array<double, 2> frame_out_covector(const BaryFrame& f, const Vec3d& g) { return {dot(f.u_hat, g), dot(f.v_hat, g)}; }

// Accessor algebra on an already computed JacobianPair (a few dozen flops on host structs, as in
// the reference; the batched device form is dg_ep_backward / dg_gfd_jacobians with g).
std::pair<std::array<double, 2>, std::array<double, 2>> pullback(const std::array<double, 2>& grad_out,
                                                                 const JacobianPair& jac) {
  if (jac.rotation_ep) {
    const Vec3d g_tan = jac.frame_out.pinv_row0 * grad_out[0] + jac.frame_out.pinv_row1 * grad_out[1];
    const Mat3& r = *jac.rotation_ep;
    const Vec3d a = r * jac.frame_in_v.e_par, b = r * jac.frame_in_v.e_perp;
    std::array<double, 2> gv{dot(a, g_tan), dot(b, g_tan)};
    gv = jac.j_v.transposed() * gv;
    return {gv, {0.0, 0.0}};
  }
  return {jac.j_v.transposed() * grad_out, jac.j_p.transposed() * grad_out};
}
PulledGradients pullback_ambient(const Vec3d& grad_at_endpoint, const JacobianPair& jac) {
  const auto [gv, gp] = pullback(frame_out_covector(jac.frame_out, grad_at_endpoint), jac);
  return {jac.frame_in_v.e_par * gv[0] + jac.frame_in_v.e_perp * gv[1],
          jac.frame_in_p.pinv_row0 * gp[0] + jac.frame_in_p.pinv_row1 * gp[1]};
}

}  // namespace digeo
