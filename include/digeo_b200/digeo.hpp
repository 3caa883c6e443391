// digeo.hpp -- host-side C++ surface of the B200 tracer, source-compatible with the reference's
// public API for the hot path (proj/include/digeo/{geometry,mesh,tracer,diff}.hpp): the same
// namespace, type names, field names, function signatures and exception types. The forwarding
// headers include/digeo/{geometry,mesh,tracer,diff}.hpp put it under the reference's include
// paths, so the reference's own callers -- gradcheck.cpp, oracles.cpp, io.cpp, opt.cpp and
// tests/acceptance.cpp, UNMODIFIED -- compile against it and link libdigeo_host.so +
// libdigeo_b200.so instead of digeo_core (tests/refdrop/Makefile builds exactly that and
// tests/test_gpu_refdrop.py runs it on the GPU).
//
// Everything that computes goes through the C-ABI in dg_b200.h (CUDA, sm_100a); there is no CPU
// tracing path behind these functions. What stays on the host is what the reference keeps in
// plain structs: the mesh arrays (filled by dg_mesh_derive), result marshalling, and the tiny
// accessor algebra on an already computed JacobianPair (pullback).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <iosfwd>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

struct dg_batch;  // include/dg_b200.h

namespace digeo {

// ---- geometry.hpp ------------------------------------------------------------------------
template <class S>
struct Vec3 {
  S x{}, y{}, z{};
  Vec3() = default;
  Vec3(S a, S b, S c) : x(a), y(b), z(c) {}
  template <class U> explicit Vec3(const Vec3<U>& o) : x(S(o.x)), y(S(o.y)), z(S(o.z)) {}
  S& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  S operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  Vec3 operator-() const { return {-x, -y, -z}; }
  Vec3 operator*(S s) const { return {x * s, y * s, z * s}; }
  Vec3 operator/(S s) const { return {x / s, y / s, z / s}; }
  Vec3& operator+=(const Vec3& o) { x += o.x; y += o.y; z += o.z; return *this; }
  Vec3& operator-=(const Vec3& o) { x -= o.x; y -= o.y; z -= o.z; return *this; }
  Vec3& operator*=(S s) { x *= s; y *= s; z *= s; return *this; }
  bool operator==(const Vec3& o) const { return x == o.x && y == o.y && z == o.z; }
};
template <class S> Vec3<S> operator*(S s, const Vec3<S>& v) { return v * s; }
template <class S> S dot(const Vec3<S>& a, const Vec3<S>& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class S> Vec3<S> cross(const Vec3<S>& a, const Vec3<S>& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class S> S norm2(const Vec3<S>& v) { return dot(v, v); }
template <class S> S norm(const Vec3<S>& v) { return std::sqrt(norm2(v)); }
template <class S> Vec3<S> normalized(const Vec3<S>& v) {
  const S n = norm(v);
  return n > S(0) ? v / n : Vec3<S>{};
}
// geometry.hpp:50-67: unsigned / signed angles (atan2 forms) and the Rodrigues rotation about a unit axis
template <class S> S angle_between(const Vec3<S>& a, const Vec3<S>& b) { return std::atan2(norm(cross(a, b)), dot(a, b)); }
template <class S> S signed_angle(const Vec3<S>& a, const Vec3<S>& b, const Vec3<S>& axis) {
  return std::atan2(dot(cross(a, b), axis), dot(a, b));
}
template <class S> Vec3<S> rotate_about(const Vec3<S>& v, const Vec3<S>& axis, S angle) {
  const S c = std::cos(angle), s = std::sin(angle);
  return v * c + cross(axis, v) * s + axis * (dot(axis, v) * (S(1) - c));
}
using Vec3d = Vec3<double>;
using Vec3f = Vec3<float>;

struct Mat3 {  // row-major
  std::array<double, 9> m{};
  static Mat3 identity() { Mat3 r; r.m = {1, 0, 0, 0, 1, 0, 0, 0, 1}; return r; }
  static Mat3 zero() { return {}; }
  static Mat3 from_columns(const Vec3d& a, const Vec3d& b, const Vec3d& c) {
    Mat3 r; r.m = {a.x, b.x, c.x, a.y, b.y, c.y, a.z, b.z, c.z}; return r;
  }
  double operator()(int r, int c) const { return m[3 * r + c]; }
  double& operator()(int r, int c) { return m[3 * r + c]; }
  Vec3d col(int c) const { return {m[c], m[3 + c], m[6 + c]}; }
  Vec3d row(int r) const { return {m[3 * r], m[3 * r + 1], m[3 * r + 2]}; }
  Vec3d operator*(const Vec3d& v) const { return {dot(row(0), v), dot(row(1), v), dot(row(2), v)}; }
  Mat3 operator*(const Mat3& o) const;
  Mat3 transposed() const;
  double det() const;
};
struct Mat2 {  // row-major
  double a = 0, b = 0, c = 0, d = 0;
  static Mat2 identity() { return {1, 0, 0, 1}; }
  static Mat2 zero() { return {}; }
  std::array<double, 2> operator*(const std::array<double, 2>& v) const { return {a * v[0] + b * v[1], c * v[0] + d * v[1]}; }
  Mat2 transposed() const { return {a, c, b, d}; }
  Mat2 operator-(const Mat2& o) const { return {a - o.a, b - o.b, c - o.c, d - o.d}; }
  double max_abs() const { return std::fmax(std::fmax(std::fabs(a), std::fabs(b)), std::fmax(std::fabs(c), std::fabs(d))); }
};

// geometry.hpp:136: coefficients of v on the in-plane basis {e1, e2} through the 2x2 Gram system
inline std::array<double, 2> plane_coefficients(const Vec3d& e1, const Vec3d& e2, const Vec3d& v) {
  const double g11 = dot(e1, e1), g12 = dot(e1, e2), g22 = dot(e2, e2);
  const double r1 = dot(e1, v), r2 = dot(e2, v);
  const double det = g11 * g22 - g12 * g12;
  return {(g22 * r1 - g12 * r2) / det, (g11 * r2 - g12 * r1) / det};
}

// geometry.hpp:146-185: the reference's deterministic generator -- xoshiro256** seeded through splitmix64, 53-bit
// uniform() -- so that samplers compiled against this header draw the reference's streams
struct Rng {
  explicit Rng(std::uint64_t seed) {
    for (auto& w : s_) {   // splitmix64
      std::uint64_t z = (seed += 0x9e3779b97f4a7c15ULL);
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      w = z ^ (z >> 31);
    }
  }
  std::uint64_t next_u64() {
    const std::uint64_t result = rotl(s_[1] * 5, 7) * 9, t = s_[1] << 17;
    s_[2] ^= s_[0]; s_[3] ^= s_[1]; s_[1] ^= s_[2]; s_[0] ^= s_[3]; s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return result;
  }
  double uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  int uniform_int(int n) { return int(next_u64() % std::uint64_t(n)); }  // in [0, n)

 private:
  static std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  std::uint64_t s_[4];
};

struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseError : Error { using Error::Error; };
struct NonManifoldError : Error { using Error::Error; };
struct DegenerateFaceError : Error { using Error::Error; };
struct NumericalStall : Error { using Error::Error; };
struct DegenerateDirection : Error { using Error::Error; };
struct NotOnSphere : Error { using Error::Error; };
struct NotTangent : Error { using Error::Error; };
struct StepTooLarge : Error { using Error::Error; };
struct MaxIterations : Error { using Error::Error; };
struct InvalidArgs : Error { using Error::Error; };
struct IOError : Error { using Error::Error; };
struct BoundaryHit : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA failure or no device (no CPU fallback)

// ---- mesh.hpp ----------------------------------------------------------------------------
inline constexpr double kBaryTol = 1e-10;
inline constexpr float kBaryTolF = 1e-6f;

struct SurfacePoint {
  int face = -1;
  Vec3d bary{0, 0, 0};
  SurfacePoint() = default;
  SurfacePoint(int f, const Vec3d& b) : face(f), bary(b) {}
  bool operator==(const SurfacePoint& o) const = default;
};
enum class PointClass { Interior, Edge, Vertex };
struct PointClassification {
  PointClass kind = PointClass::Interior;
  int local = -1;
};

class DeviceMesh;  // owns the dg_mesh handle (GPU-resident fat records)

class Mesh {
 public:
  std::vector<Vec3d> vertices;
  std::vector<std::array<int, 3>> faces;
  std::vector<std::array<int, 3>> face_adjacency;  // -1 = boundary
  std::vector<Vec3d> face_normals;
  std::vector<double> face_areas;
  std::vector<double> vertex_total_angle;
  std::vector<double> vertex_area;
  std::vector<bool> vertex_on_boundary;

  int vertex_count() const { return int(vertices.size()); }
  int face_count() const { return int(faces.size()); }
  const std::array<int, 3>& corners(int f) const { return faces[f]; }
  int corner_of(int f, int v) const {
    const auto& c = faces[f];
    return c[0] == v ? 0 : (c[1] == v ? 1 : (c[2] == v ? 2 : -1));
  }
  int neighbor(int f, int k) const { return face_adjacency[f][k]; }
  int neighbor_across(int f, int a, int b) const;
  bool edge_is_boundary(int f, int k) const { return face_adjacency[f][k] < 0; }
  double mean_edge_length() const { return mean_edge_length_; }
  double total_area() const { return total_area_; }
  std::span<const int> vertex_faces(int v) const;

  static Mesh build(std::vector<Vec3d> vertices, std::vector<std::array<int, 3>> faces);

  // GPU residency: uploaded lazily by the first compute call, shared by copies of this Mesh.
  const DeviceMesh& device() const;
  // Selects the CUDA device used by meshes uploaded afterwards (one process per GPU).
  static void set_device(int ordinal);
  // One process, several GPUs (dg_set_devices): meshes uploaded afterwards are replicated on every device of the
  // mask (bit i = CUDA device i) and trace_batch / gfd_batched_many / ep_*_batch / ResidentBatch fan each large
  // request out over them -- the GPU form of the reference's `workers` (tracer.cpp:596-603). Results stay at the
  // request index and are bitwise independent of the set.
  static void set_devices(std::uint64_t mask);
  static void set_device_list(const std::vector<int>& ordinals);  // ordered; an ordinal may repeat (tests)

 private:
  double mean_edge_length_ = 0, total_area_ = 0;
  std::vector<int> vertex_face_offsets_, vertex_face_list_;
  mutable std::shared_ptr<DeviceMesh> device_;
};

struct TangentVector {
  SurfacePoint anchor;
  Vec3d dir{0, 0, 0};
};

Mesh load_obj(std::istream& in);
Mesh load_obj_file(const std::string& path);
void write_obj(const Mesh& m, std::ostream& out);
void write_obj_file(const Mesh& m, const std::string& path);
Mesh concat_meshes(const Mesh& a, const Mesh& b);
Vec3d embed(const SurfacePoint& p, const Mesh& m);
PointClassification classify(const SurfacePoint& p, double tol = kBaryTol);
bool bary_valid(const Vec3d& b, double tol = 1e-9);
Vec3d project_to_face(const Mesh& m, int f, const Vec3d& q);  // barycentrics of the closest point of face f (mesh.cpp:233)
double total_angle(int vertex, const Mesh& m);

// ---- tracer.hpp --------------------------------------------------------------------------
enum class TraceTermination { LengthReached, Boundary, MaxSteps };
enum class TraceStatus { Ok, Stalled };

struct TraceConfig {
  int max_steps = 0;  // 0: 10*sqrt(F) + 100
  bool hole_avoidance = false;
  std::optional<Vec3d> transport_payload;
  bool want_transport_matrix = false;
  bool record_polyline = true;
  bool use_f32 = false;
};

struct GeodesicTrace {
  std::vector<SurfacePoint> points;
  std::vector<double> segment_lengths;
  SurfacePoint final_point;
  Vec3d final_dir{0, 0, 0};
  double traced_length = 0;
  double requested_length = 0;
  TraceTermination terminated_by = TraceTermination::LengthReached;
  std::optional<Vec3d> transported_payload;
  std::optional<Mat3> transport_matrix;
  TraceStatus status = TraceStatus::Ok;
  std::string error;
};
bool traces_bit_equal(const GeodesicTrace& a, const GeodesicTrace& b);

struct BatchRequest {
  const Mesh* mesh = nullptr;
  std::vector<SurfacePoint> starts;
  std::vector<TangentVector> dirs;
  std::vector<Vec3d> payloads;  // empty or one per element; a zero row means "no payload"
  TraceConfig config;
};

enum class StepEvent { Advanced, CrossedEdge, CrossedVertex, BoundarySlide, BoundaryStop };
struct StepResult {
  SurfacePoint point;
  Vec3d dir{0, 0, 0};
  double step_length = 0;
  bool finished = false;
  StepEvent event = StepEvent::Advanced;
};

StepResult geodesic_step(const Mesh& m, const SurfacePoint& p, const Vec3d& v_unit, double remaining,
                         const TraceConfig& cfg = {});
std::pair<SurfacePoint, Vec3d> transport_over_edge(const Mesh& m, int f, const Vec3d& b, const Vec3d& v);
std::pair<SurfacePoint, Vec3d> transport_over_vertex(const Mesh& m, int f, const Vec3d& b, const Vec3d& v);
std::pair<SurfacePoint, Vec3d> boundary_continue(const Mesh& m, const SurfacePoint& p, const Vec3d& v);

GeodesicTrace trace(const Mesh& m, const SurfacePoint& p, const TangentVector& v, const TraceConfig& cfg = {});
// `workers` is accepted for source compatibility; the GPU schedules the batch itself and the
// results are bitwise independent of it.
std::vector<GeodesicTrace> trace_batch(const BatchRequest& req, int workers = 0);
std::vector<GeodesicTrace> trace_batch_serial(const BatchRequest& req);
int resolve_workers(int requested);
int default_max_steps(const Mesh& m);

// SoA entry point for large batches (10^6..10^8 queries): no per-element heap objects.
struct TraceSoA {
  std::vector<int32_t> face;
  std::vector<double> bary, dir, traced, requested, payload, transport;
  std::vector<uint8_t> term, status, stall;
  std::vector<int32_t> crossings;
  uint64_t total_crossings = 0;
};
TraceSoA trace_batch_soa(const Mesh& m, std::span<const int32_t> face, std::span<const double> bary,
                         std::span<const double> dir, std::span<const double> payload, const TraceConfig& cfg);

// ---- diff.hpp ----------------------------------------------------------------------------
struct GfdConfig;

// One training step on device-resident samples (dg_batch_*): the forward exp map, then the EP or
// GFD backward of the SAME samples, without sending the forward state back to the GPU. Replaces
// the call pair trace_batch -> ep_jacobians/pullback_ambient loop | gfd_batched_many of
// gradcheck.cpp:70-89; results are bit-identical to those calls.
class ResidentBatch {
 public:
  ResidentBatch(const Mesh& m, size_t capacity);
  ~ResidentBatch();
  ResidentBatch(const ResidentBatch&) = delete;
  ResidentBatch& operator=(const ResidentBatch&) = delete;
  // plain forward exp map (cfg: max_steps / use_f32 only). gfd_follows != nullptr: the backward of this step will be
  // gfd(*gfd_follows, g) -- forward and Jacobians are then computed in one pass (the forward traces are GFD's base
  // traces, diff.cpp:288-294) and gfd() only pulls g back; same results as the separate calls.
  TraceSoA trace(std::span<const int32_t> face, std::span<const double> bary, std::span<const double> dir,
                 const TraceConfig& cfg = {}, const GfdConfig* gfd_follows = nullptr);
  // grad_v [3n] of pullback_ambient(g_i, ep_jacobians(sample_i)); grad_p is identically zero
  std::vector<double> ep_backward(std::span<const double> g);
  struct Gfd {
    std::vector<double> jv, jp;       // [4n] row-major 2x2 per sample
    std::vector<uint8_t> degraded;    // [4n] degraded_v[0..1], degraded_p[0..1]
    std::vector<double> grad_v, grad_p;  // [3n], filled when g is given
  };
  Gfd gfd(const GfdConfig& cfg, std::span<const double> g = {});
  size_t size() const;

 private:
  ::dg_batch* h_ = nullptr;
};

struct TangentFrame {
  SurfacePoint origin;
  Vec3d e_par, e_perp, normal;
};
struct BaryFrame {
  SurfacePoint origin;
  Vec3d u_hat, v_hat;
  Vec3d pinv_row0, pinv_row1;
};
struct GfdConfig {
  double eps_v = 1e-4;
  double eps_p = 1e-4;
};
GfdConfig default_gfd_config(const Mesh& m);

struct JacobianPair {
  Mat2 j_v = Mat2::identity();
  Mat2 j_p = Mat2::zero();
  TangentFrame frame_in_v;
  BaryFrame frame_in_p;
  BaryFrame frame_out;
  std::optional<Mat3> rotation_ep;
  std::array<bool, 2> degraded_v{false, false};
  std::array<bool, 2> degraded_p{false, false};
};

TangentFrame make_tangent_frame(const Mesh& m, const SurfacePoint& p, const Vec3d& v);
BaryFrame make_bary_frame(const Mesh& m, const SurfacePoint& p);
JacobianPair ep_jacobians(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace);
Mat2 gfd_jacobian_v(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace, const GfdConfig& cfg);
Mat2 gfd_jacobian_p(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace, const GfdConfig& cfg);
JacobianPair gfd_batched(const Mesh& m, const SurfacePoint& p, const Vec3d& v, const GeodesicTrace& trace,
                         const GfdConfig& cfg, int workers = 0);
struct GfdSample {
  SurfacePoint p;
  Vec3d v;
};
std::vector<JacobianPair> gfd_batched_many(const Mesh& m, const std::vector<GfdSample>& samples, const GfdConfig& cfg,
                                           int workers = 0);
std::pair<std::array<double, 2>, std::array<double, 2>> pullback(const std::array<double, 2>& grad_out,
                                                                 const JacobianPair& jac);
struct PulledGradients {
  Vec3d grad_v;
  Vec3d grad_p;
};
PulledGradients pullback_ambient(const Vec3d& grad_at_endpoint, const JacobianPair& jac);
std::array<double, 2> frame_out_covector(const BaryFrame& f, const Vec3d& g);

// Batched forms of the per-sample loop the reference runs serially (gradcheck.cpp:76-89): one
// launch for all samples.
std::vector<JacobianPair> ep_jacobians_batch(const Mesh& m, const std::vector<GfdSample>& samples,
                                             const std::vector<GeodesicTrace>& traces);
// grad_v of pullback_ambient(g, ep_jacobians(...)) for every sample, fused on the device.
std::vector<Vec3d> ep_backward_batch(const Mesh& m, const std::vector<GfdSample>& samples,
                                     const std::vector<GeodesicTrace>& traces, const std::vector<Vec3d>& g);

}  // namespace digeo
