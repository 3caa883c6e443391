// TEST INFRASTRUCTURE ONLY -- not part of the product path.
//
// C-ABI shim over the UNMODIFIED reference library (digeo, C++20/OpenMP) so that
// tests/ and bench.py's cpu_baseline / --impl reference legs can drive the real
// reference through ctypes. The reference sources are compiled where they lie
// under /root/reference/proj/src by oracle/Makefile into oracle/_ref/libdigeo_ref.so;
// nothing from the reference is copied into this repository. This file only
// marshals plain arrays <-> the reference's own types and calls its public API:
//   Mesh::build                 proj/src/mesh.cpp:34
//   trace_batch / trace         proj/src/tracer.cpp:596 / :557
//   geodesic_step & friends     proj/src/tracer.cpp:630-735
//   ep_jacobians / pullback     proj/src/diff.cpp:44 / :328 / :347
//   gfd_batched(_many), gfd_jacobian_v/p   proj/src/diff.cpp:208-326
//   make_icosphere ... make_cone           proj/src/oracles.cpp:183-316
//   sample_surface_point / sample_tangent  proj/src/io.cpp:168-197
//   run_gradcheck               proj/src/gradcheck.cpp:46
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "digeo/diff.hpp"
#include "digeo/gradcheck.hpp"
#include "digeo/io.hpp"
#include "digeo/mesh.hpp"
#include "digeo/oracles.hpp"
#include "digeo/tracer.hpp"

using namespace digeo;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

void put_err(char* buf, int len, const std::string& s) {
  g_err = s;
  if (buf && len > 0) {
    std::strncpy(buf, s.c_str(), size_t(len) - 1);
    buf[len - 1] = 0;
  }
}

// Error class ids shared with tests/refapi.py.
int classify_error(const std::exception& e) {
  if (dynamic_cast<const InvalidArgs*>(&e)) return 1;
  if (dynamic_cast<const ParseError*>(&e)) return 3;
  if (dynamic_cast<const NonManifoldError*>(&e)) return 4;
  if (dynamic_cast<const DegenerateFaceError*>(&e)) return 5;
  if (dynamic_cast<const DegenerateDirection*>(&e)) return 6;
  if (dynamic_cast<const NumericalStall*>(&e)) return 10;
  if (dynamic_cast<const BoundaryHit*>(&e)) return 11;
  if (dynamic_cast<const Error*>(&e)) return 7;
  return 99;
}

Vec3d v3(const double* p) { return {p[0], p[1], p[2]}; }
void st3(double* p, const Vec3d& v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }

using Result = std::vector<GeodesicTrace>;

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- mesh ----

REF_API void* ref_mesh_build(const double* xyz, int nv, const int32_t* tri, int nf,
                             int* err_class, char* err, int errlen) {
  try {
    std::vector<Vec3d> v(nv);
    for (int i = 0; i < nv; ++i) v[i] = v3(xyz + 3 * i);
    std::vector<std::array<int, 3>> f(nf);
    for (int i = 0; i < nf; ++i) f[i] = {tri[3 * i], tri[3 * i + 1], tri[3 * i + 2]};
    if (err_class) *err_class = 0;
    return new Mesh(Mesh::build(std::move(v), std::move(f)));
  } catch (const std::exception& e) {
    if (err_class) *err_class = classify_error(e);
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

REF_API void* ref_mesh_load_obj(const char* path, int* err_class, char* err, int errlen) {
  try {
    if (err_class) *err_class = 0;
    return new Mesh(load_obj_file(path));
  } catch (const std::exception& e) {
    if (err_class) *err_class = classify_error(e);
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

REF_API void ref_mesh_free(void* h) { delete static_cast<Mesh*>(h); }
REF_API int ref_mesh_nv(void* h) { return static_cast<Mesh*>(h)->vertex_count(); }
REF_API int ref_mesh_nf(void* h) { return static_cast<Mesh*>(h)->face_count(); }
REF_API double ref_mesh_mean_edge(void* h) { return static_cast<Mesh*>(h)->mean_edge_length(); }
REF_API double ref_mesh_total_area(void* h) { return static_cast<Mesh*>(h)->total_area(); }
REF_API int ref_default_max_steps(void* h) { return default_max_steps(*static_cast<Mesh*>(h)); }

// Any output pointer may be null.
REF_API void ref_mesh_get(void* h, double* xyz, int32_t* tri, int32_t* adj, double* fnormal,
                          double* farea, double* vangle, double* varea, uint8_t* vboundary,
                          int32_t* csr_off, int32_t* csr_list) {
  const Mesh& m = *static_cast<Mesh*>(h);
  const int nv = m.vertex_count(), nf = m.face_count();
  for (int i = 0; i < nv; ++i) {
    if (xyz) st3(xyz + 3 * i, m.vertices[i]);
    if (vangle) vangle[i] = m.vertex_total_angle[i];
    if (varea) varea[i] = m.vertex_area[i];
    if (vboundary) vboundary[i] = m.vertex_on_boundary[i] ? 1 : 0;
  }
  for (int f = 0; f < nf; ++f) {
    for (int k = 0; k < 3; ++k) {
      if (tri) tri[3 * f + k] = m.faces[f][k];
      if (adj) adj[3 * f + k] = m.face_adjacency[f][k];
    }
    if (fnormal) st3(fnormal + 3 * f, m.face_normals[f]);
    if (farea) farea[f] = m.face_areas[f];
  }
  if (csr_off || csr_list) {
    int pos = 0;
    for (int v = 0; v < nv; ++v) {
      if (csr_off) csr_off[v] = pos;
      for (int g : m.vertex_faces(v)) {
        if (csr_list) csr_list[pos] = g;
        ++pos;
      }
    }
    if (csr_off) csr_off[nv] = pos;
  }
}

REF_API void* ref_concat_meshes(void* a, void* b) {
  return new Mesh(concat_meshes(*static_cast<Mesh*>(a), *static_cast<Mesh*>(b)));
}

// -------------------------------------------------------------- fixtures ----

REF_API void* ref_make_icosphere(int subdiv) { return new Mesh(make_icosphere(subdiv)); }
REF_API void* ref_make_torus(double R, double r, int na, int nb) {
  return new Mesh(make_torus(R, r, na, nb));
}
REF_API void* ref_make_plane(int nx, int ny, double size, uint64_t seed) {
  return new Mesh(make_plane(nx, ny, size, seed));
}
REF_API void* ref_make_cylinder(double radius, double height, int na, int nh) {
  return new Mesh(make_cylinder(radius, height, na, nh));
}
REF_API void* ref_make_cone(double radius, double height, int na) {
  return new Mesh(make_cone(radius, height, na));
}

// n x { sample_surface_point, sample_tangent(min_len, max_len) } from Rng(seed), the
// reference's own query distribution (gradcheck.cpp:55-58 draws them in this order).
REF_API void ref_sample_queries(void* h, uint64_t seed, int n, double min_len, double max_len,
                                int32_t* face, double* bary, double* dir) {
  const Mesh& m = *static_cast<Mesh*>(h);
  Rng rng(seed);
  for (int i = 0; i < n; ++i) {
    SurfacePoint p = sample_surface_point(m, rng);
    TangentVector v = sample_tangent(m, p, rng, min_len, max_len);
    face[i] = p.face;
    st3(bary + 3 * i, p.bary);
    st3(dir + 3 * i, v.dir);
  }
}

REF_API void ref_sphere_exp(const double* p, const double* v, double* out) {
  st3(out, sphere_exp(v3(p), v3(v)));
}

// ----------------------------------------------------------------- trace ----

// Runs trace_batch (workers >= 0) or trace_batch_serial (workers < 0) and keeps the
// reference's own result vector behind an opaque handle.
REF_API void* ref_trace_batch(void* h, int64_t n, const int32_t* face, const double* bary,
                              const double* dir, const double* payload, int max_steps,
                              int hole_avoidance, int want_q, int record_polyline, int use_f32,
                              int workers, int* err_class, char* err, int errlen) {
  try {
    BatchRequest req;
    req.mesh = static_cast<Mesh*>(h);
    req.starts.resize(n);
    req.dirs.resize(n);
    if (payload) req.payloads.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      req.starts[i] = SurfacePoint{face[i], v3(bary + 3 * i)};
      req.dirs[i] = TangentVector{req.starts[i], v3(dir + 3 * i)};
      if (payload) req.payloads[i] = v3(payload + 3 * i);
    }
    req.config.max_steps = max_steps;
    req.config.hole_avoidance = hole_avoidance != 0;
    req.config.want_transport_matrix = want_q != 0;
    req.config.record_polyline = record_polyline != 0;
    req.config.use_f32 = use_f32 != 0;
    if (err_class) *err_class = 0;
    if (workers < 0) return new Result(trace_batch_serial(req));
    return new Result(trace_batch(req, workers));
  } catch (const std::exception& e) {
    if (err_class) *err_class = classify_error(e);
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

REF_API void ref_result_free(void* r) { delete static_cast<Result*>(r); }
REF_API int64_t ref_result_size(void* r) { return int64_t(static_cast<Result*>(r)->size()); }

// SoA view of the result; any pointer may be null. has_payload/has_q are per-element flags.
REF_API void ref_result_soa(void* r, int32_t* face, double* bary, double* dir, double* traced,
                            double* requested, uint8_t* term, uint8_t* status, double* payload,
                            uint8_t* has_payload, double* q, uint8_t* has_q, int32_t* npoints) {
  const Result& res = *static_cast<Result*>(r);
  for (size_t i = 0; i < res.size(); ++i) {
    const GeodesicTrace& t = res[i];
    if (face) face[i] = t.final_point.face;
    if (bary) st3(bary + 3 * i, t.final_point.bary);
    if (dir) st3(dir + 3 * i, t.final_dir);
    if (traced) traced[i] = t.traced_length;
    if (requested) requested[i] = t.requested_length;
    if (term) term[i] = uint8_t(t.terminated_by);
    if (status) status[i] = uint8_t(t.status);
    if (has_payload) has_payload[i] = t.transported_payload ? 1 : 0;
    if (payload) st3(payload + 3 * i, t.transported_payload.value_or(Vec3d{0, 0, 0}));
    if (has_q) has_q[i] = t.transport_matrix ? 1 : 0;
    if (q) {
      Mat3 m = t.transport_matrix.value_or(Mat3::zero());
      for (int k = 0; k < 9; ++k) q[9 * i + k] = m.m[k];
    }
    if (npoints) npoints[i] = int32_t(t.points.size());
  }
}

// Flattened polylines: point j of trace i lands at offsets[i] + j. Segment j of trace i
// (between points j and j+1) lands at offsets[i] + j + 1; slot offsets[i] holds 0.
REF_API void ref_result_polyline(void* r, const int64_t* offsets, int32_t* pface, double* pbary,
                                 double* pseg) {
  const Result& res = *static_cast<Result*>(r);
  for (size_t i = 0; i < res.size(); ++i) {
    const GeodesicTrace& t = res[i];
    int64_t o = offsets[i];
    for (size_t j = 0; j < t.points.size(); ++j) {
      pface[o + j] = t.points[j].face;
      st3(pbary + 3 * (o + j), t.points[j].bary);
      pseg[o + j] = j == 0 ? 0.0 : t.segment_lengths[j - 1];
    }
  }
}

REF_API int ref_result_error(void* r, int64_t i, char* buf, int len) {
  const Result& res = *static_cast<Result*>(r);
  put_err(buf, len, res[size_t(i)].error);
  return int(res[size_t(i)].error.size());
}

REF_API int ref_result_bit_equal(void* a, void* b) {
  const Result& x = *static_cast<Result*>(a);
  const Result& y = *static_cast<Result*>(b);
  if (x.size() != y.size()) return 0;
  for (size_t i = 0; i < x.size(); ++i)
    if (!traces_bit_equal(x[i], y[i])) return 0;
  return 1;
}

REF_API const char* ref_traces_json(void* r) {
  thread_local std::string s;
  s = traces_to_json(*static_cast<Result*>(r));
  return s.c_str();
}

// Single trace through digeo::trace (throws NumericalStall on a stall, InvalidArgs on bad input).
REF_API void* ref_trace_single(void* h, int face, const double* bary, const double* dir,
                               const double* payload, int max_steps, int hole_avoidance,
                               int want_q, int record_polyline, int use_f32, int* err_class,
                               char* err, int errlen) {
  try {
    TraceConfig cfg;
    cfg.max_steps = max_steps;
    cfg.hole_avoidance = hole_avoidance != 0;
    cfg.want_transport_matrix = want_q != 0;
    cfg.record_polyline = record_polyline != 0;
    cfg.use_f32 = use_f32 != 0;
    if (payload) cfg.transport_payload = v3(payload);
    SurfacePoint p{face, v3(bary)};
    if (err_class) *err_class = 0;
    auto* out = new Result;
    out->push_back(trace(*static_cast<Mesh*>(h), p, TangentVector{p, v3(dir)}, cfg));
    return out;
  } catch (const std::exception& e) {
    if (err_class) *err_class = classify_error(e);
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

// ---------------------------------------------- single-transition operations ----

REF_API int ref_geodesic_step(void* h, int face, const double* bary, const double* v_unit,
                              double remaining, int hole_avoidance, int32_t* out_face,
                              double* out_bary, double* out_dir, double* step_length,
                              int* finished, int* event, char* err, int errlen) {
  try {
    TraceConfig cfg;
    cfg.hole_avoidance = hole_avoidance != 0;
    StepResult r = geodesic_step(*static_cast<Mesh*>(h), {face, v3(bary)}, v3(v_unit),
                                 remaining, cfg);
    *out_face = r.point.face;
    st3(out_bary, r.point.bary);
    st3(out_dir, r.dir);
    *step_length = r.step_length;
    *finished = r.finished ? 1 : 0;
    *event = int(r.event);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return classify_error(e);
  }
}

// which: 0 = transport_over_edge, 1 = transport_over_vertex, 2 = boundary_continue
REF_API int ref_transition(void* h, int which, int face, const double* bary, const double* v,
                           int32_t* out_face, double* out_bary, double* out_v, char* err,
                           int errlen) {
  try {
    const Mesh& m = *static_cast<Mesh*>(h);
    std::pair<SurfacePoint, Vec3d> r;
    if (which == 0) r = transport_over_edge(m, face, v3(bary), v3(v));
    else if (which == 1) r = transport_over_vertex(m, face, v3(bary), v3(v));
    else r = boundary_continue(m, {face, v3(bary)}, v3(v));
    *out_face = r.first.face;
    st3(out_bary, r.first.bary);
    st3(out_v, r.second);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return classify_error(e);
  }
}

// ------------------------------------------------------------------ diff ----

namespace {

// Frame block per sample (27 doubles): e_par, e_perp, normal | u_hat, v_hat, pinv0, pinv1
// of frame_in_p (12) ... laid out by write_frames below.
constexpr int kFrameDoubles = 9 + 12 + 12;

void write_frames(double* f, const JacobianPair& j) {
  st3(f + 0, j.frame_in_v.e_par);
  st3(f + 3, j.frame_in_v.e_perp);
  st3(f + 6, j.frame_in_v.normal);
  st3(f + 9, j.frame_in_p.u_hat);
  st3(f + 12, j.frame_in_p.v_hat);
  st3(f + 15, j.frame_in_p.pinv_row0);
  st3(f + 18, j.frame_in_p.pinv_row1);
  st3(f + 21, j.frame_out.u_hat);
  st3(f + 24, j.frame_out.v_hat);
  st3(f + 27, j.frame_out.pinv_row0);
  st3(f + 30, j.frame_out.pinv_row1);
}

void write_mat2(double* o, const Mat2& m) { o[0] = m.a; o[1] = m.b; o[2] = m.c; o[3] = m.d; }

}  // namespace

REF_API int ref_frame_doubles() { return kFrameDoubles; }

// ep_jacobians + pullback_ambient looped over samples (the reference calls them in a
// serial for, gradcheck.cpp:76-89). g may be null (then grad_v/grad_p are not written).
REF_API int ref_ep(void* h, int64_t n, const int32_t* face, const double* bary, const double* v,
                   const int32_t* end_face, const double* end_bary, const double* end_dir,
                   const double* g, double* rot, double* frames, double* grad_v, double* grad_p,
                   int64_t* err_index, char* err, int errlen) {
  const Mesh& m = *static_cast<Mesh*>(h);
  for (int64_t i = 0; i < n; ++i) {
    try {
      GeodesicTrace t;
      t.final_point = SurfacePoint{end_face[i], v3(end_bary + 3 * i)};
      t.final_dir = v3(end_dir + 3 * i);
      JacobianPair j = ep_jacobians(m, {face[i], v3(bary + 3 * i)}, v3(v + 3 * i), t);
      if (rot) for (int k = 0; k < 9; ++k) rot[9 * i + k] = j.rotation_ep->m[k];
      if (frames) write_frames(frames + kFrameDoubles * i, j);
      if (g) {
        PulledGradients pg = pullback_ambient(v3(g + 3 * i), j);
        if (grad_v) st3(grad_v + 3 * i, pg.grad_v);
        if (grad_p) st3(grad_p + 3 * i, pg.grad_p);
      }
    } catch (const std::exception& e) {
      if (err_index) *err_index = i;
      put_err(err, errlen, e.what());
      return classify_error(e);
    }
  }
  return 0;
}

// mode 0: gfd_batched_many; mode 1: per-sample trace + gfd_batched; mode 2: per-sample
// trace + gfd_jacobian_v / gfd_jacobian_p (unbatched).  g may be null.
REF_API int ref_gfd(void* h, int mode, int64_t n, const int32_t* face, const double* bary,
                    const double* v, double eps_v, double eps_p, int workers, const double* g,
                    double* jv, double* jp, uint8_t* degraded, double* frames, double* grad_v,
                    double* grad_p, char* err, int errlen) {
  const Mesh& m = *static_cast<Mesh*>(h);
  try {
    GfdConfig cfg{eps_v, eps_p};
    std::vector<JacobianPair> jacs;
    if (mode == 0) {
      std::vector<GfdSample> s(n);
      for (int64_t i = 0; i < n; ++i) s[i] = {{face[i], v3(bary + 3 * i)}, v3(v + 3 * i)};
      jacs = gfd_batched_many(m, s, cfg, workers);
    } else {
      jacs.resize(n);
      TraceConfig tc;
      tc.record_polyline = false;
      for (int64_t i = 0; i < n; ++i) {
        SurfacePoint p{face[i], v3(bary + 3 * i)};
        Vec3d vv = v3(v + 3 * i);
        GeodesicTrace base = trace(m, p, {p, vv}, tc);
        if (mode == 1) {
          jacs[i] = gfd_batched(m, p, vv, base, cfg, workers);
        } else {
          jacs[i].frame_in_v = make_tangent_frame(m, p, vv);
          jacs[i].frame_in_p = make_bary_frame(m, p);
          jacs[i].frame_out = make_bary_frame(m, base.final_point);
          jacs[i].j_v = gfd_jacobian_v(m, p, vv, base, cfg);
          jacs[i].j_p = gfd_jacobian_p(m, p, vv, base, cfg);
        }
      }
    }
    for (int64_t i = 0; i < n; ++i) {
      const JacobianPair& j = jacs[i];
      if (jv) write_mat2(jv + 4 * i, j.j_v);
      if (jp) write_mat2(jp + 4 * i, j.j_p);
      if (degraded) {
        degraded[4 * i + 0] = j.degraded_v[0];
        degraded[4 * i + 1] = j.degraded_v[1];
        degraded[4 * i + 2] = j.degraded_p[0];
        degraded[4 * i + 3] = j.degraded_p[1];
      }
      if (frames) write_frames(frames + kFrameDoubles * i, j);
      if (g) {
        PulledGradients pg = pullback_ambient(v3(g + 3 * i), j);
        if (grad_v) st3(grad_v + 3 * i, pg.grad_v);
        if (grad_p) st3(grad_p + 3 * i, pg.grad_p);
      }
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return classify_error(e);
  }
}

REF_API double ref_default_gfd_eps(void* h) {
  return default_gfd_config(*static_cast<Mesh*>(h)).eps_v;
}

// run_gradcheck medians: out = {median_cos_v, median_norm_ratio_v, median_cos_p,
// median_norm_ratio_p, max_p_grad_norm}. scheme: 0 = EP, 1 = GFD.
REF_API int ref_gradcheck(void* h, int scheme, int n, uint64_t seed, double min_len,
                          double max_len, int workers, double* out, char* err, int errlen) {
  try {
    GradCheckReport r = run_gradcheck(*static_cast<Mesh*>(h),
                                      scheme ? DiffScheme::Gfd : DiffScheme::Ep, n, seed,
                                      min_len, max_len, workers);
    out[0] = r.median_cos_v;
    out[1] = r.median_norm_ratio_v;
    out[2] = r.median_cos_p;
    out[3] = r.median_norm_ratio_p;
    out[4] = r.max_p_grad_norm;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return classify_error(e);
  }
}

REF_API int ref_resolve_workers(int requested) { return resolve_workers(requested); }
