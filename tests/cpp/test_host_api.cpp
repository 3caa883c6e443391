// C++ tests of the host shim (include/digeo_b200/digeo.hpp) on a real GPU. Restates, in the
// reference's own test style (proj/tests/test_tracer.cpp, test_diff.cpp, test_mesh.cpp), the
// assertions that pin the hot path: known answers, invariants and error behaviour. Run by
// tests/test_gpu_cpp_api.py; differential parity with the reference is tests/test_gpu_*.py.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>

#include "digeo_b200/digeo.hpp"

using namespace digeo;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) { ++g_fail; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); } \
  } while (0)
template <class E, class F> bool throws(F&& f) {
  try { f(); } catch (const E&) { return true; } catch (...) { return false; }
  return false;
}
static bool near(const Vec3d& a, const Vec3d& b, double tol) { return norm(a - b) <= tol; }

static Mesh square() { return Mesh::build({{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}}, {{0, 1, 2}, {0, 2, 3}}); }

static Mesh icosphere(int subdiv) {  // via OBJ text, which also exercises load_obj
  const double t = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<Vec3d> v = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
                          {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
  for (auto& p : v) p = normalized(p);
  std::vector<std::array<int, 3>> f = {{0, 11, 5}, {0, 5, 1}, {0, 1, 7}, {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
                                       {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4}, {3, 4, 2}, {3, 2, 6}, {3, 6, 8},
                                       {3, 8, 9}, {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7}, {9, 8, 1}};
  for (int l = 0; l < subdiv; ++l) {
    std::vector<std::array<int, 3>> nf;
    std::vector<std::array<int, 3>> seen;  // (a, b, mid)
    auto mid = [&](int a, int b) {
      if (a > b) std::swap(a, b);
      for (auto& s : seen) if (s[0] == a && s[1] == b) return s[2];
      v.push_back(normalized(v[a] + v[b]));
      seen.push_back({a, b, int(v.size()) - 1});
      return int(v.size()) - 1;
    };
    for (auto& c : f) {
      int ab = mid(c[0], c[1]), bc = mid(c[1], c[2]), ca = mid(c[2], c[0]);
      nf.push_back({c[0], ab, ca}); nf.push_back({c[1], bc, ab}); nf.push_back({c[2], ca, bc}); nf.push_back({ab, bc, ca});
    }
    f = nf;
  }
  std::ostringstream obj;
  obj.precision(17);
  for (auto& p : v) obj << "v " << p.x << " " << p.y << " " << p.z << "\n";
  for (auto& c : f) obj << "f " << c[0] + 1 << "/1/1 " << c[1] + 1 << "//2 " << c[2] + 1 << "\n";
  std::istringstream in(obj.str());
  return load_obj(in);
}

static void test_mesh() {
  Mesh ico = icosphere(0);
  for (double a : ico.vertex_total_angle) CHECK(std::abs(a - 5 * M_PI / 3) < 1e-12);  // test_mesh.cpp:81-86
  for (int f = 0; f < ico.face_count(); ++f)
    for (int k = 0; k < 3; ++k) {
      int g = ico.face_adjacency[f][k];
      CHECK(g >= 0);
      bool back = false;
      for (int j = 0; j < 3; ++j) back |= ico.face_adjacency[g][j] == f;
      CHECK(back);  // adjacency symmetry, test_mesh.cpp:153-162
    }
  CHECK(throws<NonManifoldError>([] {
    Mesh::build({{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {0, -1, 0}}, {{0, 1, 2}, {0, 1, 3}, {1, 0, 4}});
  }));
  CHECK(throws<DegenerateFaceError>([] { Mesh::build({{0, 0, 0}, {1, 0, 0}, {2, 0, 0}}, {{0, 1, 2}}); }));
  CHECK(throws<ParseError>([] { Mesh::build({{0, 0, 0}, {1, 0, 0}, {0, 1, 0}}, {{0, 1, 3}}); }));
  Mesh two = concat_meshes(ico, square());
  CHECK(two.face_count() == ico.face_count() + 2 && two.vertex_count() == ico.vertex_count() + 4);
}

static void test_square_known_answers() {
  Mesh sq = square();
  SurfacePoint p{0, {.5, .25, .25}};
  GeodesicTrace t = trace(sq, p, {p, {.25, .5, 0}});
  // proj/tests/golden/trace_square.json
  CHECK(t.points.size() == 3 && t.segment_lengths.size() == 2);
  CHECK(t.final_point.face == 1);
  CHECK(t.final_point.bary == Vec3d(0.24999999999999992, 0.75000000000000011, 0));
  CHECK(t.segment_lengths[0] == 0.55901699437494734 && t.segment_lengths[1] == 1.1102230246251565e-16);
  CHECK(t.final_dir == Vec3d(0.44721359549995771, 0.89442719099991608, 0));
  CHECK(t.terminated_by == TraceTermination::LengthReached && t.status == TraceStatus::Ok);
  // boundary stop and hole avoidance
  GeodesicTrace b = trace(sq, p, {p, {2, .1, 0}});
  CHECK(b.terminated_by == TraceTermination::Boundary && b.traced_length == 0.50062460986251966);
  CHECK(b.final_point.bary == Vec3d(0, 0.72500000000000009, 0.27499999999999997));
  TraceConfig hole;
  hole.hole_avoidance = true;
  GeodesicTrace h = trace(sq, p, {p, {2, .1, 0}}, hole);
  CHECK(h.terminated_by == TraceTermination::LengthReached && std::abs(h.traced_length - h.requested_length) < 1e-12);
  // error behaviour of the single-call wrapper
  CHECK(throws<NumericalStall>([&] { trace(sq, p, {p, {0, 0, .5}}); }));
  CHECK(throws<InvalidArgs>([&] { trace(sq, {7, {.3, .3, .4}}, {p, {1, 0, 0}}); }));
  CHECK(throws<InvalidArgs>([&] { trace(sq, {0, {.5, .5, .5}}, {p, {1, 0, 0}}); }));
  // zero vector: one point, final_dir 0
  GeodesicTrace z = trace(sq, p, {p, {0, 0, 0}});
  CHECK(z.points.size() == 1 && z.final_dir == Vec3d(0, 0, 0) && z.traced_length == 0);
  // batch: per-element error slots never throw (tracer.cpp:584-591)
  BatchRequest req;
  req.mesh = &sq;
  req.starts = {p, {7, {.3, .3, .4}}, p};
  req.dirs = {{p, {.25, .5, 0}}, {p, {1, 0, 0}}, {p, {0, 0, .5}}};
  auto out = trace_batch(req);
  CHECK(out.size() == 3 && traces_bit_equal(out[0], t));
  CHECK(out[1].status == TraceStatus::Stalled && out[1].error == "trace: start face out of range" && out[1].final_point.face == -1);
  CHECK(out[2].status == TraceStatus::Stalled && out[2].error == "initial direction is normal to the anchor face");
  BatchRequest bad = req;
  bad.dirs.pop_back();
  CHECK(throws<InvalidArgs>([&] { trace_batch(bad); }));
  bad = req;
  bad.mesh = nullptr;
  CHECK(throws<InvalidArgs>([&] { trace_batch(bad); }));
}

static void test_sphere_batch_and_transport() {
  Mesh ico = icosphere(3);
  BatchRequest req;
  req.mesh = &ico;
  req.config.want_transport_matrix = true;
  unsigned s = 12345;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return double(s >> 8) / double(1u << 24); };
  const int n = 500;
  for (int i = 0; i < n; ++i) {
    int f = int(rnd() * ico.face_count()) % ico.face_count();
    double r1 = std::sqrt(rnd()), r2 = rnd();
    SurfacePoint p{f, {1 - r1, r1 * (1 - r2), r1 * r2}};
    const auto& c = ico.faces[f];
    Vec3d e1 = normalized(ico.vertices[c[1]] - ico.vertices[c[0]]);
    Vec3d e2 = cross(ico.face_normals[f], e1);
    double phi = 2 * M_PI * rnd();
    Vec3d d = (e1 * std::cos(phi) + e2 * std::sin(phi)) * (0.2 + rnd());
    req.starts.push_back(p);
    req.dirs.push_back({p, d});
    req.payloads.push_back(e1 * std::cos(phi + 1) + e2 * std::sin(phi + 1));
  }
  auto out = trace_batch(req);
  auto again = trace_batch_serial(req);
  double sphere_err = 0;
  for (int i = 0; i < n; ++i) {
    const auto& t = out[i];
    CHECK(traces_bit_equal(t, again[i]));  // determinism, test_tracer.cpp:474-497
    CHECK(t.status == TraceStatus::Ok && std::abs(t.traced_length - t.requested_length) < 1e-9);
    CHECK(bary_valid(t.final_point.bary, 1e-9));
    double seg = 0;
    for (double l : t.segment_lengths) seg += l;
    CHECK(std::abs(seg - t.traced_length) < 1e-9);  // test_tracer.cpp:289-309
    CHECK(t.transported_payload && std::abs(norm(*t.transported_payload) - norm(req.payloads[i])) < 1e-10);
    // Q reproduces the payload transport and is an isometry on the tangent plane (:337-393)
    CHECK(t.transport_matrix && near(*t.transport_matrix * req.payloads[i], *t.transported_payload, 1e-9));
    Vec3d td = *t.transport_matrix * normalized(req.dirs[i].dir);
    CHECK(near(td, t.final_dir, 1e-9));
    // single trace == batch element, bitwise
    if (i < 20) {
      TraceConfig c = req.config;
      c.transport_payload = req.payloads[i];
      CHECK(traces_bit_equal(trace(ico, req.starts[i], req.dirs[i], c), t));
    }
    Vec3d p0 = normalized(embed(req.starts[i], ico));
    Vec3d v = req.dirs[i].dir - p0 * dot(req.dirs[i].dir, p0);
    double len = norm(req.dirs[i].dir);
    Vec3d exact = p0 * std::cos(len) + normalized(v) * std::sin(len);
    sphere_err += norm(embed(t.final_point, ico) - exact) / n;
  }
  CHECK(sphere_err < 2e-2);  // ico-3 accuracy vs the closed-form sphere exponential map
  // SoA entry point agrees with the object API
  std::vector<int32_t> face(n);
  std::vector<double> bary(3 * n), dir(3 * n);
  for (int i = 0; i < n; ++i) {
    face[i] = req.starts[i].face;
    for (int k = 0; k < 3; ++k) { bary[3 * i + k] = req.starts[i].bary[k]; dir[3 * i + k] = req.dirs[i].dir[k]; }
  }
  TraceConfig quiet;
  quiet.record_polyline = false;
  TraceSoA soa = trace_batch_soa(ico, face, bary, dir, {}, quiet);
  uint64_t crossings = 0;
  for (int i = 0; i < n; ++i) {
    CHECK(soa.face[i] == out[i].final_point.face && soa.bary[3 * i] == out[i].final_point.bary.x);
    CHECK(soa.crossings[i] == int(out[i].points.size()) - 2);
    crossings += uint64_t(soa.crossings[i]);
  }
  CHECK(soa.total_crossings == crossings);
  // max_steps guard (test_tracer.cpp:604-612)
  TraceConfig three;
  three.max_steps = 3;
  SurfacePoint p{0, {.4, .3, .3}};
  GeodesicTrace m3 = trace(icosphere(2), p, {p, {5, 1, 0}}, three);
  CHECK(m3.terminated_by == TraceTermination::MaxSteps && m3.points.size() == 4);
}

static void test_single_transitions() {
  Mesh sq = square();
  StepResult r = geodesic_step(sq, {0, {.5, .25, .25}}, {1, 2, 0}, 10.0);
  CHECK(r.event == StepEvent::CrossedEdge && r.point.face == 1 && !r.finished);
  CHECK(std::abs(r.step_length - 0.55901699437494734) < 1e-15);
  auto [q, v] = transport_over_edge(sq, 0, {.5, 0, .5}, {0.3, 0.1, 0});
  CHECK(q.face == 1 && near(v, {0.3, 0.1, 0}, 1e-14));  // coplanar transport is the identity (:136-143)
  CHECK(throws<InvalidArgs>([&] { transport_over_edge(sq, 0, {.5, .25, .25}, {1, 0, 0}); }));
  CHECK(throws<InvalidArgs>([&] { transport_over_edge(sq, 0, {0, .5, .5}, {1, 0, 0}); }));  // boundary edge
  CHECK(throws<BoundaryHit>([&] { transport_over_vertex(sq, 0, {0, 1, 0}, {1, 0, 0}); }));
  auto [b, w] = boundary_continue(sq, {0, {0, .5, .5}}, {1, .2, 0});
  CHECK(b.face == 0 && norm(w) > 0);
  Mesh ico = icosphere(1);
  auto [qv, vv] = transport_over_vertex(ico, 0, {1, 0, 0}, normalized(ico.vertices[ico.faces[0][0]] - ico.vertices[ico.faces[0][1]]));
  CHECK(qv.bary[0] == 1 || qv.bary[1] == 1 || qv.bary[2] == 1);
  CHECK(std::abs(norm(vv) - 1) < 1e-12);
}

static void test_differentials() {
  Mesh ico = icosphere(3);
  std::vector<GfdSample> samples;
  BatchRequest req;
  req.mesh = &ico;
  req.config.record_polyline = false;
  unsigned s = 99;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return double(s >> 8) / double(1u << 24); };
  for (int i = 0; i < 200; ++i) {
    int f = int(rnd() * ico.face_count()) % ico.face_count();
    double r1 = std::sqrt(rnd()), r2 = rnd();
    SurfacePoint p{f, {1 - r1, r1 * (1 - r2), r1 * r2}};
    const auto& c = ico.faces[f];
    Vec3d e1 = normalized(ico.vertices[c[1]] - ico.vertices[c[0]]);
    Vec3d e2 = cross(ico.face_normals[f], e1);
    double phi = 2 * M_PI * rnd();
    Vec3d d = (e1 * std::cos(phi) + e2 * std::sin(phi)) * (0.2 + 0.8 * rnd());
    samples.push_back({p, d});
    req.starts.push_back(p);
    req.dirs.push_back({p, d});
  }
  auto traces = trace_batch(req);
  auto eps = ep_jacobians_batch(ico, samples, traces);
  std::vector<Vec3d> g(samples.size());
  for (size_t i = 0; i < g.size(); ++i) g[i] = {rnd() - .5, rnd() - .5, rnd() - .5};
  auto gv = ep_backward_batch(ico, samples, traces, g);
  auto gfd = gfd_batched_many(ico, samples, default_gfd_config(ico));
  for (size_t i = 0; i < samples.size(); ++i) {
    const Mat3& R = *eps[i].rotation_ep;
    Mat3 I = R * R.transposed();
    for (int k = 0; k < 9; ++k) CHECK(std::abs(I.m[k] - (k % 4 == 0 ? 1.0 : 0.0)) < 1e-9);  // test_diff.cpp:65-79
    CHECK(std::abs(R.det() - 1) < 1e-9);
    if (i < 10) {
      JacobianPair one = ep_jacobians(ico, samples[i].p, samples[i].v, traces[i]);
      CHECK(one.rotation_ep->m == R.m && one.frame_out.pinv_row0 == eps[i].frame_out.pinv_row0);
      TangentFrame tf = make_tangent_frame(ico, samples[i].p, samples[i].v);
      CHECK(tf.e_par == eps[i].frame_in_v.e_par && std::abs(dot(tf.e_par, tf.e_perp)) < 1e-12);
      BaryFrame bf = make_bary_frame(ico, samples[i].p);
      CHECK(bf.pinv_row1 == eps[i].frame_in_p.pinv_row1);
    }
    PulledGradients pg = pullback_ambient(g[i], eps[i]);
    CHECK(pg.grad_v == gv[i]);                       // fused kernel == struct-level pullback, bitwise
    CHECK(pg.grad_p == Vec3d(0, 0, 0));              // EP: grad_p identically zero
    PulledGradients pf = pullback_ambient(g[i], gfd[i]);
    double c = dot(pf.grad_v, pg.grad_v) / (norm(pf.grad_v) * norm(pg.grad_v) + 1e-300);
    CHECK(c > 0.9);                                  // EP approximates GFD (test_diff.cpp:350-361 uses medians)
    CHECK(!gfd[i].degraded_v[0] && !gfd[i].degraded_p[1]);
  }
  // batched == per-sample exactly (test_diff.cpp:139-171)
  for (int i = 0; i < 5; ++i) {
    JacobianPair one = gfd_batched(ico, samples[i].p, samples[i].v, traces[i], default_gfd_config(ico));
    CHECK((one.j_v - gfd[i].j_v).max_abs() == 0 && (one.j_p - gfd[i].j_p).max_abs() == 0);
    CHECK(gfd_jacobian_v(ico, samples[i].p, samples[i].v, traces[i], default_gfd_config(ico)).a == gfd[i].j_v.a);
  }
  // resident batch: forward + EP / GFD backward on device-resident samples, same bits as the calls above
  {
    const size_t n = samples.size();
    std::vector<int32_t> face(n);
    std::vector<double> bary(3 * n), dir(3 * n), gs(3 * n);
    for (size_t i = 0; i < n; ++i) {
      face[i] = samples[i].p.face;
      for (int k = 0; k < 3; ++k) { bary[3 * i + k] = samples[i].p.bary[k]; dir[3 * i + k] = samples[i].v[k]; gs[3 * i + k] = g[i][k]; }
    }
    ResidentBatch rb(ico, n);
    TraceSoA fwd = rb.trace(face, bary, dir);
    CHECK(rb.size() == n);
    std::vector<double> rgv = rb.ep_backward(gs);
    ResidentBatch::Gfd rg = rb.gfd(default_gfd_config(ico), gs);
    for (size_t i = 0; i < n; ++i) {
      CHECK(fwd.face[i] == traces[i].final_point.face && fwd.bary[3 * i + 1] == traces[i].final_point.bary.y);
      CHECK(Vec3d(rgv[3 * i], rgv[3 * i + 1], rgv[3 * i + 2]) == gv[i]);
      CHECK(rg.jv[4 * i] == gfd[i].j_v.a && rg.jp[4 * i + 3] == gfd[i].j_p.d);
      PulledGradients pf = pullback_ambient(g[i], gfd[i]);
      CHECK(near(Vec3d(rg.grad_v[3 * i], rg.grad_v[3 * i + 1], rg.grad_v[3 * i + 2]), pf.grad_v, 1e-12));
    }
    CHECK(throws<InvalidArgs>([&] { rb.ep_backward(std::vector<double>(3)); }));
    // the forward of a GFD step: forward + Jacobians in one pass, the backward is the pull-back -- same bits
    const GfdConfig gc = default_gfd_config(ico);
    TraceSoA fused = rb.trace(face, bary, dir, {}, &gc);
    ResidentBatch::Gfd pulled = rb.gfd(gc, gs);
    int diff = 0;
    for (size_t i = 0; i < n; ++i) {
      diff += fused.face[i] != fwd.face[i] || fused.bary[3 * i] != fwd.bary[3 * i] || fused.dir[3 * i + 2] != fwd.dir[3 * i + 2] ||
              fused.traced[i] != fwd.traced[i] || fused.crossings[i] != fwd.crossings[i];
      diff += pulled.jv[4 * i + 1] != rg.jv[4 * i + 1] || pulled.jp[4 * i + 2] != rg.jp[4 * i + 2] ||
              pulled.grad_v[3 * i] != rg.grad_v[3 * i] || pulled.grad_p[3 * i + 1] != rg.grad_p[3 * i + 1];
    }
    CHECK(diff == 0 && fused.total_crossings == fwd.total_crossings);
  }
  CHECK(throws<DegenerateDirection>([&] { ep_jacobians(ico, samples[0].p, {0, 0, 0}, traces[0]); }));
  CHECK(throws<DegenerateDirection>([&] { make_tangent_frame(ico, samples[0].p, ico.face_normals[samples[0].p.face]); }));
  // GFD whole-call failure when a base trace leaves the mesh (diff.cpp:121-124)
  Mesh sq = square();
  SurfacePoint p{0, {.5, .25, .25}};
  CHECK(throws<Error>([&] { gfd_batched_many(sq, {{p, {3, .1, 0}}}, default_gfd_config(sq)); }));
  // GFD on a flat mesh: j_v and j_p are frame changes of the identity -> grad_v == grad_p == g (tangent part)
  auto flat = gfd_batched_many(sq, {{p, {.2, .1, 0}}}, default_gfd_config(sq));
  PulledGradients pp = pullback_ambient({.3, -.2, 0}, flat[0]);
  CHECK(near(pp.grad_v, {.3, -.2, 0}, 1e-6) && near(pp.grad_p, {.3, -.2, 0}, 1e-6));
}

// acceptance.cpp:173-201 with devices in the place of workers: the same request on one copy of the mesh and
// fanned out over a device set (two and three copies on GPU 0 -- the whole fork/join path on a one-GPU box)
// gives bit-identical traces, polylines included, and identical GFD Jacobians.
static void test_device_set_is_bitwise_invisible() {
  auto request = [](const Mesh& m, int n, bool polyline) {
    BatchRequest req;
    req.mesh = &m;
    req.config.record_polyline = polyline;
    unsigned s = 777;
    auto rnd = [&] { s = s * 1664525u + 1013904223u; return double(s >> 8) / double(1u << 24); };
    for (int i = 0; i < n; ++i) {
      int f = int(rnd() * m.face_count()) % m.face_count();
      double r1 = std::sqrt(rnd()), r2 = rnd();
      SurfacePoint p{f, {1 - r1, r1 * (1 - r2), r1 * r2}};
      const auto& c = m.faces[f];
      Vec3d e1 = normalized(m.vertices[c[1]] - m.vertices[c[0]]);
      Vec3d e2 = cross(m.face_normals[f], e1);
      double phi = 2 * M_PI * rnd();
      req.starts.push_back(p);
      req.dirs.push_back({p, (e1 * std::cos(phi) + e2 * std::sin(phi)) * (0.05 + 0.6 * rnd() * rnd())});
    }
    return req;
  };
  const int n = 52000;
  Mesh::set_device(0);
  Mesh one = icosphere(3);
  BatchRequest r1 = request(one, n, true);
  auto base = trace_batch(r1);
  std::vector<GfdSample> samples;
  for (int i = 0; i < n; ++i) samples.push_back({r1.starts[i], r1.dirs[i].dir});
  auto jac1 = gfd_batched_many(one, samples, default_gfd_config(one));
  for (int copies = 2; copies <= 3; ++copies) {
    Mesh::set_device_list(std::vector<int>(size_t(copies), 0));
    Mesh many = icosphere(3);
    BatchRequest r2 = request(many, n, true);
    auto fan = trace_batch(r2);
    int differ = 0;
    for (int i = 0; i < n; ++i) differ += traces_bit_equal(base[i], fan[i]) ? 0 : 1;
    CHECK(differ == 0);
    auto jac2 = gfd_batched_many(many, samples, default_gfd_config(many));
    int jdiff = 0;
    for (int i = 0; i < n; ++i)
      jdiff += ((jac1[i].j_v - jac2[i].j_v).max_abs() == 0 && (jac1[i].j_p - jac2[i].j_p).max_abs() == 0) ? 0 : 1;
    CHECK(jdiff == 0);
  }
  Mesh::set_device(0);
}

int main() {
  try {
    test_mesh();
    test_device_set_is_bitwise_invisible();
    test_square_known_answers();
    test_sphere_batch_and_transport();
    test_single_transitions();
    test_differentials();
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught exception: %s\n", e.what());
    return 2;
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
