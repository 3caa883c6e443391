// Throughput of the drop-in C++ API (std::vector<GeodesicTrace> in and out, the reference's own call shape):
// trace_batch on a torus with and without polylines, against the time the GPU call itself takes (SoA entry point).
// usage: bench_api [n = 100000]
#include <chrono>
#include <cmath>
#include <cstdio>
#include "digeo_b200/digeo.hpp"
using namespace digeo;
static double now_ms() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 100000;
  const int na = 128, nb = 64;
  std::vector<Vec3d> v;
  std::vector<std::array<int, 3>> f;
  for (int i = 0; i < na; ++i)
    for (int j = 0; j < nb; ++j) {
      double a = 2 * M_PI * i / na, b = 2 * M_PI * j / nb, w = 1.0 / 3 + std::cos(b) / 6;
      v.push_back({w * std::cos(a), w * std::sin(a), std::sin(b) / 6});
    }
  auto id = [&](int i, int j) { return (i % na) * nb + (j % nb); };
  for (int i = 0; i < na; ++i)
    for (int j = 0; j < nb; ++j) {
      f.push_back({id(i, j), id(i + 1, j), id(i + 1, j + 1)});
      f.push_back({id(i, j), id(i + 1, j + 1), id(i, j + 1)});
    }
  Mesh m = Mesh::build(v, f);
  BatchRequest req;
  req.mesh = &m;
  Rng rng(7);
  std::vector<int32_t> face(n);
  std::vector<double> bary(3 * size_t(n)), dir(3 * size_t(n));
  for (int i = 0; i < n; ++i) {
    int fc = rng.uniform_int(m.face_count());
    double r1 = std::sqrt(rng.uniform()), r2 = rng.uniform();
    SurfacePoint p{fc, {1 - r1, r1 * (1 - r2), r1 * r2}};
    const auto& c = m.faces[fc];
    Vec3d e1 = normalized(m.vertices[c[1]] - m.vertices[c[0]]), e2 = cross(m.face_normals[fc], e1);
    double phi = 2 * M_PI * rng.uniform();
    Vec3d d = (e1 * std::cos(phi) + e2 * std::sin(phi)) * 0.5;
    req.starts.push_back(p);
    req.dirs.push_back({p, d});
    face[i] = fc;
    for (int k = 0; k < 3; ++k) { bary[3 * size_t(i) + k] = p.bary[k]; dir[3 * size_t(i) + k] = d[k]; }
  }
  for (int poly = 0; poly < 2; ++poly) {
    req.config.record_polyline = poly != 0;
    auto out = trace_batch(req);
    double best = 1e30;
    size_t points = 0;
    for (int r = 0; r < 5; ++r) {
      double t0 = now_ms();
      out = trace_batch(req);
      best = std::min(best, now_ms() - t0);
    }
    for (auto& t : out) points += t.points.size();
    std::printf("trace_batch n=%d record_polyline=%d: %.2f ms (%.0f ns per geodesic, %zu polyline points)\n", n, poly, best,
                best * 1e6 / n, points);
  }
  TraceConfig cfg;
  cfg.record_polyline = false;
  auto soa = trace_batch_soa(m, face, bary, dir, {}, cfg);
  double best = 1e30;
  for (int r = 0; r < 5; ++r) {
    double t0 = now_ms();
    soa = trace_batch_soa(m, face, bary, dir, {}, cfg);
    best = std::min(best, now_ms() - t0);
  }
  std::printf("trace_batch_soa n=%d: %.2f ms, %llu face crossings\n", n, best, (unsigned long long)soa.total_crossings);
  return 0;
}
