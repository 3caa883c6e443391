// Small-batch latency of the host API (the opt.cpp:298-323 use: ~50 seeds, transport matrix on).
#include <chrono>
#include <cmath>
#include <cstdio>
#include "digeo_b200/digeo.hpp"
using namespace digeo;
int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 50;
  // octahedron subdivided a few times via concat-free builder: reuse an icosphere-like mesh from a torus grid
  const int na = 64, nb = 32;
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
  req.config.want_transport_matrix = true;
  req.config.record_polyline = false;
  for (int i = 0; i < n; ++i) {
    int face = (i * 7919) % m.face_count();
    SurfacePoint p{face, {0.3, 0.3, 0.4}};
    const auto& c = m.faces[face];
    Vec3d d = normalized(m.vertices[c[1]] - m.vertices[c[0]]) * 0.3;
    req.starts.push_back(p);
    req.dirs.push_back({p, d});
  }
  auto out = trace_batch(req);
  const int reps = 200;
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) out = trace_batch(req);
  double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
  std::printf("trace_batch n=%d want_transport_matrix: %.1f us per call (status %d)\n", n, us, int(out[0].status));
  return 0;
}
