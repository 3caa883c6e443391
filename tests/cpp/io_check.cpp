// CPU-tier check of the wire formats (no GPU call): prints the JSON of the reference's golden
// trace (proj/tests/golden/trace_square.json, values restated) plus a stalled trace with a
// payload, then round-trips the CSV and points-JSON formats.
#include <cstdio>
#include <sstream>

#include "digeo_b200/io.hpp"

using namespace digeo;

int main() {
  GeodesicTrace t;
  t.points = {{0, {0.5, 0.25, 0.25}}, {0, {0.25, 0.0, 0.75}}, {1, {0.24999999999999992, 0.75000000000000011, 0.0}}};
  t.segment_lengths = {0.55901699437494734, 1.1102230246251565e-16};
  t.final_point = t.points.back();
  t.final_dir = {0.44721359549995771, 0.89442719099991608, 0.0};
  t.traced_length = 0.55901699437494745;
  t.requested_length = 0.55901699437494745;
  GeodesicTrace s;
  s.status = TraceStatus::Stalled;
  s.error = "initial direction is normal to the anchor face";
  s.final_point = {0, {0.5, 0.25, 0.25}};
  s.requested_length = 0.5;
  s.transported_payload = Vec3d{1e-5, -2.5e20, 3.0};
  std::printf("%s\n", traces_to_json({t, s}).c_str());

  std::vector<SurfacePoint> pts = {{2, {0.5, 0.25, 0.25}}, {7, {1.0 / 3, 1.0 / 3, 1.0 / 3}}};
  std::ostringstream csv;
  write_points_csv(csv, pts);
  std::istringstream in(csv.str());
  bool ok = read_points_csv(in) == pts && points_from_json(points_to_json(pts)) == pts;
  std::vector<Vec3d> vs = {{0.1, -0.2, 1e-17}, {3, 4, 5}};
  std::ostringstream vcsv;
  write_vectors_csv(vcsv, vs);
  std::istringstream vin(vcsv.str());
  ok = ok && read_vectors_csv(vin) == vs;
  bool threw = false;
  try { std::istringstream bad("face,b0,b1,b2\n1,2,3\n"); read_points_csv(bad); } catch (const ParseError&) { threw = true; }
  try { points_from_json("{\"schema\": \"other\"}"); ok = false; } catch (const ParseError&) {}
  std::fprintf(stderr, "%s\n", ok && threw ? "IO_OK" : "IO_FAIL");
  return ok && threw ? 0 : 1;
}
