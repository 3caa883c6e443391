// Wire formats of the reference (proj/src/io.cpp:26-166) without its JSON dependency: a small
// pretty-printer that emits what nlohmann::json::dump(2) emits for these documents (object keys
// in lexicographic order, two-space indent, shortest round-trip doubles with a trailing ".0" for
// integral values) and a minimal reader for the points schema.
#include "digeo_b200/io.hpp"

#include <cctype>
#include <charconv>
#include <istream>
#include <ostream>

namespace digeo {

namespace {

std::vector<std::string> split(const std::string& line, char sep) {
  std::vector<std::string> out;
  size_t a = 0;
  for (;;) {
    const size_t b = line.find(sep, a);
    if (b == std::string::npos) {
      if (a < line.size()) out.push_back(line.substr(a));
      return out;
    }
    out.push_back(line.substr(a, b - a));
    a = b + 1;
  }
}

template <class Row>
void read_csv(std::istream& in, const char* header_key, size_t ncols, const std::string& what,
              const char* columns, Row&& row) {
  std::string line;
  bool first = true;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (first) {
      first = false;
      if (line.find(header_key) != std::string::npos) continue;  // header row
    }
    const auto cols = split(line, ',');
    if (cols.size() != ncols) throw ParseError(what + " csv: expected " + columns);
    try {
      row(cols);
    } catch (const std::exception&) {
      throw ParseError(what + " csv: bad row '" + line + "'");
    }
  }
}

std::string num(double x) {  // shortest representation that round-trips, kept a JSON float
  char buf[40];
  const auto r = std::to_chars(buf, buf + sizeof buf, x);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".en") == std::string::npos) s += ".0";
  return s;
}

struct Writer {
  std::string s;
  int depth = 0;
  void nl() { s += '\n'; s.append(size_t(2 * depth), ' '); }
  void key(const char* k, bool first) {
    if (!first) s += ',';
    nl();
    s += '"'; s += k; s += "\": ";
  }
  void open(char c) { s += c; ++depth; }
  void close(char c, bool empty) {
    --depth;
    if (!empty) nl();
    s += c;
  }
  template <class Seq, class Item>
  void array(const Seq& seq, Item&& item) {
    open('[');
    bool first = true;
    for (const auto& e : seq) {
      if (!first) s += ',';
      first = false;
      nl();
      item(e);
    }
    close(']', first);
  }
  void vec3(const Vec3d& v) {
    const double c[3] = {v.x, v.y, v.z};
    array(c, [&](double x) { s += num(x); });
  }
  void point(const SurfacePoint& p) {
    open('{');
    key("bary", true); vec3(p.bary);
    key("face", false); s += std::to_string(p.face);
    close('}', false);
  }
  void str(const std::string& v) {
    s += '"';
    for (char c : v) {
      if (c == '"' || c == '\\') { s += '\\'; s += c; }
      else if (c == '\n') s += "\\n";
      else s += c;
    }
    s += '"';
  }
};

const char* termination_name(TraceTermination t) {
  switch (t) {
    case TraceTermination::LengthReached: return "length_reached";
    case TraceTermination::Boundary: return "boundary";
    case TraceTermination::MaxSteps: return "max_steps";
  }
  return "unknown";
}

// next JSON number at or after `pos` in `text`; advances pos past it
double next_number(const std::string& text, size_t& pos) {
  while (pos < text.size() && !(std::isdigit(static_cast<unsigned char>(text[pos])) || text[pos] == '-')) ++pos;
  size_t end = pos;
  while (end < text.size() && (std::isalnum(static_cast<unsigned char>(text[end])) || text[end] == '.' ||
                               text[end] == '-' || text[end] == '+'))
    ++end;
  double v = 0;
  const auto r = std::from_chars(text.data() + pos, text.data() + end, v);
  if (pos == end || r.ec != std::errc()) throw ParseError("points json: bad number");
  pos = end;
  return v;
}

}  // namespace

std::vector<SurfacePoint> read_points_csv(std::istream& in) {
  std::vector<SurfacePoint> pts;
  read_csv(in, "face", 4, "points", "face,b0,b1,b2", [&](const std::vector<std::string>& c) {
    pts.push_back({std::stoi(c[0]), {std::stod(c[1]), std::stod(c[2]), std::stod(c[3])}});
  });
  return pts;
}
void write_points_csv(std::ostream& out, const std::vector<SurfacePoint>& pts) {
  out.precision(17);
  out << "face,b0,b1,b2\n";
  for (const auto& p : pts) out << p.face << "," << p.bary[0] << "," << p.bary[1] << "," << p.bary[2] << "\n";
}
std::vector<Vec3d> read_vectors_csv(std::istream& in) {
  std::vector<Vec3d> vs;
  read_csv(in, "dx", 3, "vectors", "dx,dy,dz", [&](const std::vector<std::string>& c) {
    vs.push_back({std::stod(c[0]), std::stod(c[1]), std::stod(c[2])});
  });
  return vs;
}
void write_vectors_csv(std::ostream& out, const std::vector<Vec3d>& vs) {
  out.precision(17);
  out << "dx,dy,dz\n";
  for (const auto& v : vs) out << v.x << "," << v.y << "," << v.z << "\n";
}

std::string traces_to_json(const std::vector<GeodesicTrace>& traces) {
  Writer w;
  w.open('{');
  w.key("schema", true); w.str(kTracesSchema);
  w.key("traces", false);
  w.array(traces, [&](const GeodesicTrace& t) {
    w.open('{');
    bool first = true;
    auto k = [&](const char* name) { w.key(name, first); first = false; };
    if (t.status != TraceStatus::Ok) { k("error"); w.str(t.error); }
    k("final_dir"); w.vec3(t.final_dir);
    k("final_point"); w.point(t.final_point);
    k("ok"); w.s += t.status == TraceStatus::Ok ? "true" : "false";
    k("points"); w.array(t.points, [&](const SurfacePoint& p) { w.point(p); });
    k("requested_length"); w.s += num(t.requested_length);
    k("segment_lengths"); w.array(t.segment_lengths, [&](double x) { w.s += num(x); });
    k("terminated_by"); w.str(termination_name(t.terminated_by));
    k("traced_length"); w.s += num(t.traced_length);
    if (t.transported_payload) { k("transported_payload"); w.vec3(*t.transported_payload); }
    w.close('}', false);
  });
  w.close('}', false);
  return w.s;
}

std::string points_to_json(const std::vector<SurfacePoint>& pts) {
  Writer w;
  w.open('{');
  w.key("points", true);
  w.array(pts, [&](const SurfacePoint& p) { w.point(p); });
  w.key("schema", false); w.str(kPointsSchema);
  w.close('}', false);
  return w.s;
}

std::vector<SurfacePoint> points_from_json(const std::string& text) {
  // {"points": [{"bary": [a, b, c], "face": n}, ...], "schema": "digeo.points/1"}
  if (text.find(std::string("\"") + kPointsSchema + "\"") == std::string::npos)
    throw ParseError("points json: unexpected schema");
  size_t pos = text.find("\"points\"");
  if (pos == std::string::npos) throw ParseError("points json: missing points");
  std::vector<SurfacePoint> out;
  for (;;) {
    const size_t obj = text.find('{', pos + 1);
    if (obj == std::string::npos) break;
    const size_t close = text.find('}', obj);
    if (close == std::string::npos) throw ParseError("points json: unterminated object");
    const std::string item = text.substr(obj, close - obj + 1);
    size_t b = item.find("\"bary\""), f = item.find("\"face\"");
    if (b == std::string::npos || f == std::string::npos) throw ParseError("points json: point needs face and bary");
    SurfacePoint p;
    b += 6;
    p.bary.x = next_number(item, b);
    p.bary.y = next_number(item, b);
    p.bary.z = next_number(item, b);
    f += 6;
    p.face = int(next_number(item, f));
    out.push_back(p);
    pos = close;
  }
  return out;
}

void write_traces_obj(std::ostream& out, const Mesh& m, const std::vector<GeodesicTrace>& traces) {
  out.precision(17);
  int base = 1;
  for (const auto& t : traces) {
    for (const auto& p : t.points) {
      const Vec3d q = embed(p, m);
      out << "v " << q.x << " " << q.y << " " << q.z << "\n";
    }
    if (t.points.size() >= 2) {
      out << "l";
      for (size_t i = 0; i < t.points.size(); ++i) out << " " << base + int(i);
      out << "\n";
    }
    base += int(t.points.size());
  }
}

}  // namespace digeo
