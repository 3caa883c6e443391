// Straightest-geodesic state machine, one geodesic per thread.
//
// WHAT it computes is fixed by the reference (proj/src/tracer.cpp, struct Kernel<S>, :44-529);
// every method below cites the lines it restates. HOW it runs is different: the walker reads
// fat face records (dg_mesh_view.cuh) so that entering a face is a single gather, keeps the
// record of the current face in registers, never indexes a register array dynamically, and is
// written as a re-entrant step() so that a warp can refill finished lanes between steps
// (dg_kernels.cu). The floating-point expression trees follow the reference operation for
// operation and the library is compiled with -fmad=false, so an f64 trace that never takes a
// vertex branch (no libm calls) is bit-identical to the reference's CPU build.
#pragma once

#include "dg_mesh_view.cuh"

namespace dg {

// codes shared with include/dg_b200.h
enum : uint8_t { kTermLength = 0, kTermBoundary = 1, kTermMaxSteps = 2 };
enum : uint8_t { kStatusOk = 0, kStatusStalled = 1 };
enum : uint8_t { kStallNone = 0, kStallDegenerateDir = 1, kStallNoExit = 2, kStallNormalDir = 3,
                 kStallFaceRange = 4, kStallBaryRange = 5 };
enum : uint8_t { kEvAdvanced = 0, kEvCrossedEdge = 1, kEvCrossedVertex = 2, kEvBoundarySlide = 3,
                 kEvBoundaryStop = 4 };

enum class Outcome : int { Continue = 0, Finished = 1, Boundary = 2, Maxed = 3, Stalled = 4 };

// tracer.cpp:14-27
template <class S> struct Tol;
template <> struct Tol<double> {
  static DG_HD double bary() { return 1e-10; }
  static DG_HD double dir_rel() { return 1e-12; }
  static DG_HD double angle() { return 1e-12; }
};
template <> struct Tol<float> {
  static DG_HD float bary() { return 1e-6f; }
  static DG_HD float dir_rel() { return 1e-5f; }
  static DG_HD float angle() { return 1e-5f; }
};

template <class S> DG_HD S dg_inf();
template <> DG_HD double dg_inf<double>() { return HUGE_VAL; }
template <> DG_HD float dg_inf<float>() { return HUGE_VALF; }

// Fold isometry across an edge, tracer.cpp:33-42.
template <class S>
struct EdgeTransport {
  V3<S> edge, in_from, in_to;
  DG_HD V3<S> operator()(const V3<S>& w) const { return edge * dot(w, edge) - in_to * dot(w, in_from); }
};
template <class S> struct PlaneProject {  // w - n (w.n), tracer.cpp:332,435
  V3<S> n;
  DG_HD V3<S> operator()(const V3<S>& w) const { return w - n * dot(w, n); }
};
template <class S> struct AxisRotate {  // tracer.cpp:301
  V3<S> axis; S angle;
  DG_HD V3<S> operator()(const V3<S>& w) const { return rotate_about(w, axis, angle); }
};

// Optional polyline sink: slot j of this trace lives at base + j. cap > 0: the trace owns `cap` slots only (the
// capped first pass of one-call recording, dg_trace_polylines); points beyond them are counted, not written.
struct PolySink {
  int32_t* face;
  double* bary;
  double* seg;
  int64_t base;  // < 0: not recording
  int32_t cap;   // 0: unbounded
  DG_HD bool room(int npoints) const { return cap == 0 || npoints < cap; }
};

// kFull = payload / transport-matrix / hole-avoidance / polyline support compiled in. The lite
// instantiation is the plain forward exp map (the benchmarked path) and carries 26 fewer live
// f64 registers per thread.
// kCached = crossings read the per-half-edge transport cache (f64 only; MeshView::he != null).
template <class S, bool kFull, bool kCached = false>
struct Tracer {
  const MeshView& m;
  int max_steps;
  bool hole_avoidance;

  int face;
  V3<S> bary, dir;
  S remaining, target;
  Face<S> cur;  // record of `face`

  bool has_payload, want_q;
  V3<S> payload, q0, q1, q2;
  S payload_norm;

  double traced;
  int npoints, crossings, steps;
  uint8_t status, stall_code, term, last_event;
  PolySink sink;

  DG_HD Tracer(const MeshView& mesh, int max_steps_, bool hole)
      : m(mesh), max_steps(max_steps_), hole_avoidance(hole) {
    reset();
  }

  DG_HD void reset() {
    face = 0;
    bary = dir = V3<S>{S(0), S(0), S(0)};
    remaining = target = S(0);
    has_payload = want_q = false;
    payload = V3<S>{S(0), S(0), S(0)};
    payload_norm = S(0);
    q0 = unit_axis<S>(0); q1 = unit_axis<S>(1); q2 = unit_axis<S>(2);
    traced = 0.0;
    npoints = crossings = steps = 0;
    status = kStatusOk; stall_code = kStallNone; term = kTermLength; last_event = kEvAdvanced;
    sink.base = -1; sink.cap = 0;
  }

  DG_HD void set_face(int f) { face = f; cur = load_face<S>(m, f); }

  // tracer.cpp:75-82
  DG_HD V3<double> widened_bary() const {
    V3<double> b{double(bary.x), double(bary.y), double(bary.z)};
    double s = b.x + b.y + b.z;
    if (s > 0 && s != 1.0) b = b / s;
    return b;
  }

  // tracer.cpp:84-89
  DG_HD void push_point(S seg_len) {
    traced += double(seg_len);
    if (kFull && sink.base >= 0 && sink.room(npoints)) {
      V3<double> b = widened_bary();
      int64_t o = sink.base + npoints;
      sink.face[o] = face;
      sink.bary[3 * o] = b.x; sink.bary[3 * o + 1] = b.y; sink.bary[3 * o + 2] = b.z;
      sink.seg[o] = double(seg_len);
    }
    ++npoints;
  }
  DG_HD void push_start() {
    if (kFull && sink.base >= 0 && sink.room(npoints)) {
      V3<double> b = widened_bary();
      int64_t o = sink.base + npoints;
      sink.face[o] = face;
      sink.bary[3 * o] = b.x; sink.bary[3 * o + 1] = b.y; sink.bary[3 * o + 2] = b.z;
      sink.seg[o] = 0.0;
    }
    ++npoints;
  }

  // tracer.cpp:91-103
  template <class Map>
  DG_HD void apply_transport(const Map& t) {
    if (!kFull) return;
    if (has_payload) {
      payload = t(payload);
      S n = norm(payload);
      if (n > S(0)) payload = payload * (payload_norm / n);
    }
    if (want_q) {
      q0 = t(q0); q1 = t(q1); q2 = t(q2);
    }
  }

  // tracer.cpp:106-111 with positions already in hand.
  static DG_HD V3<S> edge_inward(const V3<S>& a, const V3<S>& e, const V3<S>& off) {
    V3<S> w = off - a;
    return normalized(w - e * dot(w, e));
  }
  // tracer.cpp:113-126. xa/xc: positions of the shared edge, off_*: the third vertex of each face.
  static DG_HD EdgeTransport<S> make_edge_transport(const V3<S>& xa, const V3<S>& xc,
                                                    const V3<S>& off_from, const V3<S>& off_to) {
    EdgeTransport<S> t;
    t.edge = normalized(xc - xa);
    t.in_from = edge_inward(xa, t.edge, off_from);
    t.in_to = edge_inward(xa, t.edge, off_to);
    return t;
  }

  // tracer.cpp:130-138
  static DG_HD void wedge_coeffs(const Face<S>& g, int k, const V3<S>& w, S* c1, S* c2) {
    V3<S> x0 = g.pos(k);
    V3<S> e1 = g.pos(k == 2 ? 0 : k + 1) - x0;
    V3<S> e2 = g.pos(k == 0 ? 2 : k - 1) - x0;
    S g11 = dot(e1, e1), g12 = dot(e1, e2), g22 = dot(e2, e2);
    S det = g11 * g22 - g12 * g12;
    S r1 = dot(e1, w), r2 = dot(e2, w);
    div_pair(g22 * r1 - g12 * r2, g11 * r2 - g12 * r1, det, c1, c2);
  }
  // tracer.cpp:140-146
  static DG_HD bool wedge_contains(const Face<S>& g, int k, const V3<S>& w) {
    S c1, c2;
    wedge_coeffs(g, k, w, &c1, &c2);
    S mag = dg_abs(c1) + dg_abs(c2);
    if (mag <= S(0)) return false;
    S tol = Tol<S>::dir_rel() * mag;
    return c1 >= -tol && c2 >= -tol;
  }

  // tracer.cpp:148-161
  DG_HD void snap_bary() {
    if (bary.x <= Tol<S>::bary()) bary.x = S(0);
    if (bary.y <= Tol<S>::bary()) bary.y = S(0);
    if (bary.z <= Tol<S>::bary()) bary.z = S(0);
    S s = bary.x + bary.y + bary.z;
    if (s > S(0)) bary = div_pos(bary, s);
    const S hi = S(1) - Tol<S>::bary();
    if (bary.x >= hi) bary = unit_axis<S>(0);
    else if (bary.y >= hi) bary = unit_axis<S>(1);
    else if (bary.z >= hi) bary = unit_axis<S>(2);
  }
  // tracer.cpp:163-167
  DG_HD int vertex_corner() const {
    if (bary.x == S(1)) return 0;
    if (bary.y == S(1)) return 1;
    if (bary.z == S(1)) return 2;
    return -1;
  }
  DG_HD Outcome stall(uint8_t why) {
    status = kStatusStalled;
    stall_code = why;
    return Outcome::Stalled;
  }

  // lambda = max(0, -b / v) of tracer.cpp:190-191 for a candidate (v < 0, b >= +0), computed so
  // that no lane ever divides a zero (CUDA's f64 division takes a long slow path for a zero
  // quotient, and b is exactly 0 for the corner opposite the entry edge): (-0)/v is +0 for v < 0.
  // Lanes without a candidate in this slot (valid == false) divide 1 by -1 and are ignored.
  static DG_HD S exit_param(S b, S v, bool valid) {
    const bool z = !valid || b == S(0);
    const S q = nonzero_numerator(valid ? -b : S(0), z) / (valid ? v : S(-1));
    S lambda = z ? S(0) : q;
    if (lambda < S(0)) lambda = S(0);
    return lambda;
  }

  // tracer.cpp:177-223
  DG_HD Outcome advance() {
    S bv1, bv2;
    wedge_coeffs(cur, 0, dir, &bv1, &bv2);
    V3<S> bv{-(bv1 + bv2), bv1, bv2};

    S scale = dg_abs(bv.x) + dg_abs(bv.y) + dg_abs(bv.z);
    if (!dg_finite(double(scale)) || scale <= S(0)) return stall(kStallDegenerateDir);
    S tol = Tol<S>::dir_rel() * scale;

    // Exit candidates are the components with bv_i < -tol, scanned in index order with a strict
    // '<' (first wins ties), tracer.cpp:186-196. The velocity sums to zero, so at most two
    // components qualify: the two candidate quotients are computed in two branch-free slots
    // (A = lowest candidate index, B = the next one) instead of three divergent branches.
    const bool c0 = !(bv.x >= -tol), c1 = !(bv.y >= -tol), c2 = !(bv.z >= -tol);
    const int ia = c0 ? 0 : (c1 ? 1 : (c2 ? 2 : -1));
    const int ib = c0 ? (c1 ? 1 : (c2 ? 2 : -1)) : ((c1 && c2) ? 2 : -1);
    S best = dg_inf<S>();
    int exit_edge = -1;
    {
      const S lambda = exit_param(get(bary, ia), get(bv, ia), ia >= 0);
      if (ia >= 0 && lambda < best) { best = lambda; exit_edge = ia; }
    }
    {
      const S lambda = exit_param(get(bary, ib), get(bv, ib), ib >= 0);
      if (ib >= 0 && lambda < best) { best = lambda; exit_edge = ib; }
    }
    if (c0 && c1 && c2) {  // unreachable for finite inputs; kept for exact reference semantics
      const S lambda = exit_param(bary.z, bv.z, true);
      if (lambda < best) { best = lambda; exit_edge = 2; }
    }
    if (exit_edge < 0) return stall(kStallNoExit);

    if (best >= remaining) {
      bary = bary + bv * remaining;
      snap_bary();
      push_point(remaining);
      remaining = S(0);
      last_event = kEvAdvanced;
      return Outcome::Finished;
    }

    bary = bary + bv * best;
    put(bary, exit_edge, S(0));
    snap_bary();
    remaining -= best;
    push_point(best);

    if (vertex_corner() >= 0) {
      last_event = kEvAdvanced;
      return Outcome::Continue;  // vertex branch on the next transition
    }
    if (get(bary, exit_edge) != S(0)) {
      last_event = kEvAdvanced;
      return Outcome::Continue;
    }
    return cross_edge(exit_edge);
  }

  // tracer.cpp:225-248
  DG_HD Outcome cross_edge(int k) {
    int g = cur.adj(k);
    if (g < 0) {
      if (kFull && hole_avoidance) return slide_from_edge(k);
      last_event = kEvBoundaryStop;
      return Outcome::Boundary;
    }
    const int ka = k == 2 ? 0 : k + 1, kc = k == 0 ? 2 : k - 1;
    const S wa = get(bary, ka), wc = get(bary, kc);
    V3<S> nb{S(0), S(0), S(0)};
    Face<S> G;
    if (kCached) {
      // the fold isometry and the corner map of this half-edge were computed at upload
      const HalfEdge h = load_halfedge(m, face, k);
      G = load_face<S>(m, g);
      EdgeTransport<S> t{cast<S>(h.edge), cast<S>(h.in_from), cast<S>(h.in_to)};
      dir = normalized(t(dir));
      apply_transport(t);
      put(nb, h.ja, wa);
      put(nb, h.jc, wc);
    } else {
      const int va = cur.id(ka), vc = cur.id(kc);
      G = load_face<S>(m, g);
      EdgeTransport<S> t =
          make_edge_transport(cur.pos(ka), cur.pos(kc), cur.pos(k), G.pos_of(G.third(va, vc)));
      dir = normalized(t(dir));
      apply_transport(t);
      put(nb, G.corner_of(va), wa);
      put(nb, G.corner_of(vc), wc);
    }
    face = g;
    cur = G;
    bary = nb;
    snap_bary();
    ++crossings;
    last_event = kEvCrossedEdge;
    return Outcome::Continue;
  }

  // tracer.cpp:252-311. Returns false when the fan ends at the boundary first.
  DG_HD bool fan_walk(int x0) {
    S theta = S(m.vangle[x0]);
    S half = theta / S(2);
    V3<S> x0p = cur.pos_of(x0);
    V3<S> rev = -dir;

    int k0 = cur.corner_of(x0);
    int p1 = cur.id(k0 == 2 ? 0 : k0 + 1);
    int p2 = cur.id(k0 == 0 ? 2 : k0 - 1);
    S a1 = angle_between(rev, cur.pos_of(p1) - x0p);
    S a2 = angle_between(rev, cur.pos_of(p2) - x0p);

    int x1 = a1 <= a2 ? p1 : p2;
    S alpha = a2 < a1 ? a2 : a1;  // std::min(a1, a2)
    int g = face;
    Face<S> G = cur;
    int near_vertex = -1;
    V3<S> near_pos{S(0), S(0), S(0)};
    V3<S> x1p = G.pos_of(x1);
    V3<S> carried = dir;

    int guard = (m.csr_off[x0 + 1] - m.csr_off[x0]) + 2;
    while (alpha < half - Tol<S>::angle()) {
      if (--guard < 0) return false;
      int gn = G.neighbor_across(x0, x1);
      if (gn < 0) return false;
      Face<S> GN = load_face<S>(m, gn);
      // the interior angle of the fan face at x0: from the table built at upload (the same function of the same
      // corner vectors -- the cross product's sign is the only thing the order of the two changes, and the angle
      // takes its norm), fetched beside the face record; computed here in the f32 lane and without a table
      const bool tabled = sizeof(S) == sizeof(double) && m.cangle != nullptr;
      V3<double> corner_angles{0.0, 0.0, 0.0};
      if (tabled) corner_angles = load_corner_angles(m, gn);
      int x2 = GN.third(x0, x1);
      V3<S> x2p = GN.pos_of(x2);
      if (tabled) alpha += S(get(corner_angles, GN.corner_of(x0)));
      else alpha += angle_between(x1p - x0p, x2p - x0p);
      EdgeTransport<S> t = make_edge_transport(x0p, x1p, G.pos_of(G.third(x0, x1)), x2p);
      carried = t(carried);
      apply_transport(t);
      near_vertex = x1;
      near_pos = x1p;
      g = gn;
      G = GN;
      x1 = x2;
      x1p = x2p;
      ++crossings;
    }

    S beta = alpha - half;
    if (!(S(0) < beta)) beta = S(0);  // std::max(S(0), alpha - half)
    V3<S> e_far = normalized(x1p - x0p);
    V3<S> n_g = load_normal<S>(m, g);
    V3<S> e_near = near_vertex >= 0 ? normalized(near_pos - x0p) : rev;
    // the reference takes the sign of signed_angle (tracer.cpp:294): only the sign is computed, the same predicate
    S side = signed_angle_nonneg(e_far, e_near, n_g) ? S(1) : S(-1);
    V3<S> outgoing = rotate_about(e_far, n_g, side * beta);
    outgoing = normalized(outgoing - n_g * dot(outgoing, n_g));

    if (kFull && (has_payload || want_q)) {
      V3<S> carried_in_plane = normalized(carried - n_g * dot(carried, n_g));
      S rho = signed_angle(carried_in_plane, outgoing, n_g);
      apply_transport(AxisRotate<S>{n_g, rho});
    }

    face = g;
    cur = G;
    bary = unit_axis<S>(G.corner_of(x0));
    dir = outgoing;
    last_event = kEvCrossedVertex;
    return true;
  }

  // ---- hole avoidance, tracer.cpp:316-405 -------------------------------------------------
  // Returns Continue with *then_advance = true when the reference calls advance() right away.
  DG_HD Outcome blue_vertex(int x0, bool* then_advance) {
    int best_face = -1;
    S best_err = dg_inf<S>();
    const int beg = m.csr_off[x0], end = m.csr_off[x0 + 1];
    for (int i = beg; i < end; ++i) {
      int g = m.csr_list[i];
      V3<S> n = load_normal<S>(m, g);
      V3<S> proj = dir - n * dot(dir, n);
      if (norm(proj) < S(1e-6)) continue;
      Face<S> G = load_face<S>(m, g);
      if (!wedge_contains(G, G.corner_of(x0), proj)) continue;
      S err = angle_between(dir, proj);
      if (err < best_err) { best_err = err; best_face = g; }
    }
    if (best_face >= 0) {
      PlaneProject<S> project{load_normal<S>(m, best_face)};
      dir = normalized(project(dir));
      apply_transport(project);
      set_face(best_face);
      bary = unit_axis<S>(cur.corner_of(x0));
      last_event = kEvBoundarySlide;
      *then_advance = true;
      return Outcome::Continue;
    }
    return slide_from_vertex(x0);
  }

  DG_HD Outcome slide_from_vertex(int x0) {
    int best_to = -1, best_face = -1;
    S best_align = -dg_inf<S>();
    const int beg = m.csr_off[x0], end = m.csr_off[x0 + 1];
    for (int i = beg; i < end; ++i) {
      int g = m.csr_list[i];
      Face<S> G = load_face<S>(m, g);
      int k0 = G.corner_of(x0);
      for (int off = 1; off <= 2; ++off) {
        int kc = (k0 + off) % 3;
        int y = G.id(kc);
        int opp = 3 - k0 - kc;  // corner opposite edge (x0, y)
        if (G.adj(opp) >= 0) continue;
        S align = dot(dir, normalized(G.pos(kc) - G.pos(k0)));
        if (align > best_align || (align == best_align && y < best_to)) {
          best_align = align;
          best_to = y;
          best_face = g;
        }
      }
    }
    if (best_to < 0) {
      last_event = kEvBoundaryStop;
      return Outcome::Boundary;
    }
    return slide_along(best_face, x0, best_to, S(0));
  }

  DG_HD Outcome slide_from_edge(int k) {
    const int ka = k == 2 ? 0 : k + 1, kc = k == 0 ? 2 : k - 1;
    int va = cur.id(ka), vc = cur.id(kc);
    V3<S> pos = cur.pos(ka) * get(bary, ka) + cur.pos(kc) * get(bary, kc);
    S da = dot(dir, normalized(cur.pos(ka) - pos));
    S dc = dot(dir, normalized(cur.pos(kc) - pos));
    int to = da >= dc ? va : vc;
    int from = to == va ? vc : va;
    S t0 = to == va ? get(bary, ka) : get(bary, kc);  // weight of `to`
    return slide_along(face, from, to, t0);
  }

  DG_HD Outcome slide_along(int g, int from, int to, S t0) {
    if (g != face) set_face(g);
    S edge_len = norm(cur.pos_of(to) - cur.pos_of(from));
    S left = edge_len * (S(1) - t0);
    S consume = remaining < left ? remaining : left;  // std::min(left, remaining)
    S t1 = t0 + consume / edge_len;

    bary = V3<S>{S(0), S(0), S(0)};
    put(bary, cur.corner_of(from), S(1) - t1);
    put(bary, cur.corner_of(to), t1);
    snap_bary();
    remaining -= consume;
    push_point(consume);
    last_event = kEvBoundarySlide;
    if (remaining <= S(0)) {
      remaining = S(0);
      return Outcome::Finished;
    }
    return Outcome::Continue;
  }

  // tracer.cpp:408-449. *then_advance is set when the reference tail-calls advance().
  DG_HD Outcome at_vertex(int k0, bool* then_advance) {
    int x0 = cur.id(k0);
    if (kFull && hole_avoidance && m.vboundary[x0]) return blue_vertex(x0, then_advance);

    // (one call site of fan_walk for both of the reference's -- arriving through this face, and no face to
    // re-anchor in: the walk is inlined, and a second copy of it is a sixth of the kernel's instructions)
    if (!wedge_contains(cur, k0, -dir)) {  // not arriving through this face
      if (wedge_contains(cur, k0, dir)) {
        *then_advance = true;
        return Outcome::Continue;
      }

      // departing into some other incident face: re-anchor with the best inward margin
      int best_face = -1;
      S best_margin = -dg_inf<S>();
      const int beg = m.csr_off[x0], end = m.csr_off[x0 + 1];
      for (int i = beg; i < end; ++i) {
        int g = m.csr_list[i];
        Face<S> G = load_face<S>(m, g);
        S c1, c2;
        wedge_coeffs(G, G.corner_of(x0), dir, &c1, &c2);
        S mag = dg_abs(c1) + dg_abs(c2);
        if (mag <= S(0)) continue;
        S margin = (c2 < c1 ? c2 : c1) / mag;  // std::min(c1, c2) / mag
        if (margin > best_margin) { best_margin = margin; best_face = g; }
      }
      if (best_face >= 0 && best_margin >= -Tol<S>::dir_rel()) {
        PlaneProject<S> project{load_normal<S>(m, best_face)};
        V3<S> proj = project(dir);
        if (norm(proj) > S(0)) {
          dir = normalized(proj);
          apply_transport(project);
          set_face(best_face);
          bary = unit_axis<S>(cur.corner_of(x0));
          *then_advance = true;
          return Outcome::Continue;
        }
      }
    }
    if (fan_walk(x0)) return Outcome::Continue;
    last_event = kEvBoundaryStop;
    return Outcome::Boundary;
  }

  // tracer.cpp:451-455. advance() is instantiated once: the vertex branches that tail-call it
  // in the reference fall through to the same call site here.
  DG_HD Outcome step() {
    int k0 = vertex_corner();
    if (k0 >= 0) {
      bool then_advance = false;
      Outcome oc = at_vertex(k0, &then_advance);
      if (!then_advance) return oc;
    }
    return advance();
  }

  // tracer.cpp:457-488 (+ run_one :578-592 for the payload rule). Returns false when the trace
  // must not run (rejected start or normal direction); status/stall are then set.
  DG_HD bool initialise(int f, const V3<double>& b, const V3<double>& v, const V3<double>& pay,
                        bool has_pay, bool want_matrix) {
    if (f < 0 || f >= m.nf) {
      face = -1;
      stall(kStallFaceRange);
      return false;
    }
    {  // bary_valid(b, 1e-6), mesh.cpp:225-231
      const double tol = 1e-6;
      double s = b.x + b.y + b.z;
      bool ok = !(fabs(s - 1.0) > tol);
      if (b.x < -tol || b.x > 1.0 + tol) ok = false;
      if (b.y < -tol || b.y > 1.0 + tol) ok = false;
      if (b.z < -tol || b.z > 1.0 + tol) ok = false;
      if (!ok) {
        face = -1;
        stall(kStallBaryRange);
        return false;
      }
    }
    set_face(f);
    bary = cast<S>(b);
    snap_bary();

    target = S(norm(v));
    remaining = target;

    V3<S> n = load_normal<S>(m, face);
    V3<S> vv = cast<S>(v);
    V3<S> in_plane = vv - n * dot(vv, n);
    if (target > S(0) && norm(in_plane) < S(1e-12) * target) {
      stall(kStallNormalDir);
      return false;
    }
    dir = normalized(in_plane);

    if (kFull && has_pay) {
      has_payload = true;
      payload = cast<S>(pay);
      payload_norm = norm(payload);
    }
    want_q = kFull && want_matrix;
    push_start();
    return true;
  }

  // One iteration of the run loop, tracer.cpp:497-504. Returns true while the trace is live.
  DG_HD bool run_step() {
    if (!(remaining > S(0))) return false;
    if (steps++ >= max_steps) {
      term = kTermMaxSteps;
      return false;
    }
    Outcome oc = step();
    if (oc == Outcome::Continue) return true;
    if (oc == Outcome::Boundary) term = kTermBoundary;
    return false;
  }
};

}  // namespace dg
