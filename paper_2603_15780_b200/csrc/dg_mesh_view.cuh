// Device mesh layout ("fat face records") and its register-resident view.
//
// The reference keeps an indexed mesh (vertices[], faces[], face_adjacency[],
// proj/include/digeo/mesh.hpp:42-49) and re-fetches positions through two dependent
// lookups on every crossing (tracer.cpp:72, :113-126). On B200 the walk is a chain of
// dependent L2 gathers, so the device layout trades capacity for chain depth: ONE 96-byte,
// 32-byte-aligned record per face holds everything a trace needs while it is inside that
// face -- the three corner positions, the three vertex ids and the three neighbour ids.
// Entering a face costs exactly one gather of three 32-B sectors; 1 M faces = 96 MB, which
// stays resident in the 126 MB L2.
//
// Word order inside the record is chosen so that it is read with six 128-bit loads
// (or three 256-bit loads): x[0..7] | x[8], v0, v1 | v2, a0, a1, a2.
#pragma once

#include "dg_math.cuh"

namespace dg {

struct alignas(32) FaceRec {
  double x[9];     // corner positions, x[3*k + c] = coordinate c of corner k (exact copies of Mesh::vertices)
  int32_t v[3];    // vertex ids of the corners                       (Mesh::faces[f])
  int32_t adj[3];  // face across the edge opposite corner k, -1 = boundary (Mesh::face_adjacency[f])
};
static_assert(sizeof(FaceRec) == 96, "FaceRec must be three 32-byte sectors");

// Optional per-directed-half-edge crossing record (slot 3 f + k = leaving face f through the
// edge opposite corner k): everything the walker needs to cross that edge and to take its next
// step inside the entered face g, in ONE 128-byte line:
//   * the fold isometry of tracer.cpp:113-126 (unit edge, in-plane edge normals of both faces).
//     It depends only on the mesh, so it is computed once at upload -- by the same device
//     functions the uncached walker runs, hence bit-identical -- and a crossing needs no sqrt /
//     normalisation of edge frames;
//   * the two corner-0 edge vectors of g, exactly as wedge_coeffs (tracer.cpp:130-138) forms them
//     (x1 - x0, x2 - x0), which is all advance() reads of a face on the fast path;
//   * g itself and the corner map of the shared edge in g.
// The walk is then a chain of single-line gathers, record(3 f + k).g -> record(3 g + k').
// The profile that led here: with 6 sectors per crossing in two records the kernel sat at 75 % of
// the L1TEX -> crossbar request rate (one sector request per cycle per SM, profiles/).
struct alignas(128) HalfEdgeRec {
  double t[9];      // edge, in_from, in_to (unit vectors)
  double e[6];      // entered face: x1 - x0, x2 - x0
  int32_t g;        // face entered (-1 = boundary)
  int32_t corners;  // ja | jc << 2 | jt << 4: corners of va, vc and of the third vertex in g
};
static_assert(sizeof(HalfEdgeRec) == 128, "HalfEdgeRec must be one 128-byte line");

// The crossing record of the TOLERANCE lane (DG_LANE_FAST): half the size. In the intrinsic form of the fold a
// crossing needs the shared edge vector E = xc - xa, the third vertex of the entered face relative to xa, W = xt - xa,
// and 1 / |E|: with e = E / |E| and in_to = unit(W - e (W.e)) the transported direction is
// e (d.e) + in_to sqrt(1 - (d.e)^2) -- the unit direction d lies in the plane of the face it leaves, so its component
// along that face's inward edge normal is -sqrt(1 - (d.e)^2) and in_from is never needed --, and the barycentric
// velocity in the entered face follows from the same numbers (v_t = beta / |W_perp|, v_c = (alpha - v_t W.e) / |E|)
// without a Gram solve. Not the reference's operation sequence: results agree to rounding (1e-13 of the diagonal),
// not to the bit, which is why only the tolerance lane reads it. One 64-byte half line = two 32-byte sectors.
struct alignas(64) HalfEdgeRec64 {
  double E[3];      // xc - xa (a, c: the end points of the crossed edge, corners (k + 1) % 3 and (k + 2) % 3 of the face left)
  double W[3];      // xt - xa (t: the third vertex of the entered face)
  double inv_len;   // 1 / |E|
  int32_t g;        // face entered (-1 = boundary)
  int32_t corners;  // ja | jc << 2 | jt << 4, as HalfEdgeRec
};
static_assert(sizeof(HalfEdgeRec64) == 64, "HalfEdgeRec64 must be two 32-byte sectors");

struct MeshView {
  const FaceRec* rec;        // [nf]
  const HalfEdgeRec* he;     // [3 nf] or null (transport cache off)
  const double* fnormal;     // [3 nf] unit face normals                  (Mesh::face_normals)
  const double* vangle;      // [nv]   total interior angle per vertex    (Mesh::vertex_total_angle)
  const int32_t* csr_off;    // [nv+1] vertex -> incident faces, face order (mesh.cpp:118-127)
  const int32_t* csr_list;   // [3 nf]
  const uint8_t* vboundary;  // [nv]   (Mesh::vertex_on_boundary)
  int32_t nf, nv;
  const HalfEdgeRec64* he64 = nullptr;  // [3 nf] or null: the tolerance lane's half-size crossing records
  // [3 nf] or null: interior angle of face f at corner k -- angle_between(x_{k+1} - x_k, x_{k+2} - x_k), computed at
  // upload by the device function the fan walk (tracer.cpp:252-311) would call per fan face; f64 lane only
  const double* cangle = nullptr;
};

// Register copy of one face record in the stepping scalar type S.
template <class S>
struct Face {
  V3<S> x0, x1, x2;
  int v0, v1, v2;
  int a0, a1, a2;

  DG_HD V3<S> pos(int k) const { return k == 0 ? x0 : (k == 1 ? x1 : x2); }
  DG_HD int id(int k) const { return sel3(k, v0, v1, v2); }
  DG_HD int adj(int k) const { return sel3(k, a0, a1, a2); }
  // Mesh::corner_of (mesh.hpp:56)
  DG_HD int corner_of(int v) const { return v0 == v ? 0 : (v1 == v ? 1 : (v2 == v ? 2 : -1)); }
  // position of the corner holding vertex id v
  DG_HD V3<S> pos_of(int v) const { return v0 == v ? x0 : (v1 == v ? x1 : x2); }
  // the vertex that is neither a nor b (the reference scans the corners and keeps the last hit,
  // tracer.cpp:115-120; ids of a face are distinct so there is exactly one)
  DG_HD int third(int a, int b) const {
    int r = -1;
    if (v0 != a && v0 != b) r = v0;
    if (v1 != a && v1 != b) r = v1;
    if (v2 != a && v2 != b) r = v2;
    return r;
  }
  // Mesh::neighbor_across (mesh.cpp:21-27)
  DG_HD int neighbor_across(int a, int b) const {
    if ((v1 == a && v2 == b) || (v1 == b && v2 == a)) return a0;
    if ((v2 == a && v0 == b) || (v2 == b && v0 == a)) return a1;
    if ((v0 == a && v1 == b) || (v0 == b && v1 == a)) return a2;
    return -1;
  }
};

template <class S>
DG_HD Face<S> load_face(const MeshView& m, int f) {
  Face<S> r;
#ifdef __CUDA_ARCH__
  const double2* p = reinterpret_cast<const double2*>(m.rec + f);
  double2 d0 = __ldg(p + 0), d1 = __ldg(p + 1), d2 = __ldg(p + 2), d3 = __ldg(p + 3);
  const int4* q = reinterpret_cast<const int4*>(p + 4);
  int4 w0 = __ldg(q + 0), w1 = __ldg(q + 1);
  double x8 = __hiloint2double(w0.y, w0.x);
  r.x0 = {S(d0.x), S(d0.y), S(d1.x)};
  r.x1 = {S(d1.y), S(d2.x), S(d2.y)};
  r.x2 = {S(d3.x), S(d3.y), S(x8)};
  r.v0 = w0.z; r.v1 = w0.w; r.v2 = w1.x;
  r.a0 = w1.y; r.a1 = w1.z; r.a2 = w1.w;
#else
  const FaceRec& c = m.rec[f];
  r.x0 = {S(c.x[0]), S(c.x[1]), S(c.x[2])};
  r.x1 = {S(c.x[3]), S(c.x[4]), S(c.x[5])};
  r.x2 = {S(c.x[6]), S(c.x[7]), S(c.x[8])};
  r.v0 = c.v[0]; r.v1 = c.v[1]; r.v2 = c.v[2];
  r.a0 = c.adj[0]; r.a1 = c.adj[1]; r.a2 = c.adj[2];
#endif
  return r;
}

struct HalfEdge {
  V3<double> edge, in_from, in_to;
  int g, ja, jc, jt;
};
DG_HD HalfEdge load_halfedge(const MeshView& m, int f, int k) {
  HalfEdge h;
  const HalfEdgeRec* r = m.he + (3 * size_t(f) + size_t(k));
#ifdef __CUDA_ARCH__
  const double2* p = reinterpret_cast<const double2*>(r);
  double2 d0 = __ldg(p + 0), d1 = __ldg(p + 1), d2 = __ldg(p + 2), d3 = __ldg(p + 3);
  const double t8 = __ldg(&r->t[8]);
  const int2 w = __ldg(reinterpret_cast<const int2*>(&r->g));
  h.edge = {d0.x, d0.y, d1.x};
  h.in_from = {d1.y, d2.x, d2.y};
  h.in_to = {d3.x, d3.y, t8};
  h.g = w.x;
  const int c = w.y;
#else
  h.edge = {r->t[0], r->t[1], r->t[2]};
  h.in_from = {r->t[3], r->t[4], r->t[5]};
  h.in_to = {r->t[6], r->t[7], r->t[8]};
  h.g = r->g;
  const int c = r->corners;
#endif
  h.ja = c & 3; h.jc = (c >> 2) & 3; h.jt = (c >> 4) & 3;
  return h;
}

// The three corner angles of face f (MeshView::cangle must be non-null).
DG_HD V3<double> load_corner_angles(const MeshView& m, int f) {
  const double* p = m.cangle + 3 * size_t(f);
#ifdef __CUDA_ARCH__
  return {__ldg(p), __ldg(p + 1), __ldg(p + 2)};
#else
  return {p[0], p[1], p[2]};
#endif
}

template <class S>
DG_HD V3<S> load_normal(const MeshView& m, int f) {
#ifdef __CUDA_ARCH__
  const double* p = m.fnormal + 3 * size_t(f);
  return {S(__ldg(p)), S(__ldg(p + 1)), S(__ldg(p + 2))};
#else
  const double* p = m.fnormal + 3 * size_t(f);
  return {S(p[0]), S(p[1]), S(p[2])};
#endif
}

}  // namespace dg
