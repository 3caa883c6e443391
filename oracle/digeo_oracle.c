/* TEST INFRASTRUCTURE ONLY -- see digeo_oracle.h. Plain C99, compiled with -ffp-contract=off so
 * every operation rounds once, like the reference's default (-O2, no -march) build. */
#include "digeo_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double x, y, z; } v3;

struct og_mesh {
  int nv, nf;
  v3* X;          /* vertices */
  int32_t* T;     /* faces, 3 per face */
  int32_t* A;     /* adjacency, 3 per face, -1 = boundary */
  v3* N;          /* unit face normals */
  double* area;
  double* vangle;
  double* varea;
  uint8_t* vbnd;
  int32_t* off;   /* CSR */
  int32_t* lst;
  double mean_edge, total_area;
};

/* ---- geometry.hpp:36-65 ---------------------------------------------------------------- */
static v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 add(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 neg(v3 a) { return V(-a.x, -a.y, -a.z); }
static v3 mul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static v3 dvd(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 cross(v3 a, v3 b) { return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
static double norm(v3 a) { return sqrt(dot(a, a)); }
static v3 unit(v3 a) { double n = norm(a); return n > 0 ? dvd(a, n) : V(0, 0, 0); }
static double angle_between(v3 a, v3 b) { return atan2(norm(cross(a, b)), dot(a, b)); }
static double signed_angle(v3 a, v3 b, v3 axis) { return atan2(dot(cross(a, b), axis), dot(a, b)); }
static v3 rotate_about(v3 v, v3 axis, double ang) {
  double c = cos(ang), s = sin(ang);
  return add(add(mul(v, c), mul(cross(axis, v), s)), mul(axis, dot(axis, v) * (1.0 - c)));
}
static double max3(double a, double b, double c) { double m = a; if (m < b) m = b; if (m < c) m = c; return m; }

/* ---- mesh.cpp:34-130 -------------------------------------------------------------------- */
typedef struct { int a, b, f, k; } half_edge;
static int he_cmp(const void* p, const void* q) {
  const half_edge* x = (const half_edge*)p; const half_edge* y = (const half_edge*)q;
  if (x->a != y->a) return x->a < y->a ? -1 : 1;
  if (x->b != y->b) return x->b < y->b ? -1 : 1;
  int sx = 3 * x->f + x->k, sy = 3 * y->f + y->k;
  return sx < sy ? -1 : (sx > sy ? 1 : 0);
}

void og_mesh_free(og_mesh* m) {
  if (!m) return;
  free(m->X); free(m->T); free(m->A); free(m->N); free(m->area); free(m->vangle); free(m->varea);
  free(m->vbnd); free(m->off); free(m->lst); free(m);
}

static og_mesh* build_fail(og_mesh* m, half_edge* he, int* err, int code, char* msg, int len, const char* fmt, int a, int b) {
  if (err) *err = code;
  if (msg && len > 0) snprintf(msg, (size_t)len, fmt, a, b);
  free(he);
  og_mesh_free(m);
  return NULL;
}

og_mesh* og_mesh_build(const double* xyz, int nv, const int32_t* tri, int nf, int* err, char* msg, int msglen) {
  og_mesh* m = (og_mesh*)calloc(1, sizeof *m);
  half_edge* he = NULL;
  if (err) *err = OG_OK;
  m->nv = nv; m->nf = nf;
  m->X = (v3*)malloc(sizeof(v3) * (size_t)(nv ? nv : 1));
  m->T = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(nf ? nf : 1));
  for (int i = 0; i < nv; ++i) m->X[i] = V(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  memcpy(m->T, tri, sizeof(int32_t) * 3 * (size_t)nf);
  for (int f = 0; f < nf; ++f) {
    const int32_t* c = m->T + 3 * f;
    for (int k = 0; k < 3; ++k)
      if (c[k] < 0 || c[k] >= nv) return build_fail(m, he, err, OG_PARSE, msg, msglen, "face %d references vertex out of range", f, 0);
    if (c[0] == c[1] || c[1] == c[2] || c[0] == c[2])
      return build_fail(m, he, err, OG_DEGENERATE_FACE, msg, msglen, "face %d has repeated vertices", f, 0);
  }
  m->N = (v3*)malloc(sizeof(v3) * (size_t)(nf ? nf : 1));
  m->area = (double*)malloc(sizeof(double) * (size_t)(nf ? nf : 1));
  m->total_area = 0;
  for (int f = 0; f < nf; ++f) {
    const int32_t* c = m->T + 3 * f;
    v3 e1 = sub(m->X[c[1]], m->X[c[0]]), e2 = sub(m->X[c[2]], m->X[c[0]]);
    v3 n = cross(e1, e2);
    double a2 = norm(n);
    v3 e3 = sub(m->X[c[2]], m->X[c[1]]);
    double longest2 = max3(dot(e1, e1), dot(e2, e2), dot(e3, e3));
    if (a2 <= 1e-14 * longest2 || longest2 == 0.0)
      return build_fail(m, he, err, OG_DEGENERATE_FACE, msg, msglen, "face %d has zero area", f, 0);
    m->N[f] = dvd(n, a2);
    m->area[f] = 0.5 * a2;
    m->total_area += m->area[f];
  }
  /* adjacency through sorted vertex pairs; the sort visits edges in the std::map's key order */
  he = (half_edge*)malloc(sizeof(half_edge) * 3 * (size_t)(nf ? nf : 1));
  for (int f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      int a = m->T[3 * f + (k + 1) % 3], b = m->T[3 * f + (k + 2) % 3];
      half_edge h = {a < b ? a : b, a < b ? b : a, f, k};
      he[3 * f + k] = h;
    }
  qsort(he, 3 * (size_t)nf, sizeof(half_edge), he_cmp);
  m->A = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(nf ? nf : 1));
  for (int i = 0; i < 3 * nf; ++i) m->A[i] = -1;
  m->vbnd = (uint8_t*)calloc((size_t)(nv ? nv : 1), 1);
  double len_sum = 0; int64_t edges = 0;
  int bad_slot = -1, bad_a = 0, bad_b = 0;
  for (int i = 0; i < 3 * nf;) {
    int j = i;
    while (j < 3 * nf && he[j].a == he[i].a && he[j].b == he[i].b) ++j;
    if (j - i >= 3) {
      int slot = 3 * he[i + 2].f + he[i + 2].k;
      if (bad_slot < 0 || slot < bad_slot) { bad_slot = slot; bad_a = he[i].a; bad_b = he[i].b; }
    } else if (j - i == 2) {
      m->A[3 * he[i].f + he[i].k] = he[i + 1].f;
      m->A[3 * he[i + 1].f + he[i + 1].k] = he[i].f;
    } else {
      m->vbnd[he[i].a] = 1; m->vbnd[he[i].b] = 1;
    }
    len_sum += norm(sub(m->X[he[i].a], m->X[he[i].b]));
    ++edges;
    i = j;
  }
  if (bad_slot >= 0) return build_fail(m, he, err, OG_NON_MANIFOLD, msg, msglen, "edge (%d,%d) incident to 3+ faces", bad_a, bad_b);
  free(he); he = NULL;
  m->mean_edge = edges ? len_sum / (double)edges : 0.0;

  m->vangle = (double*)calloc((size_t)(nv ? nv : 1), sizeof(double));
  m->varea = (double*)calloc((size_t)(nv ? nv : 1), sizeof(double));
  for (int f = 0; f < nf; ++f) {
    const int32_t* c = m->T + 3 * f;
    for (int k = 0; k < 3; ++k) {
      v3 apex = m->X[c[k]];
      m->vangle[c[k]] += angle_between(sub(m->X[c[(k + 1) % 3]], apex), sub(m->X[c[(k + 2) % 3]], apex));
      m->varea[c[k]] += m->area[f] / 3.0;
    }
  }
  m->off = (int32_t*)calloc((size_t)nv + 1, sizeof(int32_t));
  m->lst = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(nf ? nf : 1));
  for (int i = 0; i < 3 * nf; ++i) m->off[m->T[i] + 1]++;
  for (int v = 0; v < nv; ++v) m->off[v + 1] += m->off[v];
  {
    int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nv ? nv : 1));
    memcpy(cur, m->off, sizeof(int32_t) * (size_t)nv);
    for (int f = 0; f < nf; ++f)
      for (int k = 0; k < 3; ++k) m->lst[cur[m->T[3 * f + k]]++] = f;
    free(cur);
  }
  return m;
}

int og_mesh_nv(const og_mesh* m) { return m->nv; }
int og_mesh_nf(const og_mesh* m) { return m->nf; }
double og_mesh_mean_edge(const og_mesh* m) { return m->mean_edge; }
void og_mesh_get(const og_mesh* m, int32_t* adj, double* fnormal, double* farea, double* vangle, double* varea,
                 uint8_t* vboundary, int32_t* csr_off, int32_t* csr_list) {
  if (adj) memcpy(adj, m->A, sizeof(int32_t) * 3 * (size_t)m->nf);
  if (fnormal) memcpy(fnormal, m->N, sizeof(v3) * (size_t)m->nf);
  if (farea) memcpy(farea, m->area, sizeof(double) * (size_t)m->nf);
  if (vangle) memcpy(vangle, m->vangle, sizeof(double) * (size_t)m->nv);
  if (varea) memcpy(varea, m->varea, sizeof(double) * (size_t)m->nv);
  if (vboundary) memcpy(vboundary, m->vbnd, (size_t)m->nv);
  if (csr_off) memcpy(csr_off, m->off, sizeof(int32_t) * ((size_t)m->nv + 1));
  if (csr_list) memcpy(csr_list, m->lst, sizeof(int32_t) * 3 * (size_t)m->nf);
}

static int corner_of(const og_mesh* m, int f, int v) {
  const int32_t* c = m->T + 3 * f;
  return c[0] == v ? 0 : (c[1] == v ? 1 : (c[2] == v ? 2 : -1));
}
static int neighbor_across(const og_mesh* m, int f, int a, int b) {
  for (int k = 0; k < 3; ++k) {
    int u = m->T[3 * f + (k + 1) % 3], w = m->T[3 * f + (k + 2) % 3];
    if ((u == a && w == b) || (u == b && w == a)) return m->A[3 * f + k];
  }
  return -1;
}

/* ---- tracer.cpp:44-529, Kernel<double> ------------------------------------------------- */
#define TOL_BARY 1e-10
#define TOL_DIR 1e-12
#define TOL_ANGLE 1e-12
enum { OC_CONTINUE, OC_FINISHED, OC_BOUNDARY, OC_MAXED, OC_STALLED };

typedef struct {
  const og_mesh* m;
  int max_steps, hole;
  int face;
  double bary[3];
  v3 dir;
  double remaining, target;
  int has_payload, want_q;
  v3 payload, q[3];
  double payload_norm;
  double traced;
  int npoints, status, stall, term;
  int64_t poly_base;  /* <0: off */
  int32_t* pf; double* pb; double* ps;
} walker;

typedef struct { v3 e, in_from, in_to; int kind; v3 n; double ang; } transport; /* kind 0 edge, 1 project, 2 rotate */

static v3 tr_apply(const transport* t, v3 w) {
  if (t->kind == 0) return sub(mul(t->e, dot(w, t->e)), mul(t->in_to, dot(w, t->in_from)));
  if (t->kind == 1) return sub(w, mul(t->n, dot(w, t->n)));
  return rotate_about(w, t->n, t->ang);
}
static void apply_transport(walker* k, const transport* t) {
  if (k->has_payload) {
    k->payload = tr_apply(t, k->payload);
    double n = norm(k->payload);
    if (n > 0) k->payload = mul(k->payload, k->payload_norm / n);
  }
  if (k->want_q) for (int j = 0; j < 3; ++j) k->q[j] = tr_apply(t, k->q[j]);
}
static void widened(const walker* k, double* b) {
  b[0] = k->bary[0]; b[1] = k->bary[1]; b[2] = k->bary[2];
  double s = b[0] + b[1] + b[2];
  if (s > 0 && s != 1.0) { b[0] /= s; b[1] /= s; b[2] /= s; }
}
static void push_point(walker* k, double seg, int is_start) {
  if (!is_start) k->traced += seg;
  if (k->poly_base >= 0) {
    int64_t o = k->poly_base + k->npoints;
    k->pf[o] = k->face;
    widened(k, k->pb + 3 * o);
    k->ps[o] = is_start ? 0.0 : seg;
  }
  k->npoints++;
}
static v3 edge_inward(const og_mesh* m, int va, int vc, int voff) {
  v3 a = m->X[va];
  v3 e = unit(sub(m->X[vc], a));
  v3 w = sub(m->X[voff], a);
  return unit(sub(w, mul(e, dot(w, e))));
}
static transport make_edge_transport(const og_mesh* m, int f_from, int f_to, int va, int vc) {
  int off_from = -1, off_to = -1;
  for (int k = 0; k < 3; ++k) {
    int u = m->T[3 * f_from + k];
    if (u != va && u != vc) off_from = u;
    int w = m->T[3 * f_to + k];
    if (w != va && w != vc) off_to = w;
  }
  transport t;
  memset(&t, 0, sizeof t);
  t.kind = 0;
  t.e = unit(sub(m->X[vc], m->X[va]));
  t.in_from = edge_inward(m, va, vc, off_from);
  t.in_to = edge_inward(m, va, vc, off_to);
  return t;
}
static void wedge_coeffs(const og_mesh* m, int g, int k, v3 w, double* c1, double* c2) {
  v3 x0 = m->X[m->T[3 * g + k]];
  v3 e1 = sub(m->X[m->T[3 * g + (k + 1) % 3]], x0);
  v3 e2 = sub(m->X[m->T[3 * g + (k + 2) % 3]], x0);
  double g11 = dot(e1, e1), g12 = dot(e1, e2), g22 = dot(e2, e2);
  double det = g11 * g22 - g12 * g12;
  double r1 = dot(e1, w), r2 = dot(e2, w);
  *c1 = (g22 * r1 - g12 * r2) / det;
  *c2 = (g11 * r2 - g12 * r1) / det;
}
static int wedge_contains(const og_mesh* m, int g, int k, v3 w) {
  double c1, c2;
  wedge_coeffs(m, g, k, w, &c1, &c2);
  double mag = fabs(c1) + fabs(c2);
  if (mag <= 0) return 0;
  double tol = TOL_DIR * mag;
  return c1 >= -tol && c2 >= -tol;
}
static void snap_bary(walker* k) {
  for (int i = 0; i < 3; ++i) if (k->bary[i] <= TOL_BARY) k->bary[i] = 0;
  double s = k->bary[0] + k->bary[1] + k->bary[2];
  if (s > 0) for (int i = 0; i < 3; ++i) k->bary[i] = k->bary[i] / s;
  for (int i = 0; i < 3; ++i)
    if (k->bary[i] >= 1.0 - TOL_BARY) {
      k->bary[0] = k->bary[1] = k->bary[2] = 0;
      k->bary[i] = 1;
      break;
    }
}
static int vertex_corner(const walker* k) {
  for (int i = 0; i < 3; ++i) if (k->bary[i] == 1.0) return i;
  return -1;
}
static int stall(walker* k, int why) { k->status = 1; k->stall = why; return OC_STALLED; }

static int slide_along(walker* k, int g, int from, int to, double t0);
static int slide_from_edge(walker* k, int e);
static int cross_edge(walker* k, int e);

static int advance(walker* k) {
  const og_mesh* m = k->m;
  double bv[3];
  wedge_coeffs(m, k->face, 0, k->dir, &bv[1], &bv[2]);
  bv[0] = -(bv[1] + bv[2]);
  double scale = fabs(bv[0]) + fabs(bv[1]) + fabs(bv[2]);
  if (!isfinite(scale) || scale <= 0) return stall(k, 1);
  double tol = TOL_DIR * scale;
  double best = INFINITY;
  int exit_edge = -1;
  for (int i = 0; i < 3; ++i) {
    if (bv[i] >= -tol) continue;
    double lambda = -k->bary[i] / bv[i];
    if (lambda < 0) lambda = 0;
    if (lambda < best) { best = lambda; exit_edge = i; }
  }
  if (exit_edge < 0) return stall(k, 2);
  if (best >= k->remaining) {
    for (int i = 0; i < 3; ++i) k->bary[i] += bv[i] * k->remaining;
    snap_bary(k);
    push_point(k, k->remaining, 0);
    k->remaining = 0;
    return OC_FINISHED;
  }
  for (int i = 0; i < 3; ++i) k->bary[i] += bv[i] * best;
  k->bary[exit_edge] = 0;
  snap_bary(k);
  k->remaining -= best;
  push_point(k, best, 0);
  if (vertex_corner(k) >= 0) return OC_CONTINUE;
  if (k->bary[exit_edge] != 0) return OC_CONTINUE;
  return cross_edge(k, exit_edge);
}

static int cross_edge(walker* k, int e) {
  const og_mesh* m = k->m;
  int g = m->A[3 * k->face + e];
  if (g < 0) return k->hole ? slide_from_edge(k, e) : OC_BOUNDARY;
  int va = m->T[3 * k->face + (e + 1) % 3], vc = m->T[3 * k->face + (e + 2) % 3];
  double wa = k->bary[(e + 1) % 3], wc = k->bary[(e + 2) % 3];
  transport t = make_edge_transport(m, k->face, g, va, vc);
  k->dir = unit(tr_apply(&t, k->dir));
  apply_transport(k, &t);
  double nb[3] = {0, 0, 0};
  nb[corner_of(m, g, va)] = wa;
  nb[corner_of(m, g, vc)] = wc;
  k->face = g;
  memcpy(k->bary, nb, sizeof nb);
  snap_bary(k);
  return OC_CONTINUE;
}

static int fan_walk(walker* k, int x0) {
  const og_mesh* m = k->m;
  double half = m->vangle[x0] / 2;
  v3 x0p = m->X[x0];
  v3 rev = neg(k->dir);
  int k0 = corner_of(m, k->face, x0);
  int p1 = m->T[3 * k->face + (k0 + 1) % 3], p2 = m->T[3 * k->face + (k0 + 2) % 3];
  double a1 = angle_between(rev, sub(m->X[p1], x0p));
  double a2 = angle_between(rev, sub(m->X[p2], x0p));
  int x1 = a1 <= a2 ? p1 : p2;
  double alpha = a2 < a1 ? a2 : a1;
  int g = k->face, near_vertex = -1;
  v3 carried = k->dir;
  int guard = (m->off[x0 + 1] - m->off[x0]) + 2;
  while (alpha < half - TOL_ANGLE) {
    if (--guard < 0) return 0;
    int gn = neighbor_across(m, g, x0, x1);
    if (gn < 0) return 0;
    int x2 = -1;
    for (int c = 0; c < 3; ++c) {
      int u = m->T[3 * gn + c];
      if (u != x0 && u != x1) x2 = u;
    }
    alpha += angle_between(sub(m->X[x1], x0p), sub(m->X[x2], x0p));
    transport t = make_edge_transport(m, g, gn, x0, x1);
    carried = tr_apply(&t, carried);
    apply_transport(k, &t);
    near_vertex = x1; g = gn; x1 = x2;
  }
  double beta = alpha - half;
  if (!(0 < beta)) beta = 0;
  v3 e_far = unit(sub(m->X[x1], x0p));
  v3 n_g = m->N[g];
  v3 e_near = near_vertex >= 0 ? unit(sub(m->X[near_vertex], x0p)) : rev;
  double side = signed_angle(e_far, e_near, n_g) >= 0 ? 1.0 : -1.0;
  v3 outgoing = rotate_about(e_far, n_g, side * beta);
  outgoing = unit(sub(outgoing, mul(n_g, dot(outgoing, n_g))));
  if (k->has_payload || k->want_q) {
    v3 cip = unit(sub(carried, mul(n_g, dot(carried, n_g))));
    transport r;
    memset(&r, 0, sizeof r);
    r.kind = 2; r.n = n_g; r.ang = signed_angle(cip, outgoing, n_g);
    apply_transport(k, &r);
  }
  k->face = g;
  k->bary[0] = k->bary[1] = k->bary[2] = 0;
  k->bary[corner_of(m, g, x0)] = 1;
  k->dir = outgoing;
  return 1;
}

static void reanchor(walker* k, int g, int x0) {
  k->face = g;
  k->bary[0] = k->bary[1] = k->bary[2] = 0;
  k->bary[corner_of(k->m, g, x0)] = 1;
}

static int slide_from_vertex(walker* k, int x0) {
  const og_mesh* m = k->m;
  int best_to = -1, best_face = -1;
  double best_align = -INFINITY;
  for (int i = m->off[x0]; i < m->off[x0 + 1]; ++i) {
    int g = m->lst[i];
    int k0 = corner_of(m, g, x0);
    for (int o = 1; o <= 2; ++o) {
      int kc = (k0 + o) % 3;
      int y = m->T[3 * g + kc];
      int opp = 3 - k0 - kc;
      if (m->A[3 * g + opp] >= 0) continue;
      double align = dot(k->dir, unit(sub(m->X[y], m->X[x0])));
      if (align > best_align || (align == best_align && y < best_to)) { best_align = align; best_to = y; best_face = g; }
    }
  }
  if (best_to < 0) return OC_BOUNDARY;
  return slide_along(k, best_face, x0, best_to, 0.0);
}

static int blue_vertex(walker* k, int x0) {
  const og_mesh* m = k->m;
  int best_face = -1;
  double best_err = INFINITY;
  for (int i = m->off[x0]; i < m->off[x0 + 1]; ++i) {
    int g = m->lst[i];
    v3 n = m->N[g];
    v3 proj = sub(k->dir, mul(n, dot(k->dir, n)));
    if (norm(proj) < 1e-6) continue;
    if (!wedge_contains(m, g, corner_of(m, g, x0), proj)) continue;
    double e = angle_between(k->dir, proj);
    if (e < best_err) { best_err = e; best_face = g; }
  }
  if (best_face >= 0) {
    transport p;
    memset(&p, 0, sizeof p);
    p.kind = 1; p.n = m->N[best_face];
    k->dir = unit(tr_apply(&p, k->dir));
    apply_transport(k, &p);
    reanchor(k, best_face, x0);
    return advance(k);
  }
  return slide_from_vertex(k, x0);
}

static int slide_from_edge(walker* k, int e) {
  const og_mesh* m = k->m;
  int va = m->T[3 * k->face + (e + 1) % 3], vc = m->T[3 * k->face + (e + 2) % 3];
  v3 pos = add(mul(m->X[va], k->bary[(e + 1) % 3]), mul(m->X[vc], k->bary[(e + 2) % 3]));
  double da = dot(k->dir, unit(sub(m->X[va], pos)));
  double dc = dot(k->dir, unit(sub(m->X[vc], pos)));
  int to = da >= dc ? va : vc;
  int from = to == va ? vc : va;
  double t0 = to == va ? k->bary[(e + 1) % 3] : k->bary[(e + 2) % 3];
  return slide_along(k, k->face, from, to, t0);
}

static int slide_along(walker* k, int g, int from, int to, double t0) {
  const og_mesh* m = k->m;
  double edge_len = norm(sub(m->X[to], m->X[from]));
  double left = edge_len * (1.0 - t0);
  double consume = k->remaining < left ? k->remaining : left;
  double t1 = t0 + consume / edge_len;
  k->face = g;
  k->bary[0] = k->bary[1] = k->bary[2] = 0;
  k->bary[corner_of(m, g, from)] = 1.0 - t1;
  k->bary[corner_of(m, g, to)] = t1;
  snap_bary(k);
  k->remaining -= consume;
  push_point(k, consume, 0);
  if (k->remaining <= 0) { k->remaining = 0; return OC_FINISHED; }
  return OC_CONTINUE;
}

static int at_vertex(walker* k, int k0) {
  const og_mesh* m = k->m;
  int x0 = m->T[3 * k->face + k0];
  if (k->hole && m->vbnd[x0]) return blue_vertex(k, x0);
  if (wedge_contains(m, k->face, k0, neg(k->dir))) return fan_walk(k, x0) ? OC_CONTINUE : OC_BOUNDARY;
  if (wedge_contains(m, k->face, k0, k->dir)) return advance(k);
  int best_face = -1;
  double best_margin = -INFINITY;
  for (int i = m->off[x0]; i < m->off[x0 + 1]; ++i) {
    int g = m->lst[i];
    double c1, c2;
    wedge_coeffs(m, g, corner_of(m, g, x0), k->dir, &c1, &c2);
    double mag = fabs(c1) + fabs(c2);
    if (mag <= 0) continue;
    double margin = (c2 < c1 ? c2 : c1) / mag;
    if (margin > best_margin) { best_margin = margin; best_face = g; }
  }
  if (best_face >= 0 && best_margin >= -TOL_DIR) {
    transport p;
    memset(&p, 0, sizeof p);
    p.kind = 1; p.n = m->N[best_face];
    v3 proj = tr_apply(&p, k->dir);
    if (norm(proj) > 0) {
      k->dir = unit(proj);
      apply_transport(k, &p);
      reanchor(k, best_face, x0);
      return advance(k);
    }
  }
  return fan_walk(k, x0) ? OC_CONTINUE : OC_BOUNDARY;
}

static int bary_valid(const double* b, double tol) {
  double s = b[0] + b[1] + b[2];
  if (fabs(s - 1.0) > tol) return 0;
  for (int i = 0; i < 3; ++i) if (b[i] < -tol || b[i] > 1.0 + tol) return 0;
  return 1;
}

/* one full trace; returns through the walker */
static void run_trace(walker* k, int f, const double* b, v3 v, const double* pay, int want_q) {
  const og_mesh* m = k->m;
  k->face = -1; k->bary[0] = k->bary[1] = k->bary[2] = 0; k->dir = V(0, 0, 0);
  k->remaining = k->target = 0; k->has_payload = 0; k->want_q = 0; k->payload = V(0, 0, 0);
  k->q[0] = V(1, 0, 0); k->q[1] = V(0, 1, 0); k->q[2] = V(0, 0, 1);
  k->traced = 0; k->npoints = 0; k->status = 0; k->stall = 0; k->term = 0;
  if (f < 0 || f >= m->nf) { stall(k, 4); return; }
  if (!bary_valid(b, 1e-6)) { stall(k, 5); return; }
  k->face = f;
  memcpy(k->bary, b, 3 * sizeof(double));
  snap_bary(k);
  k->target = k->remaining = norm(v);
  v3 n = m->N[f];
  v3 in_plane = sub(v, mul(n, dot(v, n)));
  if (k->target > 0 && norm(in_plane) < 1e-12 * k->target) { stall(k, 3); return; }
  k->dir = unit(in_plane);
  if (pay && (pay[0] * pay[0] + pay[1] * pay[1] + pay[2] * pay[2]) > 0) {
    k->has_payload = 1;
    k->payload = V(pay[0], pay[1], pay[2]);
    k->payload_norm = norm(k->payload);
  }
  k->want_q = want_q;
  push_point(k, 0, 1);
  int oc = OC_FINISHED, steps = 0;
  while (k->remaining > 0) {
    if (steps++ >= k->max_steps) { oc = OC_MAXED; break; }
    int k0 = vertex_corner(k);
    oc = k0 >= 0 ? at_vertex(k, k0) : advance(k);
    if (oc != OC_CONTINUE) break;
  }
  if (oc == OC_BOUNDARY) k->term = 1;
  else if (oc == OC_MAXED) k->term = 2;
}

static int default_max_steps(const og_mesh* m) { return (int)(10.0 * sqrt((double)m->nf)) + 100; }

void og_trace_batch(const og_mesh* m, int64_t n, const int32_t* face, const double* bary, const double* dir,
                    const double* payload, const og_cfg* cfg, int32_t* o_face, double* o_bary, double* o_dir,
                    double* o_traced, double* o_requested, uint8_t* o_term, uint8_t* o_status, uint8_t* o_stall,
                    double* o_payload, double* o_q, int32_t* o_npoints, const int64_t* poly_off,
                    int32_t* poly_face, double* poly_bary, double* poly_seg) {
  og_cfg c = {0, 0, 0, 0};
  if (cfg) c = *cfg;
  int max_steps = c.max_steps > 0 ? c.max_steps : default_max_steps(m);
#ifdef _OPENMP
  int threads = c.threads > 0 ? c.threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
#endif
  for (int64_t i = 0; i < n; ++i) {
    walker k;
    memset(&k, 0, sizeof k);
    k.m = m; k.max_steps = max_steps; k.hole = c.hole_avoidance;
    k.poly_base = poly_off ? poly_off[i] : -1;
    k.pf = poly_face; k.pb = poly_bary; k.ps = poly_seg;
    run_trace(&k, face[i], bary + 3 * i, V(dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]),
              payload ? payload + 3 * i : NULL, c.want_q);
    if (o_face) o_face[i] = k.face;
    if (o_bary) widened(&k, o_bary + 3 * i);
    if (o_dir) {
      v3 d = k.target > 0 ? k.dir : V(0, 0, 0);
      o_dir[3 * i] = d.x; o_dir[3 * i + 1] = d.y; o_dir[3 * i + 2] = d.z;
    }
    if (o_traced) o_traced[i] = k.traced;
    if (o_requested) o_requested[i] = k.target;
    if (o_term) o_term[i] = (uint8_t)k.term;
    if (o_status) o_status[i] = (uint8_t)k.status;
    if (o_stall) o_stall[i] = (uint8_t)k.stall;
    if (o_payload) {
      v3 p = k.has_payload ? k.payload : V(0, 0, 0);
      o_payload[3 * i] = p.x; o_payload[3 * i + 1] = p.y; o_payload[3 * i + 2] = p.z;
    }
    if (o_q) {
      double* o = o_q + 9 * i;
      if (k.want_q) {
        o[0] = k.q[0].x; o[1] = k.q[1].x; o[2] = k.q[2].x;
        o[3] = k.q[0].y; o[4] = k.q[1].y; o[5] = k.q[2].y;
        o[6] = k.q[0].z; o[7] = k.q[1].z; o[8] = k.q[2].z;
      } else {
        memset(o, 0, 9 * sizeof(double));
      }
    }
    if (o_npoints) o_npoints[i] = k.npoints;
  }
}

/* ---- diff.cpp -------------------------------------------------------------------------- */
typedef struct { v3 e_par, e_perp, normal; } tframe;
typedef struct { v3 u_hat, v_hat, p0, p1; } bframe;

static int make_tangent_frame(const og_mesh* m, int f, v3 v, tframe* t) {
  if (norm(v) < 1e-12) return 0;
  t->normal = m->N[f];
  v3 in_plane = sub(v, mul(t->normal, dot(v, t->normal)));
  if (norm(in_plane) < 1e-12 * norm(v)) return 0;
  t->e_par = unit(in_plane);
  t->e_perp = cross(t->normal, t->e_par);
  return 1;
}
static bframe make_bary_frame(const og_mesh* m, int f) {
  const int32_t* c = m->T + 3 * f;
  bframe b;
  b.u_hat = unit(sub(m->X[c[1]], m->X[c[0]]));
  b.v_hat = unit(sub(m->X[c[2]], m->X[c[0]]));
  double g11 = dot(b.u_hat, b.u_hat), g12 = dot(b.u_hat, b.v_hat), g22 = dot(b.v_hat, b.v_hat);
  double det = g11 * g22 - g12 * g12;
  b.p0 = dvd(sub(mul(b.u_hat, g22), mul(b.v_hat, g12)), det);
  b.p1 = dvd(sub(mul(b.v_hat, g11), mul(b.u_hat, g12)), det);
  return b;
}
static v3 embed(const og_mesh* m, int f, const double* b) {
  const int32_t* c = m->T + 3 * f;
  return add(add(mul(m->X[c[0]], b[0]), mul(m->X[c[1]], b[1])), mul(m->X[c[2]], b[2]));
}
static void put3(double* o, v3 a) { o[0] = a.x; o[1] = a.y; o[2] = a.z; }
static void put_frames(double* o, const tframe* fv, const bframe* fp, const bframe* fo) {
  if (fv) { put3(o, fv->e_par); put3(o + 3, fv->e_perp); put3(o + 6, fv->normal); }
  if (fp) { put3(o + 9, fp->u_hat); put3(o + 12, fp->v_hat); put3(o + 15, fp->p0); put3(o + 18, fp->p1); }
  if (fo) { put3(o + 21, fo->u_hat); put3(o + 24, fo->v_hat); put3(o + 27, fo->p0); put3(o + 30, fo->p1); }
}

int og_ep(const og_mesh* m, int64_t n, const int32_t* face, const double* v, const int32_t* end_face,
          const double* end_dir, const double* g, double* rot, double* frames, double* grad_v, double* grad_p,
          int64_t* err_index) {
  for (int64_t i = 0; i < n; ++i) {
    v3 vv = V(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    tframe fv;
    if (norm(vv) < 1e-12 || !make_tangent_frame(m, face[i], vv, &fv)) {
      if (err_index) *err_index = i;
      return OG_DEGENERATE_DIRECTION;
    }
    bframe fp = make_bary_frame(m, face[i]);
    bframe fo = make_bary_frame(m, end_face[i]);
    v3 n_out = m->N[end_face[i]];
    v3 d = V(end_dir[3 * i], end_dir[3 * i + 1], end_dir[3 * i + 2]);
    v3 e_par_out = unit(sub(d, mul(n_out, dot(d, n_out))));
    v3 e_perp_out = cross(n_out, e_par_out);
    /* m_q * m_p^T with Mat3::operator* accumulation order */
    double mq[3][3] = {{e_par_out.x, e_perp_out.x, n_out.x}, {e_par_out.y, e_perp_out.y, n_out.y}, {e_par_out.z, e_perp_out.z, n_out.z}};
    double mp[3][3] = {{fv.e_par.x, fv.e_perp.x, fv.normal.x}, {fv.e_par.y, fv.e_perp.y, fv.normal.y}, {fv.e_par.z, fv.e_perp.z, fv.normal.z}};
    double r[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += mq[a][k] * mp[b][k];
        r[3 * a + b] = s;
      }
    if (rot) memcpy(rot + 9 * i, r, sizeof r);
    if (frames) put_frames(frames + 33 * i, &fv, &fp, &fo);
    if (g) {
      v3 gg = V(g[3 * i], g[3 * i + 1], g[3 * i + 2]);
      double go0 = dot(fo.u_hat, gg), go1 = dot(fo.v_hat, gg);
      v3 g_tan = add(mul(fo.p0, go0), mul(fo.p1, go1));
      v3 r0 = V(r[0], r[1], r[2]), r1 = V(r[3], r[4], r[5]), r2 = V(r[6], r[7], r[8]);
      v3 epo = V(dot(r0, fv.e_par), dot(r1, fv.e_par), dot(r2, fv.e_par));
      v3 eqo = V(dot(r0, fv.e_perp), dot(r1, fv.e_perp), dot(r2, fv.e_perp));
      double gv0 = dot(epo, g_tan), gv1 = dot(eqo, g_tan);
      double t0 = 1.0 * gv0 + 0.0 * gv1, t1 = 0.0 * gv0 + 1.0 * gv1;
      if (grad_v) put3(grad_v + 3 * i, add(mul(fv.e_par, t0), mul(fv.e_perp, t1)));
      if (grad_p) put3(grad_p + 3 * i, add(mul(fp.p0, 0.0), mul(fp.p1, 0.0)));
    }
  }
  return OG_OK;
}

typedef struct { int face; double bary[3]; v3 dir; v3 payload; int has_payload; int status, term; } endstate;

static endstate one_trace(const og_mesh* m, int f, const double* b, v3 d, const v3* pay) {
  walker k;
  memset(&k, 0, sizeof k);
  k.m = m; k.max_steps = default_max_steps(m); k.hole = 0; k.poly_base = -1;
  double pp[3] = {0, 0, 0};
  if (pay) { pp[0] = pay->x; pp[1] = pay->y; pp[2] = pay->z; }
  run_trace(&k, f, b, d, pay ? pp : NULL, 0);
  endstate e;
  e.face = k.face;
  widened(&k, e.bary);
  e.dir = k.target > 0 ? k.dir : V(0, 0, 0);
  e.payload = k.payload;
  e.has_payload = k.has_payload;
  e.status = k.status;
  e.term = k.term;
  return e;
}
static int reached(const endstate* e) { return e->status == 0 && e->term == 0; }

/* fd_column, diff.cpp:130-137. minus == NULL: the minus side could not be set up. Returns -1 when
 * the minus-side trace() would have thrown NumericalStall. */
static int fd_column(const og_mesh* m, const endstate* plus, double eps, v3 ref, const endstate* minus, uint8_t* degraded, v3* col) {
  if (reached(plus)) { *col = dvd(sub(embed(m, plus->face, plus->bary), ref), eps); return 0; }
  *degraded = 1;
  *col = V(0, 0, 0);
  if (!minus) return 0;
  if (minus->status) return -1;
  if (reached(minus)) *col = dvd(sub(ref, embed(m, minus->face, minus->bary)), eps);
  return 0;
}

int og_gfd(const og_mesh* m, int64_t n, const int32_t* face, const double* bary, const double* v, double eps_v,
           double eps_p, const double* g, double* jv, double* jp, uint8_t* degraded, double* frames,
           double* grad_v, double* grad_p, int threads, char* msg, int msglen) {
  int rc = OG_OK;
  int64_t first_bad = n;
  const char* why = "";
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
#endif
  for (int64_t i = 0; i < n; ++i) {
    int my_rc = OG_OK;
    const char* my_why = "";
    const double* b = bary + 3 * i;
    v3 vv = V(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    tframe fv;
    uint8_t dg[4] = {0, 0, 0, 0};
    do {
      if (face[i] < 0 || face[i] >= m->nf || !make_tangent_frame(m, face[i], vv, &fv)) {
        my_rc = OG_DEGENERATE_DIRECTION; my_why = "tangent frame needs a nonzero in-plane direction"; break;
      }
      bframe fp = make_bary_frame(m, face[i]);
      endstate base = one_trace(m, face[i], b, vv, NULL);
      if (!reached(&base)) { my_rc = OG_ERROR; my_why = "gfd: the base trace did not reach its requested length"; break; }
      endstate perp = one_trace(m, face[i], b, add(vv, mul(fv.e_perp, eps_v)), NULL);
      endstate seed_u = one_trace(m, face[i], b, mul(fp.u_hat, eps_p), &vv);
      endstate seed_v = one_trace(m, face[i], b, mul(fp.v_hat, eps_p), &vv);
      endstate par = one_trace(m, base.face, base.bary, mul(base.dir, eps_v), NULL);
      double zero_b[3] = {b[0], b[1], b[2]};
      endstate ret_u = reached(&seed_u) ? one_trace(m, seed_u.face, seed_u.bary, seed_u.payload, NULL)
                                        : one_trace(m, face[i], zero_b, V(0, 0, 0), NULL);
      endstate ret_v = reached(&seed_v) ? one_trace(m, seed_v.face, seed_v.bary, seed_v.payload, NULL)
                                        : one_trace(m, face[i], zero_b, V(0, 0, 0), NULL);
      bframe fo = make_bary_frame(m, base.face);
      v3 ref = embed(m, base.face, base.bary);
      v3 col[4];
      /* j_v columns */
      endstate mn; int have;
      have = 0;
      if (!reached(&par)) { mn = one_trace(m, base.face, base.bary, mul(base.dir, -eps_v), NULL); have = 1; }
      if (fd_column(m, &par, eps_v, ref, have ? &mn : NULL, &dg[0], &col[0]) < 0) { my_rc = OG_NUMERICAL_STALL; my_why = "trace: fallback stalled"; break; }
      have = 0;
      if (!reached(&perp)) { mn = one_trace(m, face[i], b, sub(vv, mul(fv.e_perp, eps_v)), NULL); have = 1; }
      if (fd_column(m, &perp, eps_v, ref, have ? &mn : NULL, &dg[1], &col[1]) < 0) { my_rc = OG_NUMERICAL_STALL; my_why = "trace: fallback stalled"; break; }
      if (!reached(&seed_u) || !reached(&seed_v)) { my_rc = OG_ERROR; my_why = "gfd: start-point perturbation seeds failed to trace"; break; }
      /* j_p columns; minus side = back-step with payload, then retrace (diff.cpp:186-194) */
      int bad = 0;
      for (int c = 0; c < 2 && !bad; ++c) {
        const endstate* plus = c == 0 ? &ret_u : &ret_v;
        v3 sd = c == 0 ? fp.u_hat : fp.v_hat;
        have = 0;
        if (!reached(plus)) {
          endstate back = one_trace(m, face[i], b, mul(sd, -eps_p), &vv);
          if (back.status) { bad = 1; break; }
          if (reached(&back)) { mn = one_trace(m, back.face, back.bary, back.payload, NULL); have = 1; }
        }
        if (fd_column(m, plus, eps_p, ref, have ? &mn : NULL, &dg[2 + c], &col[2 + c]) < 0) bad = 1;
      }
      if (bad) { my_rc = OG_NUMERICAL_STALL; my_why = "trace: fallback stalled"; break; }
      double J[4] = {dot(fo.p0, col[0]), dot(fo.p0, col[1]), dot(fo.p1, col[0]), dot(fo.p1, col[1])};
      double P[4] = {dot(fo.p0, col[2]), dot(fo.p0, col[3]), dot(fo.p1, col[2]), dot(fo.p1, col[3])};
      if (jv) memcpy(jv + 4 * i, J, sizeof J);
      if (jp) memcpy(jp + 4 * i, P, sizeof P);
      if (degraded) memcpy(degraded + 4 * i, dg, 4);
      if (frames) put_frames(frames + 33 * i, &fv, &fp, &fo);
      if (g) {
        v3 gg = V(g[3 * i], g[3 * i + 1], g[3 * i + 2]);
        double go0 = dot(fo.u_hat, gg), go1 = dot(fo.v_hat, gg);
        double gv0 = J[0] * go0 + J[2] * go1, gv1 = J[1] * go0 + J[3] * go1;
        double gp0 = P[0] * go0 + P[2] * go1, gp1 = P[1] * go0 + P[3] * go1;
        if (grad_v) put3(grad_v + 3 * i, add(mul(fv.e_par, gv0), mul(fv.e_perp, gv1)));
        if (grad_p) put3(grad_p + 3 * i, add(mul(fp.p0, gp0), mul(fp.p1, gp1)));
      }
    } while (0);
    if (my_rc != OG_OK) {
#ifdef _OPENMP
#pragma omp critical
#endif
      if (i < first_bad) { first_bad = i; rc = my_rc; why = my_why; }
    }
  }
  if (rc != OG_OK && msg && msglen > 0) snprintf(msg, (size_t)msglen, "%s", why);
  return rc;
}
