// Differentials of the exponential map: the fused extrinsic-proxy (EP) Jacobian / pullback
// kernel, the job builders and assembly kernels of geodesic finite differences (GFD), and the
// single-transition kernel. Restates proj/src/diff.cpp (EP :44-66, :328-354; GFD :116-326) and
// the public single-step wrappers of proj/src/tracer.cpp:630-735; the expression trees follow
// the reference so that, compiled with -fmad=false, the f64 results are bit-identical whenever
// the underlying traces are.
//
// GFD job layout (ours, not the reference's interleaved 4i+k): the jobs of one kind are
// contiguous so that each round is ONE launch per kernel variant --
//   round 1: [0,n) seed_u  [n,2n) seed_v                                  (payload kernel, eps-length)
//   round 2: [0,n) ret_u  [n,2n) ret_v  [2n,3n) perp  [3n,4n) par | base  (lite)
// The full-length jobs of a sample (ret_u, ret_v, perp -- and its base trace when the caller does
// not bring one) differ by an O(eps) offset and cross the same faces: round 2 runs them as a
// sibling group in one warp (TraceParams::siblings, stride n) so that they share every
// crossing-record fetch. With the caller's forward results as base traces the group has three
// members and the eps-length par jobs fill the tail of the same launch; without, the base trace is
// the fourth member and the par jobs (which start where the base ends) get a short launch of
// their own.
//   fallback rounds (only if some + perturbation left the mesh):
//   round 3: [0,n) par-  [n,2n) perp-   [2n,3n) back_u  [3n,4n) back_v    (payload)
//   round 4: [0,n) retrace of back_u    [n,2n) retrace of back_v          (lite)
#include "dg_kernels.cuh"
#include "dg_tracer_core.cuh"

namespace dg {

namespace {

using V = V3<double>;
constexpr unsigned long long kNoError = ~0ull;

__device__ __forceinline__ V ld3(const double* p, int64_t i) { return V{p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
__device__ __forceinline__ void st3(double* p, int64_t i, const V& v) {
  p[3 * i] = v.x; p[3 * i + 1] = v.y; p[3 * i + 2] = v.z;
}
__device__ __forceinline__ void note_error(unsigned long long* slot, int64_t i) {
  atomicMin(slot, (unsigned long long)i);
}

struct TangentFrame { V e_par, e_perp, normal; };
struct BaryFrame { V u_hat, v_hat, pinv0, pinv1; };

// diff.cpp:13-24. Returns false for a degenerate direction.
__device__ bool make_tangent_frame(const MeshView& m, int face, const V& v, TangentFrame* f) {
  if (norm(v) < 1e-12) return false;
  f->normal = load_normal<double>(m, face);
  V in_plane = v - f->normal * dot(v, f->normal);
  if (norm(in_plane) < 1e-12 * norm(v)) return false;
  f->e_par = normalized(in_plane);
  f->e_perp = cross(f->normal, f->e_par);
  return true;
}
// diff.cpp:26-38
__device__ BaryFrame make_bary_frame(const Face<double>& c) {
  BaryFrame f;
  f.u_hat = normalized(c.x1 - c.x0);
  f.v_hat = normalized(c.x2 - c.x0);
  double g11 = dot(f.u_hat, f.u_hat), g12 = dot(f.u_hat, f.v_hat), g22 = dot(f.v_hat, f.v_hat);
  double det = g11 * g22 - g12 * g12;
  f.pinv0 = (f.u_hat * g22 - f.v_hat * g12) / det;
  f.pinv1 = (f.v_hat * g11 - f.u_hat * g12) / det;
  return f;
}
// embed, mesh.cpp:208-212
__device__ __forceinline__ V embed(const Face<double>& c, const V& b) {
  return c.x0 * b.x + c.x1 * b.y + c.x2 * b.z;
}
__device__ void store_frames(double* frames, int64_t i, const TangentFrame* fv, const BaryFrame* fp,
                             const BaryFrame* fo) {
  double* o = frames + 33 * i;
  if (fv) { st3(o, 0, fv->e_par); st3(o, 1, fv->e_perp); st3(o, 2, fv->normal); }
  if (fp) { st3(o, 3, fp->u_hat); st3(o, 4, fp->v_hat); st3(o, 5, fp->pinv0); st3(o, 6, fp->pinv1); }
  if (fo) { st3(o, 7, fo->u_hat); st3(o, 8, fo->v_hat); st3(o, 9, fo->pinv0); st3(o, 10, fo->pinv1); }
}

// ------------------------------------------------------------------------------------- EP

// error word: (sample << 2) | kind, kind 0 = |v| too small, 1 = normal to the face, 2 = bad face
// A latency-bound gather (two face records and two normals per sample, 17 % of the issue slots busy): more
// resident warps pay -- 1 M samples, device-resident, L2 flushed: 4 blocks per SM (112 registers) 0.108 ms,
// 5 (96 registers, 40 bytes of spill) 0.095, 6 / 8 (80 / 64 registers) 0.093 / 0.094.
#ifndef DG_EP_MIN_BLOCKS
#define DG_EP_MIN_BLOCKS 5
#endif
__global__ void __launch_bounds__(128, DG_EP_MIN_BLOCKS) ep_kernel(const __grid_constant__ EpParams p) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= p.n) return;
  const int f = p.face[i], fe = p.end_face[i];
  if (f < 0 || f >= p.mesh.nf || fe < 0 || fe >= p.mesh.nf) {
    atomicMin(p.first_error, ((unsigned long long)i << 2) | 2ull);
    return;
  }
  const V v = ld3(p.v, i);
  if (norm(v) < 1e-12) {  // diff.cpp:46
    atomicMin(p.first_error, ((unsigned long long)i << 2) | 0ull);
    return;
  }
  TangentFrame fv;
  if (!make_tangent_frame(p.mesh, f, v, &fv)) {
    atomicMin(p.first_error, ((unsigned long long)i << 2) | 1ull);
    return;
  }
  const Face<double> cq = load_face<double>(p.mesh, fe);
  const BaryFrame fo = make_bary_frame(cq);

  // endpoint frame from the transported direction, diff.cpp:54-56
  const V n_out = load_normal<double>(p.mesh, fe);
  const V d_out = ld3(p.end_dir, i);
  const V e_par_out = normalized(d_out - n_out * dot(d_out, n_out));
  const V e_perp_out = cross(n_out, e_par_out);

  // rotation_ep = M_q M_p^T with the reference's accumulation order (geometry.hpp:94-103)
  double r[9];
  {
    const double qc[3][3] = {{e_par_out.x, e_perp_out.x, n_out.x},
                             {e_par_out.y, e_perp_out.y, n_out.y},
                             {e_par_out.z, e_perp_out.z, n_out.z}};  // m_q(i,k)
    const double pc[3][3] = {{fv.e_par.x, fv.e_perp.x, fv.normal.x},
                             {fv.e_par.y, fv.e_perp.y, fv.normal.y},
                             {fv.e_par.z, fv.e_perp.z, fv.normal.z}};  // m_p(j,k)
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        double s = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) s += qc[a][k] * pc[b][k];
        r[3 * a + b] = s;
      }
  }
  if (p.rot) {
#pragma unroll
    for (int k = 0; k < 9; ++k) p.rot[9 * i + k] = r[k];
  }
  const bool want_in_p = p.frames || p.grad_p;
  BaryFrame fp{};
  if (want_in_p) fp = make_bary_frame(load_face<double>(p.mesh, f));
  if (p.frames) store_frames(p.frames, i, &fv, &fp, &fo);

  if (p.g && (p.grad_v || p.grad_p)) {
    // pullback_ambient, diff.cpp:347-354 with the EP branch of pullback, :330-341
    const V g = ld3(p.g, i);
    const double go0 = dot(fo.u_hat, g), go1 = dot(fo.v_hat, g);
    const V g_tan = fo.pinv0 * go0 + fo.pinv1 * go1;
    const V r0{r[0], r[1], r[2]}, r1{r[3], r[4], r[5]}, r2{r[6], r[7], r[8]};
    const V e_par_o{dot(r0, fv.e_par), dot(r1, fv.e_par), dot(r2, fv.e_par)};
    const V e_perp_o{dot(r0, fv.e_perp), dot(r1, fv.e_perp), dot(r2, fv.e_perp)};
    double gv0 = dot(e_par_o, g_tan), gv1 = dot(e_perp_o, g_tan);
    // j_v^T (identity) applied as Mat2::operator*
    const double t0 = 1.0 * gv0 + 0.0 * gv1, t1 = 0.0 * gv0 + 1.0 * gv1;
    if (p.grad_v) st3(p.grad_v, i, fv.e_par * t0 + fv.e_perp * t1);
    if (p.grad_p) st3(p.grad_p, i, fp.pinv0 * 0.0 + fp.pinv1 * 0.0);
  }
}

// ------------------------------------------------------------------------------------ GFD

__device__ __forceinline__ bool reached(uint8_t status, uint8_t term) {  // diff.cpp:116-119
  return status == kStatusOk && term == kTermLength;
}
__device__ __forceinline__ void put_job(int32_t* jf, double* jb, double* jd, double* jp, int64_t slot, int face,
                                        const V& b, const V& d, const V& pay) {
  jf[slot] = face;
  st3(jb, slot, b);
  st3(jd, slot, d);
  if (jp) st3(jp, slot, pay);
}

__global__ void __launch_bounds__(128) gfd_round1_jobs_kernel(const __grid_constant__ GfdBuffers b) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t n = b.n;
  if (i >= n) return;
  const int f = b.face[i];
  const V p = ld3(b.bary, i), v = ld3(b.v, i);
  const V zero{0.0, 0.0, 0.0};
  TangentFrame fv;
  const bool face_ok = f >= 0 && f < b.mesh.nf;
  if (!face_ok || !make_tangent_frame(b.mesh, f, v, &fv)) {  // diff.cpp:284 throws for the whole call
    note_error(b.err + 0, i);
    for (int k = 0; k < 2; ++k) put_job(b.j1_face, b.j1_bary, b.j1_dir, b.j1_payload, k * n + i, f, p, zero, zero);
    put_job(b.j2_face, b.j2_bary, b.j2_dir, nullptr, 2 * n + i, f, p, zero, zero);
    // (the base job keeps the sample's own v: with a fused forward its record is the forward result of the sample)
    if (b.base_in_round2) put_job(b.j2_face, b.j2_bary, b.j2_dir, nullptr, 3 * n + i, f, p, v, zero);
    return;
  }
  const BaryFrame fp = make_bary_frame(load_face<double>(b.mesh, f));
  put_job(b.j1_face, b.j1_bary, b.j1_dir, b.j1_payload, i, f, p, fp.u_hat * b.eps_p, v);              // seed_u
  put_job(b.j1_face, b.j1_bary, b.j1_dir, b.j1_payload, n + i, f, p, fp.v_hat * b.eps_p, v);          // seed_v
  put_job(b.j2_face, b.j2_bary, b.j2_dir, nullptr, 2 * n + i, f, p, v + fv.e_perp * b.eps_v, zero);   // perp (runs in round 2)
  if (b.base_in_round2) put_job(b.j2_face, b.j2_bary, b.j2_dir, nullptr, 3 * n + i, f, p, v, zero);   // base (ditto)
  if (b.frames) store_frames(b.frames, i, &fv, &fp, nullptr);
}

__global__ void __launch_bounds__(128) gfd_round2_jobs_kernel(const __grid_constant__ GfdBuffers b) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t n = b.n;
  if (i >= n) return;
  const V zero{0.0, 0.0, 0.0};
  const V p = ld3(b.bary, i);
  const int f = b.face[i];
  if (!b.base_in_round2) {
    // require_base, diff.cpp:121-124
    if (!reached(b.base_status[i], b.base_term[i])) {
      note_error(b.err + 1, i);
      for (int k = 0; k < 4; ++k) put_job(b.j2_face, b.j2_bary, b.j2_dir, nullptr, k * n + i, f, p, zero, zero);
      return;
    }
    put_job(b.par_jface, b.par_jbary, b.par_jdir, nullptr, i, b.base_face[i], ld3(b.base_bary, i), ld3(b.base_dir, i) * b.eps_v, zero);
  }
  for (int k = 0; k < 2; ++k) {  // diff.cpp:302-308: ret_u, ret_v from the seeds' end states
    const int64_t s = k * n + i;
    if (reached(b.r1_status[s], b.r1_term[s]))
      put_job(b.j2_face, b.j2_bary, b.j2_dir, nullptr, s, b.r1_face[s], ld3(b.r1_bary, s), ld3(b.r1_payload, s), zero);
    else
      put_job(b.j2_face, b.j2_bary, b.j2_dir, nullptr, s, f, p, zero, zero);
  }
}

// Without a caller-provided base: the par jobs start where the base traces of round 2 ended.
__global__ void __launch_bounds__(128) gfd_par_jobs_kernel(const __grid_constant__ GfdBuffers b) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= b.n) return;
  const V zero{0.0, 0.0, 0.0};
  if (!reached(b.base_status[i], b.base_term[i])) {  // require_base, diff.cpp:121-124
    note_error(b.err + 1, i);
    put_job(b.par_jface, b.par_jbary, b.par_jdir, nullptr, i, b.face[i], ld3(b.bary, i), zero, zero);
    return;
  }
  put_job(b.par_jface, b.par_jbary, b.par_jdir, nullptr, i, b.base_face[i], ld3(b.base_bary, i), ld3(b.base_dir, i) * b.eps_v, zero);
}

// Endpoint of a finished job in ambient space.
__device__ __forceinline__ V end_point(const MeshView& m, const int32_t* rf, const double* rb, int64_t slot) {
  return embed(load_face<double>(m, rf[slot]), ld3(rb, slot));
}

// Assembly of one sample, diff.cpp:151-204 + :312-324. phase 0: forward differences only; a
// column whose + trace did not reach its length is flagged and left for the fallback rounds.
// phase 1 (after rounds 3/4): flagged samples are re-assembled with one-sided differences.
template <int kPhase>
__global__ void __launch_bounds__(128) gfd_assemble_kernel(const __grid_constant__ GfdBuffers b) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t n = b.n;
  if (i >= n) return;
  if (*(volatile unsigned long long*)(b.err + 0) != kNoError || *(volatile unsigned long long*)(b.err + 1) != kNoError) return;
  uint8_t* dflag = b.degraded + 4 * i;
  if (kPhase == 1 && !(dflag[0] | dflag[1] | dflag[2] | dflag[3])) return;

  const int f = b.face[i];
  const V v = ld3(b.v, i);
  TangentFrame fv;
  make_tangent_frame(b.mesh, f, v, &fv);
  const BaryFrame fp = make_bary_frame(load_face<double>(b.mesh, f));
  const Face<double> cb = load_face<double>(b.mesh, b.base_face[i]);
  const BaryFrame fo = make_bary_frame(cb);
  const V ref = embed(cb, ld3(b.base_bary, i));
  if (kPhase == 0 && b.frames) store_frames(b.frames, i, nullptr, nullptr, &fo);

  // seeds must have traced, diff.cpp:182-184
  if (!reached(b.r1_status[i], b.r1_term[i]) || !reached(b.r1_status[n + i], b.r1_term[n + i])) {
    note_error(b.err + 2, i);
    return;
  }

  V col[4];  // par, perp, u, v
  bool deg[4] = {false, false, false, false};
  {  // + side (fd_column :130-137)
    // par (its own result arrays, indexed by sample), perp, u, v (round 2)
    const int64_t slot[4] = {i, 2 * n + i, i, n + i};
    const uint8_t* st[4] = {b.par_status, b.r2_status, b.r2_status, b.r2_status};
    const uint8_t* tm[4] = {b.par_term, b.r2_term, b.r2_term, b.r2_term};
    const int32_t* rf[4] = {b.par_face, b.r2_face, b.r2_face, b.r2_face};
    const double* rb[4] = {b.par_bary, b.r2_bary, b.r2_bary, b.r2_bary};
    const double eps[4] = {b.eps_v, b.eps_v, b.eps_p, b.eps_p};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (reached(st[c][slot[c]], tm[c][slot[c]])) {
        col[c] = (end_point(b.mesh, rf[c], rb[c], slot[c]) - ref) / eps[c];
      } else {
        deg[c] = true;
        col[c] = V{0.0, 0.0, 0.0};
      }
    }
  }
  if (kPhase == 0) {
    dflag[0] = deg[0]; dflag[1] = deg[1]; dflag[2] = deg[2]; dflag[3] = deg[3];
    if (deg[0] | deg[1] | deg[2] | deg[3]) atomicAdd(b.err + 3, 1ull);
  } else {
    // - side: par / perp come straight from round 3, u / v from the round-4 retraces
    const double eps[4] = {b.eps_v, b.eps_v, b.eps_p, b.eps_p};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (!deg[c]) continue;
      const int64_t s3 = c * n + i;
      if (b.r3_status[s3] == kStatusStalled) { note_error(b.err + 4, i); return; }  // trace() throws, diff.cpp:161,167,190
      if (c < 2) {
        if (reached(b.r3_status[s3], b.r3_term[s3])) col[c] = (ref - end_point(b.mesh, b.r3_face, b.r3_bary, s3)) / eps[c];
      } else if (reached(b.r3_status[s3], b.r3_term[s3])) {
        const int64_t s4 = (c - 2) * n + i;
        if (b.r4_status[s4] == kStatusStalled) { note_error(b.err + 4, i); return; }
        if (reached(b.r4_status[s4], b.r4_term[s4])) col[c] = (ref - end_point(b.mesh, b.r4_face, b.r4_bary, s4)) / eps[c];
      }
      // a column that fails both ways stays zero and flagged
    }
  }

  // Mat2{a0, b0, a1, b1}, diff.cpp:172-174, :201-203
  const double jv[4] = {dot(fo.pinv0, col[0]), dot(fo.pinv0, col[1]), dot(fo.pinv1, col[0]), dot(fo.pinv1, col[1])};
  const double jp[4] = {dot(fo.pinv0, col[2]), dot(fo.pinv0, col[3]), dot(fo.pinv1, col[2]), dot(fo.pinv1, col[3])};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (b.jv) b.jv[4 * i + k] = jv[k];
    if (b.jp) b.jp[4 * i + k] = jp[k];
  }
  if (b.g) {  // pullback_ambient with the GFD branch of pullback, diff.cpp:342-354
    const V g = ld3(b.g, i);
    const double go0 = dot(fo.u_hat, g), go1 = dot(fo.v_hat, g);
    const double gv0 = jv[0] * go0 + jv[2] * go1, gv1 = jv[1] * go0 + jv[3] * go1;
    const double gp0 = jp[0] * go0 + jp[2] * go1, gp1 = jp[1] * go0 + jp[3] * go1;
    if (b.grad_v) st3(b.grad_v, i, fv.e_par * gv0 + fv.e_perp * gv1);
    if (b.grad_p) st3(b.grad_p, i, fp.pinv0 * gp0 + fp.pinv1 * gp1);
  }
}

// pullback_ambient through GFD Jacobians that are already there (diff.cpp:342-354): the last block of
// gfd_assemble_kernel on its own, same expressions, same bits. One thread per sample.
__global__ void __launch_bounds__(128) gfd_pullback_kernel(const __grid_constant__ GfdPullback b) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= b.n) return;
  const int f = b.face[i], fe = b.end_face[i];
  if (f < 0 || f >= b.mesh.nf || fe < 0 || fe >= b.mesh.nf) return;
  TangentFrame fv;
  if (!make_tangent_frame(b.mesh, f, ld3(b.v, i), &fv)) return;
  const BaryFrame fp = make_bary_frame(load_face<double>(b.mesh, f));
  const BaryFrame fo = make_bary_frame(load_face<double>(b.mesh, fe));
  const double* jv = b.jv + 4 * i;
  const double* jp = b.jp + 4 * i;
  const V g = ld3(b.g, i);
  const double go0 = dot(fo.u_hat, g), go1 = dot(fo.v_hat, g);
  const double gv0 = jv[0] * go0 + jv[2] * go1, gv1 = jv[1] * go0 + jv[3] * go1;
  const double gp0 = jp[0] * go0 + jp[2] * go1, gp1 = jp[1] * go0 + jp[3] * go1;
  if (b.grad_v) st3(b.grad_v, i, fv.e_par * gv0 + fv.e_perp * gv1);
  if (b.grad_p) st3(b.grad_p, i, fp.pinv0 * gp0 + fp.pinv1 * gp1);
}

__global__ void __launch_bounds__(128) gfd_fallback_jobs_kernel(const __grid_constant__ GfdBuffers b) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t n = b.n;
  if (i >= n) return;
  const V zero{0.0, 0.0, 0.0};
  const int f = b.face[i];
  const V p = ld3(b.bary, i), v = ld3(b.v, i);
  const uint8_t* dflag = b.degraded + 4 * i;
  for (int c = 0; c < 4; ++c) put_job(b.j3_face, b.j3_bary, b.j3_dir, b.j3_payload, c * n + i, f, p, zero, zero);
  if (!(dflag[0] | dflag[1] | dflag[2] | dflag[3])) return;
  TangentFrame fv;
  make_tangent_frame(b.mesh, f, v, &fv);
  const BaryFrame fp = make_bary_frame(load_face<double>(b.mesh, f));
  if (dflag[0])  // diff.cpp:161
    put_job(b.j3_face, b.j3_bary, b.j3_dir, b.j3_payload, i, b.base_face[i], ld3(b.base_bary, i), ld3(b.base_dir, i) * -b.eps_v, zero);
  if (dflag[1])  // diff.cpp:167
    put_job(b.j3_face, b.j3_bary, b.j3_dir, b.j3_payload, n + i, f, p, v - fv.e_perp * b.eps_v, zero);
  if (dflag[2])  // diff.cpp:187-190
    put_job(b.j3_face, b.j3_bary, b.j3_dir, b.j3_payload, 2 * n + i, f, p, fp.u_hat * -b.eps_p, v);
  if (dflag[3])
    put_job(b.j3_face, b.j3_bary, b.j3_dir, b.j3_payload, 3 * n + i, f, p, fp.v_hat * -b.eps_p, v);
}

__global__ void __launch_bounds__(128) gfd_fallback_round2_jobs_kernel(const __grid_constant__ GfdBuffers b) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t n = b.n;
  if (i >= n) return;
  const V zero{0.0, 0.0, 0.0};
  const int f = b.face[i];
  const V p = ld3(b.bary, i);
  const uint8_t* dflag = b.degraded + 4 * i;
  for (int c = 2; c < 4; ++c) {
    const int64_t s3 = c * n + i, s4 = (c - 2) * n + i;
    if (dflag[c] && reached(b.r3_status[s3], b.r3_term[s3]))  // diff.cpp:191-193
      put_job(b.j4_face, b.j4_bary, b.j4_dir, nullptr, s4, b.r3_face[s3], ld3(b.r3_bary, s3), ld3(b.r3_payload, s3), zero);
    else
      put_job(b.j4_face, b.j4_bary, b.j4_dir, nullptr, s4, f, p, zero, zero);
  }
}

// ---------------------------------------------------------------- single-transition operations

// classify, mesh.cpp:214-223: 0 interior, 1 edge, 2 vertex
__device__ int classify(const V& b, double tol, int* local) {
  int imax = 0, imin = 0;
  const double bb[3] = {b.x, b.y, b.z};
  for (int i = 1; i < 3; ++i) {
    if (bb[i] > bb[imax]) imax = i;
    if (bb[i] < bb[imin]) imin = i;
  }
  if (bb[imax] >= 1.0 - tol) { *local = imax; return 2; }
  if (bb[imin] <= tol) { *local = imin; return 1; }
  *local = -1;
  return 0;
}

__global__ void __launch_bounds__(64) transition_kernel(const __grid_constant__ TransitionParams p) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= p.n) return;
  const int f = p.face[i];
  const V b = ld3(p.bary, i), v = ld3(p.v, i);
  auto done = [&](int rc) { p.rc[i] = rc; };
  if (p.stall) p.stall[i] = kStallNone;
  if (f < 0 || f >= p.mesh.nf) return done(1);  // InvalidArgs "... face out of range"

  Tracer<double, true> T(p.mesh, 0x7fffffff, p.which == 3 ? true : p.hole_avoidance != 0);
  T.set_face(f);
  T.bary = b;
  int local = -1;
  const int kind = classify(b, 1e-10, &local);

  if (p.which == 0) {  // geodesic_step, tracer.cpp:630-654
    T.snap_bary();
    T.dir = normalized(v);
    const double rem = p.remaining[i];
    T.target = T.remaining = rem;
    const Outcome oc = T.step();
    if (oc == Outcome::Stalled) {
      if (p.stall) p.stall[i] = T.stall_code;
      return done(10);
    }
    const V wb = T.widened_bary();
    p.out_face[i] = T.face;
    st3(p.out_bary, i, wb);
    st3(p.out_v, i, T.dir);
    if (p.step_length) p.step_length[i] = rem - T.remaining;
    if (p.finished) p.finished[i] = oc == Outcome::Finished;
    if (p.event) p.event[i] = T.last_event;
    return done(0);
  }
  if (p.which == 1) {  // transport_over_edge, tracer.cpp:656-681
    if (kind != 1) return done(1);
    const int k = local;
    const int g = T.cur.adj(k);
    if (g < 0) return done(1);
    const int ka = (k + 1) % 3, kc = (k + 2) % 3;
    const int va = T.cur.id(ka), vc = T.cur.id(kc);
    const Face<double> G = load_face<double>(p.mesh, g);
    EdgeTransport<double> t = Tracer<double, true>::make_edge_transport(T.cur.pos(ka), T.cur.pos(kc), T.cur.pos(k),
                                                                        G.pos_of(G.third(va, vc)));
    V vp = t(v);
    const double nn = norm(vp);
    if (nn > 0) vp = vp * (norm(v) / nn);
    V nb{0.0, 0.0, 0.0};
    put(nb, G.corner_of(va), get(b, ka));
    put(nb, G.corner_of(vc), get(b, kc));
    p.out_face[i] = g;
    st3(p.out_bary, i, nb);
    st3(p.out_v, i, vp);
    return done(0);
  }
  if (p.which == 2) {  // transport_over_vertex, tracer.cpp:683-704
    if (kind != 2) return done(1);
    T.snap_bary();
    const double speed = norm(v);
    T.dir = normalized(v);
    T.remaining = T.target = 1.0;
    const int x0 = T.cur.id(local);
    if (!T.fan_walk(x0)) return done(11);  // BoundaryHit
    p.out_face[i] = T.face;
    st3(p.out_bary, i, T.widened_bary());
    st3(p.out_v, i, T.dir * speed);
    return done(0);
  }
  // boundary_continue, tracer.cpp:706-735
  T.snap_bary();
  const double speed = norm(v);
  T.dir = normalized(v);
  T.remaining = T.target = HUGE_VAL;
  if (kind == 2) {
    const int x0 = T.cur.id(local);
    if (!p.mesh.vboundary[x0]) return done(1);
    bool then_advance = false;
    T.blue_vertex(x0, &then_advance);
    if (then_advance) T.advance();
  } else if (kind == 1) {
    if (T.cur.adj(local) >= 0) return done(1);
    T.slide_from_edge(local);
  } else {
    return done(1);
  }
  p.out_face[i] = T.face;
  st3(p.out_bary, i, T.widened_bary());
  st3(p.out_v, i, T.dir * speed);
  return done(0);
}

inline unsigned grid_for(int64_t n, int block) { return unsigned((n + block - 1) / block); }

}  // namespace

cudaError_t launch_ep(const EpParams& p, cudaStream_t stream) {
  if (p.n <= 0) return cudaSuccess;
  ep_kernel<<<grid_for(p.n, 128), 128, 0, stream>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_gfd_round1_jobs(const GfdBuffers& b, cudaStream_t stream) {
  gfd_round1_jobs_kernel<<<grid_for(b.n, 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_gfd_round2_jobs(const GfdBuffers& b, cudaStream_t stream) {
  gfd_round2_jobs_kernel<<<grid_for(b.n, 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_gfd_par_jobs(const GfdBuffers& b, cudaStream_t stream) {
  gfd_par_jobs_kernel<<<grid_for(b.n, 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_gfd_assemble(const GfdBuffers& b, cudaStream_t stream) {
  gfd_assemble_kernel<0><<<grid_for(b.n, 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_gfd_pullback(const GfdPullback& b, cudaStream_t stream) {
  if (b.n <= 0) return cudaSuccess;
  gfd_pullback_kernel<<<unsigned((b.n + 127) / 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_gfd_fallback_jobs(const GfdBuffers& b, cudaStream_t stream) {
  gfd_fallback_jobs_kernel<<<grid_for(b.n, 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_gfd_fallback_round2_jobs(const GfdBuffers& b, cudaStream_t stream) {
  gfd_fallback_round2_jobs_kernel<<<grid_for(b.n, 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_gfd_fallback_assemble(const GfdBuffers& b, cudaStream_t stream) {
  gfd_assemble_kernel<1><<<grid_for(b.n, 128), 128, 0, stream>>>(b);
  return cudaGetLastError();
}
cudaError_t launch_transition(const TransitionParams& p, cudaStream_t stream) {
  if (p.n <= 0) return cudaSuccess;
  transition_kernel<<<grid_for(p.n, 64), 64, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace dg
