// Forward tracing kernel: persistent warps, one geodesic per lane, lane-level work stealing.
//
// Replaces the reference's `#pragma omp parallel for schedule(dynamic, 8)` over run_one
// (proj/src/tracer.cpp:596-603). Path lengths differ by orders of magnitude between queries,
// so a lane that finishes its geodesic does not wait for the rest of its warp: between two
// steps the warp ballots its idle lanes, ONE lane advances the global queue cursor by the
// number of idle lanes (warp-aggregated atomic) and every idle lane initialises the next
// query in place. The grid is sized to the resident capacity of the chip (SM count x
// resident blocks per SM), never to the batch.
#include <atomic>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "dg_fast_walk.cuh"
#include "dg_kernels.cuh"
#include "dg_tracer_core.cuh"

namespace dg {

namespace {

#ifndef DG_TRACE_BLOCK
#define DG_TRACE_BLOCK 128
#endif
// Resident CTAs per SM the register allocation is capped for. The lite f64 walker fits 128
// registers (4 CTAs x 4 warps per SM) with ~50 bytes of spill and is 17% faster there than at its
// natural 146 registers / 3 CTAs (profiles/tuning_r1.md); the full variant (212 registers) keeps 2 CTAs.
#ifndef DG_TRACE_MIN_BLOCKS
#define DG_TRACE_MIN_BLOCKS 4
#endif
#ifndef DG_TRACE_MIN_BLOCKS_FULL
#define DG_TRACE_MIN_BLOCKS_FULL 2
#endif
constexpr int kBlockThreads = DG_TRACE_BLOCK;
constexpr unsigned kFullMask = 0xffffffffu;

template <class S, bool kFull, bool kCached>
__device__ __forceinline__ void write_result(const TraceParams& p, int64_t q,
                                             const Tracer<S, kFull, kCached>& T) {
  V3<double> b = T.widened_bary();
  if (p.o_face) p.o_face[q] = T.face;
  if (p.o_bary) { p.o_bary[3 * q] = b.x; p.o_bary[3 * q + 1] = b.y; p.o_bary[3 * q + 2] = b.z; }
  if (p.o_dir) {
    // tracer.cpp:525: zero for zero-length requests
    V3<double> d = T.target > S(0) ? cast<double>(T.dir) : V3<double>{0.0, 0.0, 0.0};
    p.o_dir[3 * q] = d.x; p.o_dir[3 * q + 1] = d.y; p.o_dir[3 * q + 2] = d.z;
  }
  if (p.o_traced && q >= p.aux_from) p.o_traced[q - p.aux_from] = T.traced;
  if (p.o_requested && q >= p.aux_from) p.o_requested[q - p.aux_from] = double(T.target);
  if (p.o_term) p.o_term[q] = T.term;
  if (p.o_status) p.o_status[q] = T.status;
  if (p.o_stall && q >= p.aux_from) p.o_stall[q - p.aux_from] = T.stall_code;
  if (p.o_npoints && q >= p.aux_from) p.o_npoints[q - p.aux_from] = T.npoints;
  if (p.o_crossings && q >= p.aux_from) p.o_crossings[q - p.aux_from] = T.crossings;
  if (kFull) {
    if (p.o_payload) {
      V3<double> w = T.has_payload ? cast<double>(T.payload) : V3<double>{0.0, 0.0, 0.0};
      p.o_payload[3 * q] = w.x; p.o_payload[3 * q + 1] = w.y; p.o_payload[3 * q + 2] = w.z;
    }
    if (p.o_transport) {
      // Mat3::from_columns(q0, q1, q2), row-major (geometry.hpp:80-84)
      double* o = p.o_transport + 9 * q;
      const bool on = T.want_q;
      o[0] = on ? double(T.q0.x) : 0.0; o[1] = on ? double(T.q1.x) : 0.0; o[2] = on ? double(T.q2.x) : 0.0;
      o[3] = on ? double(T.q0.y) : 0.0; o[4] = on ? double(T.q1.y) : 0.0; o[5] = on ? double(T.q2.y) : 0.0;
      o[6] = on ? double(T.q0.z) : 0.0; o[7] = on ? double(T.q1.z) : 0.0; o[8] = on ? double(T.q2.z) : 0.0;
    }
  } else {
    // the lite kernel is only launched when neither output is requested
  }
}

template <class S, bool kFull, bool kCached>
__global__ void __launch_bounds__(kBlockThreads, kFull ? DG_TRACE_MIN_BLOCKS_FULL : DG_TRACE_MIN_BLOCKS) trace_kernel(const __grid_constant__ TraceParams p) {
  Tracer<S, kFull, kCached> T(p.mesh, p.max_steps, p.hole_avoidance != 0);
  const unsigned lane = threadIdx.x & 31u;
  const unsigned long long n = (unsigned long long)p.n;
  if (p.clear_word && blockIdx.x == 0 && threadIdx.x == 0) *p.clear_word = 0ull;
  bool live = false;
  bool exhausted = false;  // warp-uniform: the queue has no more work
  int64_t q = -1;
  unsigned long long my_crossings = 0;

  for (;;) {
    const unsigned idle = __ballot_sync(kFullMask, !live);
    if (idle != 0u && !exhausted) {
      const int n_idle = __popc(idle);
      if (n_idle >= p.refill_min || n_idle == 32) {
        const int leader = __ffs(idle) - 1;
        unsigned long long base = 0;
        if (lane == unsigned(leader)) base = atomicAdd(p.queue_head, (unsigned long long)n_idle);
        base = __shfl_sync(kFullMask, base, leader);
        if (base + (unsigned long long)n_idle >= n) exhausted = true;
        if (!live) {
          const unsigned long long slot = base + (unsigned long long)__popc(idle & ((1u << lane) - 1u));
          if (slot < n) {
            q = p.perm ? int64_t(p.perm[slot]) : int64_t(slot);
            const int f = p.face[q];
            const V3<double> b{p.bary[3 * q], p.bary[3 * q + 1], p.bary[3 * q + 2]};
            const V3<double> v{p.dir[3 * q], p.dir[3 * q + 1], p.dir[3 * q + 2]};
            V3<double> pay{0.0, 0.0, 0.0};
            bool has_pay = false;
            if (kFull && p.payload) {
              pay = V3<double>{p.payload[3 * q], p.payload[3 * q + 1], p.payload[3 * q + 2]};
              has_pay = norm2(pay) > 0.0;  // tracer.cpp:582
            }
            T.reset();
            if (kFull && (p.poly_offsets || p.poly_cap > 0)) {
              T.sink.face = p.poly_face; T.sink.bary = p.poly_bary; T.sink.seg = p.poly_seg;
              T.sink.base = p.poly_offsets ? p.poly_offsets[q] : int64_t(q) * p.poly_cap;
              T.sink.cap = p.poly_cap;
            }
            live = T.initialise(f, b, v, pay, has_pay, p.want_q != 0);
            if (!live) write_result<S, kFull, kCached>(p, q, T);
          }
        }
      }
    }
    if (__ballot_sync(kFullMask, live) == 0u) {
      if (exhausted) break;
      continue;
    }
    if (live) {
      live = T.run_step();
      if (!live) {
        if (q >= p.aux_from) my_crossings += (unsigned long long)T.crossings;
        write_result<S, kFull, kCached>(p, q, T);
      }
    }
  }

  if (p.total_crossings) {
    for (int o = 16; o > 0; o >>= 1) my_crossings += __shfl_xor_sync(kFullMask, my_crossings, o);
    if (lane == 0 && my_crossings) atomicAdd(p.total_crossings, my_crossings);
  }
}

template <class S, bool kFull, bool kCached>
cudaError_t launch_one(const TraceParams& p_in, LaunchShape shape, cudaStream_t stream) {
  TraceParams p = p_in;
  if (p.refill_min <= 0) p.refill_min = 1;  // the general walker refills a lane as soon as it is idle
  int per_sm = shape.blocks_per_sm;
  if (per_sm <= 0) {
    static std::atomic<int> cached_per_sm{0};  // per kernel variant; the query costs microseconds per call
    per_sm = cached_per_sm.load(std::memory_order_relaxed);
    if (per_sm <= 0) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trace_kernel<S, kFull, kCached>,
                                                                    kBlockThreads, 0);
      if (e != cudaSuccess) return e;
      if (per_sm < 1) per_sm = 1;
      cached_per_sm.store(per_sm, std::memory_order_relaxed);
    }
  }
  long long blocks = (long long)shape.sm_count * per_sm;
  const long long needed = (p.n + kBlockThreads - 1) / kBlockThreads;
  if (blocks > needed) blocks = needed;
  if (blocks < 1) blocks = 1;
  trace_kernel<S, kFull, kCached><<<unsigned(blocks), kBlockThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

template <bool kCached, int kTma, int kPay = 0, bool kDense = false, int kLane = 0, bool kStream = false>
cudaError_t launch_fast(const TraceParams& p_in, LaunchShape shape, cudaStream_t stream) {
  constexpr size_t smem = kTma ? size_t(kFastTmaSmemBytes) : 0;
  TraceParams p = p_in;
  // Start-ups side by side: a warp waits for 4 idle lanes, at most DG_REFILL_PATIENCE (8) transitions.
  // Measured: c2 3.97 -> 3.77 ms, c3 24.46 -> 24.63 ms (profiles/tuning_r1.md).
  if (p.refill_min <= 0) p.refill_min = 4;
  p.snap_hi = 1.0 - 1e-10;
  int per_sm = shape.blocks_per_sm;
  if (per_sm <= 0) {
    static std::atomic<int> cached_per_sm{0};
    per_sm = cached_per_sm.load(std::memory_order_relaxed);
    if (per_sm <= 0) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trace_fast_kernel<kCached, kTma, kPay, kDense, kLane, kStream>, DG_FAST_BLOCK, smem);
      if (e != cudaSuccess) return e;
      if (per_sm < 1) per_sm = 1;
      cached_per_sm.store(per_sm, std::memory_order_relaxed);
    }
  }
  long long blocks = (long long)shape.sm_count * per_sm;
  const long long needed = (p.n + DG_FAST_BLOCK - 1) / DG_FAST_BLOCK;
  if (blocks > needed) blocks = needed;
  if (blocks < 1) blocks = 1;
  trace_fast_kernel<kCached, kTma, kPay, kDense, kLane, kStream><<<unsigned(blocks), DG_FAST_BLOCK, smem, stream>>>(p);
  return cudaGetLastError();
}

// DG_FAST_WALK=0 keeps the generic walker on the plain f64 forward path (A/B measurements).
bool fast_walk_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_FAST_WALK");
    return !(e && (!strcmp(e, "0") || !strcmp(e, "off")));
  }();
  return on;
}

// How the fast walker gathers the crossing records (dg_fast_walk.cuh): 0 = four 256-bit loads per lane,
// 1 = TMA tile::gather4, 2 = cooperative 256-bit loads (four lanes per record, sectors handed to their owner
// through shared memory). Measured (profiles/tuning_r1.md; scripts/micro/gather_bench.cu):
//  * lone traces, records within 250 MB (c2): per-lane loads -- 3.80 ms against 4.01 (cooperative) and 4.37 (TMA):
//    the walker is issue-bound there and the per-lane loads cost the fewest instructions;
//  * lone traces beyond (c3 and up): per-lane loads fall off a cliff (one request and one address translation per
//    sector: 37 ms on c3); cooperative loads send one request per record like TMA and need no barrier wait:
//    c3 18.2 ms against 19.4 (TMA), 2.25 M faces 9.7 / 10.3, 7.8 M faces 19.4 / 19.8, config-4 batch 14.6 / 15.7;
//  * a sibling schedule (TraceParams::siblings, GFD round 2): per-lane loads at every size -- the lanes of a group ask
//    for the same line and the load path merges them (c3: 45.3 ms against 52.8 cooperative, 55.9 TMA).
// DG_FAST_GATHER=loads|tma|coop forces one (A/B measurements); dg_trace_cfg.walker selects one per call.
int gather_mode(const MeshView& m, int siblings, bool map_ok, int walker, bool face_order = false) {
  if (!m.he) return 0;
  static const int forced = [] {
    const char* e = getenv("DG_FAST_GATHER");
    return !e ? -1 : !strcmp(e, "loads") ? 0 : !strcmp(e, "tma") ? 1 : !strcmp(e, "coop") ? 2 : -1;
  }();
  int mode;
  if (walker == 2) mode = 0;
  else if (walker == 3) mode = 1;
  else if (walker == 4) mode = 2;
  else if (forced >= 0) mode = forced;
  // (start-face order: neighbouring lanes walk through the same neighbourhood, most sectors are L2 hits and the
  // per-lane loads lead -- c3 15.7 ms against 17.2 cooperative, c4 18.5 against 19.7 -- while the traces are short
  // for the mesh; the request layer queues long-trace batches on the cooperative gather as well and lets the
  // requested lengths, summed on the device, pick: enqueue_trace, dg_capi.cu)
  else mode = (siblings <= 1 && !face_order && size_t(m.nf) * 3 * sizeof(HalfEdgeRec) > (size_t(250) << 20)) ? 2 : 0;
  if (mode == 1 && !map_ok) mode = 2;
  return mode;
}

}  // namespace

int fast_walker_gather_mode(const MeshView& m, bool map_ok, bool face_order) { return fast_walk_enabled() ? gather_mode(m, 0, map_ok, 0, face_order) : 0; }

bool trace_streamable(const TraceParams& p, bool use_f32, bool needs_full, LaunchShape shape) {
  return !use_f32 && !needs_full && shape.walker != 1 && fast_walk_enabled() && !p.lane_fast && p.mesh.he && !p.perm &&
         p.siblings <= 1 && p.aux_from == 0 && gather_mode(p.mesh, p.siblings, p.he_map_ok != 0, shape.walker, false) == 0;
}
cudaError_t launch_trace_streamed(const TraceParams& p, LaunchShape shape, cudaStream_t stream) {
  if (p.n <= 0) return cudaSuccess;
  if (!p.stream_uploaded || !p.stream_done || !p.stream_flags || !p.stream_error || p.stream_shift < 5) return cudaErrorInvalidValue;
  return launch_fast<true, 0, 0, false, 0, true>(p, shape, stream);
}

cudaError_t launch_trace(const TraceParams& p_in, bool use_f32, bool needs_full, LaunchShape shape,
                         cudaStream_t stream) {
  if (p_in.n <= 0) return cudaSuccess;
  // The general walker has no sibling schedule: it runs such a request in plain order (and the order of the GROUPS
  // that perm then holds means nothing to it).
  TraceParams plain = p_in;
  if (plain.siblings > 1) plain.perm = nullptr;
  const bool general = use_f32 || shape.walker == 1 || !fast_walk_enabled();
  const TraceParams& p = general ? plain : p_in;
  if (use_f32) {
    return needs_full ? launch_one<float, true, false>(p, shape, stream) : launch_one<float, false, false>(p, shape, stream);
  }
  const int gather = gather_mode(p.mesh, p.siblings, p.he_map_ok != 0, shape.walker, p.perm != nullptr);
  auto fast = [&](auto pay) {
    constexpr int kPay = decltype(pay)::value;
    if (!p.mesh.he) return launch_fast<false, 0, kPay>(p, shape, stream);
    return gather == 1 ? launch_fast<true, 1, kPay>(p, shape, stream)
         : gather == 2 ? launch_fast<true, 2, kPay>(p, shape, stream)
                       : launch_fast<true, 0, kPay>(p, shape, stream);
  };
  if (!needs_full && shape.walker != 1 && fast_walk_enabled()) {
    if (p.lane_fast && p.mesh.he64 && !std::getenv("DG_LANE_FAST_128")) {
      // DG_LANE_FAST: the tolerance lane over half-size records, intrinsic fold (HalfEdgeRec64)
      if (p.siblings > 1) return launch_fast<true, 0, 0, true, 2>(p, shape, stream);
      return launch_fast<true, 0, 0, false, 2>(p, shape, stream);
    }
    if (p.lane_fast && p.mesh.he) {   // ... over the 128-byte records (no half-size records on this mesh)
      if (gather == 0 && p.siblings > 1) return launch_fast<true, 0, 0, true, 1>(p, shape, stream);
      return gather == 0 ? launch_fast<true, 0, 0, false, 1>(p, shape, stream) : launch_fast<true, 2, 0, false, 1>(p, shape, stream);
    }
    if (p.mesh.he && gather == 0 && p.siblings > 1) return launch_fast<true, 0, 0, true>(p, shape, stream);
    return fast(std::integral_constant<int, 0>{});
  }
  // a payload to transport, hole avoidance, a polyline to record -- anything but the transport matrix:
  // the fast walker carries the payload along, writes one polyline point per step and leaves boundary
  // events to the full Tracer behind it
  const bool payload_only = (p.payload || p.o_payload || p.hole_avoidance || p.poly_offsets || p.poly_cap > 0) && !p.want_q && !p.o_transport;
  if (payload_only && shape.walker != 1 && fast_walk_enabled()) {
    // no payload to carry (the reference's default call: record_polyline = true, no payload): the polyline-only
    // instantiation -- the plain walker's step plus one polyline point (TMA requests take the cooperative gather)
    if (!p.payload && !p.o_payload) {
      if (!p.mesh.he) return launch_fast<false, 0, 3>(p, shape, stream);
      return gather != 0 ? launch_fast<true, 2, 3>(p, shape, stream) : launch_fast<true, 0, 3>(p, shape, stream);
    }
    return fast(std::integral_constant<int, 1>{});
  }
  // the transport matrix as well: three more vectors through every fold isometry
  if (p.want_q && shape.walker != 1 && fast_walk_enabled()) return fast(std::integral_constant<int, 2>{});
  if (p.mesh.he) return needs_full ? launch_one<double, true, true>(p, shape, stream) : launch_one<double, false, true>(p, shape, stream);
  return needs_full ? launch_one<double, true, false>(p, shape, stream) : launch_one<double, false, false>(p, shape, stream);
}

void trace_kernel_info(bool use_f32, int variant, int* regs, int* blocks_per_sm, int* block_threads) {
  cudaFuncAttributes a{};
  int per_sm = 0, threads = kBlockThreads;
  const bool full = variant & 1, cached = (variant & 2) && !use_f32, tma = (variant & 4) != 0, coop = (variant & 8) != 0,
             dense = (variant & 16) != 0;
  auto query = [&](auto kernel, int block) {
    cudaFuncGetAttributes(&a, kernel);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0);
    threads = block;
  };
  if (use_f32) {
    if (full) query(trace_kernel<float, true, false>, kBlockThreads); else query(trace_kernel<float, false, false>, kBlockThreads);
  } else if (!full && fast_walk_enabled()) {
    if (cached && tma) {
      cudaFuncGetAttributes(&a, trace_fast_kernel<true, 1>);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trace_fast_kernel<true, 1>, DG_FAST_BLOCK, kFastTmaSmemBytes);
      threads = DG_FAST_BLOCK;
    } else if (cached && dense) {
      query(trace_fast_kernel<true, 0, 0, true>, DG_FAST_BLOCK);
    } else if (cached && coop) {
      cudaFuncGetAttributes(&a, trace_fast_kernel<true, 2>);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trace_fast_kernel<true, 2>, DG_FAST_BLOCK, kFastTmaSmemBytes);
      threads = DG_FAST_BLOCK;
    } else if (cached) {
      query(trace_fast_kernel<true, 0>, DG_FAST_BLOCK);
    } else {
      query(trace_fast_kernel<false, 0>, DG_FAST_BLOCK);
    }
  } else if (cached) {
    if (full) query(trace_kernel<double, true, true>, kBlockThreads); else query(trace_kernel<double, false, true>, kBlockThreads);
  } else {
    if (full) query(trace_kernel<double, true, false>, kBlockThreads); else query(trace_kernel<double, false, false>, kBlockThreads);
  }
  if (regs) *regs = a.numRegs;
  if (blocks_per_sm) *blocks_per_sm = per_sm;
  if (block_threads) *block_threads = threads;
}

}  // namespace dg
