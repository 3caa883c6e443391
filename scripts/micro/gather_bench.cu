// Micro-benchmark: random 128-byte record gathers from an L2-resident array, one record per lane per
// iteration, (a) four 256-bit loads per lane, (b) one cp.async.bulk (TMA) per lane into shared memory
// with a per-warp mbarrier, then eight 128-bit shared loads. Prints records/s per variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ void ldg256(const void* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

__global__ void __launch_bounds__(128, 4) gather_ldg(const char* rec, uint32_t nrec, int iters, double* out) {
  uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u % nrec;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    const char* p = rec + size_t(idx) * 128;
    double v[16];
    ldg256(p, v[0], v[1], v[2], v[3]); ldg256(p + 32, v[4], v[5], v[6], v[7]);
    ldg256(p + 64, v[8], v[9], v[10], v[11]); ldg256(p + 96, v[12], v[13], v[14], v[15]);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 15; ++k) s += v[k];
    acc += s;
    idx = uint32_t(__double2loint(v[15])) % nrec;   // dependent chain, like the walk
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// (d) 64-byte records, two 256-bit loads per lane: what a half-size crossing record would cost to gather
// (prototype measurement for a tolerance-lane layout; the next index sits in the low word of the 8th double)
__global__ void __launch_bounds__(128, 4) gather_ldg64(const char* rec, uint32_t nrec, int iters, double* out) {
  uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u % nrec;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    const char* p = rec + size_t(idx) * 64;
    double v[8];
    ldg256(p, v[0], v[1], v[2], v[3]); ldg256(p + 32, v[4], v[5], v[6], v[7]);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) s += v[k];
    acc += s;
    idx = uint32_t(__double2loint(v[7])) % nrec;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

constexpr int kStride = 144;  // bytes per lane slot in shared memory (128 + 16: conflict-free 128-bit reads)

__global__ void __launch_bounds__(128, 4) gather_tma(const char* rec, uint32_t nrec, int iters, double* out) {
  extern __shared__ __align__(128) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* slot = smem + warp * (32 * kStride) + lane * kStride;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * 32 * kStride) + warp;
  const uint32_t bar_s = uint32_t(__cvta_generic_to_shared(bar));
  const uint32_t slot_s = uint32_t(__cvta_generic_to_shared(slot));
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
  __syncwarp();
  uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u % nrec;
  double acc = 0;
  uint32_t phase = 0;
  for (int i = 0; i < iters; ++i) {
    const char* p = rec + size_t(idx) * 128;
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(32 * 128) : "memory");
    __syncwarp();
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                 ::"r"(slot_s), "l"(p), "r"(bar_s) : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(bar_s), "r"(phase) : "memory");
    }
    phase ^= 1;
    double s = 0;
    const double2* q = reinterpret_cast<const double2*>(slot);
    double2 last;
#pragma unroll
    for (int k = 0; k < 8; ++k) { double2 t = q[k]; if (k < 7) s += t.x + t.y; else { s += t.x; last = t; } }
    acc += s;
    idx = uint32_t(__double2loint(last.y)) % nrec;
    __syncwarp();   // all lanes have read their slots before the next copies land
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// (c) cooperative loads: in each of the four 256-bit load instructions, lanes 4m..4m+3 read the four
// sectors of ONE record (owner lane 8j+m), so an instruction touches 8 lines instead of 32 -- a quarter of
// the L1TEX->crossbar requests for the same bytes; the sectors reach their owner through shared memory.
__global__ void __launch_bounds__(128, 4) gather_coop(const char* rec, uint32_t nrec, int iters, double* out) {
  extern __shared__ __align__(128) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* wbase = smem + warp * (32 * kStride);
  char* slot = wbase + lane * kStride;
  uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u % nrec;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    double r[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t oi = __shfl_sync(0xffffffffu, idx, 8 * j + (lane >> 2));
      ldg256(rec + size_t(oi) * 128 + (lane & 3) * 32, r[j][0], r[j][1], r[j][2], r[j][3]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2* w = reinterpret_cast<double2*>(wbase + (8 * j + (lane >> 2)) * kStride + (lane & 3) * 32);
      w[0] = make_double2(r[j][0], r[j][1]);
      w[1] = make_double2(r[j][2], r[j][3]);
    }
    __syncwarp();
    double s = 0;
    const double2* q = reinterpret_cast<const double2*>(slot);
    double2 last;
#pragma unroll
    for (int k = 0; k < 8; ++k) { double2 t = q[k]; if (k < 7) s += t.x + t.y; else { s += t.x; last = t; } }
    acc += s;
    idx = uint32_t(__double2loint(last.y)) % nrec;
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const uint32_t nrec = argc > 1 ? atoi(argv[1]) : 245760;   // 31 MB, the c2 record array
  const int iters = argc > 2 ? atoi(argv[2]) : 2000;
  char* rec; double* out;
  cudaMalloc(&rec, size_t(nrec) * 128);
  // records: 15 doubles of payload + the next index in the low word of the 16th
  double* h = (double*)malloc(size_t(nrec) * 128);
  uint32_t x = 12345;
  for (uint32_t r = 0; r < nrec; ++r) {
    for (int k = 0; k < 15; ++k) h[size_t(r) * 16 + k] = 1e-3 * k;
    x = x * 1664525u + 1013904223u;
    uint64_t bits = x % nrec;
    memcpy(&h[size_t(r) * 16 + 15], &bits, 8);
  }
  cudaMemcpy(rec, h, size_t(nrec) * 128, cudaMemcpyHostToDevice);
  int sm; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sm * 4, threads = 128;
  cudaMalloc(&out, size_t(blocks) * threads * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t smem = 4 * 32 * kStride + 64;
  cudaFuncSetAttribute(gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(gather_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int only = argc > 3 ? atoi(argv[3]) : -1;   // one variant, machine-readable: bench.py's gather ceiling
  if (only == 3) {   // 64-byte records: the same array read as 2 nrec half-size records
    const uint32_t n64 = nrec;   // (argv[1] counts 64-byte records in this mode; the array holds nrec * 64 bytes of them)
    double* h64 = (double*)malloc(size_t(n64) * 64);
    uint32_t y = 12345;
    for (uint32_t r = 0; r < n64; ++r) {
      for (int k = 0; k < 7; ++k) h64[size_t(r) * 8 + k] = 1e-3 * k;
      y = y * 1664525u + 1013904223u;
      uint64_t bits = y % n64;
      memcpy(&h64[size_t(r) * 8 + 7], &bits, 8);
    }
    cudaMemcpy(rec, h64, size_t(n64) * 64, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      gather_ldg64<<<blocks, threads>>>(rec, n64, iters, out);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("{\"variant\": 3, \"records\": %u, \"record_bytes\": 64, \"ms\": %.4f, \"grecords_per_s\": %.4f, \"cuda\": \"%s\"}\n",
                           n64, ms, double(blocks) * threads * iters / ms / 1e6, cudaGetErrorString(err));
    }
    return 0;
  }
  for (int variant = 0; variant < 3; ++variant) {
    if (only >= 0 && variant != only) continue;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (variant == 0) gather_ldg<<<blocks, threads>>>(rec, nrec, iters, out);
      else if (variant == 1) gather_tma<<<blocks, threads, smem>>>(rec, nrec, iters, out);
      else gather_coop<<<blocks, threads, smem>>>(rec, nrec, iters, out);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2 && only >= 0) {
        printf("{\"variant\": %d, \"records\": %u, \"ms\": %.4f, \"grecords_per_s\": %.4f, \"cuda\": \"%s\"}\n", variant, nrec, ms,
               double(blocks) * threads * iters / ms / 1e6, cudaGetErrorString(err));
        continue;
      }
      if (rep == 2) printf("%s: %.3f ms, %.2f G records/s (%s)\n", variant == 0 ? "4 x LDG.256 per lane" : variant == 1 ? "1 x cp.async.bulk per lane" : "4 x LDG.256, 4 lanes per record + smem",
                           ms, double(blocks) * threads * iters / ms / 1e6, cudaGetErrorString(err));
    }
  }
  return 0;
}
