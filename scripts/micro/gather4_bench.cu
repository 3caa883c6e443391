// Micro-benchmark: random 128-byte record gathers through TMA tile::gather4 (one instruction fetches
// four rows of a 2-D tensor map [records x 16 doubles], 128B-swizzled into shared memory), eight
// ops per warp per iteration, one mbarrier per warp; each lane then reads its own row (8 x 128-bit).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_bench gather4_bench.cu   (no -lcuda: entry point via the runtime)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(128, 4) gather4(const __grid_constant__ CUtensorMap tmap, uint32_t nrec, int iters, double* out) {
  extern __shared__ __align__(1024) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* rows = smem + warp * 4096;                         // 32 rows x 128 B, 1024-aligned: swizzle phase = row & 7
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * 4096) + warp;
  const uint32_t bar_s = uint32_t(__cvta_generic_to_shared(bar));
  const uint32_t rows_s = uint32_t(__cvta_generic_to_shared(rows));
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u % nrec;
  double acc = 0;
  uint32_t phase = 0;
  for (int i = 0; i < iters; ++i) {
    const int r1 = __shfl_down_sync(0xffffffffu, int(idx), 1), r2 = __shfl_down_sync(0xffffffffu, int(idx), 2),
              r3 = __shfl_down_sync(0xffffffffu, int(idx), 3);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(4096) : "memory");
    if ((lane & 3) == 0) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(rows_s + lane * 128), "l"(&tmap), "r"(0), "r"(int(idx)), "r"(r1), "r"(r2), "r"(r3), "r"(bar_s) : "memory");
    }
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(bar_s), "r"(phase) : "memory");
    }
    phase ^= 1;
    double s = 0;
    double2 last;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 t = *reinterpret_cast<const double2*>(rows + lane * 128 + ((k ^ (lane & 7)) << 4));
      if (k < 7) s += t.x + t.y; else { s += t.x; last = t; }
    }
    acc += s;
    idx = uint32_t(__double2loint(last.y)) % nrec;
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const uint32_t nrec = argc > 1 ? atoi(argv[1]) : 245760;
  const int iters = argc > 2 ? atoi(argv[2]) : 400;
  char* rec; double* out;
  cudaMalloc(&rec, size_t(nrec) * 128);
  double* h = (double*)malloc(size_t(nrec) * 128);
  uint32_t x = 12345;
  double check = 0;
  for (uint32_t r = 0; r < nrec; ++r) {
    for (int k = 0; k < 15; ++k) h[size_t(r) * 16 + k] = 1e-3 * k;
    x = x * 1664525u + 1013904223u;
    uint64_t bits = x % nrec;
    memcpy(&h[size_t(r) * 16 + 15], &bits, 8);
  }
  for (int k = 0; k < 15; ++k) check += 1e-3 * k;
  cudaMemcpy(rec, h, size_t(nrec) * 128, cudaMemcpyHostToDevice);
  // tensor map: 2-D [nrec rows][16 doubles], box = 1 row x 16 doubles (gather4 fetches 4 such rows), 128B swizzle
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult qres;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres);
  if (!fn) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  CUtensorMap tmap;
  cuuint64_t dims[2] = {16, nrec}, strides[1] = {128};
  cuuint32_t box[2] = {16, 1}, estr[2] = {1, 1};
  CUresult cr = ((EncodeFn)fn)(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, rec, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed: %d\n", int(cr)); return 1; }
  int sm; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sm * 4, threads = 128;
  cudaMalloc(&out, size_t(blocks) * threads * 8);
  const size_t smem = 4 * 4096 + 64 + 1024;
  cudaFuncSetAttribute(gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    gather4<<<blocks, threads, smem>>>(tmap, nrec, iters, out);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double o0; cudaMemcpy(&o0, out, 8, cudaMemcpyDeviceToHost);
    if (rep == 2) printf("gather4 (8 ops per warp-iteration): %.3f ms, %.2f G records/s (%s), checksum %s\n", ms,
                         double(blocks) * threads * iters / ms / 1e6, cudaGetErrorString(err),
                         fabs(o0 - check * iters) < 1e-6 * iters ? "ok" : "WRONG");
  }
  return 0;
}
