// Probe: HBM streaming bandwidth through a shared-memory ring filled by 2D TMA boxes
// (cp.async.bulk.tensor.2d) over a row-major bf16 matrix, per box shape and swizzle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma2d_probe tma2d_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void etx(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void arr(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void wt(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@P bra D;\nbra W;\nD:\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su(d)), "l"(m), "r"(c0), "r"(c1), "r"(su(b)) : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap map, int rows_per_cta, int cols, int bc, int br, int boxes_per_stage, int nst, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  uint8_t* ring = sm + 1024;
  const int box_bytes = bc * br * 2, stage = box_bytes * boxes_per_stage;
  if (threadIdx.x == 0) { for (int i = 0; i < nst; ++i) { init(&full[i], 1); init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const int bands = rows_per_cta / br, kcols = cols / bc;
  const int nbox = bands * kcols, nstage = nbox / boxes_per_stage;
  if (threadIdx.x == 0) {
    int box = 0;
    for (int n = 0; n < nstage; ++n) {
      const int s = n % nst;
      wt(&empty[s], ((n / nst) & 1) ^ 1);
      etx(&full[s], stage);
      for (int j = 0; j < boxes_per_stage; ++j, ++box) {
        const int band = box / kcols, kc = box % kcols;
        tma2d(ring + s * stage + j * box_bytes, &map, &full[s], kc * bc, blockIdx.x * rows_per_cta + band * br);
      }
    }
  } else if (threadIdx.x >= 32 && threadIdx.x < 64) {
    unsigned long long acc = 0;
    for (int n = 0; n < nstage; ++n) {
      const int s = n % nst;
      wt(&full[s], (n / nst) & 1);
      acc += ring[s * stage + (threadIdx.x & 31)];
      __syncwarp();
      if (threadIdx.x == 32) arr(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int cols = 4096, rows_per_cta = 256, rows = 148 * rows_per_cta;
  const size_t total = (size_t)rows * cols * 2;
  void* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct Cfg { int bc, br, bps, nst, swz; };
  Cfg cfgs[] = {{256, 32, 2, 4, 0}, {256, 64, 1, 4, 0}, {256, 16, 4, 4, 0}, {128, 32, 4, 4, 0}, {256, 8, 8, 4, 0},
                {64, 128, 2, 4, 1}, {64, 256, 1, 4, 1}, {64, 32, 8, 4, 1}, {64, 16, 16, 4, 1}, {256, 32, 4, 3, 0}, {256, 64, 2, 3, 0}};
  for (auto c : cfgs) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)c.bc, (cuuint32_t)c.br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     c.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d for %d x %d\n", (int)r, c.bc, c.br); continue; }
    const int smem = 1024 + c.bc * c.br * 2 * c.bps * c.nst;
    for (int it = 0; it < 2; ++it) probe<<<148, 64, smem>>>(m, rows_per_cta, cols, c.bc, c.br, c.bps, c.nst, sink);
    cudaEventRecord(a);
    const int iters = 10;
    for (int it = 0; it < iters; ++it) probe<<<148, 64, smem>>>(m, rows_per_cta, cols, c.bc, c.br, c.bps, c.nst, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("{\"box_cols\": %d, \"box_rows\": %d, \"box_bytes\": %d, \"boxes_per_stage\": %d, \"stages\": %d, \"swizzle128\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n",
           c.bc, c.br, c.bc * c.br * 2, c.bps, c.nst, c.swz, (double)total * iters / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
