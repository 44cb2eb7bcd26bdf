// Probe: HBM streaming bandwidth through a shared-memory ring filled by 1D bulk copies
// (cp.async.bulk) as a function of the copy size and copies per stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_probe bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void etx(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void arr(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void wt(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@P bra D;\nbra W;\nD:\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void cp(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}

// Each CTA streams `per_cta` bytes: stages of `stage` bytes made of `stage/copy` copies
// (copies of a stage are `row_stride` bytes apart in global, like weight rows).
__global__ void probe(const uint8_t* src, size_t per_cta, int stage, int copy, size_t row_stride, int nst, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  uint8_t* ring = sm + 256;
  if (threadIdx.x == 0) { for (int i = 0; i < nst; ++i) { init(&full[i], 1); init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const int ncopy = stage / copy;
  const size_t nstage = per_cta / stage;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (size_t n = 0; n < nstage; ++n) {
      const int s = n % nst;
      wt(&empty[s], ((n / nst) & 1) ^ 1);
      if (lane == 0) etx(&full[s], stage);
      __syncwarp();
      // stage n covers rows [n*ncopy, (n+1)*ncopy) at column 0 .. copy of a matrix with row_stride
      for (int c = lane; c < ncopy; c += 32) {
        const size_t off = row_stride ? ((n * ncopy + c) % (per_cta / row_stride)) * row_stride + ((n * ncopy + c) / (per_cta / row_stride)) * copy
                                      : (n * stage + (size_t)c * copy);
        cp(ring + s * stage + c * copy, base + off, copy, &full[s]);
      }
    }
  } else if (threadIdx.x < 64) {
    unsigned long long acc = 0;
    for (size_t n = 0; n < nstage; ++n) {
      const int s = n % nst;
      wt(&full[s], (n / nst) & 1);
      acc += ring[s * stage + (threadIdx.x & 31)];
      __syncwarp();
      if (threadIdx.x == 32) arr(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

int main() {
  const size_t total = (size_t)148 * 16 * 1024 * 1024;  // 2.3 GiB
  uint8_t* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t per_cta = total / 148;
  struct Cfg { int stage, copy, nst; size_t row_stride; };
  Cfg cfgs[] = {
    {32768, 512, 4, 0}, {32768, 1024, 4, 0}, {32768, 2048, 4, 0}, {32768, 4096, 4, 0}, {32768, 8192, 4, 0}, {32768, 32768, 4, 0},
    {32768, 1024, 4, 8192}, {32768, 2048, 4, 16384}, {16384, 1024, 8, 8192}, {16384, 16384, 8, 0},
    {49152, 1024, 4, 8192}, {49152, 49152, 4, 0}, {24576, 24576, 8, 0}, {8192, 8192, 8, 0}, {4096, 4096, 8, 0}};
  for (auto c : cfgs) {
    const int smem = 256 + c.stage * c.nst;
    for (int it = 0; it < 2; ++it) probe<<<148, 64, smem>>>(buf, per_cta, c.stage, c.copy, c.row_stride, c.nst, sink);
    cudaEventRecord(a);
    const int iters = 5;
    for (int it = 0; it < iters; ++it) probe<<<148, 64, smem>>>(buf, per_cta, c.stage, c.copy, c.row_stride, c.nst, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("{\"stage\": %d, \"copy\": %d, \"stages\": %d, \"row_stride\": %zu, \"GBps\": %.1f, \"err\": \"%s\"}\n", c.stage, c.copy, c.nst,
           c.row_stride, (double)total * iters / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
  }
  return 0;
}
