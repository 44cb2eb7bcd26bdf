// Probe: legacy mma.sync.m16n8k16 bf16 throughput on sm_100a (independent accumulator
// chains per warp, no memory traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void probe(int iters, float* out) {
  float c[CH][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int ch : {1, 4, 8}) {
      auto run = [&]() {
        if (ch == 1) probe<1><<<148, warps * 32>>>(iters, out);
        if (ch == 4) probe<4><<<148, warps * 32>>>(iters, out);
        if (ch == 8) probe<8><<<148, warps * 32>>>(iters, out);
      };
      run();
      cudaEventRecord(a);
      run();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double flops = 148.0 * warps * ch * (double)iters * 16 * 8 * 16 * 2;
      printf("{\"warps_per_sm\": %d, \"chains\": %d, \"TFLOPs\": %.1f, \"cycles_per_mma_per_sm\": %.2f}\n", warps, ch,
             flops / (ms * 1e-3) / 1e12, (ms * 1e-3 * 1.965e9) / (warps * ch * (double)iters));
    }
  }
  return 0;
}
