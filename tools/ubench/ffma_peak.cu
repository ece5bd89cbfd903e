// FP32 pipe microbenchmark (dev tool): 3-register FFMA, FFMA with an
// immediate, and packed fma.rn.f32x2, each as 8 independent chains per
// thread; prints TFLOP/s (FMA = 2 flops) over a full-GPU grid.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_ffma_reg(float* out, float b, float c0) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  float bb = b + threadIdx.x * 1e-9f, cc = c0;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], bb, cc);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_ffma_imm(float* out, float b, float c0) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  float bb = b + threadIdx.x * 1e-9f;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], bb, 0.5f);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1.2345f) out[0] = s;
}

__device__ __forceinline__ unsigned long long f2pack(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}

__global__ void k_ffma2(float* out, float b, float c0) {
  unsigned long long a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = f2pack(threadIdx.x * 1e-3f + j, j * 0.5f);
  const unsigned long long bb = f2pack(b + threadIdx.x * 1e-9f, b);
  const unsigned long long cc = f2pack(c0, c0);
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(bb), "l"(cc));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[j]));
    s += x + y;
  }
  if (s == 1.2345f) out[0] = s;
}

template <typename K>
void run(const char* name, K k, int flops_per_fma_per_iter) {
  float* out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 grid(sms * 8), block(256);
  k<<<grid, block>>>(out, 0.999f, 0.001f);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) k<<<grid, block>>>(out, 0.999f, 0.001f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 10.0 * grid.x * block.x * (double)ITERS * 8 * flops_per_fma_per_iter;
  printf("%-10s %8.2f TFLOP/s (%s)\n", name, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run("ffma_reg", k_ffma_reg, 2);
  run("ffma_imm", k_ffma_imm, 2);
  run("ffma2", k_ffma2, 4);
  return 0;
}
