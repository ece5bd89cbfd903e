// Probe of the tcgen05 kind::tf32 operand views used by bed_backward_tc.cuh:
// X (64 x 64) stored as rows in the K-major no-swizzle core-matrix layout,
// read either K-major (D = X Y^T) or through MN-major descriptors (D = X^T Y),
// with the LBO/SBO roles as given.  Prints the max error of each variant
// against the CPU product.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -I paper_2207_04228_b200/csrc tools/ubench/umma_probe.cu -o /tmp/umma_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "bed_tc.cuh"

using namespace bed;

__global__ void probe(const float* X, const float* Y, float* D, int mn, uint32_t lbo, uint32_t sbo, uint32_t step) {
  __shared__ __align__(1024) uint8_t sm[2 * 16384 + 64];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 32768 + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 4096; e += blockDim.x) {
    const int row = e / 64, k = e % 64;
    *reinterpret_cast<float*>(sm + kmaj_off(row, k)) = tf32_hi(X[e]);
    *reinterpret_cast<float*>(sm + 16384 + kmaj_off(row, k)) = tf32_hi(Y[e]);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  proxy_fence_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 16384);
    const uint32_t idesc = mn ? kIdescTf32MN : kIdescTf32;
    for (int kk = 0; kk < 8; ++kk)
      umma_tf32(tmem, umma_desc(a + step * kk, lbo, sbo), umma_desc(b + step * kk, lbo, sbo), idesc, kk > 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  float d[16];
  for (int q = 0; q < 4; ++q) {
    tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16 * q, d);
    tmem_wait_ld();
    if (lane < 16)
      for (int j = 0; j < 16; ++j) D[(16 * warp + lane) * 64 + 16 * q + j] = d[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

int main() {
  float *X, *Y, *D;
  cudaMallocManaged(&X, 4096 * 4); cudaMallocManaged(&Y, 4096 * 4); cudaMallocManaged(&D, 4096 * 4);
  srand(1);
  for (int i = 0; i < 4096; ++i) { X[i] = (rand() % 17 - 8) / 8.0f; Y[i] = (rand() % 13 - 6) / 4.0f; }
  struct V { int mn; uint32_t lbo, sbo, step; };
  std::vector<V> vs = {{0, 128, 2048, 256}};
  const uint32_t opts[] = {64, 128, 256, 512, 1024, 2048};
  for (uint32_t l : opts)
    for (uint32_t s : opts) vs.push_back({1, l, s, 2048});
  for (auto& v : vs) {
    for (int i = 0; i < 4096; ++i) D[i] = NAN;
    probe<<<1, 128>>>(X, Y, D, v.mn, v.lbo, v.sbo, v.step);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mn %d lbo %u sbo %u: %s\n", v.mn, v.lbo, v.sbo, cudaGetErrorString(e)); return 1; }
    double worst = 0;
    int good = 0;
    for (int m = 0; m < 64; ++m)
      for (int n = 0; n < 64; ++n) {
        double ref = 0;
        for (int k = 0; k < 64; ++k) ref += v.mn ? (double)X[k * 64 + m] * Y[k * 64 + n] : (double)X[m * 64 + k] * Y[n * 64 + k];
        const double err = fabs(ref - D[m * 64 + n]);
        worst = fmax(worst, err);
        good += err < 1e-3;
      }
    printf("mn %d lbo %5u sbo %5u: max |err| %8.3g, %4d / 4096 right\n", v.mn, v.lbo, v.sbo, worst, good);
  }
  return 0;
}
