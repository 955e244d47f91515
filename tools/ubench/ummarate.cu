// tcgen05.mma issue/throughput rate (M = 128, kind::f16, operands in smem, no loads)
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#include "ptx.cuh"
using namespace onmt;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__global__ void __launch_bounds__(128, 1) k_mma(int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tmem = tslot;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_bf16(tmem, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sb + kk * 32), idesc, 1u);
    }
    tc_commit(&done);
    mbar_wait(&done, 0);
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}
int main() {
  unsigned long long* o; CK(cudaMalloc(&o, 64));
  CK(cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
  for (int grid : {1, 148}) for (int N : {32, 64, 128, 160, 192, 256}) {
    const int iters = 2000;
    k_mma<<<grid, 128, 80 * 1024>>>(N, 10, o); CK(cudaDeviceSynchronize());
    k_mma<<<grid, 128, 80 * 1024>>>(N, iters, o); CK(cudaDeviceSynchronize());
    unsigned long long h; CK(cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost));
    const double per = h / (4.0 * iters);
    const double flop = 2.0 * 128 * N * 16;
    printf("grid %3d  N=%3d: %.2f ns per MMA (128x%dx16) -> %.1f TFLOP/s per SM, x148 = %.0f TFLOP/s\n", grid, N, per, N,
           flop / per / 1e3, flop / per / 1e3 * 148);
  }
  return 0;
}
