// The generator's MMA-thread pattern (gen_step.cu): per stage, NT weight tiles x 4 K steps x (hi, lo)
// MMAs of 128 x N x 16 (N = 160 hypothesis rows), descriptors from the stage index, tiles gated by a
// runtime coverage mask.  One CTA per SM on 148 SMs; stage operands resident (no loads).
//   hoisted      descriptors loop-invariant (pipe rate)
//   gated        rolled stage loop, `if (!(cov >> j & 1)) continue;` between the tiles (as gen_step)
//   ungated      rolled, the NT tiles straight-line (NT a template parameter)
//   unroll2      ungated, stage loop unrolled x2
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1805_11462_b200/csrc umloop2.cu -lcuda -o umloop2
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#include "ptx.cuh"
using namespace onmt;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
enum { HOISTED = 0, GATED = 1, UNGATED = 2, UNROLL2 = 3 };
constexpr int kStages = 2, kReps = 64;

template <int NT>
__global__ void __launch_bounds__(512, 1) k_gen(int N, int mode, unsigned cov, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += 512) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tmem = tslot;
  const uint32_t b_bytes = N * 128, a_bytes = 16384, stage_bytes = 2 * b_bytes + NT * a_bytes;
  if (threadIdx.x == 32) {
    const uint32_t idesc = umma_idesc_bf16(128, N);
    unsigned long long t0, t1;
    auto stage = [&](int it, bool gated) {
      const uint32_t sb = smem_u32(smem) + (uint32_t)(it % kStages) * stage_bytes;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        if (gated && !((cov >> j) & 1u)) continue;
        const uint32_t sa = sb + 2 * b_bytes + j * a_bytes;
        const uint32_t d = tmem + (uint32_t)(j * 160);
        const uint32_t acc0 = it == 0 ? 0u : 1u;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t da = umma_desc_sw128(sa + kk * 32);
          tc_mma_bf16(d, da, umma_desc_sw128(sb + kk * 32), idesc, kk == 0 ? acc0 : 1u);
          tc_mma_bf16(d, da, umma_desc_sw128(sb + b_bytes + kk * 32), idesc, 1u);
        }
      }
    };
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (mode == HOISTED) {
      const uint32_t sb = smem_u32(smem), sa = sb + 2 * b_bytes;
      for (int it = 0; it < kReps * NT; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t da = umma_desc_sw128(sa + kk * 32);
          tc_mma_bf16(tmem, da, umma_desc_sw128(sb + kk * 32), idesc, 1u);
          tc_mma_bf16(tmem, da, umma_desc_sw128(sb + b_bytes + kk * 32), idesc, 1u);
        }
      }
    } else if (mode == GATED) {
#pragma unroll 1
      for (int it = 0; it < kReps; ++it) stage(it, true);
    } else if (mode == UNGATED) {
#pragma unroll 1
      for (int it = 0; it < kReps; ++it) stage(it, false);
    } else {
#pragma unroll 2
      for (int it = 0; it < kReps; ++it) stage(it, false);
    }
    tc_commit(&done);
    mbar_wait(&done, 0);
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* o; CK(cudaMalloc(&o, 64));
  CK(cudaFuncSetAttribute(k_gen<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  CK(cudaFuncSetAttribute(k_gen<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  const char* names[] = {"hoisted", "gated", "ungated", "unroll2"};
  for (int N : {160, 32})
  for (int nt = 1; nt <= 2; ++nt)
    for (int mode = 0; mode < 4; ++mode) {
      for (int w = 0; w < 2; ++w) {
        if (nt == 1) k_gen<1><<<148, 512, 210 * 1024>>>(N, mode, 3u, o);
        else k_gen<2><<<148, 512, 210 * 1024>>>(N, mode, 3u, o);
        CK(cudaDeviceSynchronize());
      }
      unsigned long long h; CK(cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost));
      printf("N=%3d tiles/stage %d  %-8s %7.1f ns per stage (%d MMAs)\n", N, nt, names[mode], h / (double)kReps, 8 * nt);
    }
  return 0;
}
