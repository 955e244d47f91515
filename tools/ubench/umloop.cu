// tcgen05.mma issue rate of a K loop whose smem descriptors change per K block (the fused cell
// kernel's MMA thread: 8 K blocks x 4 K steps of 128 x N x 16, N = 32), one CTA per SM on 80 SMs.
//   hoisted    descriptors loop-invariant (as tools/ubench/ummarate): the tensor-pipe rate
//   rolled     descriptors computed from the K block index in a rolled loop
//   unroll2    the same loop unrolled x2
//   unrolled   fully unrolled (8 K blocks)
//   unrolled+wait  fully unrolled with a (complete) mbarrier wait per K block
// (stacked is a template parameter: a runtime branch between the MMAs has the same effect.)
// Rolled, the next block's descriptors are written into the uniform registers the previous
// block's MMAs read, and the issue waits for those MMAs: ~250-330 ns per K block whether the
// block has 4 or 8 MMAs, against ~100 ns pipe time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1805_11462_b200/csrc umloop.cu -lcuda -o umloop
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#include "ptx.cuh"
using namespace onmt;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

enum { HOISTED = 0, ROLLED = 1, UNROLL2 = 2, UNROLLED = 3, UNROLLED_WAIT = 4 };
constexpr int kNkb = 8, kReps = 100;

template <bool stacked>
__global__ void __launch_bounds__(256, 1) k_loop(int N, int nkb, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kNkb], done;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += 256) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNkb; ++i) mbar_init(&full[i], 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) for (int i = 0; i < kNkb; ++i) mbar_arrive_local(&full[i]);
  __syncthreads();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    const uint32_t sA = smem_u32(smem), sB = sA + kNkb * 16384;   // A: [kb][128][64], B: [kb][hi, lo][N][64]
    const uint32_t idesc = umma_idesc_bf16(128, stacked ? 2 * N : N);
    unsigned long long t0, t1;
    auto blk = [&](int i, uint32_t acc0) {
      const uint32_t sa = sA + i * 16384, sbh = sB + i * 2 * N * 128, sbl = sbh + N * 128;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = umma_desc_sw128(sa + kk * 32);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, kk ? 1u : acc0);
        if (!stacked) tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
      }
    };
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (mode == HOISTED) {
      const uint32_t idesc1 = umma_idesc_bf16(128, N);
      for (int i = 0; i < kReps * nkb; ++i) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc_mma_bf16(tmem, umma_desc_sw128(sA + kk * 32), umma_desc_sw128(sB + kk * 32), idesc1, 1u);
      }
    } else {
      for (int rep = 0; rep < kReps; ++rep) {
        if (mode == ROLLED) {
#pragma unroll 1
          for (int i = 0; i < nkb; ++i) blk(i, (rep | i) != 0);
        } else if (mode == UNROLL2) {
#pragma unroll 2
          for (int i = 0; i < nkb; ++i) blk(i, (rep | i) != 0);
        } else if (mode == UNROLLED) {
#pragma unroll
          for (int i = 0; i < kNkb; ++i) blk(i, (rep | i) != 0);
        } else {
#pragma unroll
          for (int i = 0; i < kNkb; ++i) {
            mbar_wait(&full[i], 0);
            tc_fence_after();
            blk(i, (rep | i) != 0);
          }
        }
      }
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
  CK(cudaFuncSetAttribute(k_loop<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  CK(cudaFuncSetAttribute(k_loop<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  const char* names[] = {"hoisted (4 MMAs)", "rolled", "unroll2", "unrolled", "unrolled+wait"};
  const int N = 32;
  for (int mode = 0; mode < 5; ++mode)
    for (int st = 0; st < (mode ? 2 : 1); ++st) {
      for (int w = 0; w < 2; ++w) {
        if (st) k_loop<true><<<80, 256, 210 * 1024>>>(N, kNkb, mode, o);
        else k_loop<false><<<80, 256, 210 * 1024>>>(N, kNkb, mode, o);
        CK(cudaDeviceSynchronize());
      }
      unsigned long long h; CK(cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost));
      printf("%-18s %-22s %.1f ns per K block\n", names[mode], mode ? (st ? "4 MMAs (N = 64 stacked)" : "8 MMAs (N = 32)") : "",
             h / (double)(kReps * kNkb));
    }
  return 0;
}
