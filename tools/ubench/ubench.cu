// Microbenchmarks for the decode-step design (run on the GPU box):
//   1. launch cost of an empty PDL kernel inside a CUDA graph
//   2. a minimal split-K tcgen05 tile (barrier init, TMEM alloc, TMA ring, MMA, TMEM load)
//      with %globaltimer phase stamps per CTA
//   3. cost of a software grid barrier inside one persistent kernel
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1805_11462_b200/csrc ubench.cu -lcuda -o ubench
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

using namespace onmt;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_empty(int* p) {
  pdl_trigger();
  pdl_wait();
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0]++;
}

struct TArgs {
  int nkb, n_group, stages, n_rows_pad;
  unsigned long long* ts;   // [grid][8]
  float* out;
};

__global__ void __launch_bounds__(128, 1) k_tc(const __grid_constant__ CUtensorMap tmW,
                                               const __grid_constant__ CUtensorMap tmX, TArgs a) {
  unsigned long long t0 = gt();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t a_bytes = 128 * 128, b_bytes = a.n_group * 128;
  const uint32_t stage_bytes = a_bytes + 2 * b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
  uint64_t* empty = full + a.stages;
  uint64_t* done = empty + a.stages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = (blockIdx.x % 16) * 128;
  const int kb0 = (blockIdx.x / 16) * a.nkb;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  unsigned long long t1 = gt();
  pdl_wait();
  unsigned long long t2 = gt(), t3 = 0, t4 = 0;
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < a.nkb; ++i) {
      const int s = i % a.stages;
      if (i >= a.stages) mbar_wait(&empty[s], ((i / a.stages) & 1) ^ 1);
      uint8_t* st = smem + s * stage_bytes;
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      const int kx = (kb0 + i) * 64;
      tma_load_2d(st, &tmW, kx, m0, &full[s]);
      tma_load_2d(st + a_bytes, &tmX, kx, 0, &full[s]);
      tma_load_2d(st + a_bytes + b_bytes, &tmX, kx, a.n_rows_pad, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, a.n_group);
    for (int i = 0; i < a.nkb; ++i) {
      const int s = i % a.stages;
      mbar_wait(&full[s], (i / a.stages) & 1);
      if (i == 0) t3 = gt();
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint32_t sbh = sa + a_bytes, sbl = sa + a_bytes + b_bytes;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = umma_desc_sw128(sa + kk * 32);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, (i | kk) != 0);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
      }
      tc_commit(&empty[s]);
    }
    tc_commit(done);
    t4 = gt();
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  unsigned long long t5 = gt();
  const int q = warp & 3;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  float accv = 0.f;
  for (int c0 = 0; c0 < a.n_group; c0 += 16) {
    float v[16];
    tmem_ld16(trow + c0, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) accv += v[j];
  }
  a.out[blockIdx.x * 128 + threadIdx.x] = accv;
  unsigned long long t6 = gt();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
  unsigned long long t7 = gt();
  if (threadIdx.x == 0) {
    unsigned long long* T = a.ts + blockIdx.x * 8;
    T[0] = t0; T[1] = t1; T[2] = t2; T[5] = t5; T[6] = t6; T[7] = t7;
  }
  if (threadIdx.x == 32) { a.ts[blockIdx.x * 8 + 3] = t3; a.ts[blockIdx.x * 8 + 4] = t4; }
}

// software grid barrier: generation counter
__global__ void k_gridbar(unsigned int* bar, int iters, unsigned long long* ts) {
  unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int target = (unsigned int)(i + 1) * gridDim.x;
      __threadfence();
      atomicAdd(bar, 1u);
      while (true) {
        unsigned int v;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(bar));
        if (v >= target) break;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) { ts[0] = t0; ts[1] = gt(); }
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap make_tmap(const void* base, int k_pad, int rows, int box_rows) {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    fn = (PFN_encodeTiled_t)p;
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)k_pad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)k_pad * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tmap fail\n"); exit(1); }
  return m;
}

template <typename F>
static float time_graph(cudaStream_t st, int reps, F launch_one) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < reps; ++i) launch_one();
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaEventRecord(a, st));
  CK(cudaGraphLaunch(ge, st));
  CK(cudaEventRecord(b, st));
  CK(cudaStreamSynchronize(st));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return ms * 1000.f / reps;
}

int main() {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int* dcount;
  CK(cudaMalloc(&dcount, 4));
  auto pdl_launch = [&](auto kern, dim3 grid, dim3 block, size_t smem, auto... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, args...));
  };
  for (int grid : {1, 148, 296}) {
    float us = time_graph(st, 200, [&]() { pdl_launch(k_empty, dim3(grid), dim3(128), 0, dcount); });
    float us2 = time_graph(st, 200, [&]() { k_empty<<<grid, 128, 0, st>>>(dcount); });
    printf("empty kernel grid=%d: %.2f us/launch (PDL graph), %.2f us (plain graph)\n", grid, us, us2);
  }
  // tcgen05 tile
  const int N = 160, KP = 1536, M = 2048;
  __nv_bfloat16 *W, *X;
  CK(cudaMalloc(&W, (size_t)M * KP * 2));
  CK(cudaMalloc(&X, (size_t)2 * N * KP * 2));
  CK(cudaMemset(W, 0, (size_t)M * KP * 2));
  CK(cudaMemset(X, 0, (size_t)2 * N * KP * 2));
  CUtensorMap tmW = make_tmap(W, KP, M, 128), tmX = make_tmap(X, KP, 2 * N, N);
  float* out;
  CK(cudaMalloc(&out, 1 << 20));
  unsigned long long* ts;
  CK(cudaMalloc(&ts, 4096 * 8 * 8));
  for (int splits : {8, 4, 2}) {
    TArgs a{};
    a.nkb = 24 / splits;
    a.n_group = N;
    a.stages = std::min(a.nkb, 3);
    a.n_rows_pad = N;
    a.ts = ts;
    a.out = out;
    const int grid = 16 * splits;
    size_t smem = 1024 + a.stages * (128 * 128 + 2 * N * 128) + 256;
    CK(cudaFuncSetAttribute(k_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    float us = time_graph(st, 100, [&]() { pdl_launch(k_tc, dim3(grid), dim3(128), smem, tmW, tmX, a); });
    CK(cudaMemset(ts, 0, 4096 * 64));
    pdl_launch(k_tc, dim3(grid), dim3(128), smem, tmW, tmX, a);
    CK(cudaStreamSynchronize(st));
    std::vector<unsigned long long> h(grid * 8);
    CK(cudaMemcpy(h.data(), ts, grid * 64, cudaMemcpyDeviceToHost));
    unsigned long long tmin = ~0ull, tmax = 0;
    double avg[8] = {0};
    for (int b = 0; b < grid; ++b) {
      tmin = std::min(tmin, h[b * 8]);
      tmax = std::max(tmax, h[b * 8 + 7]);
      for (int i = 1; i < 8; ++i) avg[i] += (double)(h[b * 8 + i] - h[b * 8]) / grid;
    }
    double skew = 0;
    for (int b = 0; b < grid; ++b) skew = std::max(skew, (double)(h[b * 8] - tmin));
    printf("tc tile splits=%d grid=%d kb/cta=%d: %.2f us/launch in graph; span %.2f us; entry skew %.2f us\n", splits,
           grid, a.nkb, us, (tmax - tmin) / 1e3, skew / 1e3);
    printf("   avg from entry (us): init+alloc %.2f | pdl_wait %.2f | first data %.2f | mma issued %.2f | mma done %.2f | tmem ld %.2f | exit %.2f\n",
           avg[1] / 1e3, avg[2] / 1e3, avg[3] / 1e3, avg[4] / 1e3, avg[5] / 1e3, avg[6] / 1e3, avg[7] / 1e3);
  }
  // grid barrier
  unsigned int* bar;
  CK(cudaMalloc(&bar, 4));
  for (int grid : {148, 296}) {
    CK(cudaMemset(bar, 0, 4));
    const int iters = 1000;
    k_gridbar<<<grid, 128, 0, st>>>(bar, iters, ts);
    CK(cudaStreamSynchronize(st));
    unsigned long long h[2];
    CK(cudaMemcpy(h, ts, 16, cudaMemcpyDeviceToHost));
    printf("grid barrier grid=%d: %.3f us per barrier\n", grid, (h[1] - h[0]) / 1e3 / iters);
  }
  return 0;
}
