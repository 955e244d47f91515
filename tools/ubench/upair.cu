// CTA-pair tcgen05 check and rates (sm_100a):
//  1. correctness of cta_group::2 (M = 256): each CTA TMA-loads its 128 rows of A and its half
//     (N/2 rows) of B, the peer's loads complete on the leader's mbarrier (.cta_group::2), the
//     leader issues the MMAs, the commit is multicast to both CTAs; D rows 128r + lane in CTA r.
//  2. MMA rate, M = 128 (cta_group::1) vs M = 256 (pair), N = 160, operands in smem, with and
//     without a concurrent TMA stream into other shared memory (the generator's ring refills).
//  3. one thread streaming global -> shared: 2D tensor boxes vs 1D bulk copies, pipelined / bursts.
//  4. the generator's per-stage load pattern (weight + activation boxes, 2-stage ring) with a
//     consumer that holds each stage or issues the stage's 16 MMAs.
//  5. latency of a single 16 KB box with the tensor core idle / busy.
// Results and what they ruled out: DESIGN.md §6.2 (round-2 generator investigation).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1805_11462_b200/csrc upair.cu -lcuda -o upair
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "common.cuh"
#include "ptx.cuh"
using namespace onmt;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ void tmem_alloc2(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t t) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)), "h"(mask)
               : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const void* tmap, int x, int y, uint32_t bar_cl) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                   smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(bar_cl)
               : "memory");
}

// ---- 1. correctness: D[256][N] = A[256][64] . B[N][64]^T
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_check(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int N, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full, done;
  __shared__ uint32_t tslot;
  const uint32_t r = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(&full, 1); mbar_init(&done, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc2(&tslot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  uint8_t* sA = smem;                 // 128 x 128 B
  uint8_t* sB = smem + 16384;         // N/2 x 128 B
  const uint32_t bar0 = mapa_peer(smem_u32(&full), 0);
  if (threadIdx.x == 0) {
    if (r == 0) mbar_arrive_expect_tx(&full, 2 * (16384 + (N / 2) * 128));
    tma2(sA, &tmA, 0, 128 * r, bar0);
    tma2(sB, &tmB, 0, (N / 2) * r, bar0);
  }
  if (r == 0 && threadIdx.x == 0) {
    mbar_wait(&full, 0);
    tc_fence_after();
    const uint32_t idesc = umma_idesc_bf16(256, N);
    for (int kk = 0; kk < 4; ++kk)
      mma2(tmem, umma_desc_sw128(smem_u32(sA) + kk * 32), umma_desc_sw128(smem_u32(sB) + kk * 32), idesc, kk ? 1u : 0u);
    commit2_mc(&done, 3);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < N; c += 32) {
    uint32_t v[32];
    tmem_ld32_nw(tmem + c + ((uint32_t)(32 * w) << 16), v);
    tmem_wait_ld();
    for (int k = 0; k < 32; ++k) out[(size_t)(128 * r + 32 * w + lane) * N + c + k] = __uint_as_float(v[k]);
  }
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x < 32) tmem_dealloc2(tmem);
}

// ---- 2. rates.  pair = 0: every CTA issues M = 128 MMAs; pair = 1: leaders issue M = 256.
// tma = 1: warp 1 keeps a TMA stream of 20 KB tiles running into a separate 80 KB region.
template <int PAIR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_rate(const __grid_constant__ CUtensorMap tmS, int N, int iters, int tma, int span, unsigned long long* out, int depth = 4) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t done, tb[8];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const uint32_t r = cluster_ctarank();
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&done, 1); for (int i = 0; i < 8; ++i) mbar_init(&tb[i], 1); stop = 0; fence_mbar_init(); }
  if (threadIdx.x < 32) {
    if (PAIR) tmem_alloc2(&tslot); else tmem_alloc<512>(&tslot);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0 && (!PAIR || r == 0)) {
    const uint32_t idesc = umma_idesc_bf16(PAIR ? 256 : 128, N);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (PAIR) mma2(tmem, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sb + kk * 32), idesc, 1u);
        else tc_mma_bf16(tmem, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sb + kk * 32), idesc, 1u);
      }
    }
    if (PAIR) commit2_mc(&done, 3); else tc_commit(&done);
    mbar_wait(&done, 0);
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  }
  if (PAIR && r == 1 && threadIdx.x == 0) mbar_wait(&done, 0);
  if (PAIR && r == 1 && threadIdx.x == 0) stop = 1;
  if (threadIdx.x == 32 && tma) {       // TMA stream: 4 slots of 20 KB after the operands
    uint8_t* dst = smem + 49152;
    int it = 0;
    while (!stop) {
      const int s = it % depth;
      if (it >= depth) mbar_wait(&tb[s], ((it / depth) - 1) & 1);   // the slot's previous load landed
      mbar_arrive_expect_tx(&tb[s], 20480);
      tma_load_2d(dst + s * 20480, &tmS, 0, (int)(((long long)it * 160 + (span > 8192 ? (long long)blockIdx.x * 2621 : 0)) % (span - 160)), &tb[s]);
      ++it;
    }
    // drain: the last (up to) four loads
    for (int j = it - depth < 0 ? 0 : it - depth; j < it; ++j) mbar_wait(&tb[j % depth], (j / depth) & 1);
    if (r == 0 || !PAIR) out[1024 + blockIdx.x] = it;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32) {
    if (PAIR) tmem_dealloc2(tmem); else tmem_dealloc(tmem, 512);
  }
}


// ---- 3. one thread streaming global -> shared: 2D tensor boxes {64, rows} vs 1D bulk copies
__global__ void __launch_bounds__(32, 1)
k_tma(const __grid_constant__ CUtensorMap tm160, const __grid_constant__ CUtensorMap tm256, const uint8_t* src,
      long long span_bytes, int mode, int depth, int bytes, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t tb[8];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 8; ++i) mbar_init(&tb[i], 1);
  fence_mbar_init();
  const int rows = bytes / 128;
  const long long nrows = span_bytes / 128;
  unsigned long long t0, t1;
  long long c0 = clock64();
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  if (mode >= 2) {                          // bursts: depth loads issued back to back, then all waited
    for (int it = 0; it < iters; it += depth) {
      for (int s = 0; s < depth; ++s) {
        mbar_arrive_expect_tx(&tb[s], bytes);
        const long long row = ((long long)(it + s) * rows + (long long)blockIdx.x * 2621) % (nrows - rows);
        if (mode == 2) tma_load_2d(smem + s * bytes, rows == 160 ? (const void*)&tm160 : (const void*)&tm256, 0, (int)row, &tb[s]);
        else bulk_g2s(smem + s * bytes, src + row * 128, bytes, &tb[s]);
      }
      for (int s = 0; s < depth; ++s) mbar_wait(&tb[s], (it / depth) & 1);
    }
    iters = 0;
  }
  for (int it = 0; it < iters; ++it) {
    const int s = it % depth;
    if (it >= depth) mbar_wait(&tb[s], ((it / depth) - 1) & 1);
    mbar_arrive_expect_tx(&tb[s], bytes);
    const long long row = ((long long)it * rows + (long long)blockIdx.x * 2621) % (nrows - rows);
    if (mode == 0) tma_load_2d(smem + s * bytes, rows == 160 ? (const void*)&tm160 : (const void*)&tm256, 0, (int)row, &tb[s]);
    else bulk_g2s(smem + s * bytes, src + row * 128, bytes, &tb[s]);
  }
  for (int j = iters - depth < 0 ? 0 : iters - depth; j < iters; ++j) mbar_wait(&tb[j % depth], (j / depth) & 1);
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  long long c1 = clock64();
  out[blockIdx.x] = t1 - t0;
  out[1024 + blockIdx.x] = c1 - c0;
}

// ---- 4. the generator's load pattern without MMAs: per stage nw weight boxes {64, 128} (distinct
// rows per CTA over a wspan-row region) + na activation boxes {64, 160} (rows shared by every
// CTA), a ring of `stages`; the consumer holds each stage for hold_ns (the MMA time) then frees it.
__global__ void __launch_bounds__(512, 1)
k_pat(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx, long long wspan, int nw, int na,
      int stages, int hold_ns, int iters, unsigned long long* out, int mma = 0, int real = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[8], empty[8];
  const int stage_bytes = nw * 16384 + na * 20480;
  __shared__ uint32_t tslot;
  if (threadIdx.x >= 64) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  if (threadIdx.x >= 32) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  unsigned long long t0, t1, lat = 0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) {                       // producer
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (it >= stages) mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      uint8_t* st = smem + s * stage_bytes;
      for (int j = 0; j < nw; ++j) {
        if (real) {                             // the generator's W: [50048][512], tile rows x K block
          const int tile = (blockIdx.x * 3 + (it / 8) * nw + j) % 391;
          tma_load_2d(st + j * 16384, &tw, (it % 8) * 64, tile * 128, &full[s]);
        } else {
          const long long row = (((long long)blockIdx.x * 64 + (long long)it * nw + j) * 128) % (wspan - 128);
          tma_load_2d(st + j * 16384, &tw, 0, (int)row, &full[s]);
        }
      }
      for (int j = 0; j < na; ++j) tma_load_2d(st + nw * 16384 + j * 20480, &tx, (it % 8) * 64, j * 160, &full[s]);
    }
  } else if (threadIdx.x == 32) {               // consumer
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      unsigned long long a_, b_;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(a_));
      mbar_wait(&full[s], (it / stages) & 1);
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(b_));
      lat += b_ - a_;                          // time the consumer waited for data
      if (mma) {                               // 2 tiles x 4 kk x (hi, lo): 16 MMAs M = 128, N = 160
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(128, 160);
        const uint32_t sb = smem_u32(smem + s * stage_bytes);
        for (int j = 0; j < 2; ++j)
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = umma_desc_sw128(sb + j * 16384 + kk * 32);
            tc_mma_bf16(tslot + j * 160, da, umma_desc_sw128(sb + nw * 16384 + kk * 32), idesc, 1u);
            tc_mma_bf16(tslot + j * 160, da, umma_desc_sw128(sb + nw * 16384 + 20480 + kk * 32), idesc, 1u);
          }
        tc_commit(&empty[s]);
      } else {
        unsigned long long c_ = b_;
        while (c_ - b_ < (unsigned long long)hold_ns) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(c_));
        mbar_arrive_local(&empty[s]);
      }
    }
    if (mma) { mbar_wait(&empty[(iters - 1) % stages], ((iters - 1) / stages) & 1); }
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
    out[1024 + blockIdx.x] = lat;
  }
  __syncthreads();
  if (threadIdx.x >= 32) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

// ---- 5. latency of single TMA boxes (depth 1) while the tensor core is idle / busy (M = 128,
// N = 160 MMAs back to back from another thread on operands in the same shared memory)
__global__ void __launch_bounds__(64, 1)
k_lat(const __grid_constant__ CUtensorMap tw, long long wspan, int mma_on, int n, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); stop = 0; fence_mbar_init(); }
  if (threadIdx.x >= 32) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int i = 0; i < n; ++i) {
      unsigned long long a_, b_;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(a_));
      mbar_arrive_expect_tx(&bar, 16384);
      const long long row = (((long long)blockIdx.x * 977 + i) * 128) % (wspan - 128);
      tma_load_2d(smem + 65536, &tw, 0, (int)row, &bar);
      mbar_wait(&bar, i & 1);
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(b_));
      tot += b_ - a_;
    }
    out[blockIdx.x] = tot / n;
    stop = 1;
  } else if (threadIdx.x == 32 && mma_on) {
    const uint32_t idesc = umma_idesc_bf16(128, 160);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    while (!stop) {
      for (int kk = 0; kk < 64; ++kk)
        tc_mma_bf16(tslot, umma_desc_sw128(sa + (kk & 3) * 32), umma_desc_sw128(sb + (kk & 3) * 32), idesc, 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x >= 32) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// ---- 6. per-box cost: one thread pipelining 2D boxes {64, rows} (rows = 32 .. 256) and 3D
// boxes {64, rows, 2} (two planes), depth 4, distinct rows per CTA over a 48 MB region
__global__ void __launch_bounds__(32, 1)
k_box(const __grid_constant__ CUtensorMap tm, int is3d, int box_bytes, long long nrows, int rows, int iters,
      unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t tb[4];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 4; ++i) mbar_init(&tb[i], 1);
  fence_mbar_init();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int it = 0; it < iters; ++it) {
    const int s = it & 3;
    if (it >= 4) mbar_wait(&tb[s], ((it >> 2) - 1) & 1);
    mbar_arrive_expect_tx(&tb[s], box_bytes);
    const long long row = ((long long)it * rows + (long long)blockIdx.x * 2621) % (nrows - rows);
    if (is3d) tma_load_3d(smem + s * box_bytes, &tm, 0, (int)row, 0, &tb[s]);
    else tma_load_2d(smem + s * box_bytes, &tm, 0, (int)row, &tb[s]);
  }
  for (int j = iters - 4; j < iters; ++j) mbar_wait(&tb[j & 3], (j >> 2) & 1);
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap make_tmap(const void* base, int k, int rows, int box_rows) {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) { void* p = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q)); fn = (PFN_encodeTiled_t)p; }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)k * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("tmap\n"); exit(1); }
  return m;
}

static CUtensorMap make_tmap3p(const void* base, long long rows, int box_rows) {   // {64, rows, 2 planes}
  typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  CUtensorMap m;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {128, (cuuint64_t)rows * 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 2};
  cuuint32_t es[3] = {1, 1, 1};
  if (((F)p)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("tmap3\n"); exit(1); }
  return m;
}
int main() {
  if (getenv("UPAIR_BOX")) {                           // section 6 only
    const long long NR = 48ll * 1024 * 1024 / 128;
    __nv_bfloat16* S; CK(cudaMalloc(&S, (size_t)NR * 128)); CK(cudaMemset(S, 0, (size_t)NR * 128));
    unsigned long long* o; CK(cudaMalloc(&o, 2048 * 8));
    CK(cudaFuncSetAttribute(k_box, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int is3d : {0, 1})
      for (int rows : {32, 64, 128, 160, 256}) {
        if (is3d && rows > 160) continue;
        CUtensorMap tm = is3d ? make_tmap3p(S, NR / 2, rows) : make_tmap(S, 64, (int)NR, rows);
        const int bytes = rows * 128 * (is3d ? 2 : 1), grid = 148, iters = 2000;
        k_box<<<grid, 32, 200 * 1024>>>(tm, is3d, bytes, is3d ? NR / 2 : NR, rows, 100, o); CK(cudaDeviceSynchronize());
        k_box<<<grid, 32, 200 * 1024>>>(tm, is3d, bytes, is3d ? NR / 2 : NR, rows, iters, o); CK(cudaDeviceSynchronize());
        std::vector<unsigned long long> h(grid);
        CK(cudaMemcpy(h.data(), o, grid * 8, cudaMemcpyDeviceToHost));
        double ns = 0; for (int b = 0; b < grid; ++b) ns += h[b]; ns /= grid;
        printf("%s box %3d rows (%6d B): %.0f ns per box, %.1f GB/s per SM\n", is3d ? "3D x2 planes" : "2D         ", rows,
               bytes, ns / iters, (double)bytes * iters / ns);
      }
    return 0;
  }
  // ---- 1. correctness
  for (int N : {32, 160, 256}) {
    std::vector<__nv_bfloat16> hA(256 * 64), hB((size_t)N * 64);
    std::vector<float> fA(256 * 64), fB((size_t)N * 64);
    for (int i = 0; i < 256 * 64; ++i) { fA[i] = (float)((i * 7 + 3) % 17 - 8) / 8.f; hA[i] = __float2bfloat16(fA[i]); }
    for (int i = 0; i < N * 64; ++i) { fB[i] = (float)((i * 5 + 1) % 13 - 6) / 4.f; hB[i] = __float2bfloat16(fB[i]); }
    __nv_bfloat16 *dA, *dB; float* dO;
    CK(cudaMalloc(&dA, hA.size() * 2)); CK(cudaMalloc(&dB, hB.size() * 2)); CK(cudaMalloc(&dO, 256 * N * 4));
    CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(dO, 0, 256 * N * 4));
    CUtensorMap tA = make_tmap(dA, 64, 256, 128), tB = make_tmap(dB, 64, N, N / 2);
    CK(cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    k_check<<<2, 128, 64 * 1024>>>(tA, tB, N, dO);
    CK(cudaDeviceSynchronize());
    std::vector<float> o(256 * N);
    CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < 64; ++k) s += (double)fA[m * 64 + k] * fB[n * 64 + k];
        err = fmax(err, fabs(s - o[m * N + n]));
      }
    printf("pair check N=%d: max |D - A.B^T| = %.3g %s\n", N, err, err < 1e-3 ? "OK" : "WRONG");
  }
  // ---- 2. rates
  const int SPAN = 48 * 1024 * 1024 / 128;               // 48 MB of 128-byte rows
  __nv_bfloat16* S; CK(cudaMalloc(&S, (size_t)SPAN * 64 * 2)); CK(cudaMemset(S, 0, (size_t)SPAN * 64 * 2));
  CUtensorMap tS = make_tmap(S, 64, SPAN, 160);
  unsigned long long* o; CK(cudaMalloc(&o, 2048 * 8));
  CK(cudaFuncSetAttribute(k_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024));
  CK(cudaFuncSetAttribute(k_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024));
  for (int pair : {0, 1})
    for (int tma : {0, 1, 2}) {
      const int span = tma == 2 ? SPAN : 8192;             // 2: distinct rows per CTA over 48 MB
      const int N = 160, iters = 2000, grid = 148;
      auto run = [&](int it) {
        if (pair) k_rate<1><<<grid, 128, 140 * 1024>>>(tS, N, it, tma, span, o); else k_rate<0><<<grid, 128, 140 * 1024>>>(tS, N, it, tma, span, o);
        CK(cudaDeviceSynchronize());
      };
      run(10);
      run(iters);
      std::vector<unsigned long long> h(2048);
      CK(cudaMemcpy(h.data(), o, 2048 * 8, cudaMemcpyDeviceToHost));
      double ns = 0, tiles = 0; int n = 0;
      for (int b = 0; b < grid; ++b) if (!pair || b % 2 == 0) { ns += h[b]; tiles += tma ? h[1024 + b] : 0; ++n; }
      ns /= n; tiles /= n;
      const double per = ns / (4.0 * iters);             // ns per MMA instruction
      const double flop = 2.0 * (pair ? 256 : 128) * N * 16;
      printf("%s N=%d tma=%d: %.2f ns per MMA -> %.0f TFLOP/s chip; TMA stream %.1f GB/s per CTA\n",
             pair ? "pair M=256" : "single M=128", N, tma, per, flop / per / 1e3 * (pair ? 74 : 148),
             tiles * 20480 / ns);
    }
  // TMA stream alone (the MMA thread idles ~200 us): L2 -> SM capacity, hot 1 MB vs 48 MB distinct
  CK(cudaFuncSetAttribute(k_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (int depth : {2, 4, 8})
  for (int grid : {148, 74, 16})
  for (int span : {SPAN}) {
    k_rate<0><<<grid, 128, 220 * 1024>>>(tS, 8, 20000, 1, span, o, depth); CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(2048);
    CK(cudaMemcpy(h.data(), o, 2048 * 8, cudaMemcpyDeviceToHost));
    double ns = 0, tiles = 0;
    for (int b = 0; b < grid; ++b) { ns += h[b]; tiles += h[1024 + b]; }
    printf("TMA only, %s, depth %d x 20 KB, grid %d: %.1f GB/s per CTA, %.2f TB/s chip\n", span > 8192 ? "48 MB distinct" : "1 MB shared",
           depth, grid, tiles * 20480 / ns, tiles * 20480 / ns * grid / 1e3);
  }
  {
    CUtensorMap t160 = make_tmap(S, 64, SPAN, 160), t256 = make_tmap(S, 64, SPAN, 256);
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int mode : {0, 2, 3})
      for (int bytes : {160 * 128, 256 * 128})
        for (int depth : {1, 2, 4, 8}) {
          if (bytes * depth > 190 * 1024) continue;
          const int grid = 148, iters = 4000;
          k_tma<<<grid, 32, 200 * 1024>>>(t160, t256, (const uint8_t*)S, (long long)SPAN * 128, mode, depth, bytes, 100, o);
          CK(cudaDeviceSynchronize());
          k_tma<<<grid, 32, 200 * 1024>>>(t160, t256, (const uint8_t*)S, (long long)SPAN * 128, mode, depth, bytes, iters, o);
          CK(cudaDeviceSynchronize());
          std::vector<unsigned long long> h(2048);
          CK(cudaMemcpy(h.data(), o, 2048 * 8, cudaMemcpyDeviceToHost));
          double ns = 0, cyc = 0;
          for (int b = 0; b < grid; ++b) { ns += h[b]; cyc += h[1024 + b]; }
          ns /= grid; cyc /= grid;
          printf("%s %5d B x depth %d: %.1f GB/s per SM (%.1f B/cycle, clock %.0f MHz), %.2f TB/s chip\n",
                 mode == 0 ? "2D tensor" : mode == 2 ? "2D burst " : "1D burst ", bytes, depth, (double)bytes * iters / ns, (double)bytes * iters / cyc,
                 cyc / ns * 1e3, (double)bytes * iters / ns * grid / 1e3);
        }
  }
  {
    const long long WROWS = 56ll * 1024 * 1024 / 128;          // 56 MB of weights (rows of 128 B)
    __nv_bfloat16 *Wb, *Xb;
    CK(cudaMalloc(&Wb, (size_t)WROWS * 128)); CK(cudaMemset(Wb, 0, (size_t)WROWS * 128));
    CK(cudaMalloc(&Xb, (size_t)320 * 512 * 2)); CK(cudaMemset(Xb, 0, (size_t)320 * 512 * 2));
    CUtensorMap tw = make_tmap(Wb, 64, (int)WROWS, 128), tx = make_tmap(Xb, 512, 320, 160);
    CK(cudaFuncSetAttribute(k_pat, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    struct Cfg { long long wspan; int nw, na, stages, hold; const char* nm; int mma; int real; };
    std::vector<__nv_bfloat16> hw((size_t)50048 * 512);
    { unsigned long long st_ = 88172645463325252ull;
      for (size_t i = 0; i < hw.size(); ++i) { st_ ^= st_ << 13; st_ ^= st_ >> 7; st_ ^= st_ << 17;
        hw[i] = __float2bfloat16((float)((st_ >> 11) * (1.0 / 9007199254740992.0) * 0.2 - 0.1)); } }
    __nv_bfloat16* Wr; CK(cudaMalloc(&Wr, hw.size() * 2)); CK(cudaMemcpy(Wr, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice));
    CUtensorMap twr = make_tmap(Wr, 512, 50048, 128);
    CK(cudaFuncSetAttribute(k_pat, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
    for (int big : {0, 1}) {
      const int grid = 148, iters = 200, thr = big ? 512 : 64, sm = big ? 226 * 1024 : 200 * 1024;
      k_pat<<<grid, thr, sm>>>(twr, tx, WROWS, 2, 2, 2, 0, iters, o, 1, 1); CK(cudaDeviceSynchronize());
      k_pat<<<grid, thr, sm>>>(twr, tx, WROWS, 2, 2, 2, 0, iters, o, 1, 1); CK(cudaDeviceSynchronize());
      std::vector<unsigned long long> h(2048);
      CK(cudaMemcpy(h.data(), o, 2048 * 8, cudaMemcpyDeviceToHost));
      double ns = 0, wt = 0;
      for (int b = 0; b < grid; ++b) { ns += h[b]; wt += h[1024 + b]; }
      printf("pattern REAL, %d threads, %d KB smem: %.0f ns per stage (consumer waited %.0f ns)\n", thr, sm / 1024,
             ns / grid / iters, wt / grid / iters);
    }
    const Cfg cfgs[] = {
      {WROWS, 2, 2, 2, 0, "REAL W + act, MMAs, 2 stages", 1, 1},
      {WROWS, 2, 0, 2, 0, "REAL W only, MMAs, 2 stages", 1, 1},
      {WROWS, 2, 2, 2, 700, "REAL W + act, hold 700", 0, 1},
      {WROWS, 2, 2, 2, 0, "gen non-pair with MMAs, 2 stages", 1},
      {8192, 2, 2, 2, 0, "  same, W 1 MB", 1},
      {WROWS, 2, 0, 2, 0, "  W only (B = garbage), MMAs", 1},
      {WROWS, 2, 2, 2, 700, "gen non-pair: 2 W + 2 act, 2 stages, hold 700"},
      {WROWS, 2, 2, 2, 0, "  same, hold 0"},
      {WROWS, 2, 0, 2, 700, "W only (56 MB)"},
      {8192, 2, 0, 2, 700, "W only (1 MB)"},
      {WROWS, 0, 2, 2, 700, "act only"},
      {WROWS, 2, 2, 3, 700, "2 W + 2 act, 3 stages"},
      {WROWS, 4, 0, 2, 700, "4 W (56 MB), 2 stages"},
      {WROWS, 1, 0, 2, 700, "1 W, 2 stages"},
      {WROWS, 1, 0, 4, 700, "1 W, 4 stages"},
    };
    CK(cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    for (int grid : {1, 148})
      for (int mma_on : {0, 1}) {
        k_lat<<<grid, 64, 100 * 1024>>>(tw, WROWS, mma_on, 200, o); CK(cudaDeviceSynchronize());
        std::vector<unsigned long long> h(256);
        CK(cudaMemcpy(h.data(), o, 256 * 8, cudaMemcpyDeviceToHost));
        double a = 0; for (int b = 0; b < grid; ++b) a += h[b];
        printf("16 KB box latency, grid %3d, tensor %s: %.0f ns\n", grid, mma_on ? "busy" : "idle", a / grid);
      }
    for (const Cfg& c : cfgs) {
      if (c.stages * (c.nw * 16384 + c.na * 20480) > 199 * 1024) continue;
      const int grid = 148, iters = 200;
      k_pat<<<grid, 64, 200 * 1024>>>(c.real ? twr : tw, tx, c.wspan, c.nw, c.na, c.stages, c.hold, iters, o, c.mma, c.real);
      CK(cudaDeviceSynchronize());
      k_pat<<<grid, 64, 200 * 1024>>>(c.real ? twr : tw, tx, c.wspan, c.nw, c.na, c.stages, c.hold, iters, o, c.mma, c.real);
      CK(cudaDeviceSynchronize());
      std::vector<unsigned long long> h(2048);
      CK(cudaMemcpy(h.data(), o, 2048 * 8, cudaMemcpyDeviceToHost));
      double ns = 0, wt = 0;
      for (int b = 0; b < grid; ++b) { ns += h[b]; wt += h[1024 + b]; }
      ns /= grid; wt /= grid;
      const double bytes = (double)(c.nw * 16384 + c.na * 20480) * iters;
      printf("pattern %-44s: %.0f ns per stage (consumer waited %.0f ns), %.1f GB/s per SM, %.2f TB/s chip\n", c.nm,
             ns / iters, wt / iters, bytes / ns, bytes / ns * grid / 1e3);
    }
  }
  return 0;
}
