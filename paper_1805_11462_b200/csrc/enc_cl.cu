// A3: the encoder recurrence of one layer, every direction as ONE thread-block cluster whose
// CTAs keep the recurrent state on chip (PAPER.md P129-133; SPEC S257-265):
//
//   for t = 0 .. S_max-1:  z_t = Z_t + b + W_hh h_{t-1};  (i,f,g,o) = (σ,σ,tanh,σ)(z_t)
//                          c_t = f c_{t-1} + i g;  h_t = o tanh(c_t)
//
// per sentence over its own S_b tokens (packed semantics, R3: frozen for t >= S_b; the
// backward direction runs pos = S_b-1-t), Z = W_ih x hoisted over all t by one GEMM before.
//
// Grid = D clusters of T CTAs (T = 4 Hd / 128 <= 16): CTA `tile` of direction d owns 128
// interleaved gate rows (32 units) over the whole K = Hd, its W_hh tile resident in shared
// memory.  h_{t-1} lives in shared memory too: every CTA holds the full recurrent operand in
// 32-column K blocks (bf16 hi / lo planes, UMMA K-major 64-byte swizzle, two parity buffers), and
// the 32 units of CTA `tile` are exactly K block `tile`.  Each step a CTA writes its units' h_t
// into a local 2 x N x 64-byte staging block and pushes it with T bulk copies (shared::cta ->
// shared::cluster) into every CTA's operand buffer, completing on that CTA's per-parity
// mbarrier: the next step's MMAs wait on their own barrier for all T blocks - no cluster-wide
// barrier and no global-memory round trip on the step's critical path:
//   MMAs (M = 128 gate rows, N = 2 x sentences: both planes) -> TMEM -> cell -> staging ->
//   bulk copies -> the peers' barriers.
// WAR safety without a barrier: a CTA's step-t copies overwrite the buffer its peers' step t-1
// MMAs read, but it only gets there after receiving every peer's h_{t-1}, which each peer
// produced after its step t-1 MMAs had completed.
#include <math_constants.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

struct EncClDir {
  const float* Z;          // hoisted input projection [B*S_max rows][z_ld] (interleaved gate columns)
  int z_ld;
  const float4* bias;      // [Hd] pre-summed (i, f, g, o)
  float* h_st;             // final state (the last valid step's h / c), row stride st_ld
  float* c_st;
  int st_ld;
  XOut xnext;              // next layer's input operand (or the keys/values GEMM operand)
  int next_col;
  float* mem;              // memory bank (top layer) or nullptr
  int mem_ld, mem_col;
  int backward;
};

struct EncClArgs {
  EncClDir dir[2];
  int T, Hd, B, N, S_max, kb;   // kb: K blocks of Hd (64 each)
  const int* lens;
  unsigned long long* trace;   // (debug) per-step %globaltimer stamps of CTA 0, or nullptr
};
__device__ __forceinline__ unsigned long long ec_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float ec_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float ec_tanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

// shared memory: W tile [kb][16 KB] | h operand [2 parity][2 kb][hi, lo][N x 64 B] | h staging
// [2 parity][hi, lo][N x 64 B] | gate staging [N][128] f32 | Z [2 parity][N][128] f32 | c, h
// [N][32] f32 | bias [32] float4 | lens [N] | barriers
static size_t ec_smem_bytes(int kb, int N) {
  return 1024 + (size_t)kb * 16384 + (size_t)2 * (2 * kb) * 2 * N * 64 + (size_t)2 * 2 * N * 64 +
         (size_t)3 * N * 128 * 4 + (size_t)2 * N * 32 * 4 + 32 * 16 + (size_t)((N + 3) & ~3) * 4 + 6 * 8 + 16;
}

// byte offset of (row r, K column c < 32) inside one 32-column K block's [N x 64 B] bf16 plane,
// 64-byte swizzle (address bits 4-5 ^= bits 7-8: the 16-byte chunk index XOR (r / 2) mod 4)
__device__ __forceinline__ uint32_t ec_sw64(int r, int c) {
  return (uint32_t)(r * 64 + ((((c >> 3) ^ (r >> 1)) & 3) << 4) + ((c & 7) << 1));
}

constexpr int kEcThreads = 512;   // one (unit, sentence) cell per thread at N = 16: the cell's latency
                                   // chain (loads, transcendentals, shuffles, stores) runs once per step
__global__ void __launch_bounds__(kEcThreads, 1)
enc_cl_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1, EncClArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int T = a.T, N = a.N, kb = a.kb;
  const int tile = (int)cluster_ctarank();
  const int d = blockIdx.x / T;
  const EncClDir& dg = a.dir[d];
  const CUtensorMap* tmW = d ? &tmW1 : &tmW0;
  const uint32_t nb = (uint32_t)N * 64;                           // one plane of one 32-column K block
  const int kb32 = 2 * kb;                                        // 32-column K blocks (>= T)
  uint8_t* sW = smem;                                             // [kb][128 x 64] bf16 (SW128)
  uint8_t* sX = sW + (size_t)kb * 16384;                          // [2][kb32][hi, lo][N x 32] (SW64)
  const size_t xpar = (size_t)kb32 * 2 * nb;                      // bytes of one parity buffer
  uint8_t* sH = sX + 2 * xpar;                                    // [2][hi, lo][N x 32]: my h_t block
  float* stg = reinterpret_cast<float*>(sH + 2 * 2 * nb);         // [N][128] W_hh h_{t-1} of my rows
  float* Zs = stg + (size_t)N * 128;                              // [2][N][128] Z_t of my rows (t & 1)
  float* cst = Zs + (size_t)2 * N * 128;                          // [N][32]
  float* hst = cst + (size_t)N * 32;                              // [N][32]
  float4* s_bias = reinterpret_cast<float4*>(hst + (size_t)N * 32);
  int* s_len = reinterpret_cast<int*>(s_bias + 32);
  uint64_t* wbar = reinterpret_cast<uint64_t*>(s_len + ((N + 3) & ~3));
  uint64_t* mdone = wbar + 1;
  uint64_t* hbar = wbar + 2;                                      // [2] operand buffer b complete
  uint32_t* tslot = reinterpret_cast<uint32_t*>(hbar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t tcols = 32;
  while ((int)tcols < 2 * N) tcols <<= 1;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(tmW);
    mbar_init(wbar, 1);
    mbar_init(mdone, 1);
    mbar_init(&hbar[0], 1);
    mbar_init(&hbar[1], 1);
    fence_mbar_init();
    // h_0 (buffer 1, step 1) and h_1 (buffer 0, step 2): T blocks each (re-armed after each wait)
    if (a.S_max > 1) mbar_arrive_expect_tx(&hbar[1], (uint32_t)T * 2 * nb);
    if (a.S_max > 2) mbar_arrive_expect_tx(&hbar[0], (uint32_t)T * 2 * nb);
    mbar_arrive_expect_tx(wbar, (uint32_t)kb * 16384);            // my W_hh tile, resident for all t
    for (int i = 0; i < kb; ++i) tma_load_2d(sW + (size_t)i * 16384, tmW, i * kBK, tile * kTileM, wbar);
  }
  if (warp == 1) tmem_alloc_dyn(tslot, tcols);
  if (threadIdx.x < 32) {
    const int j = tile * 32 + threadIdx.x;
    s_bias[threadIdx.x] = j < a.Hd ? dg.bias[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int j = threadIdx.x; j < N; j += blockDim.x) s_len[j] = j < a.B ? a.lens[j] : 0;
  for (int i = threadIdx.x; i < 32 * N; i += blockDim.x) { cst[i] = 0.f; hst[i] = 0.f; }
  // K blocks past the last tile's (W_hh K padding) are never pushed: clear all once
  for (int i = threadIdx.x; i < (int)(2 * xpar / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(sX)[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");    // (read by the tensor core)
  const bool backward_ = dg.backward != 0;
  const float* const Zg = dg.Z;
  const int z_ld = dg.z_ld;
  auto prefetch_z = [&](int t) {                                 // Z_t of my gate rows, live sentences
    if (threadIdx.x < 128) return;                                // (warps 4-7: idle while the MMAs run)
    for (int i = threadIdx.x - 128; i < N * 32; i += blockDim.x - 128) {
      const int j = i >> 5, ch = i & 31;
      const int L = s_len[j];
      if (j >= a.B || t >= L) continue;
      const int pos = backward_ ? L - 1 - t : t;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Zs + ((size_t)(t & 1) * N + j) * 128 + 4 * ch)),
                   "l"(Zg + ((size_t)j * a.S_max + pos) * z_ld + (size_t)tile * 128 + 4 * ch)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  __syncthreads();                                                // (s_len before the prefetch)
  prefetch_z(0);
  tc_fence_before();
  cluster_sync_all();                                             // every CTA's buffers exist and are clear
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const XOut xnext = dg.xnext;
  float* const h_st = dg.h_st;
  float* const c_st = dg.c_st;
  float* const mem = dg.mem;
  const int st_ld = dg.st_ld, next_col = dg.next_col, mem_ld = dg.mem_ld, mem_col = dg.mem_col;
  const bool has_next = xnext.f32 || xnext.hl;

  const bool tr = a.trace && blockIdx.x == 0;
  for (int t = 0; t < a.S_max; ++t) {
    const int par = t & 1;                                        // buffer par holds h_{t-1} (t > 0)
    if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 0] = ec_now();
    // Z_{t+1} streams in during this step (its buffer's last reader, step t-1's cell, is done:
    // the cluster barrier ended step t-1)
    if (t + 1 < a.S_max) prefetch_z(t + 1);
    if (t > 0) {
      if (warp == 1 && lane == 0) {
        if (t == 1) mbar_wait(wbar, 0);
        // one MMA per 16-wide K step over both planes: a K block's hi and lo planes are adjacent
        // [N rows][N rows], one B operand of 2N rows -> D columns [0, N) = W h_hi, [N, 2N) = W h_lo
        // (summed by the stagers); half the MMA instructions of two N-row MMAs, which at N = 16
        // are issue-bound.  (Waiting per source block instead, to start on the first arrivals,
        // measured slower: 2.75 vs 1.4 us for wait + MMAs.)
        mbar_wait(&hbar[par], (uint32_t)(((t - 1) >> 1) & 1));   // every CTA's block of h_{t-1} (use (t-1)/2)
        if (t + 2 < a.S_max) mbar_arrive_expect_tx(&hbar[par], (uint32_t)T * 2 * nb);   // (step t + 2)
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(kTileM, 2 * N);
        const uint32_t xb = smem_u32(sX + (size_t)par * xpar), sw0 = smem_u32(sW);
        // straight-line issue (the K-block count as a template argument): computing descriptors
        // in a rolled loop makes each small MMA wait for the previous one
        auto issue = [&](auto kbc) {
          constexpr int KB = decltype(kbc)::value;
#pragma unroll
          for (int ks = 0; ks < 4 * KB; ++ks)
            tc_mma_bf16(tmem, umma_desc_sw128(sw0 + (uint32_t)(ks >> 2) * 16384u + (uint32_t)(ks & 3) * 32u),
                        umma_desc_sw64(xb + (uint32_t)(ks >> 1) * 2u * nb + (uint32_t)(ks & 1) * 32u), idesc, ks != 0);
        };
        switch (kb) {
          case 1: issue(std::integral_constant<int, 1>{}); break;
          case 2: issue(std::integral_constant<int, 2>{}); break;
          case 3: issue(std::integral_constant<int, 3>{}); break;
          case 4: issue(std::integral_constant<int, 4>{}); break;
          case 5: issue(std::integral_constant<int, 5>{}); break;
          case 6: issue(std::integral_constant<int, 6>{}); break;
          case 7: issue(std::integral_constant<int, 7>{}); break;
          case 8: issue(std::integral_constant<int, 8>{}); break;
          default:
            for (int ks = 0; ks < 4 * kb; ++ks)
              tc_mma_bf16(tmem, umma_desc_sw128(sw0 + (uint32_t)(ks >> 2) * 16384u + (uint32_t)(ks & 3) * 32u),
                          umma_desc_sw64(xb + (uint32_t)(ks >> 1) * 2u * nb + (uint32_t)(ks & 1) * 32u), idesc,
                          ks != 0);
        }
        tc_commit(mdone);
        if (tr && t < 64) a.trace[t * 8 + 1] = ec_now();
      }
      __syncwarp();
      if (warp < 4) {                                             // TMEM -> stg[sentence][gate row]
        mbar_wait(mdone, (t - 1) & 1);
        if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 2] = ec_now();
        tc_fence_after();
        const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
        const int row = warp * 32 + lane;
        for (int cc = 0; cc < N; cc += 8) {
          uint32_t r[8], q[8];
          tmem_ld8_nw(trow + cc, r);                              // W h_hi of sentences cc .. cc+7
          tmem_ld8_nw(trow + N + cc, q);                          // W h_lo
          tmem_wait_ld();
          tmem_fence_regs(r);
          tmem_fence_regs(q);
#pragma unroll
          for (int k = 0; k < 8; ++k) stg[(size_t)(cc + k) * 128 + row] = __uint_as_float(r[k]) + __uint_as_float(q[k]);
        }
        tc_fence_before();
      }
    }
    if (t + 1 < a.S_max) asm volatile("cp.async.wait_group 1;" ::: "memory");   // Z_t landed (my chunks;
    else asm volatile("cp.async.wait_group 0;" ::: "memory");                 //  Z_{t+1} may be in flight)
    __syncthreads();
    if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 3] = ec_now();
    // ---- the cell for (unit u = lane, sentence j); h_t (bf16 hi / lo) -> my staging block
    const float* Zt = Zs + (size_t)(t & 1) * N * 128;
    const bool send = t + 1 < a.S_max;
    uint8_t* hb = sH + (size_t)(t & 1) * 2 * nb;
    for (int i = threadIdx.x; i < 32 * N; i += blockDim.x) {
      const int u = i & 31, j = i >> 5;
      const int jj = tile * 32 + u;
      float h = hst[j * 32 + u];                                  // (finished / padding: h stays, R3)
      const int L = s_len[j];
      if (j < a.B && jj < a.Hd && t < L) {
        float4 g = *reinterpret_cast<const float4*>(Zt + (size_t)j * 128 + 4 * u);
        const float4 bb = s_bias[u];
        g.x += bb.x; g.y += bb.y; g.z += bb.z; g.w += bb.w;
        if (t > 0) {
          const float4 pv = *reinterpret_cast<const float4*>(stg + (size_t)j * 128 + 4 * u);
          g.x += pv.x; g.y += pv.y; g.z += pv.z; g.w += pv.w;
        }
        const float ig = ec_sigm(g.x), fg = ec_sigm(g.y), gg = ec_tanh(g.z), og = ec_sigm(g.w);
        const float c = fg * cst[j * 32 + u] + ig * gg;
        h = og * ec_tanh(c);
        cst[j * 32 + u] = c;
        hst[j * 32 + u] = h;
      }
      if (send) {                                                 // (the step's critical path first)
        const __nv_bfloat16 hh = __float2bfloat16_rn(h);
        const __nv_bfloat16 hl = __float2bfloat16_rn(h - __bfloat162float(hh));
        const uint32_t o = ec_sw64(j, u);
        *reinterpret_cast<__nv_bfloat16*>(hb + o) = hh;
        *reinterpret_cast<__nv_bfloat16*>(hb + nb + o) = hl;
      }
      if (j < a.B && jj < a.Hd && t < L) {
        const int pos = backward_ ? L - 1 - t : t;
        const size_t row = (size_t)j * a.S_max + pos;
        if (t == L - 1) {                                         // final state (R5: decoder init)
          h_st[(size_t)j * st_ld + jj] = h;
          c_st[(size_t)j * st_ld + jj] = cst[j * 32 + u];
        }
        if (has_next) store_x(xnext, (int)row, next_col + jj, h);
        if (mem) mem[row * mem_ld + mem_col + jj] = h;
      }
    }
    if (send) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // staging stores -> bulk-copy reads
      __syncthreads();
      if (warp == 1 && lane < T) {
        // push my block into K block `tile` of every CTA's buffer par ^ 1 (mine included): lane
        // p of warp 1 copies to CTA p
        const uint32_t dst0 = smem_u32(sX + (size_t)(par ^ 1) * xpar + (size_t)tile * 2 * nb);
        const uint32_t bar0 = smem_u32(&hbar[par ^ 1]);
        bulk_s2peer(mapa_peer(dst0, (uint32_t)lane), hb, 2 * nb, mapa_peer(bar0, (uint32_t)lane));
        bulk_commit();
        bulk_wait_read<1>();                                      // (step t-1's block may be rewritten)
      }
      if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 5] = ec_now();
    }
  }
  if (warp == 1 && lane < T) bulk_wait_read<0>();
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (threadIdx.x == 0 && a.S_max <= 1) mbar_wait(wbar, 0);       // (no MMA waited for the W load)
  tc_fence_before();
  __syncthreads();
  cluster_arrive();                                               // (no peer still writes my smem)
  cluster_wait();
  if (warp == 1) tmem_dealloc(tmem, tcols);
}

// the cluster recurrence applies when a direction's gate rows form at most 16 tiles, the
// sentences fit one MMA over both planes (2N <= 256, N a multiple of 16) and the shared memory fits; T > 8 needs a
// non-portable cluster size
int enc_cl_fits(int T, int kb, int N, int D, int num_sms) {
  if (T < 1 || T > 16 || N < 16 || N > 128 || (N % 16) != 0 || D * T > num_sms) return 0;   // (MMA N = 2N <= 256)
  if (ec_smem_bytes(kb, N) > 227 * 1024) return 0;
  if (cudaFuncSetAttribute(enc_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ec_smem_bytes(kb, N)) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (T > 8 && cudaFuncSetAttribute(enc_cl_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(D * T);
  cfg.blockDim = dim3(kEcThreads);
  cfg.dynamicSmemBytes = ec_smem_bytes(kb, N);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = T;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, enc_cl_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return ncl >= 1 ? 1 : 0;                                        // (directions are independent clusters)
}

cudaError_t launch_enc_cl(const CUtensorMap* tmW, const EncClArgs& a, int D, cudaStream_t st) {
  const size_t smem = ec_smem_bytes(a.kb, a.N);
  cudaError_t e = cudaFuncSetAttribute(enc_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.T > 8) {
    e = cudaFuncSetAttribute(enc_cl_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(D * a.T);
  cfg.blockDim = dim3(kEcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.T;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, enc_cl_kernel, tmW[0], tmW[D > 1 ? 1 : 0], a);
}

}  // namespace onmt
