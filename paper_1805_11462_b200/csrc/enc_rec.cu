// A3: the encoder recurrence of one layer as ONE persistent kernel (
// PAPER.md P129-133; SPEC S257-265):
//
//   for t = 0 .. S_max-1:  z_t = Z_t + b + W_hh h_{t-1};  (i,f,g,o) = (σ,σ,tanh,σ)(z_t)
//                          c_t = f c_{t-1} + i g;  h_t = o tanh(c_t)
//
// per sentence over its own S_b tokens (packed semantics, R3: frozen for t >= S_b; the
// backward direction runs pos = S_b-1-t), Z = W_ih x hoisted over all t by one GEMM before.
//
// Grid = D x T x S CTAs: direction, 128-row tile of the interleaved gate rows (32 units),
// split of the K = Hd reduction; the S splits of a tile form one thread-block cluster.  All
// CTAs are co-resident (one per SM).  Each CTA keeps its W_hh tile's K-slice resident in
// shared memory for the whole sequence.  Per step it TMA-loads its K-slice of h_{t-1}
// (bf16 hi/lo planes, written in the previous step by the tiles owning those units), runs
// the tcgen05 MMAs (M = 128 gate rows, N = sentences; 1/S of the MMAs a whole-K tile would
// issue - small-N MMAs are issue-bound), then the cluster reduce-scatters the partial gate
// tiles through distributed shared memory: split s owns sentence columns
// [s*N/S, (s+1)*N/S), receives the other splits' partials of those columns, sums them in
// fixed split order (deterministic), applies the cell to its 32 units x N/S sentences (their
// c state stays on chip) and stores h_t into the other parity buffer.  A software barrier
// among the direction's T*S CTAs separates the steps (h_t of every unit is needed by every
// tile).  One launch per layer replaces 2 launches per step (split-K GEMM + cell kernel).
#include <math_constants.h>

#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

struct EncRecDir {
  const float* Z;          // hoisted input projection [B*S_max rows][z_ld] (interleaved gate columns)
  int z_ld;
  const float4* bias;      // [Hd] pre-summed (i, f, g, o)
  XOut xrec[2];            // recurrent operand, parity buffers (bf16 hi/lo [rows_pad][k_pad])
  float* h_st;             // final state (the last valid step's h / c), row stride st_ld
  float* c_st;
  int st_ld;
  XOut xnext;              // next layer's input operand (or the keys/values GEMM operand)
  int next_col;
  float* mem;              // memory bank (top layer) or nullptr
  int mem_ld, mem_col;
  int backward;
};

struct EncRecArgs {
  EncRecDir dir[2];
  int T, S, Hd, B, N, S_max, kb;   // kb: K blocks of the whole reduction (S divides it)
  const int* lens;
  unsigned int* bar;       // [2 x 32] step-barrier words (one per direction, self-resetting)
  unsigned long long* trace;   // (debug) per-step %globaltimer stamps of CTA 0, or nullptr
};
__device__ __forceinline__ unsigned long long er_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// sigmoid / tanh via the fast exponential (rel. error ~2^-21, as the decoder's fused cell)
__device__ __forceinline__ float er_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float er_tanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

static size_t er_smem_bytes(int kbs, int N, int S) {
  const int NS = N / S;
  return 1024 + (size_t)kbs * 16384 + (size_t)kbs * 2 * N * 128 + (size_t)S * 128 * NS * 4 + (size_t)NS * 128 * 4 +
         (size_t)2 * 32 * NS * 4 + 32 * 16 + (size_t)NS * 4 + (2 + kbs) * 8 + 32 + 16;
}

__global__ void __launch_bounds__(256, 1)
enc_rec_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
               const __grid_constant__ CUtensorMap tmX00, const __grid_constant__ CUtensorMap tmX01,
               const __grid_constant__ CUtensorMap tmX10, const __grid_constant__ CUtensorMap tmX11,
               EncRecArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = a.S;
  const int s = (int)cluster_ctarank();                          // K split = my sentence-column group
  const int ts = blockIdx.x / S;
  const int d = ts / a.T, tile = ts % a.T;
  __shared__ EncRecDir dr;                                        // my direction's arguments (uniform)
  if (threadIdx.x == 0) dr = a.dir[d];
  const CUtensorMap* tmW = d ? &tmW1 : &tmW0;
  const CUtensorMap* tmXa = d ? &tmX10 : &tmX00;                 // parity 0 (h_{t-1} for even t)
  const CUtensorMap* tmXb = d ? &tmX11 : &tmX01;
  const int N = a.N, kbs = a.kb / S, NS = N / S;
  const int kb0 = s * kbs;                                        // my first K block
  const uint32_t nb = (uint32_t)N * 128;                          // one operand plane, one K block
  uint8_t* sW = smem;                                             // [kbs][128 x 64] bf16 (SW128)
  uint8_t* sX = sW + (size_t)kbs * 16384;                         // [kbs][hi, lo][N x 64]
  float* recv = reinterpret_cast<float*>(sX + (size_t)kbs * 2 * nb);   // [S][NS][128] partials of my columns
  float* Zs = recv + (size_t)S * 128 * NS;                        // [NS][128] Z_t of my gate rows
  float* cst = Zs + (size_t)NS * 128;                             // [NS][32] c of my units, my sentences
  float* hst = cst + 32 * NS;                                     // [NS][32] h
  float4* s_bias = reinterpret_cast<float4*>(hst + 32 * NS);     // [32]
  int* s_len = reinterpret_cast<int*>(s_bias + 32);               // [NS]
  uint64_t* wbar = reinterpret_cast<uint64_t*>(s_len + ((NS + 3) & ~3));
  uint64_t* mdone = wbar + 1;
  uint64_t* xfull = wbar + 2;                                     // [kbs] per K block (TMA -> MMA pipelining)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xfull + kbs);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t tcols = 32;
  while ((int)tcols < N) tcols <<= 1;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(tmW);
    tma_prefetch_desc(tmXa);
    tma_prefetch_desc(tmXb);
    mbar_init(wbar, 1);
    for (int i = 0; i < kbs; ++i) mbar_init(&xfull[i], 1);
    mbar_init(mdone, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(wbar, (uint32_t)kbs * 16384);           // my W_hh K-slice, resident for all t
    for (int i = 0; i < kbs; ++i) tma_load_2d(sW + (size_t)i * 16384, tmW, (kb0 + i) * kBK, tile * kTileM, wbar);
  }
  if (warp == 1) tmem_alloc_dyn(tslot, tcols);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int j = tile * 32 + threadIdx.x;
    s_bias[threadIdx.x] = j < a.Hd ? dr.bias[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int j = threadIdx.x; j < NS; j += blockDim.x) s_len[j] = s * NS + j < a.B ? a.lens[s * NS + j] : 0;
  for (int i = threadIdx.x; i < 32 * NS; i += blockDim.x) { cst[i] = 0.f; hst[i] = 0.f; }
  __syncthreads();
  const bool backward_ = dr.backward != 0;
  const float* const Zg = dr.Z;
  const int z_ld = dr.z_ld;
  // Z_t of my gate rows for my live sentences (cp.async, 16 B chunks)
  auto prefetch_z = [&](int t) {
    for (int i = threadIdx.x; i < NS * 32; i += blockDim.x) {
      const int j = i >> 5, ch = i & 31;
      const int b = s * NS + j;
      const int L = s_len[j];
      if (b >= a.B || t >= L) continue;
      const int pos = backward_ ? L - 1 - t : t;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Zs + (size_t)j * 128 + 4 * ch)),
                   "l"(Zg + ((size_t)b * a.S_max + pos) * z_ld + (size_t)tile * 128 + 4 * ch)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch_z(0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // my direction's arguments in registers (the shared copy would be re-read after every
  // shared-memory store of the cell loop)
  const XOut xrec0 = dr.xrec[0], xrec1 = dr.xrec[1], xnext = dr.xnext;
  float* const h_st = dr.h_st;
  float* const c_st = dr.c_st;
  float* const mem = dr.mem;
  const int st_ld = dr.st_ld, next_col = dr.next_col, mem_ld = dr.mem_ld, mem_col = dr.mem_col;
  const bool has_next = xnext.f32 || xnext.hl;
  const bool tr = a.trace && blockIdx.x == 0;

  for (int t = 0; t < a.S_max; ++t) {
    if (t > 0) {
      // every CTA of my direction has stored h_{t-1} (and finished reading h_{t-2}'s buffer
      // and its receive buffers of step t-1)
      __syncthreads();
      if (threadIdx.x == 0) {
        if (tr && t < 64) a.trace[t * 8 + 0] = er_now();
        cta_group_barrier(a.bar + 32 * d, (unsigned)(a.T * S));
        if (tr && t < 64) a.trace[t * 8 + 1] = er_now();
        asm volatile("fence.proxy.async;" ::: "memory");          // generic stores -> TMA reads
        const CUtensorMap* tx = (t & 1) ? tmXb : tmXa;            // buffer t & 1 holds h_{t-1}
        for (int i = 0; i < kbs; ++i) {
          mbar_arrive_expect_tx(&xfull[i], 2 * nb);
          tma_load_2d(sX + (size_t)i * 2 * nb, tx, (kb0 + i) * kBK, 0, &xfull[i]);
          tma_load_2d(sX + (size_t)i * 2 * nb + nb, tx, (kb0 + i) * kBK, N, &xfull[i]);
        }
      }
      if (warp == 1 && lane == 0) {
        if (t == 1) mbar_wait(wbar, 0);
        const uint32_t idesc = umma_idesc_bf16(kTileM, N);
        for (int i = 0; i < kbs; ++i) {
          mbar_wait(&xfull[i], (t - 1) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(sW + (size_t)i * 16384);
          const uint32_t sbh = smem_u32(sX + (size_t)i * 2 * nb), sbl = sbh + nb;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t da = umma_desc_sw128(sa + kk * 32);
            tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, (i | kk) != 0);
            tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
          }
        }
        tc_commit(mdone);
      }
      __syncwarp();
      mbar_wait(mdone, (t - 1) & 1);
      if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 3] = er_now();
      tc_fence_after();
      // reduce-scatter: my partial of split p's sentence columns -> p's recv[s] (DSMEM).
      // Warp w: TMEM lane quarter w & 3, peers p = (w >> 2), (w >> 2) + 2, ...
      {
        const int q = warp & 3;
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        const int row = q * 32 + lane;
        for (int p = warp >> 2; p < S; p += 2) {
          for (int c0 = 0; c0 < NS; c0 += 8) {
            uint32_t r[8];
            tmem_ld8_nw(trow + p * NS + c0, r);
            tmem_wait_ld();
            tmem_fence_regs(r);
            // recv[s][column][row]: a warp's store covers 32 consecutive rows (128 B)
            float* dst = recv + ((size_t)s * NS + c0) * 128 + row;
            if (p == s) {
#pragma unroll
              for (int k = 0; k < 8; ++k) dst[(size_t)k * 128] = __uint_as_float(r[k]);
            } else {
              const uint32_t pa = mapa_peer(smem_u32(dst), (uint32_t)p);
#pragma unroll
              for (int k = 0; k < 8; ++k) st_cluster_b32(pa + (uint32_t)k * 512u, r[k]);
            }
          }
        }
      }
      tc_fence_before();
      cluster_arrive();                                           // (release: my DSMEM stores)
      cluster_wait();                                             // every split's partial landed
      if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 6] = er_now();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");          // Z_t landed (my chunks)
    __syncthreads();
    if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 4] = er_now();
    // ---- the cell for (unit u, my sentence j); consecutive threads take consecutive units
    const XOut xo = (t & 1) ? xrec0 : xrec1;                     // h_t for step t+1's MMA
    for (int i = threadIdx.x; i < 32 * NS; i += blockDim.x) {
      const int u = i & 31, j = i >> 5;
      const int b = s * NS + j, jj = tile * 32 + u;
      if (b >= a.B || jj >= a.Hd) continue;
      const int L = s_len[j];
      if (t >= L) {                                               // finished: carry h forward
        store_x(xo, b, jj, hst[j * 32 + u]);
        continue;
      }
      const int pos = backward_ ? L - 1 - t : t;
      const size_t row = (size_t)b * a.S_max + pos;
      float4 g = *reinterpret_cast<const float4*>(Zs + (size_t)j * 128 + 4 * u);
      const float4 bb = s_bias[u];
      g.x += bb.x; g.y += bb.y; g.z += bb.z; g.w += bb.w;
      if (t > 0) {
        for (int p = 0; p < S; ++p) {                             // fixed split order
          const float4 pv = *reinterpret_cast<const float4*>(recv + ((size_t)p * NS + j) * 128 + 4 * u);
          g.x += pv.x; g.y += pv.y; g.z += pv.z; g.w += pv.w;
        }
      }
      const float ig = er_sigm(g.x), fg = er_sigm(g.y), gg = er_tanh(g.z), og = er_sigm(g.w);
      const float c = fg * cst[j * 32 + u] + ig * gg;
      const float h = og * er_tanh(c);
      cst[j * 32 + u] = c;
      hst[j * 32 + u] = h;
      if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 2] = er_now() + (unsigned long long)(h == 1234.5f);
      store_x(xo, b, jj, h);
      if (t == L - 1) {                                           // final state (R5: decoder init)
        h_st[(size_t)b * st_ld + jj] = h;
        c_st[(size_t)b * st_ld + jj] = c;
      }
      if (has_next) store_x(xnext, (int)row, next_col + jj, h);
      if (mem) mem[row * mem_ld + mem_col + jj] = h;
    }
    if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 7] = er_now();
    __syncthreads();                                              // Zs / recv consumed
    if (tr && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 5] = er_now();
    if (t + 1 < a.S_max) prefetch_z(t + 1);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_arrive();                                               // (no peer still writes my smem)
  cluster_wait();
  if (warp == 1) tmem_dealloc(tmem, tcols);
}

// splits per tile for this layer (0 = the persistent kernel does not fit): the largest S in
// {4, 2, 1} dividing the K blocks with N/S a multiple of 8, the grid co-resident and the
// shared memory within 227 KB
// every CTA of the grid resident at once as clusters of S (the step barrier waits for all)
static bool er_coresident(int grid, int S, size_t smem) {
  if (cudaFuncSetAttribute(enc_rec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, enc_rec_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return ncl * S >= grid;
}

int enc_rec_splits(int kb, int N, int D, int T, int num_sms) {
  if (N < 16 || N > 256 || (N % 16) != 0) return 0;
  for (int S = 4; S >= 1; S >>= 1) {
    if (kb % S != 0 || (N / S) % 8 != 0 || D * T * S > num_sms) continue;
    if (er_smem_bytes(kb / S, N, S) > 227 * 1024) continue;
    if (!er_coresident(D * T * S, S, er_smem_bytes(kb / S, N, S))) continue;
    return S;
  }
  return 0;
}

cudaError_t launch_enc_rec(const CUtensorMap* tmW, const CUtensorMap* tmX0, const CUtensorMap* tmX1,
                           const EncRecArgs& a, int D, cudaStream_t st) {
  const size_t smem = er_smem_bytes(a.kb / a.S, a.N, a.S);
  cudaError_t e = cudaFuncSetAttribute(enc_rec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int d1 = D > 1 ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(D * a.T * a.S);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, enc_rec_kernel, tmW[0], tmW[d1], tmX0[0], tmX1[0], tmX0[d1], tmX1[d1], a);
}

}  // namespace onmt
