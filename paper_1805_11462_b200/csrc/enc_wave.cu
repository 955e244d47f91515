// A3 for a unidirectional stacked encoder as ONE persistent kernel that runs the layers as a
// wavefront (PAPER.md P129-133 "stacked"; SPEC S257-265): layer l computes
// step t while layer l-1 computes step t+1, so the encoder takes S_max + L - 1 serial steps
// instead of L * S_max.
//
// Layer 0 is enc_rec.cu's recurrence (hoisted input projection Z + W_hh h).  A layer l >= 1
// cannot hoist its input projection (its input arrives step by step), so its gates are one
// reduction over [h_{l-1,t} ; h_{l,t-1}] with the weights [W_ih | W_hh] (both K parts padded
// to 64-column blocks): the input K blocks are read from layer l-1's recurrent-operand
// buffer that holds h_{l-1,t}, the recurrent ones from its own.  Each layer is a set of
// T x S CTAs (32-unit gate tiles x K splits, the S splits of a tile one cluster: DSMEM
// reduce-scatter as enc_rec.cu).  Instead of a barrier, each layer counts its finished CTAs
// per step (64-bit monotonic counters, zeroed before the launch); a CTA of layer l starts
// step t when
//   (a) layer l finished step t-1 (its own recurrence),
//   (b) layer l-1 finished step t (the input), and
//   (c) layer l+1 finished step t-2 (it no longer reads h_{l,t-2}, whose buffer step t
//       overwrites - two parity buffers per layer).
#include <math_constants.h>

#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

constexpr int kWaveMaxL = 4;

struct EncWaveLayer {
  int T, S, kb, kb_in;      // tiles, splits, K blocks (input part first), K blocks of the input part
  int cta0;                 // first grid index of this layer's CTAs
  const float* Z;           // layer 0: hoisted W_ih x [rows][z_ld]; nullptr for l >= 1
  int z_ld;
  const float4* bias;       // [Hd] pre-summed (i, f, g, o)
  XOut xrec[2];             // own recurrent-operand buffers (parity)
  float* h_st;              // final state rows (st_ld)
  float* c_st;
  int st_ld;
  XOut xnext;               // top layer: the keys / values GEMM operand (or none)
  float* mem;               // top layer: the memory bank (or nullptr)
  int mem_ld;
};

struct EncWaveArgs {
  EncWaveLayer layer[kWaveMaxL];
  int L, Hd, B, N, S_max;
  const int* lens;
  unsigned long long* cnt;  // [kWaveMaxL][16] per-layer finished-CTA counters (zeroed before launch)
};

__device__ __forceinline__ float ew_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float ew_tanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}
__device__ __forceinline__ void ew_wait_count(const unsigned long long* c, unsigned long long target) {
  const unsigned long long t0 = spin_clock();
  unsigned int it = 0;
  while (true) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(c) : "memory");
    if (v >= target) break;
    spin_check(t0, it);
  }
}

static size_t ew_smem_bytes(int kbs, int N, int S) {
  const int NS = N / S;
  return 1024 + (size_t)kbs * 16384 + (size_t)kbs * 2 * N * 128 + (size_t)S * 128 * NS * 4 + (size_t)NS * 128 * 4 +
         (size_t)2 * 32 * NS * 4 + 32 * 16 + (size_t)NS * 4 + (2 + kbs) * 8 + 32 + 16;
}

__global__ void __launch_bounds__(256, 1)
enc_wave_kernel(const __grid_constant__ CUtensorMap tw0, const __grid_constant__ CUtensorMap tw1,
                const __grid_constant__ CUtensorMap tw2, const __grid_constant__ CUtensorMap tw3,
                const __grid_constant__ CUtensorMap tx00, const __grid_constant__ CUtensorMap tx01,
                const __grid_constant__ CUtensorMap tx10, const __grid_constant__ CUtensorMap tx11,
                const __grid_constant__ CUtensorMap tx20, const __grid_constant__ CUtensorMap tx21,
                const __grid_constant__ CUtensorMap tx30, const __grid_constant__ CUtensorMap tx31,
                EncWaveArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int l = 0;
  while (l + 1 < a.L && (int)blockIdx.x >= a.layer[l + 1].cta0) ++l;
  __shared__ EncWaveLayer ly;
  if (threadIdx.x == 0) ly = a.layer[l];
  __syncthreads();
  const CUtensorMap* tws[4] = {&tw0, &tw1, &tw2, &tw3};
  const CUtensorMap* txs[4][2] = {{&tx00, &tx01}, {&tx10, &tx11}, {&tx20, &tx21}, {&tx30, &tx31}};
  const CUtensorMap* tmW = tws[l];
  const int S = ly.S, T = ly.T;
  const int s = (int)cluster_ctarank();
  const int tile = (blockIdx.x - ly.cta0) / S;
  const int N = a.N, kbs = ly.kb / S, NS = N / S, kb_in = ly.kb_in;
  const int kb0 = s * kbs;
  const uint32_t nb = (uint32_t)N * 128;
  uint8_t* sW = smem;
  uint8_t* sX = sW + (size_t)kbs * 16384;
  float* recv = reinterpret_cast<float*>(sX + (size_t)kbs * 2 * nb);   // [S][NS][128]
  float* Zs = recv + (size_t)S * 128 * NS;                             // [NS][128] (layer 0)
  float* cst = Zs + (size_t)NS * 128;                                  // [NS][32]
  float* hst = cst + 32 * NS;
  float4* s_bias = reinterpret_cast<float4*>(hst + 32 * NS);
  int* s_len = reinterpret_cast<int*>(s_bias + 32);
  uint64_t* wbar = reinterpret_cast<uint64_t*>(s_len + ((NS + 3) & ~3));
  uint64_t* mdone = wbar + 1;
  uint64_t* xfull = wbar + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xfull + kbs);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // hi and lo B tiles (adjacent) as one N = 2N operand when it fits: one MMA per K step; the lo
  // sums land in TMEM columns [N, 2N)
  const bool stk = 2 * N <= 256;
  uint32_t tcols = 32;
  while ((int)tcols < (stk ? 2 * N : N)) tcols <<= 1;
  const unsigned long long n_own = (unsigned long long)T * S;
  const unsigned long long n_prev = l > 0 ? (unsigned long long)a.layer[l - 1].T * a.layer[l - 1].S : 0;
  const unsigned long long n_next = l + 1 < a.L ? (unsigned long long)a.layer[l + 1].T * a.layer[l + 1].S : 0;
  unsigned long long* c_own = a.cnt + 16 * l;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(tmW);
    mbar_init(wbar, 1);
    for (int i = 0; i < kbs; ++i) mbar_init(&xfull[i], 1);
    mbar_init(mdone, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(wbar, (uint32_t)kbs * 16384);
    for (int i = 0; i < kbs; ++i) tma_load_2d(sW + (size_t)i * 16384, tmW, (kb0 + i) * kBK, tile * kTileM, wbar);
  }
  if (warp == 1) tmem_alloc_dyn(tslot, tcols);
  if (threadIdx.x < 32) {
    const int j = tile * 32 + threadIdx.x;
    s_bias[threadIdx.x] = j < a.Hd ? ly.bias[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int j = threadIdx.x; j < NS; j += blockDim.x) s_len[j] = s * NS + j < a.B ? a.lens[s * NS + j] : 0;
  for (int i = threadIdx.x; i < 32 * NS; i += blockDim.x) { cst[i] = 0.f; hst[i] = 0.f; }
  __syncthreads();
  const float* const Zg = ly.Z;
  const int z_ld = ly.z_ld;
  auto prefetch_z = [&](int t) {
    if (Zg) {
      for (int i = threadIdx.x; i < NS * 32; i += blockDim.x) {
        const int j = i >> 5, ch = i & 31;
        const int b = s * NS + j;
        if (b >= a.B || t >= s_len[j]) continue;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Zs + (size_t)j * 128 + 4 * ch)),
                     "l"(Zg + ((size_t)b * a.S_max + t) * z_ld + (size_t)tile * 128 + 4 * ch)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch_z(0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_arrive_relaxed();                                      // every peer CTA of the cluster has
  cluster_wait();                                                // started before any DSMEM store
  const uint32_t tmem = *tslot;
  const XOut xrec0 = ly.xrec[0], xrec1 = ly.xrec[1], xnext = ly.xnext;
  float* const h_st = ly.h_st;
  float* const c_st = ly.c_st;
  float* const mem = ly.mem;
  const int st_ld = ly.st_ld, mem_ld = ly.mem_ld;
  const bool has_next = xnext.f32 || xnext.hl;
  int n_mma = 0;                                                 // completed MMA batches (mdone phase)

  for (int t = 0; t < a.S_max; ++t) {
    // K blocks this CTA reduces at step t: the input part always (l >= 1), the recurrent part
    // from t = 1 (h_{-1} = 0); layer 0 has no input part
    int first = kb0, last = kb0 + kbs;                           // [first, last) of the concatenated K
    if (t == 0) first = max(first, 0), last = min(last, kb_in);
    const bool mma = last > first;
    const bool any_gate = t > 0 || kb_in > 0;                    // some split contributes W h
    if (any_gate) {
      __syncthreads();
      if (threadIdx.x == 0) {
        if (t > 0) ew_wait_count(c_own, (unsigned long long)t * n_own);            // (a)
        if (l > 0) ew_wait_count(a.cnt + 16 * (l - 1), (unsigned long long)(t + 1) * n_prev);   // (b)
        if (n_next && t >= 2) ew_wait_count(a.cnt + 16 * (l + 1), (unsigned long long)(t - 1) * n_next);  // (c)
        __threadfence();
        asm volatile("fence.proxy.async;" ::: "memory");        // generic stores -> TMA reads
        for (int kg = first; kg < last; ++kg) {
          const int i = kg - kb0;
          const CUtensorMap* tx = kg < kb_in ? txs[l - 1][(t + 1) & 1] : txs[l][t & 1];
          const int kk = kg < kb_in ? kg : kg - kb_in;
          mbar_arrive_expect_tx(&xfull[i], 2 * nb);
          tma_load_2d(sX + (size_t)i * 2 * nb, tx, kk * kBK, 0, &xfull[i]);
          tma_load_2d(sX + (size_t)i * 2 * nb + nb, tx, kk * kBK, N, &xfull[i]);
        }
      }
      if (mma) {
        if (warp == 1 && lane == 0) {
          if (n_mma == 0) mbar_wait(wbar, 0);
          const uint32_t idesc = umma_idesc_bf16(kTileM, stk ? 2 * N : N);
          for (int kg = first; kg < last; ++kg) {
            const int i = kg - kb0;
            // (slot i was loaded at every earlier step, the recurrent part from step 1 on)
            mbar_wait(&xfull[i], (uint32_t)(kg < kb_in ? t : t - 1) & 1u);
            tc_fence_after();
            const uint32_t sa = smem_u32(sW + (size_t)i * 16384);
            const uint32_t sbh = smem_u32(sX + (size_t)i * 2 * nb), sbl = sbh + nb;
            if (stk) {                                 // (no branch between the MMAs)
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)
                tc_mma_bf16(tmem, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sbh + kk * 32), idesc,
                            (kg != first || kk != 0) ? 1u : 0u);
            } else {
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk) {
                const uint64_t da = umma_desc_sw128(sa + kk * 32);
                tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, (kg != first || kk != 0) ? 1u : 0u);
                tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
              }
            }
          }
          tc_commit(mdone);
        }
        __syncwarp();
        mbar_wait(mdone, (uint32_t)n_mma & 1u);
        ++n_mma;
        tc_fence_after();
      }
      // reduce-scatter of the partial gate tiles (zeros when this split had no K block)
      {
        const int q = warp & 3;
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        const int row = q * 32 + lane;
        for (int p = warp >> 2; p < S; p += 2) {
          for (int c0 = 0; c0 < NS; c0 += 8) {
            uint32_t r[8];
            if (mma && stk) {
              uint32_t r2[8];
              tmem_ld8_nw(trow + p * NS + c0, r);
              tmem_ld8_nw(trow + N + p * NS + c0, r2);
              tmem_wait_ld();
              tmem_fence_regs(r);
              tmem_fence_regs(r2);
#pragma unroll
              for (int k = 0; k < 8; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(r2[k]));
            } else if (mma) {
              tmem_ld8_nw(trow + p * NS + c0, r);
              tmem_wait_ld();
              tmem_fence_regs(r);
            } else {
#pragma unroll
              for (int k = 0; k < 8; ++k) r[k] = 0u;
            }
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
      cluster_arrive();
      cluster_wait();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const XOut xo = (t & 1) ? xrec0 : xrec1;                     // h_t -> buffer (t + 1) & 1
    for (int i = threadIdx.x; i < 32 * NS; i += blockDim.x) {
      const int u = i & 31, j = i >> 5;
      const int b = s * NS + j, jj = tile * 32 + u;
      if (b >= a.B || jj >= a.Hd) continue;
      const int L = s_len[j];
      if (t >= L) {
        store_x(xo, b, jj, hst[j * 32 + u]);
        continue;
      }
      const size_t row = (size_t)b * a.S_max + t;
      float4 g = Zg ? *reinterpret_cast<const float4*>(Zs + (size_t)j * 128 + 4 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 bb = s_bias[u];
      g.x += bb.x; g.y += bb.y; g.z += bb.z; g.w += bb.w;
      if (any_gate) {
        for (int p = 0; p < S; ++p) {
          const float4 pv = *reinterpret_cast<const float4*>(recv + ((size_t)p * NS + j) * 128 + 4 * u);
          g.x += pv.x; g.y += pv.y; g.z += pv.z; g.w += pv.w;
        }
      }
      const float ig = ew_sigm(g.x), fg = ew_sigm(g.y), gg = ew_tanh(g.z), og = ew_sigm(g.w);
      const float c = fg * cst[j * 32 + u] + ig * gg;
      const float h = og * ew_tanh(c);
      cst[j * 32 + u] = c;
      hst[j * 32 + u] = h;
      store_x(xo, b, jj, h);
      if (t == L - 1) {
        h_st[(size_t)b * st_ld + jj] = h;
        c_st[(size_t)b * st_ld + jj] = c;
      }
      if (has_next) store_x(xnext, (int)row, jj, h);
      if (mem) mem[row * mem_ld + jj] = h;
    }
    __syncthreads();                                             // Zs / recv consumed, h_t stored
    if (threadIdx.x == 0) {                                      // layer l finished step t here
      __threadfence();
      atomicAdd(c_own, 1ull);
    }
    if (t + 1 < a.S_max) prefetch_z(t + 1);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_arrive();
  cluster_wait();
  if (warp == 1) tmem_dealloc(tmem, tcols);
}

// co-residency of the whole grid as clusters of S CTAs (clusters must fit inside a GPC):
// the layers' counter waits need every CTA resident at once
static bool ew_coresident(int grid, int S, size_t smem) {
  if (cudaFuncSetAttribute(enc_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
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
  if (cudaOccupancyMaxActiveClusters(&ncl, enc_wave_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return ncl * S >= grid;
}

// splits per tile (uniform over the layers: one cluster shape per launch), 0 = does not fit
int enc_wave_splits(int L, const int* kb, int N, int T, int num_sms) {
  if (L < 2 || L > kWaveMaxL || N < 16 || N > 256 || (N % 16) != 0) return 0;
  for (int S = 4; S >= 1; S >>= 1) {
    bool ok = (N / S) % 8 == 0 && L * T * S <= num_sms;
    size_t smem = 0;
    for (int l = 0; l < L && ok; ++l) {
      ok = kb[l] % S == 0 && ew_smem_bytes(kb[l] / S, N, S) <= 227 * 1024;
      if (ok) smem = std::max(smem, ew_smem_bytes(kb[l] / S, N, S));
    }
    if (ok && ew_coresident(L * T * S, S, smem)) return S;
  }
  return 0;
}

cudaError_t launch_enc_wave(const CUtensorMap* tw, const CUtensorMap (*tx)[2], const EncWaveArgs& a, int grid, int S,
                            cudaStream_t st) {
  size_t smem = 0;
  for (int l = 0; l < a.L; ++l) {
    const size_t b = ew_smem_bytes(a.layer[l].kb / S, a.N, S);
    smem = b > smem ? b : smem;
  }
  cudaError_t e = cudaMemsetAsync(a.cnt, 0, (size_t)kWaveMaxL * 16 * 8, st);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(enc_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int L1 = a.L > 1 ? 1 : 0, L2 = a.L > 2 ? 2 : L1, L3 = a.L > 3 ? 3 : L2;
  return cudaLaunchKernelEx(&cfg, enc_wave_kernel, tw[0], tw[L1], tw[L2], tw[L3], tx[0][0], tx[0][1], tx[L1][0],
                            tx[L1][1], tx[L2][0], tx[L2][1], tx[L3][0], tx[L3][1], a);
}

}  // namespace onmt
