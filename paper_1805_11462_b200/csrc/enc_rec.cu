// A3: the encoder recurrence of one layer as ONE persistent kernel (
// PAPER.md P129-133; SPEC S257-265):
//
//   for t = 0 .. S_max-1:  z_t = Z_t + b + W_hh h_{t-1};  (i,f,g,o) = (σ,σ,tanh,σ)(z_t)
//                          c_t = f c_{t-1} + i g;  h_t = o tanh(c_t)
//
// per sentence over its own S_b tokens (packed semantics, R3: frozen for t >= S_b; the
// backward direction runs pos = S_b-1-t), Z = W_ih x hoisted over all t by one GEMM before.
//
// Grid = D x T CTAs (direction, 128-row tile of the interleaved gate rows = 32 units), all
// co-resident (one per SM).  Each CTA keeps its W_hh tile (128 x K bf16) resident in shared
// memory for the whole sequence and its units' c state on chip; per step it TMA-loads
// h_{t-1} of every sentence (bf16 hi/lo planes, written by all tiles of its direction in the
// previous step), runs the tcgen05 MMAs (M = 128 gate rows, N = sentences), applies the cell
// to its 32 units and stores h_t into the other parity buffer; a software barrier among the
// direction's T CTAs separates the steps.  This replaces 2 launches per step (split-K GEMM +
// cell kernel) by one launch per layer.
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
  int T, Hd, B, N, S_max, kb;
  const int* lens;
  unsigned int* bar;       // [2 x 32] step-barrier words (one per direction, self-resetting)
  unsigned long long* trace;   // (debug) per-step %globaltimer stamps of CTA 0, or nullptr
};
__device__ __forceinline__ unsigned long long er_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int kErTr = 132;                        // transpose buffer row stride (floats)

// sigmoid / tanh via the fast exponential (rel. error ~2^-21, as the decoder's fused cell)
__device__ __forceinline__ float er_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float er_tanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

static size_t er_smem_bytes(int kb, int N) {
  return 1024 + (size_t)kb * 16384 + (size_t)kb * 2 * N * 128 + (size_t)N * 128 * 4 + (size_t)2 * 32 * N * 4 +
         32 * 16 + (size_t)N * 4 + (2 + kb) * 8 + 32 + 16;
}

__global__ void __launch_bounds__(256, 1)
enc_rec_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
               const __grid_constant__ CUtensorMap tmX00, const __grid_constant__ CUtensorMap tmX01,
               const __grid_constant__ CUtensorMap tmX10, const __grid_constant__ CUtensorMap tmX11,
               EncRecArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int d = blockIdx.x / a.T, tile = blockIdx.x % a.T;
  __shared__ EncRecDir dr;                                        // my direction's arguments (uniform)
  if (threadIdx.x == 0) dr = a.dir[d];
  const CUtensorMap* tmW = d ? &tmW1 : &tmW0;
  const CUtensorMap* tmXa = d ? &tmX10 : &tmX00;                 // parity 0 (h_{t-1} for even t)
  const CUtensorMap* tmXb = d ? &tmX11 : &tmX01;
  const int N = a.N, kb = a.kb;
  const uint32_t nb = (uint32_t)N * 128;                          // one operand plane, one K block
  uint8_t* sW = smem;                                             // [kb][128 x 64] bf16 (SW128)
  uint8_t* sX = sW + (size_t)kb * 16384;                          // [kb][hi, lo][N x 64]
  float* Tr = reinterpret_cast<float*>(sX);                       // [N][132] gates (overlays sX)
  float* Zs = reinterpret_cast<float*>(sX + (size_t)kb * 2 * nb); // [N][128] Z_t of my gate rows
  float* cst = Zs + (size_t)N * 128;                              // [N][32] c of my units
  float* hst = cst + 32 * N;                                      // [N][32] h of my units
  float4* s_bias = reinterpret_cast<float4*>(hst + 32 * N);      // [32]
  int* s_len = reinterpret_cast<int*>(s_bias + 32);               // [N]
  uint64_t* wbar = reinterpret_cast<uint64_t*>(s_len + ((N + 3) & ~3));
  uint64_t* mdone = wbar + 1;
  uint64_t* xfull = wbar + 2;                                     // [kb] per K block (TMA -> MMA pipelining)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xfull + kb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t tcols = 32;
  while ((int)tcols < N) tcols <<= 1;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(tmW);
    tma_prefetch_desc(tmXa);
    tma_prefetch_desc(tmXb);
    mbar_init(wbar, 1);
    for (int i = 0; i < kb; ++i) mbar_init(&xfull[i], 1);
    mbar_init(mdone, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(wbar, (uint32_t)kb * 16384);            // W_hh tile, resident for all t
    for (int i = 0; i < kb; ++i) tma_load_2d(sW + (size_t)i * 16384, tmW, i * kBK, tile * kTileM, wbar);
  }
  if (warp == 1) tmem_alloc_dyn(tslot, tcols);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int j = tile * 32 + threadIdx.x;
    s_bias[threadIdx.x] = j < a.Hd ? dr.bias[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int b = threadIdx.x; b < N; b += blockDim.x) s_len[b] = b < a.B ? a.lens[b] : 0;
  for (int i = threadIdx.x; i < 32 * N; i += blockDim.x) { cst[i] = 0.f; hst[i] = 0.f; }
  __syncthreads();
  // Z_t of my gate rows for every live sentence (cp.async, 16 B chunks)
  const bool backward_ = dr.backward != 0;
  const float* const Zg = dr.Z;
  const int z_ld = dr.z_ld;
  auto prefetch_z = [&](int t) {
    for (int i = threadIdx.x; i < N * 32; i += blockDim.x) {
      const int b = i >> 5, ch = i & 31;
      const int L = s_len[b];
      if (b >= a.B || t >= L) continue;
      const int pos = backward_ ? L - 1 - t : t;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Zs + (size_t)b * 128 + 4 * ch)),
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
  const bool backward = dr.backward != 0, has_next = xnext.f32 || xnext.hl;

  for (int t = 0; t < a.S_max; ++t) {
    if (t > 0) {
      // every tile of my direction has stored h_{t-1} (and finished reading h_{t-2}'s buffer)
      __syncthreads();
      if (threadIdx.x == 0) {
        if (a.trace && blockIdx.x == 0 && t < 64) a.trace[t * 8 + 0] = er_now();
        cta_group_barrier(a.bar + 32 * d, (unsigned)a.T);
        if (a.trace && blockIdx.x == 0 && t < 64) a.trace[t * 8 + 1] = er_now();
        asm volatile("fence.proxy.async;" ::: "memory");          // generic stores -> TMA reads
        const CUtensorMap* tx = (t & 1) ? tmXb : tmXa;            // buffer t & 1 holds h_{t-1}
        for (int i = 0; i < kb; ++i) {
          mbar_arrive_expect_tx(&xfull[i], 2 * nb);
          tma_load_2d(sX + (size_t)i * 2 * nb, tx, i * kBK, 0, &xfull[i]);
          tma_load_2d(sX + (size_t)i * 2 * nb + nb, tx, i * kBK, N, &xfull[i]);
        }
      }
      if (warp == 1 && lane == 0) {
        if (t == 1) mbar_wait(wbar, 0);
        if (a.trace && blockIdx.x == 0 && t < 64) a.trace[t * 8 + 2] = er_now();
        const uint32_t idesc = umma_idesc_bf16(kTileM, N);
        for (int i = 0; i < kb; ++i) {
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
      if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 3] = er_now();
      tc_fence_after();
      // W_hh h_{t-1}: TMEM [gate row][sentence] -> Tr[sentence][gate row]
      {
        const int q = warp & 3, half = warp >> 2;
        const int cb = half * (N >> 1), ce = cb + (N >> 1);
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        for (int c0 = cb; c0 < ce; c0 += 8) {
          uint32_t r[8];
          tmem_ld8_nw(trow + c0, r);
          tmem_wait_ld();
          tmem_fence_regs(r);
#pragma unroll
          for (int k = 0; k < 8; ++k) Tr[(size_t)(c0 + k) * kErTr + q * 32 + lane] = __uint_as_float(r[k]);
        }
      }
      tc_fence_before();
      if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 6] = er_now();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");          // Z_t landed (my chunks)
    __syncthreads();
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 4] = er_now();
    // ---- the cell for (unit u, sentence b); consecutive threads take consecutive units
    const XOut xo = (t & 1) ? xrec0 : xrec1;                     // h_t for step t+1's MMA
    for (int i = threadIdx.x; i < 32 * N; i += blockDim.x) {
      const int u = i & 31, b = i >> 5;
      const int j = tile * 32 + u;
      if (b >= a.B || j >= a.Hd) continue;
      const int L = s_len[b];
      if (t >= L) {                                               // finished: carry h forward
        store_x(xo, b, j, hst[b * 32 + u]);
        continue;
      }
      const int pos = backward ? L - 1 - t : t;
      const size_t row = (size_t)b * a.S_max + pos;
      float4 g = *reinterpret_cast<const float4*>(Zs + (size_t)b * 128 + 4 * u);
      const float4 bb = s_bias[u];
      g.x += bb.x; g.y += bb.y; g.z += bb.z; g.w += bb.w;
      if (t > 0) {
        const float4 p = *reinterpret_cast<const float4*>(Tr + (size_t)b * kErTr + 4 * u);
        g.x += p.x; g.y += p.y; g.z += p.z; g.w += p.w;
      }
      const float ig = er_sigm(g.x), fg = er_sigm(g.y), gg = er_tanh(g.z), og = er_sigm(g.w);
      const float c = fg * cst[b * 32 + u] + ig * gg;
      const float h = og * er_tanh(c);
      cst[b * 32 + u] = c;
      hst[b * 32 + u] = h;
      store_x(xo, b, j, h);
      h_st[(size_t)b * st_ld + j] = h;
      c_st[(size_t)b * st_ld + j] = c;
      if (has_next) store_x(xnext, (int)row, next_col + j, h);
      if (mem) mem[row * mem_ld + mem_col + j] = h;
    }
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 7] = er_now();
    __syncthreads();                                              // Zs / Tr consumed
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 64) a.trace[t * 8 + 5] = er_now();
    if (t + 1 < a.S_max) prefetch_z(t + 1);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, tcols);
}

// can this layer run as one persistent kernel? (shared memory, co-residency)
bool enc_rec_fits(int kb, int N, int D, int T, int num_sms) {
  return N >= 16 && N <= 256 && (N % 16) == 0 && D * T <= num_sms && er_smem_bytes(kb, N) <= 227 * 1024 &&
         (size_t)N * kErTr * 4 <= (size_t)kb * 2 * N * 128;
}

cudaError_t launch_enc_rec(const CUtensorMap* tmW, const CUtensorMap* tmX0, const CUtensorMap* tmX1,
                           const EncRecArgs& a, int D, cudaStream_t st) {
  const size_t smem = er_smem_bytes(a.kb, a.N);
  cudaError_t e = cudaFuncSetAttribute(enc_rec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int d1 = D > 1 ? 1 : 0;
  enc_rec_kernel<<<D * a.T, 256, smem, st>>>(tmW[0], tmW[d1], tmX0[0], tmX1[0], tmX0[d1], tmX1[d1], a);
  return cudaGetLastError();
}

}  // namespace onmt
