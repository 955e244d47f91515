// tcgen05 weight-streaming GEMM for the decode/encode contractions (bf16 models).
//
//   D[m][n] = sum_k W[m][k] * (Xhi[n][k] + Xlo[n][k])
//
// W (weights, bf16, rows padded to 128, K padded to 64) is the MMA A operand
// (M = 128 weight rows per CTA = the 128 TMEM lanes); the activations X are the B
// operand (N = up to 256 hypothesis/token rows), given as two bf16 planes so that
// hi + lo carries ~16 mantissa bits (DESIGN.md §6 H4: plain bf16 activations miss
// the 2e-3 / 1e-4 parity bars).  Both planes accumulate into the same fp32 TMEM
// accumulator.  Operands are staged by TMA (128-byte swizzle) through a ring of
// `stages` shared-memory slots; one elected thread issues tcgen05.mma.
//
// Epilogues:
//   MODE_PARTIAL: split-K partial sums P[split][n][m] (fp32), reduced in fixed order by
//                 the consumer kernel (deterministic, no float atomics).
//   MODE_GEN:     generator (PAPER.md P118-119 softmax layer): logits z = D + b for 128
//                 vocabulary rows never leave the SM; per (tile, row) the kernel emits
//                 the online (max, sum exp) and the tile top-k by logit (DESIGN.md §6 K6).
#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

enum { MODE_PARTIAL = 0, MODE_GEN = 1 };

struct TcGemmArgs {
  int n_rows_pad;   // rows of one X plane (lo plane starts at this row)
  int n_group;      // rows per CTA (multiple of 16, <= 256)
  int n_valid;      // rows < n_valid are stored
  int k_blocks;     // K_pad / 64
  int kb_per_split; // K blocks per split (blockIdx.z)
  int stages;
  int m_pad;
  int tmem_cols;    // power of two >= n_group
  float* out;       // MODE_PARTIAL: [splits][n_rows_pad][m_pad]
  StepCtl ctl;
};

template <int MODE, int KMAX>
__global__ void __launch_bounds__(128, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, TcGemmArgs a,
               GenOut g) {
  if (all_done(a.ctl)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = kTileM * 128;
  const uint32_t b_bytes = a.n_group * 128;
  const uint32_t stage_bytes = a_bytes + 2 * b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
  uint64_t* empty = full + a.stages;
  uint64_t* done = empty + a.stages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kTileM;
  const int n0 = blockIdx.y * a.n_group;
  const int kb0 = blockIdx.z * a.kb_per_split;
  int nkb = a.k_blocks - kb0;
  if (nkb > a.kb_per_split) nkb = a.kb_per_split;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(tslot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int i = 0; i < nkb; ++i) {
      const int s = i % a.stages;
      if (i >= a.stages) mbar_wait(&empty[s], ((i / a.stages) & 1) ^ 1);
      uint8_t* st = smem + s * stage_bytes;
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      const int kx = (kb0 + i) * kBK;
      tma_load_2d(st, &tmW, kx, m0, &full[s]);
      tma_load_2d(st + a_bytes, &tmX, kx, n0, &full[s]);
      tma_load_2d(st + a_bytes + b_bytes, &tmX, kx, a.n_rows_pad + n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    const uint32_t idesc = umma_idesc_bf16(kTileM, a.n_group);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % a.stages;
      mbar_wait(&full[s], (i / a.stages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint32_t sbh = sa + a_bytes, sbl = sa + a_bytes + b_bytes;
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk) {
        const uint64_t da = umma_desc_sw128(sa + kk * 32);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, (i | kk) != 0);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
      }
      tc_commit(&empty[s]);
    }
    tc_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();

  const int q = warp & 3;                       // TMEM lane quarter of this warp
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  if (MODE == MODE_PARTIAL) {
    float* out = a.out + (size_t)blockIdx.z * a.n_rows_pad * a.m_pad;
    const int m = m0 + q * 32 + lane;
    for (int c0 = 0; c0 < a.n_group; c0 += 16) {
      float v[16];
      tmem_ld16(trow + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c0 + j;
        if (n < a.n_valid) out[(size_t)n * a.m_pad + m] = v[j];
      }
    }
  } else {
    // Stage the 128 x n_group logit tile transposed in shared memory (the operand
    // ring is free now), then one thread per row scans its 128 vocabulary logits.
    __syncthreads();
    float* stg = reinterpret_cast<float*>(smem);
    const int LD = kTileM + 1;
    const int vr = q * 32 + lane;
    for (int c0 = 0; c0 < a.n_group; c0 += 16) {
      float v[16];
      tmem_ld16(trow + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) stg[(c0 + j) * LD + vr] = v[j];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < a.n_group; c += blockDim.x) {
      const int r = n0 + c;
      if (r >= g.rows_valid) continue;
      float mx, sm, tz[KMAX];
      int ti[KMAX];
      scan_tile_column<KMAX>(stg + c * LD, 1, m0, g, mx, sm, tz, ti);
      write_gen_partial<KMAX>(g, blockIdx.x, r, mx, sm, tz, ti);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

// ------------------------------------------------------------------ host launchers
static size_t tc_smem_bytes(int n_group, int stages, int mode) {
  size_t stage = kTileM * 128 + 2 * (size_t)n_group * 128;
  size_t ring = stage * stages;
  size_t stg = mode == MODE_GEN ? (size_t)n_group * (kTileM + 1) * 4 : 0;
  size_t body = ring > stg ? ring : stg;
  return 1024 + body + (2 * stages + 1) * 8 + 16;
}

int tc_pick_stages(int n_group, int k_blocks_per_cta) {
  const size_t limit = 227 * 1024;
  int st = 4;
  while (st > 1 && tc_smem_bytes(n_group, st, MODE_GEN) > limit) --st;
  if (st > k_blocks_per_cta) st = k_blocks_per_cta > 1 ? k_blocks_per_cta : 1;
  return st;
}

template <int MODE, int KMAX>
static cudaError_t launch_tc(const CUtensorMap& tmW, const CUtensorMap& tmX, const TcGemmArgs& a, const GenOut& g,
                             dim3 grid, cudaStream_t st) {
  size_t smem = tc_smem_bytes(a.n_group, a.stages, MODE);
  auto fn = tc_gemm_kernel<MODE, KMAX>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, 128, smem, st>>>(tmW, tmX, a, g);
  return cudaGetLastError();
}

cudaError_t tc_gemm_partial(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                            int n_valid, int k_blocks, int splits, float* out, StepCtl ctl, cudaStream_t st) {
  TcGemmArgs a{};
  a.n_rows_pad = n_rows_pad;
  a.n_group = n_group;
  a.n_valid = n_valid;
  a.k_blocks = k_blocks;
  a.kb_per_split = (k_blocks + splits - 1) / splits;
  a.stages = tc_pick_stages(n_group, a.kb_per_split);
  a.m_pad = m_pad;
  int tc = 32;
  while (tc < n_group) tc <<= 1;
  a.tmem_cols = tc;
  a.out = out;
  a.ctl = ctl;
  GenOut g{};
  dim3 grid(m_pad / kTileM, n_rows_pad / n_group, splits);
  return launch_tc<MODE_PARTIAL, 1>(tmW, tmX, a, g, grid, st);
}

cudaError_t tc_gemm_gen(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                        int k_blocks, const GenOut& g, StepCtl ctl, cudaStream_t st) {
  TcGemmArgs a{};
  a.n_rows_pad = n_rows_pad;
  a.n_group = n_group;
  a.n_valid = g.rows_valid;
  a.k_blocks = k_blocks;
  a.kb_per_split = k_blocks;
  a.stages = tc_pick_stages(n_group, k_blocks);
  a.m_pad = m_pad;
  int tc = 32;
  while (tc < n_group) tc <<= 1;
  a.tmem_cols = tc;
  a.out = nullptr;
  a.ctl = ctl;
  dim3 grid(m_pad / kTileM, n_rows_pad / n_group, 1);
  if (g.K <= 1) return launch_tc<MODE_GEN, 1>(tmW, tmX, a, g, grid, st);
  if (g.K <= 2) return launch_tc<MODE_GEN, 2>(tmW, tmX, a, g, grid, st);
  if (g.K <= 4) return launch_tc<MODE_GEN, 4>(tmW, tmX, a, g, grid, st);
  if (g.K <= 8) return launch_tc<MODE_GEN, 8>(tmW, tmX, a, g, grid, st);
  return launch_tc<MODE_GEN, 16>(tmW, tmX, a, g, grid, st);
}

}  // namespace onmt
