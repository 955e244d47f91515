// Split-K tcgen05 GEMM with the split reduction and the consumer fused into the same
// kernel: the decoder LSTM cell (PAPER.md P129-136, gates = W [x; h] + b) or the
// attentional vector h~ = tanh(W_out [c; h]) (P69) - SURVEY §8(a) rows A6 / A8.
//
// Grid = tiles x S (tile = 128 weight rows x one N-group of hypothesis rows, S = split-K
// ways), one CTA per SM and grid <= #SMs, so every CTA is co-resident.
//   1. The producer thread TMA-loads the CTA's whole weight K-slice BEFORE
//      griddepcontrol.wait (weights are constants: the loads overlap the previous kernel),
//      then the hi/lo activation planes after it.  The slice stays resident (one smem
//      slot per K block).
//   2. One thread issues tcgen05.mma (M = 128 weight rows, N = n_group, hi and lo planes
//      accumulate into one fp32 TMEM accumulator).  Meanwhile warps 2-3 prefetch the
//      epilogue's side inputs (bias, gathered c_prev) into shared memory.
//   3. The partial tile goes TMEM -> registers -> global scratch [tile][S][n][128]
//      (coalesced, L2-resident), then a per-tile arrival barrier (release / acquire)
//      waits for the tile's S splits.
//   4. CTA s owns hypothesis columns [s*NC, (s+1)*NC): one bulk copy per split pulls
//      those columns of every partial into shared memory, they are summed in fixed split
//      order (deterministic) and the epilogue runs on them.
// A DSMEM exchange inside a cluster was measured slower (~20 B/clk per SM) than this L2
// round trip for 80 KB partial tiles.
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

enum { EPI_CELL = 0, EPI_TANH = 1 };

struct FusedArgs {
  int n_rows_pad, n_group, n_valid, k_blocks, kb_per_split, stages, tmem_cols, S;
  int NC;                  // hypothesis columns owned per split (multiple of 4)
  int M;                   // valid weight rows (4H for the cell, H for tanh)
  float* scratch;          // [tiles][S][n_group][128] fp32 partial tiles
  unsigned int* counters;  // [tiles][2] arrival barrier {count, generation}
  // EPI_CELL
  const float4* bias;      // [H] interleaved (i,f,g,o) pre-summed biases
  const float* cg;         // [rows_pad][H] c_prev gathered by parent
  float* c_out;
  float* h_out;
  int H;
  CellDst dst;
  // EPI_TANH
  float* htilde;
  XOut xg;
  // EPI_CELL of the top decoder layer with W_out folded into attention:
  // woh = W_out[:, H:2H] per 32-unit tile: [fold_mo(H) outputs][32 units] bf16, K-major with the
  // 64-byte swizzle already applied (the shared-memory image of the MMA A operand); the CTA
  // writes its units' share  W_out[:, units] h[units, cols]  to woh_part[m_tile][row][H] (fp32)
  const __nv_bfloat16* woh;
  float* woh_part;
  // EPI_CELL, recurrent-split step: per-row gate pre-activations added to
  // the GEMM result (gb[row * gb_ld + 4j .. 4j + 3] for unit j: W_hh h[parent] + bias), or null
  const float* gb;
  int gb_ld;
  StepCtl ctl;
  int stack;               // 2 n_group <= 256: the hi and lo B tiles (adjacent in shared memory) form
                           // one N = 2 n_group operand, one MMA per K step instead of two; the hi /
                           // lo sums land in TMEM columns [0, n) / [n, 2n) and are added in the
                           // epilogue
  int dbg;                 // microbenchmark ablations (ONMT_KTRACE builds only)
};

// sigmoid / tanh via the fast exponential (ex2.approx, rel. error ~2^-21): well inside the
// fp32 (1e-5) and bf16 (2e-3) log-prob bars; avoids the IEEE-division / tanhf slow paths
__device__ __forceinline__ float sigmf(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float tanhfast(float x) {
  const float e = __expf(-2.f * fabsf(x));
  const float t = __fdividef(1.f - e, 1.f + e);
  return copysignf(t, x);
}



// folded W_out slice: row stride (bf16 elements) of W_out[:, units]^T in shared memory -
// 16-byte rows for ldmatrix, +8 so the 8 rows of an 8x8 matrix hit distinct banks
__host__ __device__ __forceinline__ int fold_mo(int H) { return (H + 127) / 128 * 128; }   // outputs, padded
__host__ __device__ __forceinline__ size_t fold_tile_bytes(int H) { return (size_t)fold_mo(H) * 64; }
__host__ __device__ __forceinline__ int fold_chunks(int NC) { return (NC + 31) / 32; }      // 32-column chunks
// byte offset of (row r, column c < 32) in a [rows][32] bf16 K-major tile with the 64-byte swizzle
// (address bits 4-5 ^= bits 7-8): the layout the host packs woh in and the kernel writes h in
__host__ __device__ __forceinline__ uint32_t fold_sw64(int r, int c) {
  return (uint32_t)(r * 64 + ((((c >> 3) ^ (r >> 1)) & 3) << 4) + ((c & 7) << 1));
}

// D += A B, m16n8k16, bf16 inputs, fp32 accumulate (A: 4 regs, B: 2 regs, row.col)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// RING = 0: the split's whole K-slice is resident (one stage per K block, loaded once);
// RING = 1: fewer stages than K blocks, reloaded through empty barriers (separate instances:
// the two loop shapes compiled into one kernel measured slower for both)
template <int EPI, int RING>
__global__ void __launch_bounds__(256, 1)
tc_gemm_fused_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     FusedArgs a) {
  KT(0);
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t a_bytes = kTileM * 128, b_bytes = a.n_group * 128;
  const uint32_t stage_bytes = a_bytes + 2 * b_bytes;
  const size_t ring = (size_t)a.stages * stage_bytes;
  size_t recv_bytes = (size_t)(a.S + 1) * a.NC * kTileM * 4;         // recv [S][NC][128] + red [NC][128]
  float* recv = reinterpret_cast<float*>(smem);                  // [S][NC][128], overlays the ring
  uint8_t* tail = smem + (ring > recv_bytes ? ring : recv_bytes);
  float4* s_bias = reinterpret_cast<float4*>(tail);               // [32] (cell)
  float* s_cg = reinterpret_cast<float*>(tail + 32 * 16);         // [NC][32] (cell)
  uint64_t* full = reinterpret_cast<uint64_t*>(tail + 32 * 16 + (size_t)a.NC * 32 * 4);
  uint64_t* done = full + a.stages;
  uint64_t* rbar = done + 1;
  uint64_t* wbar = rbar + 1;
  uint64_t* empty = wbar + 1;                                      // [stages] (ring: stages < K blocks)
  uint64_t* fbar = empty + a.stages;                               // fold MMAs of a column chunk done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(fbar + 1);
  // (offsets from smem keep the shared address space visible to the compiler: LDS, not LD.E)
  const size_t woh_off = ((size_t)(reinterpret_cast<uint8_t*>(tslot) - smem) + 16 + 1023) & ~(size_t)1023;
  uint8_t* woh_s = smem + woh_off;                                 // [fold_mo][32] bf16, SW64 (A operand)
  uint8_t* s_hb = woh_s + fold_tile_bytes(a.H);                    // [chunk][hi, lo][32 cols][32 units] (B)
  float4* s_gb = reinterpret_cast<float4*>(smem + woh_off +
                                           (a.woh ? fold_tile_bytes(a.H) + (size_t)fold_chunks(a.NC) * 4096 : 0));
                                                                  // [NC][32] (16-byte aligned offsets)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x / a.S;
  const int split = blockIdx.x % a.S;
  const int n_groups = a.n_rows_pad / a.n_group;
  const int mt = tile / n_groups, grp = tile % n_groups;
  const int m0 = mt * kTileM;
  const int n0 = grp * a.n_group;
  const int kb0 = split * a.kb_per_split;
  int nkb = a.k_blocks - kb0;
  if (nkb > a.kb_per_split) nkb = a.kb_per_split;
  if (nkb < 0) nkb = 0;
  const int c_own = split * a.NC;                                  // first hypothesis column I own
  const int ncols = max(0, min(a.NC, a.n_group - c_own));

  // ---- prologue (overlaps the predecessor under PDL): barriers, TMEM, weight prefetch
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    mbar_init(rbar, 1);
    mbar_init(wbar, 1);
    mbar_init(fbar, 1);
    fence_mbar_init();
    for (int i = 0; i < nkb && i < a.stages; ++i) {                // the first ring stages' weights
      mbar_expect_tx(&full[i], a_bytes);
      tma_load_2d(smem + i * stage_bytes, &tmW, (kb0 + i) * kBK, m0, &full[i]);
    }
    if (EPI == EPI_CELL && a.woh) {                                // W_out[:, tile's units] (constant)
      const uint32_t wb = (uint32_t)fold_tile_bytes(a.H);
      mbar_arrive_expect_tx(wbar, wb);
      bulk_g2s(woh_s, reinterpret_cast<const uint8_t*>(a.woh) + (size_t)mt * wb, wb, wbar);
    }
  }
  if (warp == 0) tmem_alloc_dyn(tslot, a.tmem_cols);
  tc_fence_before();
  pdl_wait();                                    // activations / c_prev / n_done now visible
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const bool quit = all_done(a.ctl);             // uniform over the grid
  KT(1);

  if (warp == 0 && lane == 0) {
    if (!RING) {
      for (int i = 0; i < nkb; ++i) {
        uint8_t* st = smem + i * stage_bytes;
        if (quit) {
          mbar_arrive_local(&full[i]);
        } else {
          mbar_arrive_expect_tx(&full[i], 2 * b_bytes);
          tma_load_2d(st + a_bytes, &tmX, (kb0 + i) * kBK, n0, &full[i]);
          tma_load_2d(st + a_bytes + b_bytes, &tmX, (kb0 + i) * kBK, a.n_rows_pad + n0, &full[i]);
        }
      }
    } else {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % a.stages;
        uint8_t* st = smem + s * stage_bytes;
        if (quit) {
          if (i < a.stages) mbar_arrive_local(&full[s]);
          continue;
        }
        if (i >= a.stages) {                                       // ring: slot s free again
          mbar_wait(&empty[s], ((i / a.stages) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], a_bytes + 2 * b_bytes);
          tma_load_2d(st, &tmW, (kb0 + i) * kBK, m0, &full[s]);
        } else {
          mbar_arrive_expect_tx(&full[s], 2 * b_bytes);
        }
        tma_load_2d(st + a_bytes, &tmX, (kb0 + i) * kBK, n0, &full[s]);
        tma_load_2d(st + a_bytes + b_bytes, &tmX, (kb0 + i) * kBK, a.n_rows_pad + n0, &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(kTileM, a.stack ? 2 * a.n_group : a.n_group);
    for (int i = 0; i < nkb; ++i) {
      const int s = RING ? i % a.stages : i;
      if (RING && quit && i >= a.stages) break;
      mbar_wait(&full[s], RING ? (i / a.stages) & 1 : 0);
      tc_fence_after();
      if (quit) continue;
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint32_t sbh = sa + a_bytes, sbl = sa + a_bytes + b_bytes;
      if (a.stack) {                             // (no branch between the MMAs)
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          tc_mma_bf16(tmem, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sbh + kk * 32), idesc, (i | kk) != 0);
      } else {
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          const uint64_t da = umma_desc_sw128(sa + kk * 32);
          tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, (i | kk) != 0);
          tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
        }
      }
      if (RING) tc_commit(&empty[s]);            // slot s reusable once these MMAs retire
    }
    tc_commit(done);                             // also fires with no MMA issued
  } else if (warp >= 2 && EPI == EPI_CELL && !quit) {
    // side inputs of my columns: bias of the tile's 32 units, c_prev[r][j]
    const int t = threadIdx.x - 64;               // 192 threads
    if (t < 32) {
      const int j = m0 / 4 + t;
      s_bias[t] = j < a.H ? __ldg(&a.bias[j]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (a.gb)
      for (int i = t; i < ncols * 32; i += 192) {
        const int c = i / 32, ul = i % 32;
        const int r = n0 + c_own + c, j = m0 / 4 + ul;
        s_gb[i] = (r < a.n_valid && j < a.H) ? __ldcg(reinterpret_cast<const float4*>(a.gb + (size_t)r * a.gb_ld) + j)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    for (int i0 = t; i0 < ncols * 32; i0 += 192 * 8) {   // 8 loads in flight per thread
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + 192 * u;
        const int c = i / 32, ul = i % 32;
        const int r = n0 + c_own + c, j = m0 / 4 + ul;
        v[u] = (i < ncols * 32 && r < a.n_valid && j < a.H) ? __ldg(&a.cg[(size_t)r * a.H + j]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + 192 * u < ncols * 32) s_cg[i0 + 192 * u] = v[u];
    }
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  KT(2);
  if (quit) {                                    // every TMA landed (waited above); nothing else in flight
    if (EPI == EPI_CELL && a.woh) mbar_wait(wbar, 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
    return;
  }
  float* red;
  if (a.S == 1) {
    // ---- (3') no split: the accumulator goes straight to red[c][128] in shared memory (the
    //      ring is free: every MMA retired); a warp writes 128 contiguous bytes per column
    red = recv;
    const int q = warp & 3, half = warp >> 2;
    const int m = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    for (int c0 = half * 16; c0 < a.n_group; c0 += 32) {
      uint32_t r[16];
      if (nkb > 0 && a.stack) {
        uint32_t r2[16];
        tmem_ld16_nw(trow + c0, r);
        tmem_ld16_nw(trow + a.n_group + c0, r2);
        tmem_wait_ld();
        tmem_fence_regs(r);
        tmem_fence_regs(r2);
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(r2[k]));
      } else if (nkb > 0) {
        tmem_ld16_nw(trow + c0, r);
        tmem_wait_ld();
        tmem_fence_regs(r);
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = 0u;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (c0 + k < a.n_group) red[(size_t)(c0 + k) * kTileM + m] = __uint_as_float(r[k]);
    }
    tc_fence_before();
  } else {
  // ---- (3) partial tile: TMEM -> registers -> global scratch [tile][split][n/4][128][4]
    //      (each thread stores float4 = 4 consecutive columns of its row: a warp writes 512
    //      contiguous bytes), then release the tile counter
    {
      const int q = warp & 3, half = warp >> 2;                    // warps q and q+4 share a lane quarter
      const int m = q * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
      const int hcols = (a.n_group / 2 + 3) & ~3;
      const int cb = half * hcols, ce = half ? a.n_group : hcols;
      float4* out = reinterpret_cast<float4*>(a.scratch + ((size_t)(tile * a.S + split) * a.n_group) * kTileM) + m;
      for (int c0 = cb; c0 < ce; c0 += 32) {
        uint32_t r[32];
  #pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (c0 + 4 * k < ce && nkb > 0)
            tmem_ld4_nw(trow + c0 + 4 * k, r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
          else
            r[4 * k] = r[4 * k + 1] = r[4 * k + 2] = r[4 * k + 3] = 0u;
        }
        tmem_wait_ld();
        tmem_fence_regs(r);
        if (a.stack) {
          uint32_t r2[32];
  #pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (c0 + 4 * k < ce && nkb > 0)
              tmem_ld4_nw(trow + a.n_group + c0 + 4 * k, r2[4 * k], r2[4 * k + 1], r2[4 * k + 2], r2[4 * k + 3]);
            else
              r2[4 * k] = r2[4 * k + 1] = r2[4 * k + 2] = r2[4 * k + 3] = 0u;
          }
          tmem_wait_ld();
          tmem_fence_regs(r2);
  #pragma unroll
          for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(r2[k]));
        }
  #pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c0 + 4 * k < ce)
            __stcg(out + (size_t)((c0 >> 2) + k) * kTileM,
                   make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]), __uint_as_float(r[4 * k + 2]),
                               __uint_as_float(r[4 * k + 3])));
      }
    }
    tc_fence_before();
    __syncthreads();        // (thread 0's gpu-scope fence in cta_group_barrier is cumulative over
    KT(3);                  //  the CTA's stores ordered before it by the barrier: release pattern)
    if (threadIdx.x == 0) {
      cta_group_barrier(a.counters + 2 * tile, (unsigned)a.S);   // the tile's S splits are stored
      asm volatile("fence.proxy.async;" ::: "memory");
      KT(4);
      // (4) my columns of every split's partial: S contiguous blocks of NC/4 x 128 x 4 floats
      if (ncols > 0) {
        const uint32_t bytes = (uint32_t)ncols * kTileM * 4;
        mbar_arrive_expect_tx(rbar, bytes * a.S);
        for (int p = 0; p < a.S; ++p)
          bulk_g2s(recv + (size_t)p * a.NC * kTileM,
                   a.scratch + ((size_t)(tile * a.S + p) * a.n_group + c_own) * kTileM, bytes, rbar);
      } else {
        mbar_arrive_local(rbar);
      }
    }
    mbar_wait(rbar, 0);
    KT(5);
    // fixed-order split sum, written transposed into red[c][128] (conflict-free epilogue reads)
    red = recv + (size_t)a.S * a.NC * kTileM;
    if (ncols > 0) {
      const size_t slot = (size_t)a.NC * kTileM;
      const int nit = (ncols / 4) * kTileM;       // (c4 block, m) items, float4 each
      for (int it0 = threadIdx.x; it0 < nit; it0 += 2 * blockDim.x) {
        float4 v[2][16];                           // 2 items x up to 16 splits in flight
  #pragma unroll
        for (int u = 0; u < 2; ++u) {
          const size_t off = (size_t)min(it0 + u * (int)blockDim.x, nit - 1) * 4;
  #pragma unroll
          for (int p = 0; p < 16; ++p)
            v[u][p] = p < a.S ? *reinterpret_cast<const float4*>(recv + p * slot + off) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
  #pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int it = it0 + u * blockDim.x;
          float4 acc = v[u][0];                    // fixed split order: deterministic
  #pragma unroll
          for (int p = 1; p < 16; ++p) { acc.x += v[u][p].x; acc.y += v[u][p].y; acc.z += v[u][p].z; acc.w += v[u][p].w; }
          if (it < nit) {
            const int c4 = it / kTileM, m = it % kTileM;
            float* o = red + (size_t)(4 * c4) * kTileM + m;
            o[0] = acc.x; o[kTileM] = acc.y; o[2 * kTileM] = acc.z; o[3 * kTileM] = acc.w;
          }
        }
      }
    }
  }
  KT(8);
  __syncthreads();
  KT(9);
  if (ncols > 0) {
    if (EPI == EPI_CELL) {
      // rows m = 4u + g (gate-interleaved): unit j = m0/4 + ul, 32 units per tile
      const int nit = 32 * ncols;
      // fold B operand: chunk q of 32 columns holds nc8 hi rows then nc8 lo rows (nc8 = 32, or the
      // last chunk's column count rounded to 8: a small chunk runs N = 2 nc8 MMAs)
      const int qlast = (ncols - 1) >> 5, nc8_last = min(32, ((ncols - 32 * qlast) + 7) & ~7);
      for (int it0 = threadIdx.x; it0 < nit; it0 += 2 * blockDim.x) {
        float4 gz[2], bb[2];
        float cp[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int it = min(it0 + u * (int)blockDim.x, nit - 1);
          const int ul = it % 32, c = it / 32;
          gz[u] = *reinterpret_cast<const float4*>(red + (size_t)c * kTileM + 4 * ul);
          bb[u] = s_bias[ul];
          if (a.gb) {                                     // (GEMM + per-row gate bias) + unit bias
            const float4 g2 = s_gb[it];
            gz[u].x += g2.x; gz[u].y += g2.y; gz[u].z += g2.z; gz[u].w += g2.w;
          }
          cp[u] = s_cg[it];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int it = it0 + u * blockDim.x;
          const int ul = it % 32, c = it / 32;
          const int r = n0 + c_own + c, j = m0 / 4 + ul;
          const float i_ = sigmf(gz[u].x + bb[u].x), f_ = sigmf(gz[u].y + bb[u].y),
                      g_ = tanhfast(gz[u].z + bb[u].z), o_ = sigmf(gz[u].w + bb[u].w);
          const float cn = f_ * cp[u] + i_ * g_;
          const float h = o_ * tanhfast(cn);
          if (a.woh && it < nit) {                                 // h (bf16 hi / lo) -> fold B operand
            const float hv = (r < a.n_valid && j < a.H) ? h : 0.f;
            const __nv_bfloat16 hh = __float2bfloat16_rn(hv), hl = __float2bfloat16_rn(hv - __bfloat162float(hh));
            const int nc8 = (c >> 5) == qlast ? nc8_last : 32;
            uint8_t* cb = s_hb + (size_t)(c >> 5) * 4096;
            *reinterpret_cast<__nv_bfloat16*>(cb + fold_sw64(c & 31, ul)) = hh;
            *reinterpret_cast<__nv_bfloat16*>(cb + fold_sw64(nc8 + (c & 31), ul)) = hl;
          }
          if (it >= nit || r >= a.n_valid || j >= a.H) continue;
#ifdef ONMT_KTRACE
          if (a.dbg == 2) { if (h == 12345.f) a.c_out[0] = cn; continue; }
          if (a.dbg == 3) { a.c_out[(size_t)r * a.H + j] = cn; continue; }
#endif
          a.c_out[(size_t)r * a.H + j] = cn;
          a.h_out[(size_t)r * a.H + j] = h;
#ifdef ONMT_KTRACE
          if (a.dbg == 1) continue;
#endif
          for (int d = 0; d < a.dst.n; ++d) store_x(a.dst.x[d], r, a.dst.col[d] + j, h);
        }
      }
      if (a.woh) {
        // W_out[:, units] h[units, my columns] -> woh_part[mt][row][o] with tcgen05: A = the
        // tile's [outputs x 32 units] slice, B = a chunk of h as [hi rows ; lo rows] (N = 2 nc8:
        // both planes in one MMA, the two column halves summed below); accumulators in TMEM
        // columns 256.. (the GEMM's use < 256); fixed order, deterministic
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // h stores -> MMA operand reads
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        const int mo_n = fold_mo(a.H) / kTileM;                    // output tiles (<= 4: H <= 512)
        const uint32_t fcol = tmem + 256u;
        for (int q = 0; q * 32 < ncols; ++q) {
          const int nc8 = q == qlast ? nc8_last : 32;
          if (threadIdx.x == 0) {
            if (q == 0) mbar_wait(wbar, 0);
            tc_fence_after();
            const uint32_t idesc = umma_idesc_bf16(kTileM, 2 * nc8);
            const uint32_t sa = smem_u32(woh_s), sb = smem_u32(s_hb + (size_t)q * 4096);
            for (int mo = 0; mo < mo_n; ++mo)
#pragma unroll
              for (int ks = 0; ks < 2; ++ks)
                tc_mma_bf16(fcol + (uint32_t)(mo * 64), umma_desc_sw64(sa + (uint32_t)mo * 8192u + (uint32_t)ks * 32u),
                            umma_desc_sw64(sb + (uint32_t)ks * 32u), idesc, (uint32_t)ks);
            tc_commit(fbar);
          }
          __syncwarp();
          mbar_wait(fbar, (uint32_t)(q & 1));
          tc_fence_after();
          // warp w: TMEM lane quarter w & 3 (outputs), output tiles w / 4, w / 4 + 2
          const int qd = warp & 3;
          for (int mo = warp >> 2; mo < mo_n; mo += 2) {
            const int o = mo * kTileM + qd * 32 + lane;
            const uint32_t trow = fcol + (uint32_t)(mo * 64) + ((uint32_t)(qd * 32) << 16);
#pragma unroll
            for (int cc = 0; cc < 32; cc += 8) {
              if (cc >= nc8) break;
              uint32_t hv[8], lv[8];
              tmem_ld8_nw(trow + cc, hv);
              tmem_ld8_nw(trow + nc8 + cc, lv);
              tmem_wait_ld();
              tmem_fence_regs(hv);
              tmem_fence_regs(lv);
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int c = q * 32 + cc + k;
                if (o < a.H && c < ncols)
                  __stcg(a.woh_part + ((size_t)mt * a.n_rows_pad + n0 + c_own + c) * a.H + o,
                         __uint_as_float(hv[k]) + __uint_as_float(lv[k]));
              }
            }
          }
          tc_fence_before();
          __syncthreads();                                        // (the next chunk reuses the columns)
          tc_fence_after();
        }
      }
    } else {
      for (int it = threadIdx.x; it < kTileM * ncols; it += blockDim.x) {
        const int m = it % kTileM, c = it / kTileM;
        const int r = n0 + c_own + c, j = m0 + m;
        if (r >= a.n_valid || j >= a.M) continue;
        const float h = tanhfast(red[(size_t)c * kTileM + m]);
        a.htilde[(size_t)r * a.M + j] = h;
        store_x(a.xg, r, j, h);
      }
    }
  }
  KT(6);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
  KT(7);
}

static size_t fused_smem_bytes(int n_group, int stages, int S, int NC, int fold_H, bool gb = false) {
  const size_t ring = (size_t)stages * (kTileM * 128 + 2 * (size_t)n_group * 128);
  const size_t recv = (size_t)(S + 1) * kTileM * NC * 4;
  const size_t fold = fold_H ? 1024 + fold_tile_bytes(fold_H) + (size_t)fold_chunks(NC) * 4096 : 0;
  const size_t gbb = gb ? 128 + 16 + (size_t)NC * 32 * 16 : 0;
  return 1024 + (ring > recv ? ring : recv) + 32 * 16 + (size_t)NC * 32 * 4 + (2 * stages + 4) * 8 + 16 + fold + gbb;
}

// Split S: the largest S <= 16 such that every split has >= 1 K block, the split's whole
// K-slice fits the shared-memory ring, and tiles * S <= #SMs (one co-resident wave: the
// tile counter wait needs every split resident).  1 CTA per SM (smem > half an SM).
static bool fill_common(FusedArgs& a, int n_rows_pad, int n_group, int n_valid, int k_blocks, int M, int m_tiles,
                        int num_sms, int fold_H = 0, bool gb = false) {
  a.n_rows_pad = n_rows_pad;
  a.n_group = n_group;
  a.n_valid = n_valid;
  a.k_blocks = k_blocks;
  const int tiles = m_tiles * (n_rows_pad / n_group);
  const size_t limit = 227 * 1024;
  int s_max = 16;
  if (const char* e = std::getenv("ONMT_FUSED_SMAX")) s_max = std::atoi(e);   // (tuning experiments)
  for (int S = s_max; S >= 1; --S) {
    const int kbps = (k_blocks + S - 1) / S;
    if ((k_blocks + kbps - 1) / kbps != S) continue;     // no empty split
    if (tiles * S > num_sms) continue;
    int NC = (n_group + S - 1) / S;
    NC = (NC + 3) / 4 * 4;
    // the split's whole K-slice resident if it fits, else a ring of >= 2 stages
    int stages = kbps;
    while (stages > 2 && fused_smem_bytes(n_group, stages, S, NC, fold_H, gb) > limit) --stages;
    const size_t sm = fused_smem_bytes(n_group, stages, S, NC, fold_H, gb);
    if (sm > limit) continue;
    a.S = S;
    a.NC = NC;
    a.kb_per_split = kbps;
    a.stages = stages;
    a.stack = 2 * n_group <= 256;
    if (const char* e = std::getenv("ONMT_FUSED_NOSTACK")) a.stack = a.stack && !std::atoi(e);   // (A/B runs)
    int tc = 32;
    while (tc < (a.stack ? 2 * n_group : n_group)) tc <<= 1;
    if (fold_H) tc = 512;                                  // (fold accumulators at columns 256..)
    a.tmem_cols = tc;
    a.M = M;
    return true;
  }
  return false;
}

template <int EPI>
static cudaError_t launch_fused(const CUtensorMap& tmW, const CUtensorMap& tmX, const FusedArgs& a, int tiles,
                                cudaStream_t st) {
  // at least 116 KB of shared memory: never two CTAs of this kernel on one SM (the tile wait
  // relies on one CTA per SM with grid <= #SMs)
  size_t smem = fused_smem_bytes(a.n_group, a.stages, a.S, a.NC, a.woh ? a.H : 0, a.gb != nullptr);
  if (smem < 116 * 1024) smem = 116 * 1024;
  auto fn = a.stages < a.kb_per_split ? tc_gemm_fused_kernel<EPI, 1> : tc_gemm_fused_kernel<EPI, 0>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(fn, dim3(tiles * a.S), dim3(256), smem, st, tmW, tmX, a);
}

// scratch floats a fused call needs (0 = no fused configuration fits)
size_t fused_scratch_floats(int m_pad, int n_rows_pad, int n_group, int k_blocks, int num_sms) {
  FusedArgs a{};
  const int m_tiles = m_pad / kTileM;
  if (!fill_common(a, n_rows_pad, n_group, n_group, k_blocks, 1, m_tiles, num_sms)) return 0;
  return (size_t)m_tiles * (n_rows_pad / n_group) * a.S * n_group * kTileM;
}

// decoder LSTM layer: gates = W [x; h] (+ bias), cell update, h written to dst operands
int g_fused_dbg = 0;
cudaError_t tc_gemm_cell(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                         int n_valid, int k_blocks, const float* bias, const float* cg, float* c_out, float* h_out,
                         int H, CellDst dst, float* scratch, unsigned int* counters, int num_sms, StepCtl ctl,
                         cudaStream_t st, const __nv_bfloat16* woh, float* woh_part, const float* gb, int gb_ld) {
  FusedArgs a{};
  a.dbg = g_fused_dbg;
  if (!fill_common(a, n_rows_pad, n_group, n_valid, k_blocks, 4 * H, m_pad / kTileM, num_sms, woh ? H : 0,
                   gb != nullptr))
    return cudaErrorInvalidConfiguration;
  a.gb = gb;
  a.gb_ld = gb_ld;
  a.woh = woh;
  a.woh_part = woh_part;
  if (const char* e = std::getenv("ONMT_FUSED_DBG")) a.dbg = std::atoi(e);   // (ablations; wrong results)
  a.scratch = scratch;
  a.counters = counters;
  a.bias = reinterpret_cast<const float4*>(bias);
  a.cg = cg;
  a.c_out = c_out;
  a.h_out = h_out;
  a.H = H;
  a.dst = dst;
  a.ctl = ctl;
  return launch_fused<EPI_CELL>(tmW, tmX, a, m_pad / kTileM * (n_rows_pad / n_group), st);
}

// attentional vector: h~ = tanh(W_out [c; h])
cudaError_t tc_gemm_tanh(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                         int n_valid, int k_blocks, int H, float* htilde, XOut xg, float* scratch,
                         unsigned int* counters, int num_sms, StepCtl ctl, cudaStream_t st) {
  FusedArgs a{};
  if (!fill_common(a, n_rows_pad, n_group, n_valid, k_blocks, H, m_pad / kTileM, num_sms))
    return cudaErrorInvalidConfiguration;
  a.scratch = scratch;
  a.counters = counters;
  a.htilde = htilde;
  a.xg = xg;
  a.ctl = ctl;
  return launch_fused<EPI_TANH>(tmW, tmX, a, m_pad / kTileM * (n_rows_pad / n_group), st);
}

// does the top-layer cell kernel with the folded W_out share fit (shared memory, co-residency)?
bool tc_cell_fold_fits(int m_pad, int n_rows_pad, int n_group, int k_blocks, int H, int num_sms, bool gb) {
  FusedArgs a{};
  if (fold_mo(H) > 512 || n_group > 256) return false;   // (fold accumulators: TMEM columns 256..511)
  return fill_common(a, n_rows_pad, n_group, n_group, k_blocks, 4 * H, m_pad / kTileM, num_sms, H, gb);
}
// does a (non-top) cell kernel with per-row gate biases fit?
bool tc_cell_fits(int m_pad, int n_rows_pad, int n_group, int k_blocks, int H, int num_sms, bool gb) {
  FusedArgs a{};
  return fill_common(a, n_rows_pad, n_group, n_group, k_blocks, 4 * H, m_pad / kTileM, num_sms, 0, gb);
}

// split the fused kernels use for a shape (tests / DESIGN numbers; 0 = unfused)
int fused_split(int n_group, int n_rows_pad, int k_blocks, int m_tiles, int num_sms) {
  FusedArgs a{};
  return fill_common(a, n_rows_pad, n_group, n_group, k_blocks, 1, m_tiles, num_sms) ? a.S : 0;
}

}  // namespace onmt
