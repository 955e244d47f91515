// One persistent kernel for the tail of a decoder step (SURVEY §8(a) A9 + A10 + A5):
//
//   phase A  generator + log-softmax statistics + per-CTA top-K (PAPER.md P118-119):
//            z = W_gen h~ + b for every vocabulary id, logits never written to HBM.
//
// Grid = groups x C CTAs, one per SM.  Phase A is "K-outer": CTA (g, i) owns a contiguous run of nt
// vocabulary tiles (128 rows each) of N-group g and keeps all nt accumulators in TMEM
// (nt * n_group <= 512 columns), so every activation K-block (hi/lo planes, the MMA B
// operand) crosses L2 -> SM once per CTA instead of once per tile.
//   warp 0   TMA producer: per K-block the hi/lo activation tiles + nt weight tiles
//   warp 1   TMEM allocator + single-thread tcgen05.mma issuer (hi and lo into one fp32
//            accumulator per tile)
//   warps 2+ epilogue: TMEM -> registers (+bias) -> transposed shared staging (double
//            buffered across tiles) -> two threads per hypothesis row keep a running
//            (max, sum exp, top-K) over the CTA's vocabulary; one partial per (CTA, row).
#include <math_constants.h>

#include <cstdio>
#include <cstdlib>

#include "beam_device.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

constexpr int kGsStageWarps = 4;               // TMEM -> smem stagers (one per TMEM lane quarter)
constexpr int kGsScanWarps = 10;                // scanners (2 threads x 160 hypothesis rows)
constexpr int kGsThreads = 32 * (2 + kGsStageWarps + kGsScanWarps);
constexpr int kGsSLD = 136;                     // staging row stride (floats; = 8 mod 32 banks: with the
                                                // scanners' interleaved groups a quarter warp's float4
                                                // reads hit distinct banks)
constexpr int kGsMaxCh = 10;                    // 32-row staging chunks per buffer (n_group <= 320)

struct GenStepArgs {
  int n_rows_pad, n_group, groups, k_blocks, n_vt, C, nt_max, stages;
  int P;                                        // threads per hypothesis row in the scan (1 or 2)
  const float* bias;
  int V, K, R, rows_pad;
  float2* ms;                                   // partials [rows_pad][C]
  float* tz;                                    // [rows_pad][C][K]
  int* ti;
  float* row_lse;                               // [R]
  float* row_z;                                 // [R][K]
  int* row_i;
  int t;
  unsigned int* thr;                            // [2][rows_pad] shared top-K thresholds (ordered
                                                // uint keys; buffer t & 1, the other one is reset),
                                                // then [2][rows_pad][16] running-max slots
  StepCtl ctl;
  int dbg;                                      // microbenchmark ablations (ONMT_KTRACE builds)
  int ovl;                                      // 1: staging has its own smem and every tile of the
                                                //    CTA its own TMEM columns, so batch b+1's MMAs
                                                //    overlap batch b's epilogue (batches of nt_max)
  int nbuf;                                     // staging buffers (1 or 2)
  int srows_alloc;                              // staging rows per buffer (min(n_group, R))
  // gate tiles (the recurrent halves of the NEXT step's LSTM gates): 128 rows
  // of Wg (tensor map tmWg) over K blocks [q * gkbh, (q + 1) * gkbh) of the same activation
  // operand, q = tile / gt_per_q; the accumulator goes to gout[q][row][tile % gt_per_q * 128 + m]
  // (row stride gld floats).  One gate tile per CTA with the smaller vocabulary share (appended
  // after its vocabulary tiles: no scan, a plain store).
  int n_gt, gt_per_q, gkbh, gld;
  float* gout;
  // vocabulary-parallel ranks (VpOut): this launch runs CTAs [ci0, ci0 + C) of a Ct-CTA split
  int ci0, Ct;
  VpOut vp;
};

// TMEM columns per accumulator (n_group rounded to 32)
__host__ __device__ constexpr int gs_tstride(int n_group) { return (n_group + 31) & ~31; }

__device__ __forceinline__ float gs_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void gs_named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }


// order-preserving float <-> uint keys (atomicMax on the key = max on the float)
__device__ __forceinline__ unsigned int f2key(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned int k) {
  return k == 0u ? -INFINITY : __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// sorted (z desc, id asc) insertion into a register list (branch-free network)
template <int KMAX>
__device__ __forceinline__ void gs_insert(float (&tz)[KMAX], int (&ti)[KMAX], float x, int xi) {
  bool gt[KMAX];
#pragma unroll
  for (int q = 0; q < KMAX; ++q) gt[q] = better(x, xi, tz[q], ti[q]);
#pragma unroll
  for (int q = KMAX - 1; q >= 1; --q) {
    const float nz = gt[q - 1] ? tz[q - 1] : x;
    const int ni = gt[q - 1] ? ti[q - 1] : xi;
    tz[q] = gt[q] ? nz : tz[q];
    ti[q] = gt[q] ? ni : ti[q];
  }
  tz[0] = gt[0] ? x : tz[0];
  ti[0] = gt[0] ? xi : ti[0];
}

// same list, for the scan: every list entry has a smaller id than x (each thread scans its
// vocabulary rows in increasing order), so "better" reduces to a value compare
template <int KMAX>
__device__ __forceinline__ void gs_insert_scan(float (&tz)[KMAX], int (&ti)[KMAX], float x, int xi) {
  bool gt[KMAX];
#pragma unroll
  for (int q = 0; q < KMAX; ++q) gt[q] = x > tz[q];
#pragma unroll
  for (int q = KMAX - 1; q >= 1; --q) {
    tz[q] = gt[q] ? (gt[q - 1] ? tz[q - 1] : x) : tz[q];
    ti[q] = gt[q] ? (gt[q - 1] ? ti[q - 1] : xi) : ti[q];
  }
  tz[0] = gt[0] ? x : tz[0];
  ti[0] = gt[0] ? xi : ti[0];
}

// packed fp32 pairs (FFMA2 / FADD2): same rounding as two scalar operations
__device__ __forceinline__ unsigned long long gs_pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void gs_upk(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long gs_ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long gs_fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int KMAX>
__global__ void __launch_bounds__(kGsThreads, 1)
gen_step_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmWg, GenStepArgs a) {
  KT(0);
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t a_bytes = kTileM * 128, b_bytes = a.n_group * 128;
  const uint32_t stage_bytes = 2 * b_bytes + a.nt_max * a_bytes;
  const size_t ring = (size_t)a.stages * stage_bytes;
  const size_t stg_bytes = (size_t)a.nbuf * a.srows_alloc * kGsSLD * 4;
  const size_t body = a.ovl ? ring + stg_bytes : (ring > stg_bytes ? ring : stg_bytes);
  float* stg = reinterpret_cast<float*>(a.ovl ? smem + ring : smem);  // nbuf x [srows][132] (overlays the ring unless ovl)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + body);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 1;
  uint64_t* sfull = tempty + 1;                                    // [2][kGsMaxCh] staged chunk filled (stagers)
  uint64_t* sempty = sfull + 2 * kGsMaxCh;                         // [2][kGsMaxCh] staged chunk scanned (scanners)
  uint64_t* sdone = sempty + 2 * kGsMaxCh;                         // every scanner warp finished a batch
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sdone + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = blockIdx.x / a.C, ci = a.ci0 + blockIdx.x % a.C;   // (global CTA index of the split)
  const int tb = ci * a.n_vt / a.Ct, te = (ci + 1) * a.n_vt / a.Ct;  // (n_vt * Ct < 2^31)
  const int n0 = grp * a.n_group;
  // local tiles i = 0 .. ntot-1: vocabulary tiles tb + i (i < nv), then the CTA's gate tile (if
  // any).  Batch bt = local tiles [bt * nt_max, min(ntot, (bt + 1) * nt_max)), all accumulators of
  // a batch in TMEM at once (K-outer over the union of its tiles' K-block ranges).  ovl: every
  // tile its own TMEM columns, so batch bt + 1's MMAs overlap batch bt's epilogue.
  const int nv = te - tb;
  int gi = -1;                                                     // my gate tile
  if (a.n_gt > 0 && nv == a.n_vt / a.Ct) {                         // (gate tiles: single rank, Ct == C)
    // CTAs of my group before me with the smaller share: tb = ci * floor + (#larger shares before me)
    const int idx = ci - (tb - ci * (a.n_vt / a.Ct));
    if (idx < a.n_gt) gi = idx;
  }
  const int ntot = nv + (gi >= 0 ? 1 : 0);
  const int nbatch = (ntot + a.nt_max - 1) / a.nt_max;
  auto bfirst = [&](int bt) { return bt * a.nt_max; };
  auto bsize = [&](int bt) { return min(a.nt_max, ntot - bfirst(bt)); };
  // accumulators start on 32-column boundaries: the stagers' tcgen05.ld.32x32b.x32 reads
  // must not straddle (a 144-row group at column 144 read wrong data)
  const int tstride = gs_tstride(a.n_group);
  auto tcol = [&](int bt, int j) { return (uint32_t)((a.ovl ? bt * a.nt_max + j : j) * tstride); };
  auto is_gate = [&](int i) { return i >= nv; };
  const int g_lo = gi >= 0 ? (gi / a.gt_per_q) * a.gkbh : 0, g_hi = g_lo + a.gkbh;
  // per-batch tile table, computed once per batch (the single producer / MMA threads must not
  // redo index arithmetic per K block): K-block range, weight row and map of every tile slot
  struct Bat {
    int klo, khi;
    int lo[4], hi[4], row[4];
    bool gate[4];
  };
  auto make_bat = [&](int bt) {
    Bat B;
    B.klo = 1 << 30;
    B.khi = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = bfirst(bt) + j;
      const bool v = j < bsize(bt), g = is_gate(i);
      B.gate[j] = g;
      B.lo[j] = v ? (g ? g_lo : 0) : 0;
      B.hi[j] = v ? (g ? g_hi : a.k_blocks) : 0;
      B.row[j] = (g ? gi : tb + i) * kTileM;
      if (v) { B.klo = min(B.klo, B.lo[j]); B.khi = max(B.khi, B.hi[j]); }
    }
    return B;
  };
  auto cover_mask = [](const Bat& B, int kb) {
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) m |= (kb >= B.lo[j] && kb < B.hi[j]) ? (1u << j) : 0u;
    return m;
  };
  // staging is split into 32-hypothesis-row chunks with their own full/empty barriers: the
  // scanners of a chunk start as soon as it is staged and the stagers refill a chunk as soon
  // as its scanners are done (instead of whole-tile hand-offs)
  const int srows = min(a.n_group, a.R - n0);                      // staged hypothesis rows (valid ones)
  // TMEM columns staged: whole 32-column x32 loads (columns past srows are garbage; their stores
  // are predicated off and the scanners skip those rows).  A half-chunk tcgen05.ld .x16 path was
  // removed: rows of such chunks came out wrong intermittently in multi-group launches.
  const int ncols = srows > 0 ? min((srows + 31) & ~31, tstride) : 0;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    if (gi >= 0) tma_prefetch_desc(&tmWg);
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, kGsStageWarps);
    // only scanner warps with rows to scan arrive on sdone: an idle warp (rows past ncols: a
    // ragged last row group, or P = 1) runs through every batch at once and its arrivals would
    // complete later batches' phases before the active warps finished (the producer then
    // reloaded the ring under the staged tile they were still scanning)
    const int n_act = min(kGsScanWarps, (ncols * a.P + 31) >> 5);   // (warp sw scans rows from 32 sw / P; P | 32)
    mbar_init(sdone, n_act > 0 ? n_act : 1);
  }
  if (threadIdx.x >= 32 && threadIdx.x < 32 + 2 * kGsMaxCh) {      // chunk barriers (warp 1)
    const int i = threadIdx.x - 32, k = i % kGsMaxCh;
    int cnt = 0;                                                   // scanner warps of chunk k
    for (int sw = 0; sw < kGsScanWarps; ++sw) {
      const int r0 = 32 * sw / a.P;
      cnt += (r0 < ncols && (r0 >> 5) == k) ? 1 : 0;
    }
    mbar_init(&sfull[i], kGsStageWarps);
    mbar_init(&sempty[i], cnt > 0 ? cnt : 1);
  }
  if (threadIdx.x == 0 || threadIdx.x == 32) fence_mbar_init();
  // the weight tiles of the first ring stages are constants of the translation: their TMA loads
  // are issued before griddepcontrol.wait (the activation halves follow after it)
  auto load_act = [&](int it, int kb) {
    uint8_t* st = smem + (size_t)(it % a.stages) * stage_bytes;
    tma_load_2d(st, &tmX, kb * kBK, n0, &full[it % a.stages]);
    tma_load_2d(st + b_bytes, &tmX, kb * kBK, a.n_rows_pad + n0, &full[it % a.stages]);
  };
  // weight tiles of batch B that cover kb (mask cov) -> stage slot j (their position); gate
  // weights are stored compactly (K block kb - lo of the tile's block)
  auto load_w = [&](const Bat& B, unsigned cov, int kb, uint8_t* st, uint64_t* bar) {
    mbar_arrive_expect_tx(bar, 2 * b_bytes + (uint32_t)__popc(cov) * a_bytes);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((cov >> j) & 1u)
        tma_load_2d(st + 2 * b_bytes + j * a_bytes, B.gate[j] ? &tmWg : &tmW, (kb - B.lo[j]) * kBK, B.row[j], bar);
  };
  // the weight tiles of the first ring stages are constants of the translation: their TMA loads
  // are issued before griddepcontrol.wait (the activation halves follow after it)
  int npre = 0;
  if (threadIdx.x == 0 && nbatch > 0) {
    const Bat B0 = make_bat(0);
    for (int kb = B0.klo; kb < B0.khi && npre < a.stages; ++kb) {
      const unsigned cov = cover_mask(B0, kb);
      if (!cov) continue;
      load_w(B0, cov, kb, smem + (size_t)npre * stage_bytes, &full[npre]);
      ++npre;
    }
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  pdl_wait();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (a.thr && blockIdx.x == 0) {                                  // next step's thresholds start empty
    for (int i = threadIdx.x; i < a.rows_pad; i += blockDim.x) a.thr[(size_t)((a.t + 1) & 1) * a.rows_pad + i] = 0u;
    uint4* sl = reinterpret_cast<uint4*>(a.thr + (size_t)2 * a.rows_pad + (size_t)((a.t + 1) & 1) * a.rows_pad * 16);
    for (int i = threadIdx.x; i < a.rows_pad * 4; i += blockDim.x) sl[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (all_done(a.ctl)) {                                           // uniform over the grid
    if (threadIdx.x == 0 && npre > 0) {                              // (no TMA may land after exit)
      const Bat B0 = make_bat(0);
      int it = 0;
      for (int kb = B0.klo; kb < B0.khi && it < npre; ++kb)
        if (cover_mask(B0, kb)) { load_act(it, kb); mbar_wait(&full[it], 0); ++it; }
    }
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
    return;
  }
  KT(1);

  // ================================================================ phase A
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int bt = 0; bt < nbatch; ++bt) {
        if (bt > 0 && !a.ovl) {                                   // the staging overlays the ring: the
          mbar_wait(tempty, (bt - 1) & 1);                         // previous batch is staged AND scanned
          mbar_wait(sdone, (bt - 1) & 1);                          // before its stages are reloaded
        }
        const Bat B = make_bat(bt);
        for (int kb = B.klo; kb < B.khi; ++kb) {
          const unsigned cov = cover_mask(B, kb);
          if (!cov) continue;
          const int s = it % a.stages;
          if (it >= a.stages) mbar_wait(&empty[s], ((it / a.stages) & 1) ^ 1);
          if (it >= npre) load_w(B, cov, kb, smem + (size_t)s * stage_bytes, &full[s]);   // (else: in flight)
          load_act(it, kb);
          ++it;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(kTileM, a.n_group);
      int it = 0;
      for (int bt = 0; bt < nbatch; ++bt) {
        const Bat B = make_bat(bt);
        const uint32_t tc0 = tmem + tcol(bt, 0);
        for (int kb = B.klo; kb < B.khi; ++kb) {
          const unsigned cov = cover_mask(B, kb);
          if (!cov) continue;
          const int s = it % a.stages;
          mbar_wait(&full[s], (it / a.stages) & 1);
          tc_fence_after();
          KTX(7, it == 0);
          const uint32_t sb = smem_u32(smem + (size_t)s * stage_bytes);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (!((cov >> j) & 1u)) continue;
            const uint32_t sa = sb + 2 * b_bytes + j * a_bytes;
            const uint32_t d = tc0 + (uint32_t)(j * tstride);
            const uint32_t acc0 = kb == B.lo[j] ? 0u : 1u;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              const uint64_t da = umma_desc_sw128(sa + kk * 32);
              tc_mma_bf16(d, da, umma_desc_sw128(sb + kk * 32), idesc, kk == 0 ? acc0 : 1u);
              tc_mma_bf16(d, da, umma_desc_sw128(sb + b_bytes + kk * 32), idesc, 1u);
            }
          }
          tc_commit(&empty[s]);
          ++it;
        }
        tc_commit(tfull);
      }
    }
    __syncwarp();
  } else if (warp < 2 + kGsStageWarps) {
    // ---------------- stagers: accumulator j -> (+bias) -> smem buf[j & 1][c][v] (transposed)
    const int q = warp & 3;                                        // TMEM lane quarter of this warp
    const int vr = q * 32 + lane;                                  // vocabulary row this thread stages
    for (int bt = 0; bt < nbatch; ++bt) {
      const int t0 = bfirst(bt);
      const int nt = bsize(bt);
      float bias_r[4];                                             // bias of my vocabulary row, loaded
#pragma unroll                                                     // while the MMAs run
      for (int j = 0; j < 4; ++j) {
        const int vid = (tb + t0 + j) * kTileM + vr;
        bias_r[j] = (j < nt && !is_gate(t0 + j) && vid < a.V) ? __ldg(&a.bias[vid]) : -INFINITY;
      }
      mbar_wait(tfull, bt & 1);
      tc_fence_after();
      KTX(2, threadIdx.x == 64 && bt == 0);
      for (int j = 0; j < nt; ++j) {
        if (is_gate(t0 + j)) {
          // gate tile: accumulator row vr (gate row of the tile) -> gout, 32 hypothesis rows per load
          const uint32_t trow = tmem + tcol(bt, j) + ((uint32_t)(q * 32) << 16);
          const int qb = gi / a.gt_per_q, col = (gi % a.gt_per_q) * kTileM + vr;
          float* go = a.gout + ((size_t)qb * a.rows_pad + n0) * a.gld + col;
          for (int c0 = 0; c0 < ncols; c0 += 32) {
            uint32_t r[32];
            tmem_ld32_nw(trow + c0, r);                          // (ncols: a multiple of 32)
            tmem_wait_ld();
            tmem_fence_regs(r);
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (c0 + k < srows) __stcg(go + (size_t)(c0 + k) * a.gld, __uint_as_float(r[k]));
          }
          continue;
        }
        const int jj = t0 + j;                                     // staging sequence number
        const int buf = jj % a.nbuf, use = jj / a.nbuf;
        KTX(6, threadIdx.x == 64 && jj == 2);
        {
          const float bias = j == 0 ? bias_r[0] : j == 1 ? bias_r[1] : j == 2 ? bias_r[2] : bias_r[3];
          const uint32_t trow = tmem + tcol(bt, j) + ((uint32_t)(q * 32) << 16);
          float* dst = stg + (size_t)buf * a.srows_alloc * kGsSLD + vr;
          // 32-column chunks, software-pipelined: the load of chunk i+1 is in flight while
          // chunk i is stored
          auto issue = [&](int c0, uint32_t* r) {
            tmem_ld32_nw(trow + c0, r);                          // (ncols: a multiple of 32)
          };
          auto put = [&](int c0, uint32_t* r) {                    // c0: a multiple of 32 (one chunk)
            const int ch = buf * kGsMaxCh + (c0 >> 5);
            if (use > 0) mbar_wait(&sempty[ch], (use - 1) & 1);     // its scanners are done with it
            float* d = dst + (size_t)c0 * kGsSLD;
            if (c0 + 32 <= srows) {                                // whole chunk: immediate offsets
#pragma unroll
              for (int k = 0; k < 32; ++k) d[k * kGsSLD] = __uint_as_float(r[k]) + bias;
            } else {
#pragma unroll
              for (int k = 0; k < 32; ++k)
                if (c0 + k < srows) d[k * kGsSLD] = __uint_as_float(r[k]) + bias;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&sfull[ch]);
          };
          uint32_t ra[32], rb[32];
          if (ncols > 0) {
            issue(0, ra);
            tmem_wait_ld();
            tmem_fence_regs(ra);
          }
          for (int c0 = 0; c0 < ncols; c0 += 64) {
            if (c0 + 32 < ncols) issue(c0 + 32, rb);
            put(c0, ra);
            tmem_wait_ld();
            tmem_fence_regs(rb);
            if (c0 + 32 >= ncols) break;
            if (c0 + 64 < ncols) issue(c0 + 64, ra);
            put(c0 + 32, rb);
            tmem_wait_ld();
            tmem_fence_regs(ra);
          }
        }
        KTX(10, threadIdx.x == 64 && bt == 0 && j == 0);
      }
      tc_fence_before();                                           // batch's accumulators drained
      // (ring overlay: the staging stores - generic proxy - must be ordered before the next
      //  batch's TMA writes to the same bytes - async proxy - that this arrival releases)
      if (!a.ovl) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_local(tempty);
    }
  } else {
    // ---------------- scanners: P threads per hypothesis row keep (max, sum exp, top-K)
    const int et = threadIdx.x - 32 * (2 + kGsStageWarps);         // 0 .. 32*kGsScanWarps-1
    const int P = a.P;
    const int c = et / P, part = et % P;                           // hypothesis row (column) and part
    const int nv = kTileM / P;                                     // vocabulary rows scanned per tile
    // logits per register chunk: 64 (16 groups of 4); 32 for wide beams, whose longer top-K
    // lists would otherwise spill the scan state to local memory
    constexpr int ZC = KMAX <= 5 ? 64 : 32, NG = ZC / 4;
    const bool row_ok = c < a.n_group && n0 + c < a.R;
    const int wrow0 = 32 * (warp - 2 - kGsStageWarps) / P;         // first row of this warp
    const bool wact = wrow0 < ncols;                               // its chunk is staged at all
    const int wch = wrow0 >> 5;
    constexpr float L2E = 1.4426950408889634f;
    float run_m = -INFINITY, run_s = 0.f;
    float tz[KMAX];
    int ti[KMAX];
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {                               // sentinels: effective length K
      const bool sent = i < KMAX - a.K;
      tz[i] = sent ? INFINITY : -INFINITY;
      ti[i] = sent ? -1 : 0x7fffffff;
    }
    int jj = 0;
    for (int bt = 0; bt < nbatch; ++bt) {
      const int t0 = tb + bfirst(bt);                              // (vocabulary tile of local index bfirst)
      const int nt = bsize(bt);
      for (int j = 0; j < nt; ++j, ++jj) {
        if (is_gate(bfirst(bt) + j)) break;                        // (the gate tile comes last: no scan)
        const int buf = jj % a.nbuf, use = jj / a.nbuf;
        // the row's shared threshold: the largest list tail any scanner of any CTA published
        // so far - a K-th best of a subset of the row, so a lower bound of the row's K-th best
        // logit; values below it cannot reach the row's top-K.  Loaded before
        // the wait for the staged tile so the L2 round trip overlaps it.
        // (step 1 does not read: its buffer may still hold the previous call's last step)
        // A second bound: slot s of the row holds the running maximum of the scanners of the
        // CTAs ci with ci % K == s - disjoint element sets, so the K slots are K distinct
        // elements and their minimum is a lower bound of the row's K-th best (an empty slot
        // reads as -inf).  It is far tighter than the largest list tail once every CTA has
        // scanned one tile.
        float gth = -INFINITY;
        const unsigned int* slot = a.thr + (size_t)2 * a.rows_pad + ((size_t)(a.t & 1) * a.rows_pad + n0 + c) * 16;
        if (row_ok && a.thr && a.t != 1
#ifdef ONMT_KTRACE
            && a.dbg != 5
#endif
        ) {
          unsigned int kmin = 0xffffffffu;
#pragma unroll
          for (int q = 0; q < (KMAX + 3) / 4; ++q) {
            const uint4 v = __ldcg(reinterpret_cast<const uint4*>(slot) + q);
            if (4 * q < a.K) kmin = min(kmin, v.x);
            if (4 * q + 1 < a.K) kmin = min(kmin, v.y);
            if (4 * q + 2 < a.K) kmin = min(kmin, v.z);
            if (4 * q + 3 < a.K) kmin = min(kmin, v.w);
          }
          gth = fmaxf(key2f(__ldcg(a.thr + (size_t)(a.t & 1) * a.rows_pad + n0 + c)), key2f(kmin));
        }
        if (wact) mbar_wait(&sfull[buf * kGsMaxCh + wch], use & 1);
        KTX(4, et == 0 && jj == 0);
#ifdef ONMT_KTRACE
        if (a.dbg == 2) { __syncwarp(); if (wact && lane == 0) mbar_arrive_local(&sempty[buf * kGsMaxCh + wch]); continue; }
#endif
        if (row_ok) {
          // part p of the row owns the tile's float4 groups p, p + P, p + 2P, ... (interleaved, ids
          // increasing along the scan); chunk u0 / 64 covers 16 of them
          const float* col = stg + (size_t)buf * a.srows_alloc * kGsSLD + (size_t)c * kGsSLD + 4 * part;
          const int vbase = (t0 + j) * kTileM + 4 * part;
          for (int u0 = 0; u0 < nv; u0 += ZC) {                    // ZC logits per chunk, in registers
            float z[ZC];
#pragma unroll
            for (int k = 0; k < NG; ++k) {
              const float4 w = *reinterpret_cast<const float4*>(col + P * (u0 + 4 * k));
              z[4 * k] = w.x; z[4 * k + 1] = w.y; z[4 * k + 2] = w.z; z[4 * k + 3] = w.w;
            }
            float g[NG];                                           // group maxima (groups of 4)
#pragma unroll
            for (int k = 0; k < NG; ++k) g[k] = fmaxf(fmaxf(z[4 * k], z[4 * k + 1]), fmaxf(z[4 * k + 2], z[4 * k + 3]));
            float cmax = g[0];
#pragma unroll
            for (int k = 1; k < NG; ++k) cmax = fmaxf(cmax, g[k]);
            const float mn = fmaxf(run_m, cmax);
#ifdef ONMT_KTRACE
            if (a.dbg == 4) { run_m = mn; } else
#endif
            if (mn != -INFINITY) {
              const float mo = mn * L2E;
              // s0..s3 accumulate z[k], z[k+1], z[k+2], z[k+3] as packed pairs (FFMA2 / FADD2)
              const unsigned long long l2 = gs_pk(L2E, L2E), mo2 = gs_pk(-mo, -mo);
              unsigned long long s01 = gs_pk(0.f, 0.f), s23 = gs_pk(0.f, 0.f);
#pragma unroll
              for (int k = 0; k < ZC; k += 4) {
                float e0, e1, e2, e3;
                gs_upk(gs_ffma2(gs_pk(z[k], z[k + 1]), l2, mo2), e0, e1);
                gs_upk(gs_ffma2(gs_pk(z[k + 2], z[k + 3]), l2, mo2), e2, e3);
                s01 = gs_fadd2(s01, gs_pk(gs_ex2(e0), gs_ex2(e1)));
                s23 = gs_fadd2(s23, gs_pk(gs_ex2(e2), gs_ex2(e3)));
              }
              float s0, s1, s2, s3;
              gs_upk(s01, s0, s1);
              gs_upk(s23, s2, s3);
              run_s = (run_m == -INFINITY ? 0.f : run_s * gs_ex2((run_m - mn) * L2E)) + ((s0 + s1) + (s2 + s3));
              run_m = mn;
            }
#ifdef ONMT_KTRACE
            if (a.dbg == 3) continue;
#endif
            // top-K.  Candidates: z > list tail, and z >= the K-th largest group maximum of
            // this chunk (a lower bound of the chunk's K-th value - it is the K-th largest of
            // a subset - so nothing below it can enter).  The bound matters on the first
            // chunks, when the list is still cold.  Ids increase along the scan, so a value
            // compare decides every insertion (a tie never displaces an earlier id).
            const float th = fmaxf(tz[KMAX - 1], gth);
            if (cmax >= th && cmax > tz[KMAX - 1]) {
              if (tz[KMAX - 1] == -INFINITY) {
                // cold list: extract the chunk's K best exactly - K rounds of (largest group
                // maximum, its first element, the group's maximum without it) - uniform work
                // instead of inserting every element of every group above the K-th group max
                float gg[NG];
#pragma unroll
                for (int k = 0; k < NG; ++k) gg[k] = g[k];
                unsigned long long rm = 0ull;                      // extracted: bit 4 * group + element
#pragma unroll
                for (int rnd = 0; rnd < KMAX; ++rnd) {
                  if (rnd < a.K) {
                    float mx = gg[0];
#pragma unroll
                    for (int k = 1; k < NG; ++k) mx = fmaxf(mx, gg[k]);
                    if (mx != -INFINITY) {
                      int sel = NG - 1;
#pragma unroll
                      for (int k = NG - 2; k >= 0; --k) sel = gg[k] == mx ? k : sel;
                      const float4 w = *reinterpret_cast<const float4*>(col + P * (u0 + 4 * sel));
                      const unsigned gone = (unsigned)(rm >> (4 * sel)) & 15u;
                      const float v0 = (gone & 1u) ? -INFINITY : w.x, v1 = (gone & 2u) ? -INFINITY : w.y;
                      const float v2 = (gone & 4u) ? -INFINITY : w.z, v3 = (gone & 8u) ? -INFINITY : w.w;
                      const int e = v0 == mx ? 0 : v1 == mx ? 1 : v2 == mx ? 2 : 3;
                      gs_insert_scan<KMAX>(tz, ti, mx, vbase + P * (u0 + 4 * sel) + e);
                      rm |= 1ull << (4 * sel + e);
                      const float nm = fmaxf(fmaxf(e == 0 ? -INFINITY : v0, e == 1 ? -INFINITY : v1),
                                             fmaxf(e == 2 ? -INFINITY : v2, e == 3 ? -INFINITY : v3));
#pragma unroll
                      for (int k = 0; k < NG; ++k) gg[k] = k == sel ? nm : gg[k];
                    }
                  }
                }
              } else {
                unsigned gm = 0;                                   // groups holding a candidate
#pragma unroll
                for (int k = 0; k < NG; ++k) gm |= (g[k] >= th) ? (1u << k) : 0u;
                while (gm) {                                       // candidates in id order
                  const int gi = __ffs(gm) - 1;
                  gm &= gm - 1;
                  const float4 w = *reinterpret_cast<const float4*>(col + P * (u0 + 4 * gi));
                  const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    if (wv[e] >= th && wv[e] > tz[KMAX - 1]) gs_insert_scan<KMAX>(tz, ti, wv[e], vbase + P * (u0 + 4 * gi) + e);
                }
              }
            }
          }
        }
#ifdef ONMT_KTRACE
        if (a.dbg != 6)
#endif
        if (row_ok && a.thr) {                                     // publish my list tail and running max
          if (tz[KMAX - 1] != -INFINITY) atomicMax(a.thr + (size_t)(a.t & 1) * a.rows_pad + n0 + c, f2key(tz[KMAX - 1]));
          if (run_m != -INFINITY) atomicMax(const_cast<unsigned int*>(slot) + ci % a.K, f2key(run_m));
        }
        __syncwarp();
        if (wact && lane == 0) mbar_arrive_local(&sempty[buf * kGsMaxCh + wch]);
        KTX(5, et == 0 && jj == 0);
        KTX(11, et == 0 && jj == 1);
      }
      if (!a.ovl) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // (reads before the reload)
      __syncwarp();
      if (lane == 0 && (wact || (ncols == 0 && warp == 2 + kGsStageWarps)))
        mbar_arrive_local(sdone);                                  // (ring overlay: batch bt scanned)
    }
    KTX(8, et == 0);
    // ---- combine the P parts of a row (adjacent lanes, butterfly) and write the CTA's partial
    for (int o = 1; o < P; o <<= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, run_m, o), os = __shfl_xor_sync(0xffffffffu, run_s, o);
      const float M = fmaxf(run_m, om);
      float S = 0.f;
      if (run_m != -INFINITY) S += run_s * gs_ex2((run_m - M) * L2E);
      if (om != -INFINITY) S += os * gs_ex2((om - M) * L2E);
      run_m = M;
      run_s = S;
      float oz[KMAX];
      int oi[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        oz[i] = __shfl_xor_sync(0xffffffffu, tz[i], o);
        oi[i] = __shfl_xor_sync(0xffffffffu, ti[i], o);
      }
#pragma unroll
      for (int i = KMAX - 1; i >= 0; --i)                         // both lists hold K real entries at the tail
        if (i >= KMAX - a.K && better(oz[i], oi[i], tz[KMAX - 1], ti[KMAX - 1])) gs_insert<KMAX>(tz, ti, oz[i], oi[i]);
    }
    KTX(9, et == 0);
#ifdef ONMT_GS_DEBUG
    if (c == 0 && blockIdx.x == 0)
      printf("final part %d [%f %f %f %f] [%d %d %d %d]\n", part, tz[0], tz[1 % KMAX], tz[2 % KMAX], tz[3 % KMAX], ti[0],
             ti[1 % KMAX], ti[2 % KMAX], ti[3 % KMAX]);
#endif
    if (row_ok && part == 0) {
      const int r = n0 + c;
      const size_t base = ((size_t)r * a.Ct + ci) * a.K;
      if (a.vp.world == 0) {
        a.ms[(size_t)r * a.Ct + ci] = make_float2(run_m, run_s);
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
          if (i >= KMAX - a.K) {
            a.tz[base + i - (KMAX - a.K)] = tz[i];
            a.ti[base + i - (KMAX - a.K)] = ti[i];
          }
      } else {
        for (int w = 0; w < a.vp.world; ++w) {                     // every rank's exchange buffer
          __stcg(a.vp.ms[w] + (size_t)r * a.Ct + ci, make_float2(run_m, run_s));
#pragma unroll
          for (int i = 0; i < KMAX; ++i)
            if (i >= KMAX - a.K) {
              __stcg(a.vp.tz[w] + base + i - (KMAX - a.K), tz[i]);
              __stcg(a.vp.ti[w] + base + i - (KMAX - a.K), ti[i]);
            }
        }
      }
    }
  }
  KT(3);
  tc_fence_before();
  __syncthreads();
  if (a.vp.world > 0 && threadIdx.x == 0) {
    // my partials are stored everywhere (the barrier orders every thread's stores before this
    // thread's system-scope fence): raise my flag in every rank's buffer with the step epoch
    __threadfence_system();
    const unsigned long long ep = vp_epoch(a.vp.seq, a.t);
    for (int w = 0; w < a.vp.world; ++w)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.vp.flag[w] + (size_t)grp * a.Ct + ci), "l"(ep)
                   : "memory");
  }
  if (warp == 1) tmem_dealloc(tmem, 512);
}

static size_t gs_body_bytes(int n_group, int nt_max, int stages, int ovl, int nbuf, int srows) {
  const size_t ring = (size_t)stages * (2 * (size_t)n_group * 128 + (size_t)nt_max * kTileM * 128);
  const size_t stg = (size_t)nbuf * srows * kGsSLD * 4;
  return ovl ? ring + stg : (ring > stg ? ring : stg);
}
static size_t gs_smem_bytes(size_t body, int stages) { return 1024 + body + (2 * stages + 3 + 4 * kGsMaxCh) * 8 + 16; }

struct GsPlan {
  int C, nt_max, stages, P, ovl, nbuf, srows;
  size_t body;
};
// static shared memory of the kernel instance for beam width K: the dynamic part gets the rest
template <int KMAX>
static size_t gs_static_of() {
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, gen_step_kernel<KMAX>) == cudaSuccess ? fa.sharedSizeBytes : 12288;
}
static size_t gs_static_smem(int K) {
  static size_t v[7] = {0, 0, 0, 0, 0, 0, 0};
  const int i = K <= 1 ? 0 : K <= 2 ? 1 : K <= 4 ? 2 : K == 5 ? 3 : K <= 8 ? 4 : K == 10 ? 5 : 6;
  if (!v[i]) {
    switch (i) {
      case 0: v[i] = gs_static_of<1>(); break;
      case 1: v[i] = gs_static_of<2>(); break;
      case 2: v[i] = gs_static_of<4>(); break;
      case 3: v[i] = gs_static_of<5>(); break;
      case 4: v[i] = gs_static_of<8>(); break;
      case 5: v[i] = gs_static_of<10>(); break;
      default: v[i] = gs_static_of<16>(); break;
    }
  }
  return v[i];
}
static bool gs_plan(int n_vt, int n_group, int groups, int num_sms, int R, int K, GsPlan& p) {
  p.C = num_sms / groups;
  if (p.C > n_vt) p.C = n_vt;
  if (p.C < 1) return false;
  if (n_group > 32 * kGsScanWarps) return false;
  p.P = 2 * n_group <= 32 * kGsScanWarps ? 2 : 1;
  p.srows = n_group < R ? n_group : R;
  if (p.srows < 1) p.srows = 1;
  const size_t limit = 227 * 1024 - gs_static_smem(K);
  const int need = (n_vt + p.C - 1) / p.C;                          // most tiles of a CTA
  // overlapped batches: the CTA's tiles in K-outer batches of ONMT_GEN_OVL tiles
  // (every tile its own TMEM columns, staging outside the ring): batch b+1's MMAs run while
  // batch b is staged and scanned
  static const int ovl_env = getenv("ONMT_GEN_OVL") ? atoi(getenv("ONMT_GEN_OVL")) : 2;
  if (ovl_env > 0 && need >= 2 && need * gs_tstride(n_group) <= 512) {
    p.ovl = 1;
    p.stages = 2;
    // tiles per batch: ONMT_GEN_OVL (2), fewer when the ring + staging do not fit (c5's 160
    // staged rows: 1-tile batches, 30.3 vs 34.1 us for the non-overlapped plan)
    for (p.nt_max = ovl_env < need ? ovl_env : need - 1; p.nt_max >= 1; --p.nt_max)
      for (p.nbuf = 2; p.nbuf >= 1; --p.nbuf) {
        p.body = gs_body_bytes(n_group, p.nt_max, p.stages, 1, p.nbuf, p.srows);
        if (gs_smem_bytes(p.body, p.stages) <= limit && p.nt_max <= 4) return true;
      }
  }
  p.ovl = 0;
  p.nbuf = 2;
  p.nt_max = 512 / gs_tstride(n_group);                              // accumulators in TMEM
  if (p.nt_max > 4) p.nt_max = 4;                                    // (bias registers of the stagers)
  if (p.nt_max > need) p.nt_max = need;
  if (p.nt_max < 1) return false;
  p.stages = 4;
  auto fits = [&]() {
    p.body = gs_body_bytes(n_group, p.nt_max, p.stages, 0, p.nbuf, p.srows);
    return gs_smem_bytes(p.body, p.stages) <= limit;
  };
  const int nt0 = p.nt_max;
  while (p.stages > 2 && !fits()) --p.stages;
  while (p.nt_max > 1 && !fits()) --p.nt_max;
  if (fits()) return true;
  // wide row groups (> 160 rows: one scanner thread per row): one staging buffer - the stagers
  // refill a chunk once its scanners are done with it (per-chunk barriers)
  p.nbuf = 1;
  p.nt_max = nt0;
  p.stages = 4;
  while (p.stages > 2 && !fits()) --p.stages;
  while (p.nt_max > 1 && !fits()) --p.nt_max;
  return fits();
}

// parts per row written by the step kernel's phase A (0 = not applicable)
int g_gs_dbg = 0;
// is the plan the non-overlapped one-buffer plan of wide row groups?
bool gen_step_wide_plan(int n_vt, int n_group, int groups, int num_sms) {
  GsPlan p;
  return gs_plan(n_vt, n_group, groups, num_sms, n_group * groups, 16, p) && !p.ovl && p.nbuf == 1;
}
int gen_step_parts(int n_vt, int n_group, int groups, int num_sms) {
  GsPlan p;
  return gs_plan(n_vt, n_group, groups, num_sms, n_group * groups, 16, p) ? p.C : 0;
}

// gate tiles the step kernel can take per row group without raising any CTA's tile count:
// one each for the CTAs holding the smaller vocabulary share (0 if the split is even)
int gen_step_gate_capacity(int n_vt, int n_group, int groups, int num_sms) {
  GsPlan p;
  if (!gs_plan(n_vt, n_group, groups, num_sms, n_group * groups, 16, p)) return 0;
  return n_vt % p.C == 0 ? 0 : p.C - n_vt % p.C;
}

template <int KMAX>
static cudaError_t launch_gs(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmWg,
                             const GenStepArgs& a, int grid, size_t smem, cudaStream_t st) {
  auto fn = gen_step_kernel<KMAX>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(fn, dim3(grid), dim3(kGsThreads), smem, st, tmW, tmX, tmWg, a);
}

// generator partials of decode step t (t selects the threshold buffers)
cudaError_t gen_step(const CUtensorMap& tmW, const CUtensorMap& tmX, int n_vt, int n_rows_pad, int n_group,
                     int k_blocks, int num_sms, const GenOut& g, float* row_lse, float* row_z, int* row_i, int t,
                     unsigned int* thr, StepCtl ctl, cudaStream_t st, const GateTiles& gt, const VpOut* vp,
                     int vp_rank, int vp_C) {
  const int groups = n_rows_pad / n_group;
  GsPlan p;
  // vocabulary-parallel: plan for this rank's CTA count (vp_C per group), split Ct = world x vp_C
  if (!gs_plan(vp ? (n_vt + vp->ranks - 1) / vp->ranks : n_vt, n_group, groups, vp ? vp_C * groups : num_sms,
               g.rows_valid, g.K, p))
    return cudaErrorInvalidConfiguration;
  if (vp) p.C = vp_C;
  if (gt.n_gt > 0 && (n_vt % p.C == 0 || gt.n_gt > p.C - n_vt % p.C)) return cudaErrorInvalidConfiguration;
  GenStepArgs a{};
  a.n_rows_pad = n_rows_pad;
  a.n_group = n_group;
  a.groups = groups;
  a.k_blocks = k_blocks;
  a.n_vt = n_vt;
  a.C = p.C;
  a.nt_max = p.nt_max;
  a.stages = p.stages;
  a.P = p.P;
  a.bias = g.bias;
  a.V = g.V;
  a.K = g.K;
  a.R = g.rows_valid;
  a.rows_pad = g.rows_pad;
  a.ms = g.ms;
  a.tz = g.tz;
  a.ti = g.ti;
  a.row_lse = row_lse;
  a.row_z = row_z;
  a.row_i = row_i;
  a.t = t;
  a.thr = thr;
  a.ctl = ctl;
  a.dbg = g_gs_dbg;
  const int grid = p.C * groups;
  const size_t smem = gs_smem_bytes(p.body, p.stages);
  a.ci0 = vp ? vp_rank * p.C : 0;
  a.Ct = vp ? p.C * vp->ranks : p.C;
  if (vp) {
    if (gt.n_gt > 0 || p.C * vp->ranks > n_vt || vp->ranks < 1) return cudaErrorInvalidConfiguration;
    a.vp = *vp;
  }
  if (getenv("ONMT_GEN_DEBUG") && t <= 1)
    fprintf(stderr, "gen_step plan: C=%d groups=%d n_group=%d nt_max=%d stages=%d ovl=%d nbuf=%d srows=%d smem=%zu "
            "static=%zu gates=%d\n", p.C, groups, n_group, p.nt_max, p.stages, p.ovl, p.nbuf, p.srows, smem,
            gs_static_smem(g.K), gt.n_gt);
  a.ovl = p.ovl;
  a.nbuf = p.nbuf;
  a.srows_alloc = p.srows;
  a.n_gt = gt.n_gt;
  a.gt_per_q = gt.gt_per_q > 0 ? gt.gt_per_q : 1;
  a.gkbh = gt.gkbh;
  a.gld = gt.gld;
  a.gout = gt.gout;
  const CUtensorMap& tmWg = gt.n_gt > 0 ? *gt.tmWg : tmW;
  if (g.K <= 1) return launch_gs<1>(tmW, tmX, tmWg, a, grid, smem, st);
  if (g.K <= 2) return launch_gs<2>(tmW, tmX, tmWg, a, grid, smem, st);
  if (g.K <= 4) return launch_gs<4>(tmW, tmX, tmWg, a, grid, smem, st);
  if (g.K == 5) return launch_gs<5>(tmW, tmX, tmWg, a, grid, smem, st);     // (the paper's beam size)
  if (g.K <= 8) return launch_gs<8>(tmW, tmX, tmWg, a, grid, smem, st);
  if (g.K == 10) return launch_gs<10>(tmW, tmX, tmWg, a, grid, smem, st);   // (BASELINE c5)
  return launch_gs<16>(tmW, tmX, tmWg, a, grid, smem, st);
}

}  // namespace onmt
