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
#include <cstdlib>

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
  pdl_trigger();
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
  pdl_wait();                                   // predecessor's outputs (X, flags) now visible
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (all_done(a.ctl)) {                        // uniform: every thread read the same flag
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
    return;
  }

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
    if (g.gold) {
      // teacher-forced scoring: per row the tile's (max, sum exp) and the gold logit only
      // (no top-K); two register-light passes, ex2.approx (rel. error ~2^-22)
      constexpr float L2E = 1.4426950408889634f;
      const int nv = min(kTileM, g.V - m0);
      for (int c = threadIdx.x; c < a.n_group; c += blockDim.x) {
        const int r = n0 + c;
        if (r >= g.rows_valid) continue;
        const float* col = stg + c * LD;
        float m0v = -INFINITY, m1v = -INFINITY;
        for (int v = 0; v < nv; v += 2) {
          m0v = fmaxf(m0v, col[v] + __ldg(&g.bias[m0 + v]));
          if (v + 1 < nv) m1v = fmaxf(m1v, col[v + 1] + __ldg(&g.bias[m0 + v + 1]));
        }
        const float mx = fmaxf(m0v, m1v);
        float s0 = 0.f, s1 = 0.f;
        const float mo = mx * L2E;
        for (int v = 0; v < nv; v += 2) {
          float e0, e1 = 0.f;
          asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(fmaf(col[v] + __ldg(&g.bias[m0 + v]), L2E, -mo)));
          if (v + 1 < nv)
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(fmaf(col[v + 1] + __ldg(&g.bias[m0 + v + 1]), L2E, -mo)));
          s0 += e0;
          s1 += e1;
        }
        g.ms[(size_t)blockIdx.x * g.rows_pad + r] = make_float2(mx, s0 + s1);
        const int gid = g.gold[r];
        if (gid >= m0 && gid < m0 + kTileM && gid < g.V) g.zgold[r] = col[gid - m0] + g.bias[gid];
      }
    } else {
      for (int c = threadIdx.x; c < a.n_group; c += blockDim.x) {
        const int r = n0 + c;
        if (r >= g.rows_valid) continue;
        float mx, sm, tz[KMAX];
        int ti[KMAX];
        scan_tile_column<KMAX>(stg + c * LD, 1, m0, g, mx, sm, tz, ti);
        write_gen_partial<KMAX>(g, blockIdx.x, r, mx, sm, tz, ti);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

// ------------------------------------------------------------------ persistent generator
// One CTA per SM (grid = groups x C).  CTA (g, i) owns the hypothesis rows of N-group g
// and the contiguous vocabulary tiles [i*n_vt/C, (i+1)*n_vt/C).  Warp roles:
//   warp 0      TMA producer (A = 128 W_gen rows x 64 K, B = hi/lo activation planes)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; accumulators are
//               double-buffered in TMEM (2 x 256 columns) so the epilogue of tile j
//               overlaps the MMAs of tile j+1
//   warps 2-9   epilogue: TMEM -> registers (+bias) -> transposed smem staging (two warps
//               per TMEM lane quarter split the column chunks), then one thread per
//               hypothesis row keeps a running (max, sum exp, top-k) over all of the
//               CTA's vocabulary tiles; logits never reach HBM.
// Output: one partial per (CTA, row) - C partials per row instead of V/128.
struct GenPArgs {
  int n_rows_pad, n_group, k_blocks, stages, n_vt, C;
  int sc;         // staged columns per pass (n_group or half of it)
  StepCtl ctl;
  unsigned long long* dbg;   // optional timeline (%globaltimer) of CTA 0, debug builds only
  int epi_mode;              // ablation (ONMT_GEN_EPI_MODE): 0 full, 1 stage only, 2 drain only
};
#ifdef ONMT_GEN_TRACE
#define GEN_DBG(stmt) stmt
#else
#define GEN_DBG(stmt)
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- epilogue building blocks (4 lanes per hypothesis row, 32 logits each per tile)
constexpr int kEpiWarps = 10;      // epilogue warps
constexpr int kLPR = 4;            // lanes per hypothesis row
constexpr int kVPL = kTileM / kLPR;  // logits per lane per tile (32)
constexpr int kColsPerPass = kEpiWarps * 32 / kLPR;   // 80 rows staged per pass
constexpr int kSLD = 132;          // staging row stride: (row*132 + part) % 32 distinct across a warp

// branch-free sorted insertion of (x, xi) into a (z desc, id asc) list
template <int KMAX>
__device__ __forceinline__ void list_insert(float (&tz)[KMAX], int (&ti)[KMAX], float x, int xi) {
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

template <int KMAX>
__device__ __forceinline__ int list_count(const float (&tz)[KMAX]) {
  int n = 0;
#pragma unroll
  for (int q = 0; q < KMAX; ++q) n += tz[q] != -INFINITY;
  return n;
}

// One row's update with one tile: the 4 lanes of a group each scan 32 logits
// (v = part + 4i, increasing ids), then combine (max, sum exp) and top-k by butterfly
// shuffles.  The row's running state lives in shared memory (st: [m, s, z[KMAX], id[KMAX]])
// so the pass loop stays rolled (instruction-cache footprint).  All shuffles are executed
// by the whole warp (rows without work feed neutral values).
template <int KMAX>
__device__ __forceinline__ void list_shift_pop(float (&z)[KMAX], int (&id)[KMAX]) {
#pragma unroll
  for (int q = 0; q < KMAX - 1; ++q) { z[q] = z[q + 1]; id[q] = id[q + 1]; }
  z[KMAX - 1] = -INFINITY;
  id[KMAX - 1] = 0x7fffffff;
}

// One row's update with one tile: the kLPR lanes of a row each hold kVPL logits in
// registers (v = part + kLPR*i, increasing ids).  (max, sum exp) are combined by
// shuffles; top-k by threshold filtering: theta = max(running K-th best, K-th largest of
// the lanes' top-3 - computed on cold tiles only) is a lower bound of the K-th best of
// (running list U tile) - both are K-th bests of subsets - so only logits >= theta can
// enter; the leader (part 0) inserts the row's candidates (partner masks via shuffles,
// values re-read from staging).  Scans use independent sub-chains for ILP.
template <int KMAX>
__device__ __forceinline__ void top3_merge(float& a1, float& a2, float& a3, float b1, float b2, float b3) {
  // top-3 of two sorted triples
  const float x1 = fmaxf(a1, b1);
  const float y1 = fminf(a1, b1);                      // the other head
  const float x2 = fmaxf(y1, fmaxf(a2, b2));
  const float x3 = fmaxf(fminf(y1, fmaxf(a2, b2)), fmaxf(fminf(a2, b2), fmaxf(a3, b3)));
  a1 = x1; a2 = x2; a3 = x3;
}

template <int KMAX>
__device__ __forceinline__ void group_update(const float* __restrict__ col, bool valid, int part, int vbase,
                                             float* __restrict__ st, int K, unsigned long long* dbg) {
  constexpr float L2E = 1.4426950408889634f;
  const unsigned FULL = 0xffffffffu;
  const int gbase = (threadIdx.x & 31) & ~(kLPR - 1);
  GEN_DBG(if (dbg) dbg[0] = gtimer();)
  float z[kVPL];
#pragma unroll
  for (int i = 0; i < kVPL; ++i) z[i] = valid ? col[part + kLPR * i] : -INFINITY;
  // row max (4 independent chains)
  float x0 = -INFINITY, x1 = -INFINITY, x2 = -INFINITY, x3 = -INFINITY;
#pragma unroll
  for (int i = 0; i < kVPL; i += 4) {
    x0 = fmaxf(x0, z[i]); x1 = fmaxf(x1, z[i + 1]); x2 = fmaxf(x2, z[i + 2]); x3 = fmaxf(x3, z[i + 3]);
  }
  float lm = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
#pragma unroll
  for (int lvl = 1; lvl < kLPR; lvl <<= 1) lm = fmaxf(lm, __shfl_xor_sync(FULL, lm, lvl));
  const float m = valid ? st[0] : -INFINITY;
  const float mn = fmaxf(m, lm);
  float ls = 0.f;
  if (mn != -INFINITY) {
    const float mo = mn * L2E;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int i = 0; i < kVPL; i += 4) {
      a0 += ex2(fmaf(z[i], L2E, -mo)); a1 += ex2(fmaf(z[i + 1], L2E, -mo));
      a2 += ex2(fmaf(z[i + 2], L2E, -mo)); a3 += ex2(fmaf(z[i + 3], L2E, -mo));
    }
    ls = (a0 + a1) + (a2 + a3);
  }
#pragma unroll
  for (int lvl = 1; lvl < kLPR; lvl <<= 1) ls += __shfl_xor_sync(FULL, ls, lvl);
  float rz[KMAX];
  int ri[KMAX];
  float tk = INFINITY;
  if (valid && part == 0) {
    const float s0 = st[1];
    st[0] = mn;
    st[1] = (m == -INFINITY ? 0.f : s0 * ex2((m - mn) * L2E)) + ls;
#pragma unroll
    for (int q = 0; q < KMAX; ++q) { rz[q] = st[2 + q]; ri[q] = __float_as_int(st[2 + KMAX + q]); }
    tk = rz[KMAX - 1];
  }
  tk = __shfl_sync(FULL, tk, gbase);
  float theta = tk;
  GEN_DBG(if (dbg) dbg[1] = gtimer();)
  if (__any_sync(FULL, tk == -INFINITY) && K <= 3 * kLPR) {
    // cold row(s): K-th largest of the lanes' top-3 (two independent sub-chains)
    float p1 = -INFINITY, p2 = -INFINITY, p3 = -INFINITY, q1 = -INFINITY, q2 = -INFINITY, q3 = -INFINITY;
#pragma unroll
    for (int i = 0; i < kVPL; i += 2) {
      const float u = z[i], w = z[i + 1];
      p3 = fmaxf(p3, fminf(p2, u)); p2 = fmaxf(p2, fminf(p1, u)); p1 = fmaxf(p1, u);
      q3 = fmaxf(q3, fminf(q2, w)); q2 = fmaxf(q2, fminf(q1, w)); q1 = fmaxf(q1, w);
    }
    top3_merge<KMAX>(p1, p2, p3, q1, q2, q3);
    // rank each of my three values among the row's 3*kLPR values ((value, lane, slot) order)
    int r[3] = {0, 1, 2};
    const float mine[3] = {p1, p2, p3};
#pragma unroll
    for (int o = 1; o < kLPR; ++o) {
      const int srcl = gbase + ((part + o) & (kLPR - 1));
      const int op = (part + o) & (kLPR - 1);
      const float o1 = __shfl_sync(FULL, p1, srcl), o2 = __shfl_sync(FULL, p2, srcl), o3 = __shfl_sync(FULL, p3, srcl);
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const float v = mine[u];
        r[u] += (o1 > v || (o1 == v && op < part)) + (o2 > v || (o2 == v && op < part)) +
                (o3 > v || (o3 == v && op < part));
      }
    }
    float kth = -INFINITY;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const unsigned h = __ballot_sync(FULL, r[u] == K - 1);
      const unsigned gm = (h >> gbase) & ((1u << kLPR) - 1);
      const float v = __shfl_sync(FULL, mine[u], gm ? gbase + __ffs(gm) - 1 : gbase);
      if (gm) kth = v;
    }
    if (tk == -INFINITY) theta = kth;
  }
  unsigned cm = 0;
#pragma unroll
  for (int i = 0; i < kVPL; ++i) cm |= (valid && z[i] >= theta) ? (1u << i) : 0u;
  unsigned pm[kLPR];
#pragma unroll
  for (int o = 0; o < kLPR; ++o) pm[o] = __shfl_sync(FULL, cm, gbase + o);
  if (!valid || part != 0) return;
  bool dirty = false;
#pragma unroll
  for (int src = 0; src < kLPR; ++src) {
    unsigned w = pm[src];
    while (w) {
      const int i = __ffs(w) - 1;
      w &= w - 1;
      const int off = src + kLPR * i;
      const float zc = col[off];
      const int idc = vbase + off;
      if (better(zc, idc, rz[KMAX - 1], ri[KMAX - 1])) {
        list_insert<KMAX>(rz, ri, zc, idc);
        dirty = true;
      }
    }
  }
  GEN_DBG(if (dbg) dbg[2] = gtimer();)
  if (!dirty) return;
#pragma unroll
  for (int q = 0; q < KMAX; ++q) { st[2 + q] = rz[q]; st[2 + KMAX + q] = __int_as_float(ri[q]); }
}

template <int KMAX, int CS>
__global__ void __launch_bounds__(64 + 32 * kEpiWarps, 1)
gen_persistent_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GenPArgs a,
                      GenOut g) {
  // CS > 1: thread-block cluster of CS CTAs sharing the activation (B) tiles by TMA
  // multicast - CTA rank r loads rows [r*n_group/CS, (r+1)*n_group/CS) of each B tile for
  // all CS CTAs - so the B operand crosses L2 -> SM once per cluster instead of once per CTA.
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t a_bytes = kTileM * 128, b_bytes = a.n_group * 128;
  const uint32_t stage_bytes = a_bytes + 2 * b_bytes;
  float* stg = reinterpret_cast<float*>(smem + a.stages * stage_bytes);
  float* rstate = stg + (size_t)kColsPerPass * kSLD;            // [n_group][2 + 2*KMAX]
  constexpr int SW = 2 + 2 * KMAX;
  uint64_t* full = reinterpret_cast<uint64_t*>(rstate + (size_t)a.n_group * SW);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = blockIdx.x / a.C, ci = blockIdx.x % a.C;
  const int rank = CS > 1 ? (int)cluster_ctarank() : 0;
  const int Q = a.C / CS, qi = ci / CS;                       // cluster index within the group
  const int tb = (int)((long long)qi * a.n_vt / Q), te = (int)((long long)(qi + 1) * a.n_vt / Q);
  const int rounds = (te - tb + CS - 1) / CS;                 // lock-step rounds of the cluster
  const int ntiles = max(0, (te - tb - rank + CS - 1) / CS);  // this CTA's real tiles: tb + rank + CS*j
  const int n0 = grp * a.n_group;
  const uint16_t cmask = (uint16_t)((1u << CS) - 1);
  const int slice_rows = a.n_group / CS;
  const uint32_t slice_bytes = slice_rows * 128;

  GEN_DBG(if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0) a.dbg[200] = gtimer();)
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CS); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], kEpiWarps); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  pdl_wait();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (all_done(a.ctl)) {                     // uniform over the grid: no cluster traffic happened yet
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
    return;
  }
  if (CS > 1) cluster_sync_all();            // peers' barriers initialised before any multicast

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int j = 0; j < rounds; ++j) {
        const bool has = tb + rank + CS * j < te;
        const int m0 = (tb + rank + CS * j) * kTileM;
        for (int kb = 0; kb < a.k_blocks; ++kb, ++it) {
          const int s = it % a.stages;
          if (it >= a.stages) mbar_wait(&empty[s], ((it / a.stages) & 1) ^ 1);
          GEN_DBG(if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[it] = gtimer();)
          uint8_t* st = smem + s * stage_bytes;
          const bool ldA = has && a.epi_mode != 4, ldB = a.epi_mode != 3;   // (ablation modes 3/4)
          mbar_arrive_expect_tx(&full[s], (ldA ? a_bytes : 0u) + (ldB ? 2 * b_bytes : 0u));
          if (ldA) tma_load_2d(st, &tmW, kb * kBK, m0, &full[s]);
          if (!ldB) {
          } else if (CS > 1) {
            tma_load_2d_mc(st + a_bytes + rank * slice_bytes, &tmX, kb * kBK, n0 + rank * slice_rows, &full[s], cmask);
            tma_load_2d_mc(st + a_bytes + b_bytes + rank * slice_bytes, &tmX, kb * kBK,
                           a.n_rows_pad + n0 + rank * slice_rows, &full[s], cmask);
          } else {
            tma_load_2d(st + a_bytes, &tmX, kb * kBK, n0, &full[s]);
            tma_load_2d(st + a_bytes + b_bytes, &tmX, kb * kBK, a.n_rows_pad + n0, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(kTileM, a.n_group);
      int it = 0, jj = 0;
      for (int j = 0; j < rounds; ++j) {
        const bool has = tb + rank + CS * j < te;
        const int acc = jj & 1;
        if (has && jj >= 2) mbar_wait(&tempty[acc], ((jj >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int kb = 0; kb < a.k_blocks; ++kb, ++it) {
          const int s = it % a.stages;
          mbar_wait(&full[s], (it / a.stages) & 1);
          GEN_DBG(if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[64 + it] = gtimer();)
          tc_fence_after();
          if (has && a.epi_mode != 5) {
            const uint32_t sa = smem_u32(smem + s * stage_bytes);
            const uint32_t sbh = sa + a_bytes, sbl = sa + a_bytes + b_bytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              const uint64_t da = umma_desc_sw128(sa + kk * 32);
              tc_mma_bf16(d, da, umma_desc_sw128(sbh + kk * 32), idesc, (kb | kk) != 0);
              tc_mma_bf16(d, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
            }
          }
          if (CS > 1) tc_commit_mc(&empty[s], cmask);      // stage s free in every peer's view
          else tc_commit(&empty[s]);
        }
        if (has) {
          tc_commit(&tfull[acc]);
          GEN_DBG(if (a.dbg && blockIdx.x == 0 && jj < 8) a.dbg[128 + jj] = gtimer();)
          ++jj;
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..(2+kEpiWarps)
    const int et = threadIdx.x - 64;                     // 0..32*kEpiWarps-1
    const int q = warp & 3;                              // TMEM lane quarter of this warp
    const int par = (warp - 2 - ((q - 2) & 3)) >> 2;     // index among the warps sharing quarter q
    const int nwq = (kEpiWarps - ((q - 2) & 3) + 3) >> 2; // warps sharing quarter q
    const int vr = q * 32 + lane;                        // vocabulary row (TMEM lane) this thread drains
    const int gcol = et / kLPR;                          // row (column) within a pass (et < 160 scan)
    const int part = lane % kLPR;
    const int npass = (a.n_group + kColsPerPass - 1) / kColsPerPass;
    for (int i = et; i < a.n_group; i += 32 * kEpiWarps) {
      float* st = rstate + (size_t)i * SW;
      st[0] = -INFINITY; st[1] = 0.f;
      for (int qq = 0; qq < KMAX; ++qq) {
        const bool sentinel = qq < KMAX - g.K;
        st[2 + qq] = sentinel ? INFINITY : -INFINITY;
        st[2 + KMAX + qq] = __int_as_float(sentinel ? -1 : 0x7fffffff);
      }
    }
    named_bar(1, 32 * kEpiWarps);
    for (int j = 0; j < ntiles; ++j) {
      const int acc = j & 1;
      const int vt = tb + rank + CS * j;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      GEN_DBG(if (a.dbg && blockIdx.x == 0 && et == 0 && j < 8) a.dbg[144 + j] = gtimer();)
      tc_fence_after();
      const int vid = vt * kTileM + vr;
      const float bias = vid < g.V ? g.bias[vid] : -INFINITY;
      const uint32_t trow = tmem + acc * 256 + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int h = 0; h < npass; ++h) {
        const int cbeg = h * kColsPerPass;
        const int cend = min(a.n_group, cbeg + kColsPerPass);
        for (int c0 = cbeg + par * 16; c0 < cend && a.epi_mode != 2 && a.epi_mode < 3 && a.epi_mode != 5; c0 += 16 * nwq) {
          float v[16];
          tmem_ld16(trow + c0, v);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) stg[(c0 - cbeg + jj) * kSLD + vr] = v[jj] + bias;
        }
        if (h == npass - 1) {                          // accumulator drained: hand it back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        named_bar(1, 32 * kEpiWarps);
        GEN_DBG(if (a.dbg && blockIdx.x == 0 && et == 0 && j < 8 && h < 2) a.dbg[160 + 2 * j + h] = gtimer();)
        const int c = cbeg + gcol;
        const bool valid = gcol < kColsPerPass && c < cend && n0 + c < g.rows_valid;
#ifdef ONMT_GEN_TRACE
        unsigned long long* gd = (a.dbg && blockIdx.x == 0 && et == 0 && j < 2 && h < 2) ? a.dbg + 210 + 8 * (2 * j + h) : nullptr;
#else
        unsigned long long* gd = nullptr;
#endif
        if (a.epi_mode == 0)
          group_update<KMAX>(stg + min(gcol, kColsPerPass - 1) * kSLD, valid, part, vt * kTileM,
                             rstate + (size_t)min(c, a.n_group - 1) * SW, g.K, gd);
        named_bar(1, 32 * kEpiWarps);
        GEN_DBG(if (a.dbg && blockIdx.x == 0 && et == 0 && j < 8 && h < 2) a.dbg[176 + 2 * j + h] = gtimer();)
      }
    }
    for (int c = et; c < a.n_group; c += 32 * kEpiWarps) {
      const int r = n0 + c;
      if (r >= g.rows_valid) continue;
      const float* st = rstate + (size_t)c * SW;
      g.ms[(size_t)ci * g.rows_pad + r] = make_float2(st[0], st[1]);
      const size_t base = ((size_t)ci * g.rows_pad + r) * g.K;
      for (int qq = 0; qq < g.K; ++qq) {
        g.tz[base + qq] = st[2 + KMAX - g.K + qq];
        g.ti[base + qq] = __float_as_int(st[2 + 2 * KMAX - g.K + qq]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CS > 1) cluster_sync_all();            // no peer may still multicast into / arrive on us
  GEN_DBG(if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0) { a.dbg[201] = gtimer(); a.dbg[202] = ntiles; a.dbg[203] = a.stages; })
  if (warp == 1) tmem_dealloc(tmem, 512);
}

static size_t genp_smem_bytes(int n_group, int stages, int kmax) {
  return 1024 + (size_t)stages * (kTileM * 128 + 2 * (size_t)n_group * 128) + (size_t)kColsPerPass * kSLD * 4 +
         (size_t)n_group * (2 + 2 * kmax) * 4 + (2 * stages + 4) * 8 + 16;
}

// does the tile-outer generator fit for this row group at any beam width (<= 16)?
bool gen_persistent_fits(int n_group) { return genp_smem_bytes(n_group, 2, 16) <= 227 * 1024; }

// number of partials per row the persistent generator writes (C = CTAs per N-group)
int gen_persistent_parts(int n_vt, int n_groups, int num_sms, int cs) {
  int C = num_sms / n_groups;
  if (C > n_vt) C = n_vt;
  C = C / cs * cs;
  if (C < cs) C = cs;
  return C;
}

template <int KMAX, int CS>
static cudaError_t launch_genp(const CUtensorMap& tmW, const CUtensorMap& tmX, const GenPArgs& a, const GenOut& g,
                               int grid, cudaStream_t st) {
  size_t smem = genp_smem_bytes(a.n_group, a.stages, KMAX);
  auto fn = gen_persistent_kernel<KMAX, CS>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64 + 32 * kEpiWarps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CS;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fn, tmW, tmX, a, g);
}

unsigned long long* g_gen_dbg = nullptr;   // set by the runtime when ONMT_GEN_TRACE is on

// tmX: activation planes with box rows n_group (CS = 1) or n_group / CS (multicast slices)
cudaError_t tc_gen_persistent(const CUtensorMap& tmW, const CUtensorMap& tmX, int n_vt, int n_rows_pad, int n_group,
                              int k_blocks, int num_sms, int cs, const GenOut& g, StepCtl ctl, cudaStream_t st) {
  GenPArgs a{};
  a.dbg = g_gen_dbg;
  if (const char* em = std::getenv("ONMT_GEN_EPI_MODE")) a.epi_mode = std::atoi(em);
  a.n_rows_pad = n_rows_pad;
  a.n_group = n_group;
  a.k_blocks = k_blocks;
  a.n_vt = n_vt;
  const int groups = n_rows_pad / n_group;
  if (cs != 1) return cudaErrorInvalidValue;                 // (the multicast variant was removed)
  a.C = gen_persistent_parts(n_vt, groups, num_sms, cs);
  a.ctl = ctl;
  const size_t limit = 227 * 1024;
  const int kmax = g.K <= 1 ? 1 : g.K <= 2 ? 2 : g.K <= 4 ? 4 : g.K <= 8 ? 8 : 16;
  a.sc = n_group;
  int stages = 8;
  while (stages > 2 && genp_smem_bytes(n_group, stages, kmax) > limit) --stages;
  if (stages > k_blocks * 2) stages = k_blocks * 2;
  a.stages = stages;
  if (genp_smem_bytes(n_group, stages, kmax) > limit) return cudaErrorInvalidConfiguration;
  const int grid = a.C * groups;
#define ONMT_GENP(KM)                                                     \
  return launch_genp<KM, 1>(tmW, tmX, a, g, grid, st)
  if (g.K <= 1) ONMT_GENP(1);
  if (g.K <= 2) ONMT_GENP(2);
  if (g.K <= 4) ONMT_GENP(4);
  if (g.K <= 8) ONMT_GENP(8);
  ONMT_GENP(16);
#undef ONMT_GENP
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
  return launch_pdl(fn, grid, dim3(128), smem, st, tmW, tmX, a, g);
  return cudaGetLastError();
}

cudaError_t tc_gemm_partial(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                            int n_valid, int k_blocks, int splits, float* out, StepCtl ctl, cudaStream_t st,
                            bool groups_from_valid) {
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
  // groups_from_valid: row groups of a re-grouped box (tmX's box rows = n_group need not divide
  // n_rows_pad); rows past n_valid are never stored
  dim3 grid(m_pad / kTileM, groups_from_valid ? (n_valid + n_group - 1) / n_group : n_rows_pad / n_group, splits);
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
