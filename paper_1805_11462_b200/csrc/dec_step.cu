// The decoder step up to the generator as ONE persistent kernel (
// PAPER.md P115-122, P129-136, P299-301):
//
//   phase L_l (l < L)  decoder LSTM layer l: split-K tcgen05 GEMM  gates = W_l [x_l; h_l]
//                      with the split reduction and the LSTM cell fused (as gemm_fused.cu)
//   phase A1           attention chunks: per (sentence, source chunk) online softmax
//                      statistics and unnormalised context of the K beam rows
//   phase A2           attention combine: per (sentence, column slice) the context
//   phase O            h~ = tanh(W_out [c; h]) (split-K GEMM + tanh)
//
// Grid = #SMs CTAs, one per SM, all co-resident: the phases are separated by software grid
// barriers (common.cuh cta_group_barrier) instead of kernel boundaries, the TMEM allocation
// and the mbarriers are set up once, and every phase's weight K-slice is TMA-prefetched into
// its own shared-memory slots at kernel start - before griddepcontrol.wait - because the
// weights are constants.  Phase data flow through L2: activation operands written by one
// phase (generic proxy) are TMA-read by the next after fence.proxy.async + the barrier.
// Everything is deterministic (fixed reduction orders).
#include <math_constants.h>

#include <algorithm>

#include "dec_step.cuh"
#include "ptx.cuh"

namespace onmt {

__device__ __forceinline__ float ds_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float ds_tanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

__device__ __forceinline__ void ds_grid_sync(unsigned int* bar) {
  asm volatile("fence.proxy.async;" ::: "memory");   // generic writes -> later TMA reads
  __syncthreads();
  if (threadIdx.x == 0) cta_group_barrier(bar, gridDim.x);
  __syncthreads();
  asm volatile("fence.proxy.async;" ::: "memory");
}

// ---------------------------------------------------------------- split-K GEMM phase
__device__ __forceinline__ void ds_gemm_phase(const DsGemm& g, uint8_t* smem, uint64_t* bars, uint32_t tmem,
                                              uint32_t b_off, uint32_t side_off) {
  const int cta = blockIdx.x;
  if (cta >= g.tiles * g.S) return;                               // (uniform over the CTA)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t a_bytes = kTileM * 128, b_bytes = g.n_group * 128;
  uint8_t* bring = smem + b_off;
  uint64_t* wbar = bars;
  uint64_t* full = bars + 1;
  uint64_t* done = bars + 1 + kDsMaxKbps;
  uint64_t* rbar = done + 1;
  float4* s_bias = reinterpret_cast<float4*>(smem + side_off);
  float* s_cg = reinterpret_cast<float*>(smem + side_off + 32 * 16);
  const int tile = cta / g.S, split = cta % g.S;
  const int n_groups = g.n_rows_pad / g.n_group;
  const int mt = tile / n_groups, grp = tile % n_groups;
  const int m0 = mt * kTileM, n0 = grp * g.n_group;
  const int kb0 = split * g.kbps;
  const int nkb = max(0, min(g.kbps, g.k_blocks - kb0));
  const int c_own = split * g.NC;
  const int ncols = max(0, min(g.NC, g.n_group - c_own));

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < nkb; ++i) {
      uint8_t* st = bring + (size_t)i * 2 * b_bytes;
      mbar_arrive_expect_tx(&full[i], 2 * b_bytes);
      tma_load_2d(st, &g.tmX, (kb0 + i) * kBK, n0, &full[i]);
      tma_load_2d(st + b_bytes, &g.tmX, (kb0 + i) * kBK, g.n_rows_pad + n0, &full[i]);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(kTileM, g.n_group);
    if (nkb > 0) mbar_wait(wbar, 0);                              // weight slots (prefetched)
    for (int i = 0; i < nkb; ++i) {
      mbar_wait(&full[i], 0);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + g.w_off + (size_t)i * a_bytes);
      const uint32_t sbh = smem_u32(bring + (size_t)i * 2 * b_bytes), sbl = sbh + b_bytes;
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk) {
        const uint64_t da = umma_desc_sw128(sa + kk * 32);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, (i | kk) != 0);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
      }
    }
    tc_commit(done);
  } else if (warp >= 2 && g.epi == 0) {
    const int t = threadIdx.x - 64;                               // 192 threads: epilogue side inputs
    if (t < 32) {
      const int j = m0 / 4 + t;
      s_bias[t] = j < g.H ? __ldg(&g.bias[j]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int i0 = t; i0 < ncols * 32; i0 += 192 * 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + 192 * u;
        const int c = i / 32, ul = i % 32;
        const int r = n0 + c_own + c, j = m0 / 4 + ul;
        v[u] = (i < ncols * 32 && r < g.n_valid && j < g.H) ? __ldcg(&g.cg[(size_t)r * g.H + j]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + 192 * u < ncols * 32) s_cg[i0 + 192 * u] = v[u];
    }
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  // ---- partial tile -> global scratch [tile][split][n/4][128][4]
  {
    const int q = warp & 3, half = warp >> 2;
    const int m = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int hcols = (g.n_group / 2 + 3) & ~3;
    const int cb = half * hcols, ce = half ? g.n_group : hcols;
    float4* out = reinterpret_cast<float4*>(g.scratch + ((size_t)(tile * g.S + split) * g.n_group) * kTileM) + m;
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
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + 4 * k < ce)
          __stcg(out + (size_t)((c0 >> 2) + k) * kTileM,
                 make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]), __uint_as_float(r[4 * k + 2]),
                             __uint_as_float(r[4 * k + 3])));
    }
  }
  tc_fence_before();
  __threadfence();
  __syncthreads();
  float* recv = reinterpret_cast<float*>(bring);                  // [S][NC][128], overlays the (dead) ring
  if (threadIdx.x == 0) {
    cta_group_barrier(g.counters + 2 * tile, (unsigned)g.S);      // the tile's S splits are stored
    asm volatile("fence.proxy.async;" ::: "memory");
    if (ncols > 0) {
      const uint32_t bytes = (uint32_t)ncols * kTileM * 4;
      mbar_arrive_expect_tx(rbar, bytes * g.S);
      for (int p = 0; p < g.S; ++p)
        bulk_g2s(recv + (size_t)p * g.NC * kTileM, g.scratch + ((size_t)(tile * g.S + p) * g.n_group + c_own) * kTileM,
                 bytes, rbar);
    } else {
      mbar_arrive_local(rbar);
    }
  }
  mbar_wait(rbar, 0);
  float* red = recv + (size_t)g.S * g.NC * kTileM;                // [NC][128] fixed-order split sums
  if (ncols > 0) {
    const size_t slot = (size_t)g.NC * kTileM;
    const int nit = (ncols / 4) * kTileM;
    for (int it0 = threadIdx.x; it0 < nit; it0 += 2 * blockDim.x) {
      float4 v[2][16];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const size_t off = (size_t)min(it0 + u * (int)blockDim.x, nit - 1) * 4;
#pragma unroll
        for (int p = 0; p < 16; ++p)
          v[u][p] = p < g.S ? *reinterpret_cast<const float4*>(recv + p * slot + off) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int it = it0 + u * blockDim.x;
        float4 acc = v[u][0];
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
  __syncthreads();
  if (ncols > 0) {
    if (g.epi == 0) {
      const int nit = 32 * ncols;
      for (int it0 = threadIdx.x; it0 < nit; it0 += 2 * blockDim.x) {
        float4 gz[2], bb[2];
        float cp[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int it = min(it0 + u * (int)blockDim.x, nit - 1);
          const int ul = it % 32, c = it / 32;
          gz[u] = *reinterpret_cast<const float4*>(red + (size_t)c * kTileM + 4 * ul);
          bb[u] = s_bias[ul];
          cp[u] = s_cg[it];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int it = it0 + u * blockDim.x;
          const int ul = it % 32, c = it / 32;
          const int r = n0 + c_own + c, j = m0 / 4 + ul;
          const float i_ = ds_sigm(gz[u].x + bb[u].x), f_ = ds_sigm(gz[u].y + bb[u].y),
                      g_ = ds_tanh(gz[u].z + bb[u].z), o_ = ds_sigm(gz[u].w + bb[u].w);
          const float cn = f_ * cp[u] + i_ * g_;
          const float h = o_ * ds_tanh(cn);
          if (it >= nit || r >= g.n_valid || j >= g.H) continue;
          g.c_out[(size_t)r * g.H + j] = cn;
          g.h_out[(size_t)r * g.H + j] = h;
          for (int d = 0; d < g.dst.n; ++d) store_x(g.dst.x[d], r, g.dst.col[d] + j, h);
        }
      }
    } else {
      for (int it = threadIdx.x; it < kTileM * ncols; it += blockDim.x) {
        const int m = it % kTileM, c = it / kTileM;
        const int r = n0 + c_own + c, j = m0 + m;
        if (r >= g.n_valid || j >= g.M) continue;
        const float h = ds_tanh(red[(size_t)c * kTileM + m]);
        g.htilde[(size_t)r * g.M + j] = h;
        store_x(g.xg, r, j, h);
      }
    }
  }
  tc_fence_before();
}

// ---------------------------------------------------------------- attention phases
__device__ __forceinline__ void ds_cp_rows(float* dst, const float* src, int n) {
  const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 && (n & 3) == 0;
  if (al) {
    for (int i = threadIdx.x; i < (n >> 2); i += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 4 * i)), "l"(src + 4 * i)
                   : "memory");
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + i)), "l"(src + i) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// A1: CTA (b, chunk r): online softmax over positions [r*CH, min(S_b, (r+1)*CH)) for the K rows
template <int KMAX, int JPT>
__device__ __forceinline__ void ds_att_chunks(const DsAtt& a, uint8_t* buf8) {
  const int cta = blockIdx.x;
  if (cta >= a.B * a.nch) return;
  const int b = cta / a.nch, r = cta % a.nch;
  if (a.done && __ldcg(&a.done[b])) return;
  float* part = a.part + ((size_t)b * a.nch + r) * a.K * (2 + a.H);
  const int L = __ldg(&a.lens[b]);
  const int s_beg = r * a.CH, s_end = min(L, s_beg + a.CH);
  const bool same = a.keys == a.mem;
  const int H = a.H, K = a.K, SC = a.SC;
  const int kl = same ? H : a.key_ld;
  auto r4 = [](size_t n) { return (n + 3) & ~(size_t)3; };
  float* q = reinterpret_cast<float*>(buf8);
  float* s_m = q + r4((size_t)K * H);
  float* s_l = s_m + 16;
  float* s_scale = s_l + 16;
  float* e = s_scale + 16;                                        // [16][SC]
  float* bufs = e + 16 * 16;
  const size_t mb = r4((size_t)SC * H), kb = same ? 0 : r4((size_t)SC * kl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (s_end <= s_beg) {                                           // empty chunk
    for (int i = threadIdx.x; i < K * (2 + H); i += blockDim.x) {
      const int k = i / (2 + H), c = i % (2 + H);
      part[(size_t)k * (2 + H) + c] = c == 0 ? -INFINITY : 0.f;
    }
    return;
  }
  const int nsub = (s_end - s_beg + SC - 1) / SC;
  auto stage = [&](int i) {
    const int s0 = s_beg + i * SC;
    const int ns = min(SC, s_end - s0);
    float* mbp = bufs + (size_t)(i & 1) * (mb + kb);
    ds_cp_rows(mbp, a.mem + ((size_t)b * a.S_max + s0) * H, ns * H);
    if (!same) ds_cp_rows(mbp + mb, a.keys + ((size_t)b * a.S_max + s0) * a.key_ld, ns * a.key_ld);
  };
  ds_cp_rows(q, a.htop + (size_t)b * K * H, K * H);
  stage(0);
  if (nsub > 1) stage(1);
  if (threadIdx.x < 16) { s_m[threadIdx.x] = -INFINITY; s_l[threadIdx.x] = 0.f; }
  float acc[KMAX][JPT];
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int u = 0; u < JPT; ++u) acc[k][u] = 0.f;
  for (int i = 0; i < nsub; ++i) {
    if (i + 1 < nsub) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int s0 = s_beg + i * SC;
    const int ns = min(SC, s_end - s0);
    const float* ms = bufs + (size_t)(i & 1) * (mb + kb);
    const float* ks = same ? ms : ms + mb;
    for (int pos = warp; pos < ns; pos += nw) {                  // scores: one warp per position
      float d[KMAX];
#pragma unroll
      for (int k = 0; k < KMAX; ++k) d[k] = 0.f;
      const float* kr = ks + (size_t)pos * kl;
      for (int j = lane; j < H; j += 32) {
        const float kv = kr[j];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < K) d[k] = fmaf(q[(size_t)k * H + j], kv, d[k]);
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d[k] += __shfl_xor_sync(0xffffffffu, d[k], o);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < K) e[k * SC + pos] = d[k];
      }
    }
    __syncthreads();
    for (int k = warp; k < K; k += nw) {                         // online softmax per beam row
      const float v = lane < ns ? e[k * SC + lane] : -INFINITY;
      float mx = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mo = s_m[k];
      const float mn = fmaxf(mo, mx);
      const float w = lane < ns ? expf(v - mn) : 0.f;
      float sum = w;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane < SC) e[k * SC + lane] = w;
      if (lane == 0) {
        const float sc = mo == -INFINITY ? 0.f : expf(mo - mn);
        s_scale[k] = sc;
        s_l[k] = s_l[k] * sc + sum;
        s_m[k] = mn;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < JPT; ++u) {                              // context: thread owns columns j
      const int j = threadIdx.x + u * blockDim.x;
      if (j >= H) continue;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) acc[k][u] *= s_scale[k];
      for (int s = 0; s < ns; ++s) {
        const float mv = ms[(size_t)s * H + j];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < K) acc[k][u] = fmaf(e[k * SC + s], mv, acc[k][u]);
      }
    }
    __syncthreads();
    if (i + 2 < nsub) stage(i + 2);
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    part[(size_t)k * (2 + H)] = s_m[k];
    part[(size_t)k * (2 + H) + 1] = s_l[k];
  }
#pragma unroll
  for (int u = 0; u < JPT; ++u) {
    const int j = threadIdx.x + u * blockDim.x;
    if (j >= H) continue;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) part[(size_t)k * (2 + H) + 2 + j] = acc[k][u];
  }
}

// A2: CTA (b, slice r): context columns [j0, j1) of the K rows over the nch chunks (fixed order)
__device__ __forceinline__ void ds_att_combine(const DsAtt& a) {
  const int cta = blockIdx.x;
  if (cta >= a.B * a.nch) return;
  const int b = cta / a.nch, r = cta % a.nch;
  if (a.done && __ldcg(&a.done[b])) return;
  const int H = a.H, K = a.K, nch = a.nch;
  __shared__ float s_coef[8][16];
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    float mp[8], lp[8];
    float M = -INFINITY;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const float* pp = a.part + (((size_t)b * nch + p) * K + k) * (2 + H);
      mp[p] = p < nch ? __ldcg(pp) : -INFINITY;
      lp[p] = p < nch ? __ldcg(pp + 1) : 0.f;
      M = fmaxf(M, mp[p]);
    }
    float Ls = 0.f;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      mp[p] = mp[p] == -INFINITY ? 0.f : expf(mp[p] - M);
      Ls += lp[p] * mp[p];
    }
    const float inv = 1.f / Ls;
#pragma unroll
    for (int p = 0; p < 8; ++p) s_coef[p][k] = mp[p] * inv;
  }
  __syncthreads();
  const int j0 = (int)((long long)H * r / nch), j1 = (int)((long long)H * (r + 1) / nch);
  const int wj = j1 - j0;
  for (int it = threadIdx.x; it < K * wj; it += blockDim.x) {
    const int k = it / wj, j = j0 + it % wj;
    float v[8];
#pragma unroll
    for (int p = 0; p < 8; ++p)
      v[p] = p < nch ? __ldcg(a.part + (((size_t)b * nch + p) * K + k) * (2 + H) + 2 + j) : 0.f;
    float c = 0.f;
#pragma unroll
    for (int p = 0; p < 8; ++p) c = fmaf(s_coef[p][k], v[p], c);
    store_x(a.xo, b * K + k, j, c);
  }
}

// ---------------------------------------------------------------- the kernel
template <int KMAX, int JPT>
__global__ void __launch_bounds__(256, 1) dec_step_kernel(const __grid_constant__ DsArgs a) {
  KT(0);
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  __shared__ uint32_t s_tslot;
  const int warp = threadIdx.x >> 5;
  const int n_gemm = a.n_cell + 1;
  // ---- prologue (overlaps the predecessor): barriers, TMEM, every phase's weight slots
  if (threadIdx.x == 0) {
    for (int p = 0; p < n_gemm; ++p) {
      tma_prefetch_desc(&a.g[p].tmW);
      tma_prefetch_desc(&a.g[p].tmX);
      for (int i = 0; i < kDsBarsPerPhase; ++i) mbar_init(bars + p * kDsBarsPerPhase + i, 1);
    }
    fence_mbar_init();
    for (int p = 0; p < n_gemm; ++p) {
      const DsGemm& g = a.g[p];
      if ((int)blockIdx.x >= g.tiles * g.S) continue;
      const int tile = blockIdx.x / g.S, split = blockIdx.x % g.S;
      const int mt = tile / (g.n_rows_pad / g.n_group);
      const int kb0 = split * g.kbps;
      const int nkb = max(0, min(g.kbps, g.k_blocks - kb0));
      if (nkb == 0) continue;
      uint64_t* wbar = bars + p * kDsBarsPerPhase;
      mbar_arrive_expect_tx(wbar, nkb * kTileM * 128);
      for (int i = 0; i < nkb; ++i)
        tma_load_2d(smem + g.w_off + (size_t)i * kTileM * 128, &g.tmW, (kb0 + i) * kBK, mt * kTileM, wbar);
    }
  }
  if (warp == 0) tmem_alloc_dyn(&s_tslot, 256);
  tc_fence_before();
  pdl_wait();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tslot;
  if (all_done(a.ctl)) {                                          // uniform: drain the prefetches, leave
    if (threadIdx.x == 0)
      for (int p = 0; p < n_gemm; ++p) {
        const DsGemm& g = a.g[p];
        if ((int)blockIdx.x >= g.tiles * g.S) continue;
        const int nkb = max(0, min(g.kbps, g.k_blocks - (int)(blockIdx.x % g.S) * g.kbps));
        if (nkb > 0) mbar_wait(bars + p * kDsBarsPerPhase, 0);
      }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
    return;
  }
  KT(1);
  for (int l = 0; l < a.n_cell; ++l) {
    ds_gemm_phase(a.g[l], smem, bars + l * kDsBarsPerPhase, tmem, a.b_off, a.side_off);
    KT(2 + 2 * (l & 1));
    ds_grid_sync(a.gbar);
    KT(3 + 2 * (l & 1));
    tc_fence_after();
  }
  ds_att_chunks<KMAX, JPT>(a.att, smem + a.b_off);
  KT(6);
  ds_grid_sync(a.gbar);
  KT(7);
  ds_att_combine(a.att);
  KT(8);
  ds_grid_sync(a.gbar);
  KT(9);
  tc_fence_after();
  ds_gemm_phase(a.g[a.n_cell], smem, bars + a.n_cell * kDsBarsPerPhase, tmem, a.b_off, a.side_off);
  KT(10);
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
  KT(11);
}

#ifdef ONMT_KTRACE
void dec_step_set_trace(unsigned long long* p) { cudaMemcpyToSymbol(g_ktrace, &p, sizeof(p)); }
#else
void dec_step_set_trace(unsigned long long*) {}
#endif

// ---------------------------------------------------------------- host side
struct DsPlanOut {
  bool ok;
  size_t smem;
};

// choose split S for a GEMM phase (tiles * S <= num_sms, K blocks per split <= kDsMaxKbps)
static bool ds_split(DsGemm& g, int num_sms) {
  for (int S = 16; S >= 1; --S) {
    const int kbps = (g.k_blocks + S - 1) / S;
    if ((g.k_blocks + kbps - 1) / kbps != S) continue;
    if (g.tiles * S > num_sms) continue;
    if (kbps > kDsMaxKbps) continue;
    int NC = (g.n_group + S - 1) / S;
    NC = (NC + 3) / 4 * 4;
    g.S = S;
    g.kbps = kbps;
    g.NC = NC;
    return true;
  }
  return false;
}



static bool ds_build(DsArgs& a, const DsGemmSpec* specs, int n_cell, const DsAtt& att, unsigned int* gbar,
                     StepCtl ctl, int num_sms, size_t& smem_out, size_t* scratch_floats) {
  if (n_cell + 1 > kDsMaxGemm) return false;
  a = DsArgs{};
  a.n_cell = n_cell;
  size_t off = 0;
  size_t bneed = 0;
  int nc_max = 0;
  for (int p = 0; p <= n_cell; ++p) {
    const DsGemmSpec& sp = specs[p];
    DsGemm& g = a.g[p];
    g.tmW = *sp.tmW;
    g.tmX = *sp.tmX;
    g.k_blocks = sp.k_blocks;
    g.n_group = sp.n_group;
    g.n_rows_pad = sp.n_rows_pad;
    g.n_valid = sp.n_valid;
    g.tiles = sp.m_pad / kTileM * (sp.n_rows_pad / sp.n_group);
    g.M = sp.M;
    if (g.n_group > 256) return false;
    if (!ds_split(g, num_sms)) return false;
    g.w_off = (uint32_t)off;
    off += (size_t)g.kbps * kTileM * 128;
    const size_t ring = (size_t)g.kbps * 2 * g.n_group * 128;
    const size_t recv = (size_t)(g.S + 1) * g.NC * kTileM * 4;
    bneed = std::max(bneed, std::max(ring, recv));
    nc_max = std::max(nc_max, g.NC);
    g.scratch = sp.scratch;
    g.counters = sp.counters;
    g.epi = sp.epi;
    g.bias = reinterpret_cast<const float4*>(sp.bias);
    g.cg = sp.cg;
    g.c_out = sp.c_out;
    g.h_out = sp.h_out;
    g.H = sp.H;
    g.dst = sp.dst;
    g.htilde = sp.htilde;
    g.xg = sp.xg;
    if (scratch_floats) *scratch_floats = std::max(*scratch_floats, (size_t)g.tiles * g.S * g.n_group * kTileM);
  }
  a.att = att;
  if (att.B * att.nch > num_sms) return false;
  {
    auto r4 = [](size_t n) { return (n + 3) & ~(size_t)3; };
    const bool same = att.keys == att.mem;
    const int kl = same ? att.H : att.key_ld;
    const size_t abytes = (r4((size_t)att.K * att.H) + 3 * 16 + 16 * 16 +
                           2 * (r4((size_t)att.SC * att.H) + (same ? 0 : r4((size_t)att.SC * kl)))) * 4;
    bneed = std::max(bneed, abytes);
  }
  off = (off + 1023) & ~(size_t)1023;
  a.b_off = (uint32_t)off;
  off += (bneed + 1023) & ~(size_t)1023;
  a.side_off = (uint32_t)off;
  off += 32 * 16 + (size_t)nc_max * 32 * 4;
  off = (off + 15) & ~(size_t)15;
  a.bar_off = (uint32_t)off;
  off += (size_t)kDsMaxGemm * kDsBarsPerPhase * 8;
  smem_out = off + 1024;
  a.gbar = gbar;
  a.ctl = ctl;
  return smem_out <= 227 * 1024 - 1024;
}

int dec_step_att_chunks(int B, int S_max, int num_sms) {
  int nch = num_sms / (B > 0 ? B : 1);
  nch = nch > 8 ? 8 : nch < 1 ? 1 : nch;
  const int cap = (S_max + 3) / 4;
  return nch > cap ? (cap < 1 ? 1 : cap) : nch;
}

// Plans (and, with st != nullptr, launches) the fused decoder step.  Returns
// cudaErrorInvalidConfiguration when the shapes do not fit (the caller then uses the
// per-layer kernels).
cudaError_t dec_step(const DsGemmSpec* specs, int n_cell, const DsAtt& att_in, unsigned int* gbar, StepCtl ctl,
                     int num_sms, size_t* scratch_floats, cudaStream_t st) {
  DsAtt att = att_in;
  att.nch = dec_step_att_chunks(att.B, att.S_max, num_sms);
  att.CH = (att.S_max + att.nch - 1) / att.nch;
  att.SC = 8;
  if (att.K > kKMax || att.H > 4 * 256) return cudaErrorInvalidConfiguration;
  DsArgs a;
  size_t smem = 0;
  if (!ds_build(a, specs, n_cell, att, gbar, ctl, num_sms, smem, scratch_floats)) return cudaErrorInvalidConfiguration;
  if (st == nullptr) return cudaSuccess;                          // (plan only)
#define ONMT_DS(KM, JP)                                                                                  \
  {                                                                                                     \
    auto fn = dec_step_kernel<KM, JP>;                                                                  \
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    if (e != cudaSuccess) return e;                                                                     \
    return launch_pdl(fn, dim3(num_sms), dim3(256), smem, st, a);                                       \
  }
  const bool wide = att.H > 512;
  if (att.K <= 1) { if (wide) ONMT_DS(1, 4) else ONMT_DS(1, 2) }
  if (att.K <= 2) { if (wide) ONMT_DS(2, 4) else ONMT_DS(2, 2) }
  if (att.K <= 4) { if (wide) ONMT_DS(4, 4) else ONMT_DS(4, 2) }
  if (att.K <= 8) { if (wide) ONMT_DS(8, 4) else ONMT_DS(8, 2) }
  if (wide) ONMT_DS(16, 4) else ONMT_DS(16, 2)
#undef ONMT_DS
}

}  // namespace onmt
