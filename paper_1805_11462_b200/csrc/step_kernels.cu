// Element-wise, attention and beam-bookkeeping kernels of the encoder and of one
// decoder step (DESIGN.md §2 rows A1-A11).  All reductions run in a fixed order, so a
// repeated call is bitwise identical.
#include <math_constants.h>

#include "beam_device.cuh"
#include "common.cuh"

namespace onmt {

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }
__device__ __forceinline__ float cell_sigm_fast(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float cell_tanh_fast(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

// Asynchronous global -> shared copy of n floats (cp.async, 16 B granules when aligned).
__device__ __forceinline__ void stage_async(float* dst, const float* src, int n) {
  const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (al) {
    const int n4 = n >> 2;
    for (int i = threadIdx.x; i < n4; i += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + 4 * i)),
                   "l"(src + 4 * i)
                   : "memory");
    for (int i = (n4 << 2) + threadIdx.x; i < n; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + i)),
                   "l"(src + i)
                   : "memory");
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + i)),
                   "l"(src + i)
                   : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Sum of `splits` split-K partials P[s*stride + off] with all loads in flight (up to 16).
__device__ __forceinline__ float sum_splits(const float* __restrict__ P, size_t stride, size_t off, int splits) {
  if (splits == 1) return __ldg(P + off);          // (one split: the sum is the partial itself)
  float v[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) v[s] = s < splits ? __ldg(P + s * stride + off) : 0.f;
  float a = 0.f;
#pragma unroll
  for (int s = 0; s < 16; ++s) a += v[s];
  return a;
}
__device__ __forceinline__ float4 sum_splits4(const float* __restrict__ P, size_t stride, size_t off, int splits) {
  if (splits == 1) return __ldg(reinterpret_cast<const float4*>(P + off));   // (c4's gate GEMMs: one split)
  float4 v[16];
#pragma unroll
  for (int s = 0; s < 16; ++s)
    v[s] = s < splits ? __ldg(reinterpret_cast<const float4*>(P + s * stride + off)) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int s = 0; s < 16; ++s) { a.x += v[s].x; a.y += v[s].y; a.z += v[s].z; a.w += v[s].w; }
  return a;
}


// ------------------------------------------------------------------ encoder (A1-A4)
// A1: source embedding gather into the layer-0 input operand, rows b*S_max + s.
__global__ void embed_gather_kernel(const float* __restrict__ emb, int E, const int* __restrict__ ids,
                                    const int* __restrict__ lens, int S_max, XOut x) {
  const int row = blockIdx.x;
  const int b = row / S_max, s = row % S_max;
  if (s >= lens[b]) return;
  const int id = ids[row];
  const float* e = emb + (size_t)id * E;
  for (int c = threadIdx.x; c < E; c += blockDim.x) store_x(x, row, c, e[c]);
}

// A3: one recurrence step of one direction for every sentence (P129-133; AMB-3 packed
// semantics: sentence b is frozen for t >= S_b, the backward direction starts at
// S_b - 1).  Gate pre-activations: Z (hoisted input projection, A2) + recurrent
// partials + (b_ih + b_hh); gate rows are interleaved as 4*j + {i,f,g,o}.
__global__ void enc_cell_kernel(const float* __restrict__ Z, int z_ld, const float* __restrict__ P, int splits,
                                int p_rows_pad, int p_ld, const float4* __restrict__ bias, int Hd, int B,
                                const int* __restrict__ lens, int S_max, int t, int backward, float* h_st,
                                float* c_st, int st_ld, XOut xrec, XOut xnext, int next_col, float* mem,
                                int mem_ld, int mem_col) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * Hd) return;
  const int b = idx / Hd, j = idx % Hd;
  const int L = lens[b];
  if (t >= L) return;
  const int pos = backward ? L - 1 - t : t;
  const int row = b * S_max + pos;
  float4 g = reinterpret_cast<const float4*>(Z + (size_t)row * z_ld)[j];
  const float4 bb = bias[j];
  g.x += bb.x; g.y += bb.y; g.z += bb.z; g.w += bb.w;
  if (P) {
    const float4 p = sum_splits4(P, (size_t)p_rows_pad * p_ld, (size_t)b * p_ld + 4 * j, splits);
    g.x += p.x; g.y += p.y; g.z += p.z; g.w += p.w;
  }
  const float i = sigm(g.x), f = sigm(g.y), gg = tanhf(g.z), o = sigm(g.w);
  float* cp = c_st + (size_t)b * st_ld + j;
  float* hp = h_st + (size_t)b * st_ld + j;
  const float c = f * (t == 0 ? 0.f : *cp) + i * gg;
  const float h = o * tanhf(c);
  *cp = c;
  *hp = h;
  store_x(xrec, b, j, h);
  if (xnext.f32 || xnext.hl) store_x(xnext, row, next_col + j, h);
  if (mem) mem[(size_t)row * mem_ld + mem_col + j] = h;
}

// ------------------------------------------------------------------ decoder step
// A6: LSTM cell of decoder layer l over all R rows; c_prev already gathered by parent.

template <bool ONE>   // ONE: a single split (c4's gate GEMMs): no 16-way split-sum registers
__global__ void dec_cell_kernel(const float* __restrict__ P, int splits, int p_rows_pad, int p_ld,
                                const float4* __restrict__ bias, const float* __restrict__ cg, float* c_out,
                                float* h_out, int H, int R, CellDst dst, StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  if (all_done(ctl)) return;
  // two (row, unit) items per thread, idx and idx + half, with both items' loads issued before
  // either's math (one wave at c4 instead of two, twice the loads in flight per thread)
  const int n = R * H, half = (n + 1) / 2;
  const int idx0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx0 >= half) return;
  const bool fast = dst.n > 0 && dst.x[0].hl;
  float4 g[2];
  float cp[2];
  int rr[2], jj[2];
  bool ok[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int idx = idx0 + e * half;
    ok[e] = idx < n;
    rr[e] = ok[e] ? idx / H : 0;
    jj[e] = ok[e] ? idx % H : 0;
    g[e] = bias[jj[e]];
    const size_t off = (size_t)rr[e] * p_ld + 4 * jj[e];
    const float4 p = ONE ? __ldg(reinterpret_cast<const float4*>(P + off))
                         : sum_splits4(P, (size_t)p_rows_pad * p_ld, off, splits);
    g[e].x += p.x; g[e].y += p.y; g[e].z += p.z; g[e].w += p.w;
    cp[e] = cg[(size_t)rr[e] * H + jj[e]];
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    if (!ok[e]) continue;
    const int r = rr[e], j = jj[e];
    // bf16 models: the fused cell's fast exponentials (rel. error ~2^-21; IEEE expf / tanhf made
    // this kernel instruction-bound: 570 instructions per thread at c4); fp32 models keep them
    float i, f, gg, o, c, h;
    if (fast) {
      i = cell_sigm_fast(g[e].x); f = cell_sigm_fast(g[e].y); gg = cell_tanh_fast(g[e].z); o = cell_sigm_fast(g[e].w);
      c = f * cp[e] + i * gg;
      h = o * cell_tanh_fast(c);
    } else {
      i = sigm(g[e].x); f = sigm(g[e].y); gg = tanhf(g[e].z); o = sigm(g[e].w);
      c = f * cp[e] + i * gg;
      h = o * tanhf(c);
    }
    c_out[(size_t)r * H + j] = c;
    h_out[(size_t)r * H + j] = h;
#pragma unroll
    for (int d = 0; d < 2; ++d)                    // (static indices: no local-memory copy of dst)
      if (d < dst.n) store_x(dst.x[d], r, dst.col[d] + j, h);
  }
}

// A8: h~ = tanh(W_out [c ; h]) (P69; AMB-9) from split-K partials; writes h~ (fp32, for
// the next step's input feed) and the generator operand.
__global__ void attn_out_kernel(const float* __restrict__ P, int splits, int p_rows_pad, int p_ld, float* htilde,
                                int H, int R, XOut xg, StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  if (all_done(ctl)) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * H) return;
  const int r = idx / H, j = idx % H;
  const float v = sum_splits(P, (size_t)p_rows_pad * p_ld, (size_t)r * p_ld + j, splits);
  const float h = xg.hl ? cell_tanh_fast(v) : tanhf(v);       // (bf16 models: as the fused tanh epilogue)
  htilde[(size_t)r * H + j] = h;
  store_x(xg, r, j, h);
}

// ------------------------------------------------------------------ beam state

// A4 + O7: slot 0 live with cum 0, y = BOS; decoder state of every slot = the encoder's
// final state of its sentence (layer-wise, [fwd;bwd]); h~_0 = 0.
__global__ void init_decode_kernel(BeamState bs, int B, int K, const float* __restrict__ enc_h,
                                   const float* __restrict__ enc_c, int L, int H, float* dec_h, float* dec_c,
                                   int dec_rows_pad, float* htilde) {
  const int r = blockIdx.x;       // row b*K + k
  const int b = r / K, k = r % K;
  if (threadIdx.x == 0) {
    const int R = gridDim.x;
    bs.cum[R + r] = k == 0 ? 0.0 : -CUDART_INF;     // slot state of step t lives in buffer t & 1
    bs.live[R + r] = k == 0;
    bs.y[r] = 2;  // BOS
    bs.prow[r] = r;
    if (k == 0) {
      bs.done[b] = 0;
      const int nb = bs.nbest > 0 ? bs.nbest : 1;
      for (int i = 0; i < nb; ++i) {
        bs.best_t[b * nb + i] = 0;
        bs.best_r[b * nb + i] = 0;
        bs.best_raw[b * nb + i] = -CUDART_INF;
        bs.best_norm[b * nb + i] = -CUDART_INF;
      }
      if (b == 0) *bs.n_done = 0;
    }
  }
  if (bs.catt)                                       // step 1 reads buffer 1 (empty history)
    for (int s = threadIdx.x; s < bs.S_max; s += blockDim.x) bs.catt[((size_t)gridDim.x + r) * bs.S_max + s] = 0.f;
  for (int l = 0; l < L; ++l) {
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
      dec_h[((size_t)l * dec_rows_pad + r) * H + j] = enc_h[((size_t)l * B + b) * H + j];
      dec_c[((size_t)l * dec_rows_pad + r) * H + j] = enc_c[((size_t)l * B + b) * H + j];
    }
  }
  for (int j = threadIdx.x; j < H; j += blockDim.x) htilde[(size_t)r * H + j] = 0.f;
}

// A5: the next step's decoder inputs, gathered by parent row: x1 = [E_tgt[y]; h~[p];
// h_0[p]], x_l = [. ; h_l[p]] for l >= 1, c_prev of every layer.

__global__ void gather_kernel(BeamState bs, GatherArgs g, int K, StepCtl ctl) {
  if (all_done(ctl)) return;
  const int r = blockIdx.x;
  if (bs.done[r / K]) return;
  const int p = bs.prow[r];
  const int y = bs.y[r];
  const float* e = g.emb_tgt + (size_t)y * g.E;
  for (int c = threadIdx.x; c < g.E; c += blockDim.x) store_x(g.x[0], r, c, e[c]);
  for (int j = threadIdx.x; j < g.H; j += blockDim.x) {
    store_x(g.x[0], r, g.E + j, g.htilde[(size_t)p * g.H + j]);
    for (int l = 0; l < g.L; ++l) {
      const size_t src = ((size_t)l * g.rows_pad + p) * g.H + j;
      const size_t dst = ((size_t)l * g.rows_pad + r) * g.H + j;
      const float hv = g.h[src];
      if (l == 0) store_x(g.x[0], r, g.E + g.H + j, hv);
      else store_x(g.x[l], r, g.H + j, hv);
      g.cg[dst] = g.c[src];
    }
  }
}

// A10 + O8-O10: per sentence, combine the generator partials into the row LSE and the
// row top-K, select the K best (raw desc, slot asc, token asc) over live slots with
// fp64 cumulative scores, bank EOS picks and everything at t = max_len, update the
// stop flag and the histories.  One CTA per sentence, one warp per beam row.
// A10a: per hypothesis row, combine the generator partials (one per generator CTA) into
// the row log-sum-exp and the row top-K (z desc, id asc).  One 128-thread CTA per row;
// every thread issues all loads of its partials before using any of them.
template <int KMAX>
__global__ void __launch_bounds__(128) row_reduce_topk_kernel(const float2* __restrict__ ms,
                                                              const float* __restrict__ tz,
                                                              const int* __restrict__ ti, int n_parts, int ps, int rs,
                                                              int K, const int* __restrict__ live,
                                                              float* __restrict__ row_lse, float* __restrict__ row_z,
                                                              int* __restrict__ row_i, StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  if (all_done(ctl)) return;
  const int r = blockIdx.x;
  if (live && !live[r]) return;                 // (live = this step's buffer)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float s_m[4], s_s[4];
  __shared__ float s_wz[4];
  __shared__ int s_wi[4];
  // ---- loads: up to 2 partials per thread, all in flight
  float2 p[2];
  float cz[2][KMAX];
  int cid[2][KMAX];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int v = threadIdx.x + u * 128;
    const bool ok = v < n_parts;
    p[u] = ok ? __ldg(&ms[(size_t)v * ps + (size_t)r * rs]) : make_float2(-INFINITY, 0.f);
    const size_t base = ((size_t)v * ps + (size_t)r * rs) * K;
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
      cz[u][c] = (ok && c < K) ? __ldg(&tz[base + c]) : -INFINITY;
      cid[u][c] = (ok && c < K) ? __ldg(&ti[base + c]) : 0x7fffffff;
    }
  }
  for (int v = threadIdx.x + 256; v < n_parts; v += 128) {       // (more than 256 partials: rare)
    const float2 q = __ldg(&ms[(size_t)v * ps + (size_t)r * rs]);
    if (q.x > p[0].x) { p[0].y = p[0].y * expf(p[0].x - q.x) + q.y; p[0].x = q.x; }
    else if (q.x > -INFINITY) p[0].y += q.y * expf(q.x - p[0].x);
    const size_t base = ((size_t)v * ps + (size_t)r * rs) * K;
    for (int c = 0; c < K; ++c) {
      float z = __ldg(&tz[base + c]);
      int id = __ldg(&ti[base + c]);
#pragma unroll
      for (int i = 0; i < KMAX; ++i)
        if (better(z, id, cz[0][i], cid[0][i])) {
          const float a1 = cz[0][i]; const int a2 = cid[0][i];
          cz[0][i] = z; cid[0][i] = id; z = a1; id = a2;
        }
    }
  }
  // ---- log-sum-exp
  float m = fmaxf(p[0].x, p[1].x), sum = 0.f;
#pragma unroll
  for (int u = 0; u < 2; ++u)
    if (p[u].x > -INFINITY) sum += p[u].y * expf(p[u].x - m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
    const float M = fmaxf(m, m2);
    sum = (m == -INFINITY ? 0.f : sum * expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - M));
    m = M;
  }
  if (lane == 0) { s_m[warp] = m; s_s[warp] = sum; }
  // ---- top-K: each thread merges its two sorted lists, then K rounds of block argmax
  float lz[KMAX];
  int li[KMAX];
  {
    int a = 0, b2 = 0;
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      const bool ta = better(cz[0][a < KMAX ? a : KMAX - 1], cid[0][a < KMAX ? a : KMAX - 1],
                             cz[1][b2 < KMAX ? b2 : KMAX - 1], cid[1][b2 < KMAX ? b2 : KMAX - 1]);
      // (static-index selects over the two heads keep the lists in registers)
      float za = -INFINITY, zb = -INFINITY;
      int ia = 0x7fffffff, ib = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < KMAX; ++q) {
        if (q == a) { za = cz[0][q]; ia = cid[0][q]; }
        if (q == b2) { zb = cz[1][q]; ib = cid[1][q]; }
      }
      (void)ta;
      const bool takea = better(za, ia, zb, ib);
      lz[i] = takea ? za : zb;
      li[i] = takea ? ia : ib;
      a += takea;
      b2 += !takea;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = s_m[0];
    for (int w = 1; w < 4; ++w) M = fmaxf(M, s_m[w]);
    float S = 0.f;
    for (int w = 0; w < 4; ++w)
      if (s_m[w] > -INFINITY) S += s_s[w] * expf(s_m[w] - M);
    row_lse[r] = M + logf(S);
  }
  for (int c = 0; c < K; ++c) {
    float bz = lz[0];
    int bi = li[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float z2 = __shfl_xor_sync(0xffffffffu, bz, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(z2, i2, bz, bi)) { bz = z2; bi = i2; }
    }
    if (lane == 0) { s_wz[warp] = bz; s_wi[warp] = bi; }
    __syncthreads();
    float wz = s_wz[0];
    int wi = s_wi[0];
#pragma unroll
    for (int w = 1; w < 4; ++w)
      if (better(s_wz[w], s_wi[w], wz, wi)) { wz = s_wz[w]; wi = s_wi[w]; }
    if (threadIdx.x == 0) { row_z[(size_t)r * K + c] = wz; row_i[(size_t)r * K + c] = wi; }
    if (li[0] == wi && lz[0] == wz) {                            // the owner pops its head
#pragma unroll
      for (int i = 0; i < KMAX - 1; ++i) { lz[i] = lz[i + 1]; li[i] = li[i + 1]; }
      lz[KMAX - 1] = -INFINITY; li[KMAX - 1] = 0x7fffffff;
    }
    __syncthreads();
  }
}

template <int KMAX>
__global__ void __launch_bounds__(128) beam_select_gather_kernel(const float* __restrict__ row_lse,
                                                                 const float* __restrict__ row_z,
                                                                 const int* __restrict__ row_i, int K, int t,
                                                                 int max_len, double lp, BeamState bs, GatherArgs ga,
                                                                 int nslice, StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  // no all_done() here: another CTA of this launch may finish the last sentence; only
  // completions of earlier steps (done[b] < t) may skip work
  (void)ctl;
  select_gather_row<KMAX>(blockIdx.x, blockIdx.y, nslice, gridDim.x, row_lse, row_z, row_i, K, t, max_len, lp, bs, ga);
}

// A11 + O11: backtrack the banked best entry of each sentence.
__global__ void finalize_kernel(BeamState bs, int B, int K, int max_len, int* hyps, int* lens, float* scores,
                                float* raw, float* tlogp, int* unk_pos) {
  // one thread per (sentence b, n-best rank i); output row o = b * nbest + i
  const int nb = bs.nbest > 0 ? bs.nbest : 1;
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= B * nb) return;
  const int b = o / nb;
  const int T = bs.best_t[o];                        // 0: fewer than i + 1 entries were banked
  int r = bs.best_r[o];
  for (int t = max_len; t > T; --t) {
    hyps[(size_t)o * max_len + t - 1] = 0;
    if (tlogp) tlogp[(size_t)o * max_len + t - 1] = 0.f;
    if (unk_pos) unk_pos[(size_t)o * max_len + t - 1] = -1;
  }
  for (int t = T; t >= 1; --t) {
    const size_t h = (size_t)(t - 1) * B * K + (size_t)b * K + r;
    const int w = bs.hist_token[h];
    hyps[(size_t)o * max_len + t - 1] = w;
    if (tlogp) tlogp[(size_t)o * max_len + t - 1] = bs.hist_logp[h];
    // S448: an <unk> emitted at step t is replaced by the source word at argmax_s a_{t,s}
    if (unk_pos) unk_pos[(size_t)o * max_len + t - 1] = (w == 1 && bs.hist_amax) ? bs.hist_amax[h] : -1;
    r = bs.hist_parent[h];
  }
  lens[o] = T;
  scores[o] = T ? (float)bs.best_norm[o] : -INFINITY;
  if (raw) raw[o] = T ? (float)bs.best_raw[o] : -INFINITY;
}

// ------------------------------------------------------------------ host launchers
void launch_embed_gather(const float* emb, int E, const int* ids, const int* lens, int B, int S_max, XOut x,
                         cudaStream_t st) {
  embed_gather_kernel<<<B * S_max, 128, 0, st>>>(emb, E, ids, lens, S_max, x);
}

void launch_enc_cell(const float* Z, int z_ld, const float* P, int splits, int p_rows_pad, int p_ld,
                     const float* bias, int Hd, int B, const int* lens, int S_max, int t, int backward, float* h_st,
                     float* c_st, int st_ld, XOut xrec, XOut xnext, int next_col, float* mem, int mem_ld,
                     int mem_col, cudaStream_t st) {
  const int n = B * Hd;
  enc_cell_kernel<<<(n + 255) / 256, 256, 0, st>>>(Z, z_ld, P, splits, p_rows_pad, p_ld, (const float4*)bias, Hd, B,
                                                   lens, S_max, t, backward, h_st, c_st, st_ld, xrec, xnext,
                                                   next_col, mem, mem_ld, mem_col);
}

void launch_dec_cell(const float* P, int splits, int p_rows_pad, int p_ld, const float* bias, const float* cg,
                     float* c_out, float* h_out, int H, int R, CellDst dst, StepCtl ctl, cudaStream_t st) {
  const int n = (R * H + 1) / 2;                    // (two items per thread)
  launch_pdl(splits == 1 ? dec_cell_kernel<true> : dec_cell_kernel<false>, dim3((n + 255) / 256), dim3(256), 0, st, P,
             splits, p_rows_pad, p_ld, (const float4*)bias, cg, c_out, h_out, H, R, dst, ctl);
}



void launch_attn_out(const float* P, int splits, int p_rows_pad, int p_ld, float* htilde, int H, int R, XOut xg,
                     StepCtl ctl, cudaStream_t st) {
  const int n = R * H;
  launch_pdl(attn_out_kernel, dim3((n + 255) / 256), dim3(256), 0, st, P, splits, p_rows_pad, p_ld, htilde, H, R, xg,
             ctl);
}

void launch_init_decode(const BeamState& bs, int B, int K, const float* enc_h, const float* enc_c, int L, int H,
                        float* dec_h, float* dec_c, int dec_rows_pad, float* htilde, cudaStream_t st) {
  init_decode_kernel<<<B * K, 128, 0, st>>>(bs, B, K, enc_h, enc_c, L, H, dec_h, dec_c, dec_rows_pad, htilde);
}

void launch_gather(const BeamState& bs, const GatherArgs& g, int R, int K, StepCtl ctl, cudaStream_t st) {
  gather_kernel<<<R, 128, 0, st>>>(bs, g, K, ctl);
}

constexpr size_t kBeamStageBytes = 216 * 1024;  // shared staging of the gathered / prefetched rows

template <int KMAX>
__global__ void __launch_bounds__(512) beam_step_kernel(const float2* __restrict__ ms, const float* __restrict__ tz,
                                                        const int* __restrict__ ti, int n_parts, int ps, int rs, int K,
                                                        int t, int max_len, double lp, BeamState bs, GatherArgs ga,
                                                        StepCtl ctl, VpWait vw) {
  KT(0);
  pdl_trigger();
  pdl_wait();
  (void)ctl;
  if (vw.flags) {
    // vocabulary-parallel: every rank's generator CTAs raised their flag for this step in my
    // exchange buffer (their partials landed before it: release / acquire at system scope)
    if (threadIdx.x < 32) {
      const unsigned long long ep = vp_epoch(vw.seq, t);
      const unsigned long long t0 = spin_clock();
      unsigned int it = 0;
      for (int i = threadIdx.x; i < vw.n; i += 32)
        while (true) {
          unsigned long long v;
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(vw.flags + i) : "memory");
          if (v == ep) break;
          spin_check(t0, it);
        }
    }
    __syncthreads();
  }
  extern __shared__ __align__(16) float gbuf_dyn[];
  beam_step_sentence<KMAX>(blockIdx.x, ms, tz, ti, n_parts, ps, rs, K, gridDim.x * K, t, max_len, lp, bs, ga,
                           gbuf_dyn, (int)(kBeamStageBytes / 4), blockIdx.y, gridDim.y);
}

void launch_beam_merge(const float2* ms, const float* tz, const int* ti, int n_parts, int ps, int rs, int B, int K,
                       int t, int max_len, double lp, const BeamState& bs, const GatherArgs& ga, float* row_lse,
                       float* row_z, int* row_i, StepCtl ctl, cudaStream_t st, int nslice, const VpWait* vw) {
  const VpWait vwv = vw ? *vw : VpWait{nullptr, 0, nullptr};
  const int R = B * K;
  // one CTA per sentence (row reduce + select + gather) when its lanes hold every partial;
  // otherwise (SIMT generator over many tiles) a row-reduce launch + a select/gather launch
#define ONMT_MERGE(KM)                                                                                            \
  if (n_parts <= 256) {                                                                                           \
    cudaFuncSetAttribute(beam_step_kernel<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBeamStageBytes); \
    launch_pdl(beam_step_kernel<KM>, dim3(B, nslice), dim3(512), kBeamStageBytes, st, ms, tz, ti, n_parts, ps, rs,  \
               K, t,                                                                                              \
               max_len, lp, bs, ga, ctl, vwv);                                                                    \
  } else {                                                                                                        \
    launch_pdl(row_reduce_topk_kernel<KM>, dim3(R), dim3(128), 0, st, ms, tz, ti, n_parts, ps, rs, K,             \
               bs.live + (size_t)(t & 1) * R, row_lse, row_z, row_i, ctl);                                        \
    launch_pdl(beam_select_gather_kernel<KM>, dim3(R, 4), dim3(128), 0, st, row_lse, row_z, row_i, K, t, max_len, \
               lp, bs, ga, 4, ctl);                                                                               \
  }
  if (K <= 1) { ONMT_MERGE(1) }
  else if (K <= 2) { ONMT_MERGE(2) }
  else if (K <= 4) { ONMT_MERGE(4) }
  else if (K == 5) { ONMT_MERGE(5) }
  else if (K <= 8) { ONMT_MERGE(8) }
  else if (K == 10) { ONMT_MERGE(10) }
  else { ONMT_MERGE(16) }
#undef ONMT_MERGE
}

// vocabulary-parallel: the call's sequence number (step epochs of the exchange flags)
__global__ void vp_seq_kernel(unsigned long long* seq) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *seq += 1ull;
}
void launch_vp_seq(unsigned long long* seq, cudaStream_t st) { vp_seq_kernel<<<1, 32, 0, st>>>(seq); }

// A11 with the sentence's history staged in shared memory: one CTA per sentence loads the
// (token, parent, log p, attention argmax) entries of its K slots for every step (coalesced),
// one thread per n-best rank walks the parent pointers on chip, then the CTA writes the
// outputs in parallel.  The thread-per-sentence walk over global memory paid one dependent
// L2 round trip per step (~144 us at max_len 100).
__global__ void __launch_bounds__(256) finalize_smem_kernel(BeamState bs, int B, int K, int max_len, int* hyps,
                                                            int* lens, float* scores, float* raw, float* tlogp,
                                                            int* unk_pos) {
  extern __shared__ int fz[];
  const int nb = bs.nbest > 0 ? bs.nbest : 1;
  const int b = blockIdx.x, R = B * K;
  const int n_hist = max_len * K;
  int* ptok = fz;
  int* ppar = ptok + n_hist;
  float* plp = reinterpret_cast<float*>(ppar + n_hist);
  int* pam = reinterpret_cast<int*>(plp + n_hist);
  int* path = pam + n_hist;                                      // [nb][max_len] slot per step
  __shared__ int s_T;
  if (threadIdx.x == 0) {
    int T = 0;
    for (int i = 0; i < nb; ++i) T = max(T, bs.best_t[b * nb + i]);
    s_T = T;
  }
  __syncthreads();
  const int T = s_T;
  for (int i = threadIdx.x; i < T * K; i += blockDim.x) {
    const int t = i / K, k = i % K;
    const size_t h = (size_t)t * R + (size_t)b * K + k;
    ptok[i] = bs.hist_token[h];
    ppar[i] = bs.hist_parent[h];
    plp[i] = bs.hist_logp[h];
    pam[i] = bs.hist_amax ? bs.hist_amax[h] : -1;
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    const int o = b * nb + threadIdx.x;
    const int Ti = bs.best_t[o];
    int r = bs.best_r[o];
    for (int t = Ti; t >= 1; --t) {
      path[threadIdx.x * max_len + t - 1] = r;
      r = ppar[(t - 1) * K + r];
    }
    lens[o] = Ti;
    scores[o] = Ti ? (float)bs.best_norm[o] : -INFINITY;
    if (raw) raw[o] = Ti ? (float)bs.best_raw[o] : -INFINITY;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb * max_len; i += blockDim.x) {
    const int rank = i / max_len, t = i % max_len;
    const int o = b * nb + rank;
    const int Ti = bs.best_t[o];
    const size_t oi = (size_t)o * max_len + t;
    if (t < Ti) {
      const int e = t * K + path[rank * max_len + t];
      const int w = ptok[e];
      hyps[oi] = w;
      if (tlogp) tlogp[oi] = plp[e];
      // S448: an <unk> emitted at step t is replaced by the source word at argmax_s a_{t,s}
      if (unk_pos) unk_pos[oi] = (w == 1 && bs.hist_amax) ? pam[e] : -1;
    } else {
      hyps[oi] = 0;
      if (tlogp) tlogp[oi] = 0.f;
      if (unk_pos) unk_pos[oi] = -1;
    }
  }
}

// the two halves of the split beam merge, separately (copy models run copy_rows_kernel between)
void launch_row_topk(const float2* ms, const float* tz, const int* ti, int n_parts, int ps, int rs, int B, int K, int t,
                     const BeamState& bs, float* row_lse, float* row_z, int* row_i, StepCtl ctl, cudaStream_t st) {
  const int R = B * K;
#define ONMT_RT(KM)                                                                                                \
  launch_pdl(row_reduce_topk_kernel<KM>, dim3(R), dim3(128), 0, st, ms, tz, ti, n_parts, ps, rs, K,                \
             bs.live + (size_t)(t & 1) * R, row_lse, row_z, row_i, ctl);
  if (K <= 1) { ONMT_RT(1) }
  else if (K <= 2) { ONMT_RT(2) }
  else if (K <= 4) { ONMT_RT(4) }
  else if (K == 5) { ONMT_RT(5) }
  else if (K <= 8) { ONMT_RT(8) }
  else if (K == 10) { ONMT_RT(10) }
  else { ONMT_RT(16) }
#undef ONMT_RT
}

void launch_select_gather(int B, int K, int t, int max_len, double lp, const BeamState& bs, const GatherArgs& ga,
                          const float* row_lse, const float* row_z, const int* row_i, StepCtl ctl, cudaStream_t st) {
  const int R = B * K;
#define ONMT_SG(KM)                                                                                                \
  launch_pdl(beam_select_gather_kernel<KM>, dim3(R, 4), dim3(128), 0, st, row_lse, row_z, row_i, K, t, max_len, lp, \
             bs, ga, 4, ctl);
  if (K <= 1) { ONMT_SG(1) }
  else if (K <= 2) { ONMT_SG(2) }
  else if (K <= 4) { ONMT_SG(4) }
  else if (K == 5) { ONMT_SG(5) }
  else if (K <= 8) { ONMT_SG(8) }
  else if (K == 10) { ONMT_SG(10) }
  else { ONMT_SG(16) }
#undef ONMT_SG
}

void launch_finalize(const BeamState& bs, int B, int K, int max_len, int* hyps, int* lens, float* scores, float* raw,
                     float* tlogp, int* unk_pos, cudaStream_t st) {
  const int nb = bs.nbest > 0 ? bs.nbest : 1;
  const size_t smem = ((size_t)4 * max_len * K + (size_t)nb * max_len) * 4;
  if (smem <= 200 * 1024) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(finalize_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    finalize_smem_kernel<<<B, 256, smem, st>>>(bs, B, K, max_len, hyps, lens, scores, raw, tlogp, unk_pos);
    return;
  }
  const int n = B * nb;
  finalize_kernel<<<(n + 127) / 128, 128, 0, st>>>(bs, B, K, max_len, hyps, lens, scores, raw, tlogp, unk_pos);
}

// Test helper (onmt_test_gen): per row, combine generator partials into the LSE and
// the top-k (z, id), one thread per row, sequential over tiles.
__global__ void row_reduce_kernel(const float2* __restrict__ ms, const float* __restrict__ tz,
                                  const int* __restrict__ ti, int n_vt, int ps, int rs, int R, int K, float* lse,
                                  float* oz, int* oi) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  float m = -INFINITY, s = 0.f;
  for (int v = 0; v < n_vt; ++v) {
    const float2 p = ms[(size_t)v * ps + (size_t)r * rs];
    if (p.x > m) { s = s * expf(m - p.x) + p.y; m = p.x; }
    else s += p.y * expf(p.x - m);
  }
  lse[r] = m + logf(s);
  float bz[kKMax];
  int bi[kKMax];
  for (int i = 0; i < K; ++i) { bz[i] = -INFINITY; bi[i] = 0x7fffffff; }
  for (int v = 0; v < n_vt; ++v)
    for (int c = 0; c < K; ++c) {
      float cz = tz[((size_t)v * ps + (size_t)r * rs) * K + c];
      int ci = ti[((size_t)v * ps + (size_t)r * rs) * K + c];
      for (int i = 0; i < K; ++i)
        if (better(cz, ci, bz[i], bi[i])) {
          float t1 = bz[i]; int t2 = bi[i];
          bz[i] = cz; bi[i] = ci; cz = t1; ci = t2;
        }
    }
  for (int i = 0; i < K; ++i) { oz[(size_t)r * K + i] = bz[i]; oi[(size_t)r * K + i] = bi[i]; }
}

void launch_row_reduce(const float2* ms, const float* tz, const int* ti, int n_vt, int ps, int rs, int R, int K,
                       float* lse, float* oz, int* oi, cudaStream_t st) {
  row_reduce_kernel<<<(R + 127) / 128, 128, 0, st>>>(ms, tz, ti, n_vt, ps, rs, R, K, lse, oz, oi);
}

}  // namespace onmt
