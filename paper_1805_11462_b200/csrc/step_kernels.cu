// Element-wise, attention and beam-bookkeeping kernels of the encoder and of one
// decoder step (DESIGN.md §2 rows A1-A11).  All reductions run in a fixed order, so a
// repeated call is bitwise identical.
#include <math_constants.h>

#include "common.cuh"

namespace onmt {

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }

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
  float v[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) v[s] = s < splits ? __ldg(P + s * stride + off) : 0.f;
  float a = 0.f;
#pragma unroll
  for (int s = 0; s < 16; ++s) a += v[s];
  return a;
}
__device__ __forceinline__ float4 sum_splits4(const float* __restrict__ P, size_t stride, size_t off, int splits) {
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

__global__ void dec_cell_kernel(const float* __restrict__ P, int splits, int p_rows_pad, int p_ld,
                                const float4* __restrict__ bias, const float* __restrict__ cg, float* c_out,
                                float* h_out, int H, int R, CellDst dst, StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  if (all_done(ctl)) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * H) return;
  const int r = idx / H, j = idx % H;
  float4 g = bias[j];
  const float4 p = sum_splits4(P, (size_t)p_rows_pad * p_ld, (size_t)r * p_ld + 4 * j, splits);
  g.x += p.x; g.y += p.y; g.z += p.z; g.w += p.w;
  const float i = sigm(g.x), f = sigm(g.y), gg = tanhf(g.z), o = sigm(g.w);
  const float c = f * cg[(size_t)r * H + j] + i * gg;
  const float h = o * tanhf(c);
  c_out[(size_t)r * H + j] = c;
  h_out[(size_t)r * H + j] = h;
  for (int d = 0; d < dst.n; ++d) store_x(dst.x[d], r, dst.col[d] + j, h);
}

// A7: Luong global attention (P119-122, P299-301).  'general' scores are
// e_s = (W_in h) . m_s = h . (W_in^T m_s): the key k_s = W_in^T m_s is computed once per
// batch right after the encoder (one tcgen05 GEMM over all source positions), so no
// per-step query GEMM exists; 'dot' uses k_s = m_s.  CTA (b, c) stages the keys and
// memory rows of its chunk of kAttCH source positions in shared memory (cp.async) and
// computes, for all K rows of sentence b, the scores, the chunk's (max, sum exp) and
// partial context.  The last CTA of the sentence (atomic ticket) combines the chunks in
// fixed order - softmax over s < S_b only, pads excluded - and writes the context into
// the first H columns of the W_out operand.
constexpr int kAttCH = 16;

template <int KMAX>
__global__ void __launch_bounds__(256) attention_kernel(const float* __restrict__ htop,
                                                        const float* __restrict__ keys, int key_ld,
                                                        const float* __restrict__ mem, const int* __restrict__ lens,
                                                        int S_max, int H, int K, XOut xo, const int* __restrict__ done,
                                                        float* __restrict__ part_m, float* __restrict__ part_s,
                                                        float* __restrict__ part_c, int* __restrict__ tickets,
                                                        StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  if (all_done(ctl)) return;
  const int b = blockIdx.x, ch = blockIdx.y, nch = gridDim.y;
  if (done && done[b]) return;
  extern __shared__ __align__(16) float sh[];
  const bool same = keys == mem;
  float* q = sh;                                  // [K][H]
  float* e = q + K * H;                           // [K][kAttCH]
  float* ms = e + K * kAttCH;                     // [kAttCH][H]
  float* ks = same ? ms : ms + kAttCH * H;        // [kAttCH][key_ld]
  __shared__ int s_last;
  const int L = lens[b];
  const int s0 = ch * kAttCH;
  const int ns = max(0, min(kAttCH, L - s0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const size_t pbase = ((size_t)b * nch + ch) * K;
  if (ns > 0) {
    stage_async(ms, mem + ((size_t)b * S_max + s0) * H, ns * H);
    if (!same) stage_async(ks, keys + ((size_t)b * S_max + s0) * key_ld, ns * key_ld);
    const float* __restrict__ hq = htop + (size_t)b * K * H;
    for (int i0 = threadIdx.x; i0 < K * H; i0 += 4 * blockDim.x) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * blockDim.x;
        v[u] = i < K * H ? __ldg(&hq[i]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * blockDim.x < K * H) q[i0 + u * blockDim.x] = v[u];
    }
    stage_wait();
    __syncthreads();
    const int kl = same ? H : key_ld;
    for (int s0w = 2 * warp; s0w < ns; s0w += 2 * nw) {   // one warp: 2 positions x K rows at once
      const bool two = s0w + 1 < ns;
      float acc0[KMAX], acc1[KMAX];
#pragma unroll
      for (int k = 0; k < KMAX; ++k) { acc0[k] = 0.f; acc1[k] = 0.f; }
      for (int j = lane; j < H; j += 32) {
        const float k0 = ks[s0w * kl + j];
        const float k1 = two ? ks[(s0w + 1) * kl + j] : 0.f;
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < K) {
            const float qv = q[k * H + j];
            acc0[k] = fmaf(qv, k0, acc0[k]);
            acc1[k] = fmaf(qv, k1, acc1[k]);
          }
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc0[k] += __shfl_xor_sync(0xffffffffu, acc0[k], o);
          acc1[k] += __shfl_xor_sync(0xffffffffu, acc1[k], o);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < K) {
            e[k * kAttCH + s0w] = acc0[k];
            if (two) e[k * kAttCH + s0w + 1] = acc1[k];
          }
      }
    }
    __syncthreads();
    for (int k = warp; k < K; k += nw) {              // chunk softmax statistics
      const float v = lane < ns ? e[k * kAttCH + lane] : -INFINITY;
      float mx = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float w = lane < ns ? expf(v - mx) : 0.f;
      float sum = w;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane < kAttCH) e[k * kAttCH + lane] = w;
      if (lane == 0) { part_m[pbase + k] = mx; part_s[pbase + k] = sum; }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
      float acc[KMAX];
#pragma unroll
      for (int k = 0; k < KMAX; ++k) acc[k] = 0.f;
      for (int sidx = 0; sidx < ns; ++sidx) {
        const float mv = ms[sidx * H + j];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < K) acc[k] = fmaf(e[k * kAttCH + sidx], mv, acc[k]);
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) part_c[(pbase + k) * H + j] = acc[k];
    }
  } else {
    for (int k = threadIdx.x; k < K; k += blockDim.x) { part_m[pbase + k] = -INFINITY; part_s[pbase + k] = 0.f; }
  }
  // last CTA of the sentence combines the chunks (deterministic order)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&tickets[b], 1) == nch - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const size_t b0 = (size_t)b * nch * K;
  float* s_w = e;                                 // reuse: [nch][K] normalised chunk weights
  if (nch * K > K * kAttCH + K * H) return;       // (cannot happen: nch <= 128)
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    float Mx = -INFINITY;
    for (int c = 0; c < nch; ++c) Mx = fmaxf(Mx, __ldcg(&part_m[b0 + c * K + k]));
    float S = 0.f;
    for (int c = 0; c < nch; ++c) {
      const float pm = __ldcg(&part_m[b0 + c * K + k]);
      const float w = pm == -INFINITY ? 0.f : expf(pm - Mx);
      s_w[c * K + k] = w;
      S += w * __ldcg(&part_s[b0 + c * K + k]);
    }
    const float inv = 1.f / S;
    for (int c = 0; c < nch; ++c) s_w[c * K + k] *= inv;
  }
  __syncthreads();
  for (int i0 = threadIdx.x; i0 < K * H; i0 += 2 * blockDim.x) {
    float C[2] = {0.f, 0.f};
    for (int c0 = 0; c0 < nch; c0 += 8) {           // 2 items x 8 chunks of L2 loads in flight
      float v[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = min(i0 + u * (int)blockDim.x, K * H - 1);
        const int k = i / H, j = i % H;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          v[u][cc] = c0 + cc < nch ? __ldcg(&part_c[(b0 + (c0 + cc) * K + k) * H + j]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = min(i0 + u * (int)blockDim.x, K * H - 1);
        const int k = i / H;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          if (c0 + cc < nch) C[u] += s_w[(c0 + cc) * K + k] * v[u][cc];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < K * H) store_x(xo, b * K + i / H, i % H, C[u]);
    }
  }
  if (threadIdx.x == 0) tickets[b] = 0;
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
  const float h = tanhf(v);
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
      bs.best_t[b] = 0;
      bs.best_r[b] = 0;
      bs.best_raw[b] = -CUDART_INF;
      bs.best_norm[b] = -CUDART_INF;
      if (b == 0) *bs.n_done = 0;
    }
  }
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
                                                              const int* __restrict__ ti, int n_parts, int rows_pad,
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
    p[u] = ok ? __ldg(&ms[(size_t)v * rows_pad + r]) : make_float2(-INFINITY, 0.f);
    const size_t base = ((size_t)v * rows_pad + r) * K;
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
      cz[u][c] = (ok && c < K) ? __ldg(&tz[base + c]) : -INFINITY;
      cid[u][c] = (ok && c < K) ? __ldg(&ti[base + c]) : 0x7fffffff;
    }
  }
  for (int v = threadIdx.x + 256; v < n_parts; v += 128) {       // (more than 256 partials: rare)
    const float2 q = __ldg(&ms[(size_t)v * rows_pad + r]);
    if (q.x > p[0].x) { p[0].y = p[0].y * expf(p[0].x - q.x) + q.y; p[0].x = q.x; }
    else if (q.x > -INFINITY) p[0].y += q.y * expf(q.x - p[0].x);
    const size_t base = ((size_t)v * rows_pad + r) * K;
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

// A10b + A5: per sentence b, the K best (raw desc, slot asc, token asc) of the K x K row
// candidates with fp64 cumulative scores (O8); EOS / max_len banking, stop flag,
// histories (O9, O10) - computed redundantly by every CTA of the sentence from a few
// hundred bytes of state - then each CTA gathers one column slice of the next step's
// decoder inputs of one row (x1 = [E_tgt[y]; h~[p]; h_0[p]], x_l = [.; h_l[p]], c_l[p]).
// CTA (row k, slice 0) of each sentence writes the beam state.
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
  const int r = blockIdx.x, slice = blockIdx.y;
  const int b = r / K, kr = r % K;
  const int dn = bs.done[b];
  if (dn != 0 && dn < t) return;
  const int R = gridDim.x;
  const int* __restrict__ live_in = bs.live + (size_t)(t & 1) * R;
  const double* __restrict__ cum_in = bs.cum + (size_t)(t & 1) * R;
  int* live_out = bs.live + (size_t)((t + 1) & 1) * R;
  double* cum_out = bs.cum + (size_t)((t + 1) & 1) * R;
  __shared__ int s_live[KMAX];
  __shared__ double s_cum[KMAX];
  __shared__ float s_lse[KMAX];
  __shared__ float s_z[KMAX][KMAX];
  __shared__ int s_id[KMAX][KMAX];
  __shared__ int s_prow, s_y, s_cont;
  if (threadIdx.x < K) {
    const int rr = b * K + threadIdx.x;
    s_live[threadIdx.x] = live_in[rr];
    s_cum[threadIdx.x] = cum_in[rr];
    s_lse[threadIdx.x] = row_lse[rr];
  }
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) {
    s_z[i / K][i % K] = row_z[(size_t)b * K * K + i];
    s_id[i / K][i % K] = row_i[(size_t)b * K * K + i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int head[KMAX];
    int sel_k[KMAX], sel_w[KMAX];
    double sel_s[KMAX];
    float sel_lp[KMAX];
    for (int k = 0; k < K; ++k) head[k] = 0;
    int n_sel = 0;
    for (int q = 0; q < K; ++q) {
      int bk = -1, bw = 0x7fffffff;
      double bsv = -CUDART_INF;
      for (int k = 0; k < K; ++k) {
        if (!s_live[k] || head[k] >= K) continue;
        const float z = s_z[k][head[k]];
        if (z == -INFINITY) continue;
        const double sc = s_cum[k] + ((double)z - (double)s_lse[k]);
        if (bk < 0 || sc > bsv) { bk = k; bsv = sc; bw = s_id[k][head[k]]; }
      }
      if (bk < 0) break;
      sel_k[n_sel] = bk; sel_w[n_sel] = bw; sel_s[n_sel] = bsv;
      sel_lp[n_sel] = (float)((double)s_z[bk][head[bk]] - (double)s_lse[bk]);
      ++n_sel;
      ++head[bk];
    }
    bool any_live = false;
    for (int q = 0; q < n_sel; ++q) any_live |= !(sel_w[q] == 3 || t == max_len);
    const bool stop = !any_live || t == max_len || (n_sel > 0 && sel_w[0] == 3);
    const bool mine_sel = kr < n_sel;
    const bool mine_live = mine_sel && !(sel_w[kr] == 3 || t == max_len);
    s_prow = mine_live ? b * K + sel_k[kr] : r;
    s_y = mine_live ? sel_w[kr] : 0;
    s_cont = !stop;
    if (slice == 0) {
      // this CTA owns slot kr of sentence b: slot state + history entry
      const size_t hb = (size_t)(t - 1) * (size_t)gridDim.x + (size_t)r;
      live_out[r] = mine_live;
      cum_out[r] = mine_live ? sel_s[kr] : -CUDART_INF;
      bs.prow[r] = s_prow;
      bs.y[r] = s_y;
      bs.hist_parent[hb] = mine_sel ? sel_k[kr] : -1;
      bs.hist_token[hb] = mine_sel ? sel_w[kr] : 0;
      bs.hist_logp[hb] = mine_sel ? sel_lp[kr] : 0.f;
      if (bs.sel_parent) { bs.sel_parent[hb] = mine_sel ? sel_k[kr] : -1; bs.sel_score[hb] = mine_sel ? sel_s[kr] : -CUDART_INF; }
      if (kr == 0) {                                   // sentence-level banking and stop flag
        int bt = bs.best_t[b], br = bs.best_r[b];
        double braw = bs.best_raw[b], bnorm = bs.best_norm[b];
        for (int q = 0; q < n_sel; ++q) {
          if (sel_w[q] == 3 || t == max_len) {
            const double norm = sel_s[q] / lp;
            if (bt == 0 || norm > bnorm) { bt = t; br = q; braw = sel_s[q]; bnorm = norm; }
          }
        }
        bs.best_t[b] = bt; bs.best_r[b] = br; bs.best_raw[b] = braw; bs.best_norm[b] = bnorm;
        if (stop) { bs.done[b] = t; atomicAdd(bs.n_done, 1); }
      }
    }
  }
  __syncthreads();
  if (!s_cont) return;
  // ---- gather this CTA's column slice of row r (all loads first)
  const int p = s_prow, y = s_y;
  const int E = ga.E, H = ga.H, L = ga.L;
  const int e0 = (E * slice) / nslice, e1 = (E * (slice + 1)) / nslice;
  const int h0 = (H * slice) / nslice, h1 = (H * (slice + 1)) / nslice;
  const float* __restrict__ emb = ga.emb_tgt + (size_t)y * E;
  for (int c0 = e0 + threadIdx.x; c0 < e1; c0 += 2 * blockDim.x) {
    const int c1 = c0 + blockDim.x;
    const float v0 = __ldg(&emb[c0]);
    const float v1 = c1 < e1 ? __ldg(&emb[c1]) : 0.f;
    store_x(ga.x[0], r, c0, v0);
    if (c1 < e1) store_x(ga.x[0], r, c1, v1);
  }
  for (int j = h0 + threadIdx.x; j < h1; j += blockDim.x) {
    float hv[8], cv[8];
#pragma unroll
    for (int l = 0; l < 8; ++l)
      if (l < L) {
        hv[l] = __ldg(&ga.h[((size_t)l * ga.rows_pad + p) * H + j]);
        cv[l] = __ldg(&ga.c[((size_t)l * ga.rows_pad + p) * H + j]);
      }
    const float ht = __ldg(&ga.htilde[(size_t)p * H + j]);
    store_x(ga.x[0], r, E + j, ht);
#pragma unroll
    for (int l = 0; l < 8; ++l)
      if (l < L) {
        if (l == 0) store_x(ga.x[0], r, E + H + j, hv[l]);
        else store_x(ga.x[l], r, H + j, hv[l]);
        ga.cg[((size_t)l * ga.rows_pad + r) * H + j] = cv[l];
      }
  }
}

// A11 + O11: backtrack the banked best entry of each sentence.
__global__ void finalize_kernel(BeamState bs, int B, int K, int max_len, int* hyps, int* lens, float* scores,
                                float* raw, float* tlogp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int T = bs.best_t[b];
  int r = bs.best_r[b];
  for (int t = max_len; t > T; --t) {
    hyps[(size_t)b * max_len + t - 1] = 0;
    if (tlogp) tlogp[(size_t)b * max_len + t - 1] = 0.f;
  }
  for (int t = T; t >= 1; --t) {
    const size_t h = (size_t)(t - 1) * B * K + (size_t)b * K + r;
    hyps[(size_t)b * max_len + t - 1] = bs.hist_token[h];
    if (tlogp) tlogp[(size_t)b * max_len + t - 1] = bs.hist_logp[h];
    r = bs.hist_parent[h];
  }
  lens[b] = T;
  scores[b] = (float)bs.best_norm[b];
  if (raw) raw[b] = (float)bs.best_raw[b];
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
  const int n = R * H;
  launch_pdl(dec_cell_kernel, dim3((n + 255) / 256), dim3(256), 0, st, P, splits, p_rows_pad, p_ld,
             (const float4*)bias, cg, c_out, h_out, H, R, dst, ctl);
}

cudaError_t launch_attention(const float* htop, const float* keys, int key_ld, const float* mem, const int* lens,
                             int B, int S_max, int H, int K, XOut xo, const int* done, float* part_m, float* part_s,
                             float* part_c, int* tickets, StepCtl ctl, cudaStream_t st) {
  const int nch = (S_max + kAttCH - 1) / kAttCH;
  const bool same = keys == mem;
  const size_t smem = (size_t)(K * H + K * kAttCH + kAttCH * H + (same ? 0 : kAttCH * key_ld)) * sizeof(float);
  dim3 grid(B, nch);
#define ONMT_ATT(KM)                                                                                        \
  {                                                                                                         \
    cudaFuncSetAttribute(attention_kernel<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    launch_pdl(attention_kernel<KM>, grid, dim3(256), smem, st, htop, keys, key_ld, mem, lens, S_max, H, K, xo, \
               done, part_m, part_s, part_c, tickets, ctl);                                                 \
  }
  if (K <= 1) ONMT_ATT(1)
  else if (K <= 2) ONMT_ATT(2)
  else if (K <= 4) ONMT_ATT(4)
  else if (K <= 8) ONMT_ATT(8)
  else ONMT_ATT(16)
#undef ONMT_ATT
  return cudaGetLastError();
}

int attention_chunks(int S_max) { return (S_max + kAttCH - 1) / kAttCH; }

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

void launch_beam_merge(const float2* ms, const float* tz, const int* ti, int n_parts, int rows_pad, int B, int K,
                       int t, int max_len, double lp, const BeamState& bs, const GatherArgs& ga, float* row_lse,
                       float* row_z, int* row_i, StepCtl ctl, cudaStream_t st) {
  const int R = B * K;
  const int nslice = 4;
#define ONMT_MERGE(KM)                                                                                         \
  launch_pdl(row_reduce_topk_kernel<KM>, dim3(R), dim3(128), 0, st, ms, tz, ti, n_parts, rows_pad, K,          \
             bs.live + (size_t)(t & 1) * R, row_lse, row_z, row_i, ctl);                                       \
  launch_pdl(beam_select_gather_kernel<KM>, dim3(R, nslice), dim3(128), 0, st, row_lse, row_z, row_i, K, t,    \
             max_len, lp, bs, ga, nslice, ctl)
  if (K <= 1) { ONMT_MERGE(1); }
  else if (K <= 2) { ONMT_MERGE(2); }
  else if (K <= 4) { ONMT_MERGE(4); }
  else if (K <= 8) { ONMT_MERGE(8); }
  else { ONMT_MERGE(16); }
#undef ONMT_MERGE
}

void launch_finalize(const BeamState& bs, int B, int K, int max_len, int* hyps, int* lens, float* scores, float* raw,
                     float* tlogp, cudaStream_t st) {
  finalize_kernel<<<(B + 127) / 128, 128, 0, st>>>(bs, B, K, max_len, hyps, lens, scores, raw, tlogp);
}

// Test helper (onmt_test_gen): per row, combine generator partials into the LSE and
// the top-k (z, id), one thread per row, sequential over tiles.
__global__ void row_reduce_kernel(const float2* __restrict__ ms, const float* __restrict__ tz,
                                  const int* __restrict__ ti, int n_vt, int rows_pad, int R, int K, float* lse,
                                  float* oz, int* oi) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  float m = -INFINITY, s = 0.f;
  for (int v = 0; v < n_vt; ++v) {
    const float2 p = ms[(size_t)v * rows_pad + r];
    if (p.x > m) { s = s * expf(m - p.x) + p.y; m = p.x; }
    else s += p.y * expf(p.x - m);
  }
  lse[r] = m + logf(s);
  float bz[kKMax];
  int bi[kKMax];
  for (int i = 0; i < K; ++i) { bz[i] = -INFINITY; bi[i] = 0x7fffffff; }
  for (int v = 0; v < n_vt; ++v)
    for (int c = 0; c < K; ++c) {
      float cz = tz[((size_t)v * rows_pad + r) * K + c];
      int ci = ti[((size_t)v * rows_pad + r) * K + c];
      for (int i = 0; i < K; ++i)
        if (better(cz, ci, bz[i], bi[i])) {
          float t1 = bz[i]; int t2 = bi[i];
          bz[i] = cz; bi[i] = ci; cz = t1; ci = t2;
        }
    }
  for (int i = 0; i < K; ++i) { oz[(size_t)r * K + i] = bz[i]; oi[(size_t)r * K + i] = bi[i]; }
}

void launch_row_reduce(const float2* ms, const float* tz, const int* ti, int n_vt, int rows_pad, int R, int K,
                       float* lse, float* oz, int* oi, cudaStream_t st) {
  row_reduce_kernel<<<(R + 127) / 128, 128, 0, st>>>(ms, tz, ti, n_vt, rows_pad, R, K, lse, oz, oi);
}

}  // namespace onmt
