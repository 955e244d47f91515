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

// A7: Luong global attention (P119-122, P299-301), split over source chunks of CH
// positions: CTA (b, c) stages m_s for s in its chunk in shared memory once, computes
// q = W_in h (general: split-K partials summed here) or q = h (dot), the scores
// e_s = q.m_s, the chunk's (max, sum exp) and partial context for all K rows of
// sentence b.  The last CTA of a sentence (atomic ticket) combines the chunks in fixed
// order - a = softmax over s < S_b only, pads excluded - and writes the context into
// the first H columns of the W_out operand.
constexpr int kAttCH = 32;

template <int KMAX>
__global__ void __launch_bounds__(256) attention_kernel(const float* __restrict__ Pq, int splits, int p_rows_pad,
                                                        int p_ld, const float* __restrict__ htop,
                                                        const float* __restrict__ mem, const int* __restrict__ lens,
                                                        int S_max, int H, int K, XOut xo, const int* __restrict__ done,
                                                        float* __restrict__ part_m, float* __restrict__ part_s,
                                                        float* __restrict__ part_c, int* __restrict__ tickets,
                                                        StepCtl ctl) {
  if (all_done(ctl)) return;
  const int b = blockIdx.x, ch = blockIdx.y, nch = gridDim.y;
  if (done && done[b]) return;
  extern __shared__ float sh[];
  float* q = sh;                          // [K][H]
  float* ms = q + K * H;                  // [kAttCH][H]
  float* e = ms + kAttCH * H;             // [K][kAttCH]
  __shared__ int s_last;
  const int L = lens[b];
  const int s0 = ch * kAttCH;
  const int ns = max(0, min(kAttCH, L - s0));
  const float* M = mem + ((size_t)b * S_max + s0) * H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const size_t pbase = ((size_t)b * nch + ch) * K;
  if (ns > 0) {
    stage_async(ms, M, ns * H);                      // memory-bank chunk -> smem, in flight
    const size_t pstride = (size_t)p_rows_pad * p_ld;
    for (int i0 = threadIdx.x; i0 < K * H; i0 += 2 * blockDim.x) {
      float v[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = i0 + u * blockDim.x;
        v[u] = 0.f;
        if (i < K * H) {
          const int k = i / H, j = i % H;
          const int r = b * K + k;
          v[u] = Pq ? sum_splits(Pq, pstride, (size_t)r * p_ld + j, splits) : __ldg(&htop[(size_t)r * H + j]);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (i0 + u * blockDim.x < K * H) q[i0 + u * blockDim.x] = v[u];
    }
    stage_wait();
    __syncthreads();
    for (int p = warp; p < K * ns; p += nw) {         // one warp per (row, position) score
      const int k = p / ns, sidx = p % ns;
      float acc = 0.f;
      for (int j = lane; j < H; j += 32) acc = fmaf(q[k * H + j], ms[sidx * H + j], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) e[k * kAttCH + sidx] = acc;
    }
    __syncthreads();
    for (int k = warp; k < K; k += nw) {              // chunk softmax statistics
      float v = lane < ns ? e[k * kAttCH + lane] : -INFINITY;
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
  __shared__ float s_w[64][kKMax];               // per (chunk, row) weight exp(m_c - M) / S
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    float Mx = -INFINITY;
    for (int c = 0; c < nch; ++c) Mx = fmaxf(Mx, __ldcg(&part_m[b0 + c * K + k]));
    float S = 0.f;
    for (int c = 0; c < nch; ++c) {
      const float pm = __ldcg(&part_m[b0 + c * K + k]);
      const float w = pm == -INFINITY ? 0.f : expf(pm - Mx);
      s_w[c][k] = w;
      S += w * __ldcg(&part_s[b0 + c * K + k]);
    }
    for (int c = 0; c < nch; ++c) s_w[c][k] /= S;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K * H; i += blockDim.x) {
    const int k = i / H, j = i % H;
    float C = 0.f;
    for (int c = 0; c < nch; ++c) C += s_w[c][k] * __ldcg(&part_c[(b0 + c * K + k) * H + j]);
    store_x(xo, b * K + k, j, C);
  }
  if (threadIdx.x == 0) tickets[b] = 0;
}

// A8: h~ = tanh(W_out [c ; h]) (P69; AMB-9) from split-K partials; writes h~ (fp32, for
// the next step's input feed) and the generator operand.
__global__ void attn_out_kernel(const float* __restrict__ P, int splits, int p_rows_pad, int p_ld, float* htilde,
                                int H, int R, XOut xg, StepCtl ctl) {
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
    bs.cum[r] = k == 0 ? 0.0 : -CUDART_INF;
    bs.live[r] = k == 0;
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
template <int KMAX>
__global__ void __launch_bounds__(256) beam_merge_kernel(const float2* __restrict__ ms, const float* __restrict__ tz,
                                                         const int* __restrict__ ti, int n_vt, int rows_pad, int K,
                                                         int t, int max_len, float alpha, BeamState bs,
                                                         GatherArgs ga, StepCtl ctl) {
  if (all_done(ctl)) return;
  const int b = blockIdx.x;
  if (bs.done[b]) return;
  __shared__ float s_lse[KMAX];
  __shared__ float s_z[KMAX][KMAX];
  __shared__ int s_id[KMAX][KMAX];
  __shared__ int s_live[KMAX];
  __shared__ double s_cum[KMAX];
  __shared__ int s_sel_k[KMAX], s_sel_w[KMAX], s_newlive[KMAX], s_prow[KMAX], s_y[KMAX];
  __shared__ double s_sel_s[KMAX];
  __shared__ float s_sel_lp[KMAX];
  __shared__ int s_nsel, s_cont;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (threadIdx.x < K) {
    s_live[threadIdx.x] = bs.live[b * K + threadIdx.x];
    s_cum[threadIdx.x] = bs.cum[b * K + threadIdx.x];
  }
  __syncthreads();
  for (int k = warp; k < K; k += nw) {
    const int r = b * K + k;
    if (!s_live[k]) continue;
    // log-sum-exp over all partials (each lane: parts lane, lane+32, ...; loads in flight)
    float m = -INFINITY, s = 0.f;
    for (int v0 = 0; v0 < n_vt; v0 += 128) {
      float2 p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = v0 + u * 32 + lane;
        p[u] = v < n_vt ? __ldg(&ms[(size_t)v * rows_pad + r]) : make_float2(-INFINITY, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (p[u].x == -INFINITY) continue;
        if (p[u].x > m) { s = s * expf(m - p[u].x) + p[u].y; m = p[u].x; }
        else s += p[u].y * expf(p[u].x - m);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const float M = fmaxf(m, m2);
      s = (m == -INFINITY ? 0.f : s * expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - M));
      m = M;
    }
    if (lane == 0) s_lse[k] = m + logf(s);
    // row top-K over the per-part sorted lists: lane-local merge, then K warp-argmax rounds
    float lz[KMAX];
    int li[KMAX];
#pragma unroll
    for (int i = 0; i < KMAX; ++i) { lz[i] = -INFINITY; li[i] = 0x7fffffff; }
    for (int v = lane; v < n_vt; v += 32) {
      const size_t base = ((size_t)v * rows_pad + r) * K;
      float cz[KMAX];
      int cid[KMAX];
#pragma unroll
      for (int c = 0; c < KMAX; ++c) {
        cz[c] = c < K ? __ldg(&tz[base + c]) : -INFINITY;
        cid[c] = c < K ? __ldg(&ti[base + c]) : 0x7fffffff;
      }
#pragma unroll
      for (int c = 0; c < KMAX; ++c) {
        float z = cz[c];
        int id = cid[c];
        if (!better(z, id, lz[KMAX - 1], li[KMAX - 1])) break;  // per-part lists are sorted
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          if (better(z, id, lz[i], li[i])) {
            const float tzz = lz[i]; const int tii = li[i];
            lz[i] = z; li[i] = id; z = tzz; id = tii;
          }
        }
      }
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
      if (lane == 0) { s_z[k][c] = bz; s_id[k][c] = bi; }
      if (li[0] == bi && lz[0] == bz) {  // the owner pops its head
#pragma unroll
        for (int i = 0; i < KMAX - 1; ++i) { lz[i] = lz[i + 1]; li[i] = li[i + 1]; }
        lz[KMAX - 1] = -INFINITY; li[KMAX - 1] = 0x7fffffff;
      }
    }
  }
  __syncthreads();
  const size_t hb = (size_t)(t - 1) * (size_t)gridDim.x * K + (size_t)b * K;
  if (threadIdx.x == 0) {
    // sentence-level K-way merge of the per-row sorted lists (O8, AMB-13), all in smem
    int head[KMAX];
    for (int k = 0; k < K; ++k) head[k] = 0;
    int n_sel = 0;
    for (int r = 0; r < K; ++r) {
      int bk = -1, bw = 0x7fffffff;
      double bsv = -CUDART_INF;
      for (int k = 0; k < K; ++k) {
        if (!s_live[k] || head[k] >= K) continue;
        const float z = s_z[k][head[k]];
        if (z == -INFINITY) continue;
        const int w = s_id[k][head[k]];
        const double sc = s_cum[k] + ((double)z - (double)s_lse[k]);
        if (bk < 0 || sc > bsv) { bk = k; bsv = sc; bw = w; }
      }
      if (bk < 0) break;
      s_sel_k[n_sel] = bk;
      s_sel_w[n_sel] = bw;
      s_sel_s[n_sel] = bsv;
      s_sel_lp[n_sel] = (float)((double)s_z[bk][head[bk]] - (double)s_lse[bk]);
      ++n_sel;
      ++head[bk];
    }
    // O8-O9 bookkeeping: banking of EOS picks and of everything at t = max_len
    const double lp = pow((5.0 + t) / 6.0, (double)alpha);
    int bt = bs.best_t[b], br = bs.best_r[b];
    double braw = bs.best_raw[b], bnorm = bs.best_norm[b];
    bool any_live = false;
    for (int r = 0; r < K; ++r) {
      s_newlive[r] = 0; s_prow[r] = b * K + r; s_y[r] = 0;
      if (r >= n_sel) continue;
      const int w = s_sel_w[r];
      if (w == 3 || t == max_len) {
        const double norm = s_sel_s[r] / lp;
        if (bt == 0 || norm > bnorm) { bt = t; br = r; braw = s_sel_s[r]; bnorm = norm; }
      } else {
        s_newlive[r] = 1; s_prow[r] = b * K + s_sel_k[r]; s_y[r] = w;
        any_live = true;
      }
    }
    bs.best_t[b] = bt; bs.best_r[b] = br; bs.best_raw[b] = braw; bs.best_norm[b] = bnorm;
    // O10: stop after this step
    const bool stop = !any_live || t == max_len || (n_sel > 0 && s_sel_w[0] == 3);
    if (stop) {
      bs.done[b] = 1;
      atomicAdd(bs.n_done, 1);
    }
    s_nsel = n_sel;
    s_cont = !stop;
  }
  __syncthreads();
  if (threadIdx.x < K) {                          // parallel write-back of slot state + histories
    const int r = threadIdx.x, row = b * K + r;
    const bool sel = r < s_nsel;
    bs.live[row] = s_newlive[r];
    bs.cum[row] = s_newlive[r] ? s_sel_s[r] : -CUDART_INF;
    bs.prow[row] = s_prow[r];
    bs.y[row] = s_y[r];
    bs.hist_parent[hb + r] = sel ? s_sel_k[r] : -1;
    bs.hist_token[hb + r] = sel ? s_sel_w[r] : 0;
    bs.hist_logp[hb + r] = sel ? s_sel_lp[r] : 0.f;
    if (bs.sel_parent) { bs.sel_parent[hb + r] = sel ? s_sel_k[r] : -1; bs.sel_score[hb + r] = sel ? s_sel_s[r] : -CUDART_INF; }
  }
  if (!s_cont) return;
  // A5 fused: the next step's decoder inputs of this sentence's K rows, gathered by parent
  const float* __restrict__ emb = ga.emb_tgt;
  const float* __restrict__ hti = ga.htilde;
  const float* __restrict__ hs = ga.h;
  const float* __restrict__ cs = ga.c;
  const int E = ga.E, H = ga.H, L = ga.L;
  for (int i = threadIdx.x; i < K * E; i += blockDim.x) {
    const int k = i / E, c = i % E;
    store_x(ga.x[0], b * K + k, c, __ldg(&emb[(size_t)s_y[k] * E + c]));
  }
  for (int i0 = threadIdx.x; i0 < K * H; i0 += 2 * blockDim.x) {
    float hv[2][8], cv[2][8], ht[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = min(i0 + u * (int)blockDim.x, K * H - 1);
      const int k = i / H, j = i % H;
      const int p = s_prow[k];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        if (l < L) {
          hv[u][l] = __ldg(&hs[((size_t)l * ga.rows_pad + p) * H + j]);
          cv[u][l] = __ldg(&cs[((size_t)l * ga.rows_pad + p) * H + j]);
        }
      }
      ht[u] = __ldg(&hti[(size_t)p * H + j]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i >= K * H) break;
      const int k = i / H, j = i % H;
      const int r = b * K + k;
      store_x(ga.x[0], r, E + j, ht[u]);
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        if (l < L) {
          if (l == 0) store_x(ga.x[0], r, E + H + j, hv[u][l]);
          else store_x(ga.x[l], r, H + j, hv[u][l]);
          ga.cg[((size_t)l * ga.rows_pad + r) * H + j] = cv[u][l];
        }
      }
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
  dec_cell_kernel<<<(n + 255) / 256, 256, 0, st>>>(P, splits, p_rows_pad, p_ld, (const float4*)bias, cg, c_out,
                                                   h_out, H, R, dst, ctl);
}

cudaError_t launch_attention(const float* Pq, int splits, int p_rows_pad, int p_ld, const float* htop,
                             const float* mem, const int* lens, int B, int S_max, int H, int K, XOut xo,
                             const int* done, float* part_m, float* part_s, float* part_c, int* tickets, StepCtl ctl,
                             cudaStream_t st) {
  const int nch = (S_max + kAttCH - 1) / kAttCH;
  const size_t smem = (size_t)(K * H + kAttCH * H + K * kAttCH) * sizeof(float);
  dim3 grid(B, nch);
#define ONMT_ATT(KM)                                                                                          \
  {                                                                                                           \
    cudaFuncSetAttribute(attention_kernel<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
    attention_kernel<KM><<<grid, 256, smem, st>>>(Pq, splits, p_rows_pad, p_ld, htop, mem, lens, S_max, H, K, \
                                                  xo, done, part_m, part_s, part_c, tickets, ctl);            \
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
  attn_out_kernel<<<(n + 255) / 256, 256, 0, st>>>(P, splits, p_rows_pad, p_ld, htilde, H, R, xg, ctl);
}

void launch_init_decode(const BeamState& bs, int B, int K, const float* enc_h, const float* enc_c, int L, int H,
                        float* dec_h, float* dec_c, int dec_rows_pad, float* htilde, cudaStream_t st) {
  init_decode_kernel<<<B * K, 128, 0, st>>>(bs, B, K, enc_h, enc_c, L, H, dec_h, dec_c, dec_rows_pad, htilde);
}

void launch_gather(const BeamState& bs, const GatherArgs& g, int R, int K, StepCtl ctl, cudaStream_t st) {
  gather_kernel<<<R, 128, 0, st>>>(bs, g, K, ctl);
}

void launch_beam_merge(const float2* ms, const float* tz, const int* ti, int n_vt, int rows_pad, int B, int K, int t,
                       int max_len, float alpha, const BeamState& bs, const GatherArgs& ga, StepCtl ctl,
                       cudaStream_t st) {
#define ONMT_MERGE(KM) beam_merge_kernel<KM><<<B, 256, 0, st>>>(ms, tz, ti, n_vt, rows_pad, K, t, max_len, alpha, bs, ga, ctl)
  if (K <= 1) ONMT_MERGE(1);
  else if (K <= 2) ONMT_MERGE(2);
  else if (K <= 4) ONMT_MERGE(4);
  else if (K <= 8) ONMT_MERGE(8);
  else ONMT_MERGE(16);
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
