// Element-wise, attention and beam-bookkeeping kernels of the encoder and of one
// decoder step (DESIGN.md §2 rows A1-A11).  All reductions run in a fixed order, so a
// repeated call is bitwise identical.
#include <math_constants.h>

#include "common.cuh"

namespace onmt {

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }

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
    for (int s = 0; s < splits; ++s) {
      const float4 p = reinterpret_cast<const float4*>(P + ((size_t)s * p_rows_pad + b) * p_ld)[j];
      g.x += p.x; g.y += p.y; g.z += p.z; g.w += p.w;
    }
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
  for (int s = 0; s < splits; ++s) {
    const float4 p = reinterpret_cast<const float4*>(P + ((size_t)s * p_rows_pad + r) * p_ld)[j];
    g.x += p.x; g.y += p.y; g.z += p.z; g.w += p.w;
  }
  const float i = sigm(g.x), f = sigm(g.y), gg = tanhf(g.z), o = sigm(g.w);
  const float c = f * cg[(size_t)r * H + j] + i * gg;
  const float h = o * tanhf(c);
  c_out[(size_t)r * H + j] = c;
  h_out[(size_t)r * H + j] = h;
  for (int d = 0; d < dst.n; ++d) store_x(dst.x[d], r, dst.col[d] + j, h);
}

// A7: Luong global attention for the K rows of one sentence (P119-122, P299-301):
// q = W_in h (general; split-K partials summed here) or q = h (dot); e_s = q.m_s for
// s < S_b; a = softmax with pads excluded; context c = sum_s a_s m_s, written into the
// first H columns of the W_out operand.  One CTA per sentence; the memory bank rows
// are read coalesced, scores and weights live in shared memory.
template <int KMAX>
__global__ void __launch_bounds__(256) attention_kernel(const float* __restrict__ Pq, int splits, int p_rows_pad,
                                                        int p_ld, const float* __restrict__ htop,
                                                        const float* __restrict__ mem, const int* __restrict__ lens,
                                                        int S_max, int H, int K, XOut xo, const int* __restrict__ done,
                                                        StepCtl ctl) {
  if (all_done(ctl)) return;
  const int b = blockIdx.x;
  if (done && done[b]) return;
  extern __shared__ float sh[];
  float* q = sh;                  // [K][H]
  float* a = sh + K * H;          // [K][S_max]
  const int L = lens[b];
  const float* M = mem + (size_t)b * S_max * H;
  for (int e = threadIdx.x; e < K * H; e += blockDim.x) {
    const int k = e / H, j = e % H;
    const int r = b * K + k;
    float v;
    if (Pq) {
      v = 0.f;
      for (int s = 0; s < splits; ++s) v += Pq[((size_t)s * p_rows_pad + r) * p_ld + j];
    } else {
      v = htop[(size_t)r * H + j];
    }
    q[e] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int s = warp; s < L; s += nw) {
    float acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = 0.f;
    for (int j = lane; j < H; j += 32) {
      const float m = M[(size_t)s * H + j];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) acc[k] = fmaf(q[k * H + j], m, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      float v = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && k < K) a[k * S_max + s] = v;
    }
  }
  __syncthreads();
  // length-masked softmax, one warp per row (warp-shuffle max / sum)
  for (int k = warp; k < K; k += nw) {
    float mx = -INFINITY;
    for (int s = lane; s < L; s += 32) mx = fmaxf(mx, a[k * S_max + s]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int s = lane; s < L; s += 32) {
      const float e = expf(a[k * S_max + s] - mx);
      a[k * S_max + s] = e;
      sum += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv = 1.f / sum;
    for (int s = lane; s < L; s += 32) a[k * S_max + s] *= inv;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    float acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = 0.f;
    for (int s = 0; s < L; ++s) {
      const float m = M[(size_t)s * H + j];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) acc[k] = fmaf(a[k * S_max + s], m, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) store_x(xo, b * K + k, j, acc[k]);
  }
}

// A8: h~ = tanh(W_out [c ; h]) (P69; AMB-9) from split-K partials; writes h~ (fp32, for
// the next step's input feed) and the generator operand.
__global__ void attn_out_kernel(const float* __restrict__ P, int splits, int p_rows_pad, int p_ld, float* htilde,
                                int H, int R, XOut xg, StepCtl ctl) {
  if (all_done(ctl)) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * H) return;
  const int r = idx / H, j = idx % H;
  float v = 0.f;
  for (int s = 0; s < splits; ++s) v += P[((size_t)s * p_rows_pad + r) * p_ld + j];
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
                                                         StepCtl ctl) {
  if (all_done(ctl)) return;
  const int b = blockIdx.x;
  if (bs.done[b]) return;
  __shared__ float s_lse[KMAX];
  __shared__ float s_z[KMAX][KMAX];
  __shared__ int s_id[KMAX][KMAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < K; k += nw) {
    const int r = b * K + k;
    if (!bs.live[r]) continue;
    // log-sum-exp over all vocabulary tiles (fixed-order reduction)
    float m = -INFINITY, s = 0.f;
    for (int v = lane; v < n_vt; v += 32) {
      const float2 p = ms[(size_t)v * rows_pad + r];
      if (p.x > m) { s = s * expf(m - p.x) + p.y; m = p.x; }
      else if (p.x > -INFINITY) s += p.y * expf(p.x - m);
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
    // row top-K over the per-tile lists: lane-local lists then K warp-argmax rounds
    float lz[KMAX];
    int li[KMAX];
#pragma unroll
    for (int i = 0; i < KMAX; ++i) { lz[i] = -INFINITY; li[i] = 0x7fffffff; }
    for (int v = lane; v < n_vt; v += 32) {
      const size_t base = ((size_t)v * rows_pad + r) * K;
      for (int c = 0; c < K; ++c) {
        float cz = tz[base + c];
        int ci = ti[base + c];
        if (!better(cz, ci, lz[KMAX - 1], li[KMAX - 1])) break;  // per-tile lists are sorted
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          if (better(cz, ci, lz[i], li[i])) {
            const float tzz = lz[i]; const int tii = li[i];
            lz[i] = cz; li[i] = ci; cz = tzz; ci = tii;
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
  if (threadIdx.x != 0) return;
  // sentence-level K-way merge of the per-row sorted lists (O8, AMB-13)
  int head[KMAX];
  double cum[KMAX];
  int lv[KMAX];
  for (int k = 0; k < K; ++k) {
    head[k] = 0;
    lv[k] = bs.live[b * K + k];
    cum[k] = bs.cum[b * K + k];
  }
  int n_live = 0;
  for (int k = 0; k < K; ++k) n_live += lv[k];
  int sel_k[KMAX], sel_w[KMAX];
  double sel_s[KMAX];
  float sel_lp[KMAX];
  int n_sel = 0;
  for (int r = 0; r < K; ++r) {
    int bk = -1;
    double bsv = -CUDART_INF;
    int bw = 0x7fffffff;
    for (int k = 0; k < K; ++k) {
      if (!lv[k] || head[k] >= K) continue;
      const float z = s_z[k][head[k]];
      const int w = s_id[k][head[k]];
      if (z == -INFINITY) continue;
      const double sc = cum[k] + ((double)z - (double)s_lse[k]);
      if (bk < 0 || sc > bsv || (sc == bsv && (k < bk || (k == bk && w < bw)))) { bk = k; bsv = sc; bw = w; }
    }
    if (bk < 0) break;
    sel_k[n_sel] = bk;
    sel_w[n_sel] = bw;
    sel_s[n_sel] = bsv;
    sel_lp[n_sel] = (float)((double)s_z[bk][head[bk]] - (double)s_lse[bk]);
    ++n_sel;
    ++head[bk];
  }
  // O8-O9 bookkeeping
  const size_t hb = (size_t)(t - 1) * (size_t)gridDim.x * K + (size_t)b * K;
  const double lp = pow((5.0 + t) / 6.0, (double)alpha);
  bool any_live = false;
  for (int r = 0; r < K; ++r) {
    const int row = b * K + r;
    if (r >= n_sel) {
      bs.live[row] = 0;
      bs.cum[row] = -CUDART_INF;
      bs.prow[row] = row;
      bs.y[row] = 0;
      bs.hist_parent[hb + r] = -1;
      bs.hist_token[hb + r] = 0;
      bs.hist_logp[hb + r] = 0.f;
      if (bs.sel_parent) { bs.sel_parent[hb + r] = -1; bs.sel_score[hb + r] = -CUDART_INF; }
      continue;
    }
    const int k = sel_k[r], w = sel_w[r];
    bs.hist_parent[hb + r] = k;
    bs.hist_token[hb + r] = w;
    bs.hist_logp[hb + r] = sel_lp[r];
    if (bs.sel_parent) { bs.sel_parent[hb + r] = k; bs.sel_score[hb + r] = sel_s[r]; }
    if (w == 3 || t == max_len) {
      const double norm = sel_s[r] / lp;
      if (bs.best_t[b] == 0 || norm > bs.best_norm[b]) {
        bs.best_t[b] = t;
        bs.best_r[b] = r;
        bs.best_raw[b] = sel_s[r];
        bs.best_norm[b] = norm;
      }
      bs.live[row] = 0;
      bs.cum[row] = -CUDART_INF;
      bs.prow[row] = row;
      bs.y[row] = 0;
    } else {
      bs.live[row] = 1;
      bs.cum[row] = sel_s[r];
      bs.prow[row] = b * K + k;
      bs.y[row] = w;
      any_live = true;
    }
  }
  (void)n_live;
  // O10: stop after this step
  if (!any_live || t == max_len || (n_sel > 0 && sel_w[0] == 3)) {
    bs.done[b] = 1;
    atomicAdd(bs.n_done, 1);
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
                             const int* done, StepCtl ctl, cudaStream_t st) {
  const size_t smem = (size_t)(K * H + K * S_max) * sizeof(float);
#define ONMT_ATT(KM)                                                                                      \
  {                                                                                                       \
    cudaFuncSetAttribute(attention_kernel<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    attention_kernel<KM><<<B, 256, smem, st>>>(Pq, splits, p_rows_pad, p_ld, htop, mem, lens, S_max, H, K, \
                                               xo, done, ctl);                                            \
  }
  if (K <= 1) ONMT_ATT(1)
  else if (K <= 2) ONMT_ATT(2)
  else if (K <= 4) ONMT_ATT(4)
  else if (K <= 8) ONMT_ATT(8)
  else ONMT_ATT(16)
#undef ONMT_ATT
  return cudaGetLastError();
}

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
                       int max_len, float alpha, const BeamState& bs, StepCtl ctl, cudaStream_t st) {
  if (K <= 1) beam_merge_kernel<1><<<B, 256, 0, st>>>(ms, tz, ti, n_vt, rows_pad, K, t, max_len, alpha, bs, ctl);
  else if (K <= 2) beam_merge_kernel<2><<<B, 256, 0, st>>>(ms, tz, ti, n_vt, rows_pad, K, t, max_len, alpha, bs, ctl);
  else if (K <= 4) beam_merge_kernel<4><<<B, 256, 0, st>>>(ms, tz, ti, n_vt, rows_pad, K, t, max_len, alpha, bs, ctl);
  else if (K <= 8) beam_merge_kernel<8><<<B, 256, 0, st>>>(ms, tz, ti, n_vt, rows_pad, K, t, max_len, alpha, bs, ctl);
  else beam_merge_kernel<16><<<B, 256, 0, st>>>(ms, tz, ti, n_vt, rows_pad, K, t, max_len, alpha, bs, ctl);
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
