// Device-side beam step (SURVEY §8(a) A10b + A5), shared by the stand-alone select/gather
// kernel (fp32 / SIMT path) and the persistent generator step kernel (gen_step.cu).
#pragma once
#include <math_constants.h>

#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

// A10b + A5 for hypothesis row r, executed by one whole CTA (beam_device.cuh users):
// the K best (raw desc, slot asc, token asc) of sentence b's K x K row candidates with
// fp64 cumulative scores (O8); EOS / max_len banking, stop flag, histories (O9, O10) -
// computed redundantly by every CTA of the sentence from a few hundred bytes of state -
// then the CTA gathers column slice `slice` of `nslice` of row r's next-step decoder
// inputs (x1 = [E_tgt[y]; h~[p]; h_0[p]], x_l = [.; h_l[p]], c_l[p]).  The slice-0 CTA of
// row r writes slot r's beam state.  Row results (row_lse/z/i) may come from the same
// kernel (read with L2-coherent loads).
template <int KMAX>
__device__ __forceinline__ void select_gather_row(int r, int slice, int nslice, int R, const float* row_lse,
                                                  const float* row_z, const int* row_i, int K, int t, int max_len,
                                                  double lp, const BeamState& bs, const GatherArgs& ga) {
  const int b = r / K, kr = r % K;
  const int dn = __ldcg(&bs.done[b]);
  if (dn != 0 && dn < t) return;
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
    s_live[threadIdx.x] = __ldcg(&live_in[rr]);
    s_cum[threadIdx.x] = __ldcg(&cum_in[rr]);
    s_lse[threadIdx.x] = __ldcg(&row_lse[rr]);
  }
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) {
    s_z[i / K][i % K] = __ldcg(&row_z[(size_t)b * K * K + i]);
    s_id[i / K][i % K] = __ldcg(&row_i[(size_t)b * K * K + i]);
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
      const size_t hb = (size_t)(t - 1) * (size_t)R + (size_t)r;
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
  KT(4);
  if (!s_cont) return;
  // ---- gather this CTA's column slice of row r (all loads first)
  const int p = s_prow, y = s_y;
  const int E = ga.E, H = ga.H, L = ga.L;
  const int e0 = (E * slice) / nslice, e1 = (E * (slice + 1)) / nslice;
  const int h0 = (H * slice) / nslice, h1 = (H * (slice + 1)) / nslice;
  const float* __restrict__ emb = ga.emb_tgt + (size_t)feed_id(ga, y) * E;
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

__device__ __forceinline__ float rs_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float rs_tanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

// Recurrent-split step (GatherArgs::rsplit): layer 1's LSTM cell for the
// sentence's new slots from the embedding-projection table and the generator's gate tiles,
// plus the gate-bias / c_prev gathers of layers >= 2.  c_1[p] is read by every slot that
// continues p, so the new states are computed into shared memory first (gbuf: 2 K H floats)
// and written after a CTA barrier (a sentence's slots and parents are all in this CTA).
template <int KMAX>
__device__ __forceinline__ void rsplit_cell(int b, int K, const int* s_go, const int* s_prow, const int* s_y,
                                            const GatherArgs& ga, float* gbuf) {
  const int H = ga.H, G = ga.G, L = ga.L;
  const size_t PQ = (size_t)ga.rows_pad * G;
  float* cn = gbuf;
  float* hn = gbuf + (size_t)K * H;
  constexpr int U = KMAX < 4 ? KMAX : 4;                         // slots per batch of independent loads
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float4 bb = __ldg(ga.bias[0] + j);
    for (int k0 = 0; k0 < K; k0 += U) {
      float4 tv[U], pa[U], pb[U];
      float cp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {                              // every load of the batch in flight at once
        const int kr = k0 + u;
        if (kr < K && s_go[kr]) {
          const int p = s_prow[kr];
          tv[u] = __ldg(reinterpret_cast<const float4*>(ga.T + (size_t)s_y[kr] * G) + j);
          pa[u] = __ldcg(reinterpret_cast<const float4*>(ga.P + (size_t)p * G) + j);
          pb[u] = __ldcg(reinterpret_cast<const float4*>(ga.P + PQ + (size_t)p * G) + j);
          cp[u] = __ldcg(ga.c + (size_t)p * H + j);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kr = k0 + u;
        if (kr < K && s_go[kr]) {
          // gates of unit j (rows 4j..4j+3 = i, f, g, o); same summation order for every slot
          const float zi = ((tv[u].x + pa[u].x) + pb[u].x) + bb.x, zf = ((tv[u].y + pa[u].y) + pb[u].y) + bb.y;
          const float zg = ((tv[u].z + pa[u].z) + pb[u].z) + bb.z, zo = ((tv[u].w + pa[u].w) + pb[u].w) + bb.w;
          const float c = rs_sigm(zf) * cp[u] + rs_sigm(zi) * rs_tanh(zg);
          cn[kr * H + j] = c;
          hn[kr * H + j] = rs_sigm(zo) * rs_tanh(c);
        }
      }
    }
    for (int l = 1; l < L; ++l) {                                // layers >= 2: W_hh h_l[p] + c_prev gathers
      for (int k0 = 0; k0 < K; k0 += U) {
        float4 pl[U];
        float cl[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kr = k0 + u;
          if (kr < K && s_go[kr]) {
            const int p = s_prow[kr];
            pl[u] = __ldcg(reinterpret_cast<const float4*>(ga.P + (size_t)(l + 1) * PQ + (size_t)p * G) + j);
            cl[u] = __ldcg(ga.c + ((size_t)l * ga.rows_pad + p) * H + j);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kr = k0 + u;
          if (kr < K && s_go[kr]) {
            const int r = b * K + kr;
            reinterpret_cast<float4*>(ga.gb + (size_t)(l - 1) * PQ + (size_t)r * G)[j] = pl[u];
            ga.cg[((size_t)l * ga.rows_pad + r) * H + j] = cl[u];
          }
        }
      }
    }
  }
  __syncthreads();                                               // every c_1[p] read before any write
  const int H4 = H >> 2;
  for (int it = threadIdx.x; it < K * H4; it += blockDim.x) {
    const int kr = it / H4, j4 = 4 * (it - kr * H4);
    if (!s_go[kr]) continue;
    const int r = b * K + kr;
    const float4 c = *reinterpret_cast<const float4*>(cn + kr * H + j4);
    const float4 h = *reinterpret_cast<const float4*>(hn + kr * H + j4);
    *reinterpret_cast<float4*>(ga.c1_out + (size_t)r * H + j4) = c;
    store_x4(ga.xh1[0], r, ga.col_h1[0] + j4, h);
    store_x4(ga.xh1[1], r, ga.col_h1[1] + j4, h);
  }
}

// warp-wide max / min of 32-bit unsigned values in one instruction (redux.sync), and the
// order-preserving float <-> uint key (max of keys = max of floats; -inf is the smallest key
// of any non-NaN value) - the row reduce's K-round selections use these instead of 5-step
// shuffle trees
__device__ __forceinline__ unsigned warp_max_u32(unsigned v) {
  unsigned r;
  asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ unsigned warp_min_u32(unsigned v) {
  unsigned r;
  asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ unsigned fkey(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// rsplit_cell with every input staged in shared memory: parent k's block at gbuf + k * PR
// (P[0..L] rows of 4H, then c_0..c_{L-1} rows of H), new slot kr's T[y] row at gbuf + K * PR + kr * 4H;
// the new c_1 / h_1 go to gbuf + K * PR + K * 4H (2 K H floats) before the write-out.
#ifdef ONMT_KTRACE
__device__ int g_rs_dbg;      // microbenchmark ablations (tools/ubench/ubeam): 1 no layer-2 gathers, 2 no math
#endif
__device__ __forceinline__ void rsplit_cell_smem(int b, int K, const int* s_go, const int* s_prow,
                                                 const GatherArgs& ga, float* gbuf, int PR, int j0, int nj) {
  // this CTA's units [j0, j0 + nj) (a slice of the sentence's cell: grid.y CTAs per sentence);
  // staged rows hold only the slice (4 nj gate floats, nj state floats)
  const int H = ga.H, G = ga.G, L = ga.L, G4 = 4 * nj, H4 = nj >> 2;
  const size_t PQ = (size_t)ga.rows_pad * G;
  const float* tb = gbuf + (size_t)K * PR;
  float* cn = gbuf + (size_t)K * PR + (size_t)K * G4;
  float* hn = cn + (size_t)K * nj;
  const float4* s_b1 = reinterpret_cast<const float4*>(hn + (size_t)K * nj);  // layer 1's bias (staged)
  for (int it = threadIdx.x; it < K * nj; it += blockDim.x) {
    const int kr = it / nj, jl = it - kr * nj, j = j0 + jl;
    if (!s_go[kr]) continue;
    const int r = b * K + kr, pk = s_prow[kr] - b * K;
    const float* pb = gbuf + (size_t)pk * PR;
#ifdef ONMT_KTRACE
    if (g_rs_dbg == 3) { cn[it] = pb[jl]; continue; }
    if (g_rs_dbg != 1)
#endif
    for (int l = 1; l < L; ++l) {                                // layers >= 2: W_hh h_l[parent] and c_l[parent]
      reinterpret_cast<float4*>(ga.gb + (size_t)(l - 1) * PQ + (size_t)r * G)[j] =
          reinterpret_cast<const float4*>(pb + (size_t)(l + 1) * G4)[jl];
      ga.cg[((size_t)l * ga.rows_pad + r) * H + j] = pb[(size_t)(L + 1) * G4 + (size_t)l * nj + jl];
    }
    const float4 tv = reinterpret_cast<const float4*>(tb + (size_t)kr * G4)[jl];
    const float4 pa = reinterpret_cast<const float4*>(pb)[jl];
    const float4 pc = reinterpret_cast<const float4*>(pb + G4)[jl];
    const float4 bb = s_b1[jl];
    const float cp = pb[(size_t)(L + 1) * G4 + jl];
#ifdef ONMT_KTRACE
    if (g_rs_dbg == 2) { cn[it] = tv.x + pa.y + pc.z + bb.w + cp; hn[it] = 0.f; continue; }
#endif
    // gates of unit j (rows 4j..4j+3 = i, f, g, o); same summation order as rsplit_cell
    const float zi = ((tv.x + pa.x) + pc.x) + bb.x, zf = ((tv.y + pa.y) + pc.y) + bb.y;
    const float zg = ((tv.z + pa.z) + pc.z) + bb.z, zo = ((tv.w + pa.w) + pc.w) + bb.w;
    const float c = rs_sigm(zf) * cp + rs_sigm(zi) * rs_tanh(zg);
    cn[it] = c;
    hn[it] = rs_sigm(zo) * rs_tanh(c);
  }
  KT(10);
  __syncthreads();                                               // (c_1 rows were staged: no hazard, but
  KT(11);
  for (int it = threadIdx.x; it < K * H4; it += blockDim.x) {    //  cn / hn must be complete)
    const int kr = it / H4, j4 = 4 * (it - kr * H4);
    if (!s_go[kr]) continue;
    const int r = b * K + kr;
    const float4 c = *reinterpret_cast<const float4*>(cn + kr * nj + j4);
    const float4 h = *reinterpret_cast<const float4*>(hn + kr * nj + j4);
    *reinterpret_cast<float4*>(ga.c1_out + (size_t)r * H + j0 + j4) = c;
    store_x4(ga.xh1[0], r, ga.col_h1[0] + j0 + j4, h);
    store_x4(ga.xh1[1], r, ga.col_h1[1] + j0 + j4, h);
  }
}

// A10 + A5 for one whole sentence b per CTA (512 threads): the generator partials of its K
// hypothesis rows are combined (one warp per row: log-sum-exp and row top-K), thread 0
// selects the K survivors (raw desc, slot asc, token asc; fp64 scores) with EOS / max_len
// banking, histories and the stop flag, then the CTA gathers all K rows' next-step decoder
// inputs.  Partial (p, r) of the generator lives at index p * ps + r * rs (ms) and
// (p * ps + r * rs) * K (tz, ti).  Replaces a row-reduce launch plus a select/gather launch.
template <int KMAX>
__device__ __forceinline__ void beam_step_sentence(int b, const float2* __restrict__ ms, const float* __restrict__ tz,
                                                   const int* __restrict__ ti, int n_parts, int ps, int rs, int K,
                                                   int R, int t, int max_len, double lp, const BeamState& bs,
                                                   const GatherArgs& ga, float* gbuf, int gbuf_floats, int slice = 0,
                                                   int nslice = 1) {
  KT(1);
  const int dn = __ldcg(&bs.done[b]);                            // (checked after the row reduce:
  const int* __restrict__ live_in = bs.live + (size_t)(t & 1) * R;   //  its loads overlap these)
  const double* __restrict__ cum_in = bs.cum + (size_t)(t & 1) * R;
  int* live_out = bs.live + (size_t)((t + 1) & 1) * R;
  double* cum_out = bs.cum + (size_t)((t + 1) & 1) * R;
  __shared__ int s_live[KMAX];
  __shared__ double s_cum[KMAX];
  __shared__ float s_lse[KMAX];
  __shared__ float s_z[KMAX][KMAX];
  __shared__ int s_id[KMAX][KMAX];
  __shared__ int s_prow[KMAX], s_y[KMAX], s_go[KMAX], s_src[KMAX];
  __shared__ int s_cont;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int E = ga.E, H = ga.H, L = ga.L;
  const int state_f = H * (1 + 2 * L);                           // h~ | h_l, c_l (l < L)
  const int emb_f = (E + 3) & ~3, st_f = (state_f + 3) & ~3;
  // Every possible gather source is prefetched into shared memory while the rows are reduced
  // and the survivors selected: the state rows of the live slots (issued by the last warp,
  // idle during the row reduce) and, as soon as a row's top-K is known, the embedding rows of
  // its K candidates (issued by that row's warp).  Each issuer raises the expected bytes of
  // s_bar before its copies; thread 0 arrives once all rows are reduced.
  const bool pre = !ga.rsplit && gbuf != nullptr && (E & 3) == 0 && (H & 3) == 0 &&
                   (K * K * emb_f + K * st_f) <= gbuf_floats && !(dn != 0 && dn < t);
  // recurrent split (GatherArgs::rsplit): the rows layer 1's cell reads are prefetched too - the
  // live parents' gate-tile rows P[0..L][p] and cell states c_l[p] at entry, the new slots'
  // embedding-projection rows T[y] as soon as the selection is known (s_bar2)
  // (grid.y = nslice CTAs per sentence: every one reduces and selects - identical results - and
  //  runs the cell for its slice of units [j0, j0 + nj); only slice 0 writes the beam state)
  const int nq = ((H >> 2) + nslice - 1) / nslice;
  const int j0 = min(H, 4 * nq * slice), nj = min(H, 4 * nq * (slice + 1)) - j0;
  const int G4 = 4 * nj, PR = (L + 1) * G4 + L * nj;               // floats per parent block (my slice)
  const bool rpre = ga.rsplit && gbuf != nullptr && (H & 3) == 0 && nj > 0 &&
                    (size_t)K * PR + (size_t)(K + 1) * G4 + (size_t)2 * K * nj <= (size_t)gbuf_floats &&
                    !(dn != 0 && dn < t);
  __shared__ __align__(8) uint64_t s_bar, s_bar2;
  if (threadIdx.x == 0) { mbar_init(&s_bar, 1); mbar_init(&s_bar2, 1); fence_mbar_init(); }
  if (threadIdx.x < K) {
    s_live[threadIdx.x] = __ldcg(&live_in[b * K + threadIdx.x]);
    s_cum[threadIdx.x] = __ldcg(&cum_in[b * K + threadIdx.x]);
  }
  __syncthreads();
  if (rpre && warp == nw - 2 && lane == 0) {                     // layer 1's bias (a constant)
    mbar_expect_tx(&s_bar, (uint32_t)G4 * 4);
    bulk_g2s(gbuf + (size_t)K * PR + (size_t)K * G4 + (size_t)2 * K * nj, ga.bias[0] + j0, G4 * 4, &s_bar);
  }
  if (rpre && warp == nw - 1) {
    const int nseg = 2 * L + 1;                                   // P[0..L] (4H each), c_0..c_{L-1} (H each)
    const size_t PQ = (size_t)ga.rows_pad * ga.G;
    for (int c = lane; c < K * nseg; c += 32) {
      const int k = c / nseg, w = c % nseg;
      if (!s_live[k]) continue;
      const int p = b * K + k;
      float* d = gbuf + (size_t)k * PR + (w <= L ? (size_t)w * G4 : (size_t)(L + 1) * G4 + (size_t)(w - L - 1) * nj);
      const float* src = w <= L ? ga.P + (size_t)w * PQ + (size_t)p * ga.G + 4 * j0
                                : ga.c + ((size_t)(w - L - 1) * ga.rows_pad + p) * H + j0;
      const uint32_t bytes = (uint32_t)(w <= L ? G4 : nj) * 4;
      mbar_expect_tx(&s_bar, bytes);
      bulk_g2s(d, src, bytes, &s_bar);
    }
  }
  if (pre && warp == nw - 1) {
    const int nst = 1 + 2 * L;
    for (int c = lane; c < K * nst; c += 32) {                   // c -> slot c / nst, row kind c % nst
      const int k = c / nst, w = c % nst;
      if (!s_live[k]) continue;
      const int p = b * K + k;
      float* d = gbuf + (size_t)K * K * emb_f + (size_t)k * st_f + (size_t)w * H;
      const float* src = w == 0 ? ga.htilde + (size_t)p * H
                                : (((w - 1) & 1) ? ga.c : ga.h) + ((size_t)((w - 1) >> 1) * ga.rows_pad + p) * H;
      mbar_expect_tx(&s_bar, (uint32_t)H * 4);
      bulk_g2s(d, src, H * 4, &s_bar);
    }
  }
  KT(2);
  // ---- row reduce: warp k -> row b*K + k (dead slots are masked afterwards)
  for (int k = warp; k < K; k += nw) {
    const int r = b * K + k;
    // (1) every partial's (max, sum) and best logit in one round trip
    constexpr int PPL = 8;                                       // partials per lane (n_parts <= 256)
    float2 v[PPL];
    float hz[PPL];
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      const int p = lane + 32 * u;
      const size_t ix = (size_t)p * ps + (size_t)r * rs;
      v[u] = p < n_parts ? __ldcg(&ms[ix]) : make_float2(-INFINITY, 0.f);
      hz[u] = p < n_parts ? __ldcg(&tz[ix * K]) : -INFINITY;
    }

#ifdef ONMT_KTRACE
    if (g_ktrace && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && k == 0) {
      unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); g_ktrace[34000 + 0] = t_; }
#endif
    // LSE: the row maximum first (warp), then every partial's sum rescaled to it - independent
    // terms instead of a running (max, sum) chain
    float m = -INFINITY;
#pragma unroll
    for (int u = 0; u < PPL; ++u) m = fmaxf(m, v[u].x);
    m = fkey_inv(warp_max_u32(fkey(m)));
    float sm = 0.f;
#pragma unroll
    for (int u = 0; u < PPL; ++u) sm += v[u].x == -INFINITY ? 0.f : v[u].y * __expf(v[u].x - m);
    // (2) theta = K-th largest of the LANES' partial maxima (one per lane): K distinct partials
    //     have a best logit >= theta, so a partial whose best logit is below it holds no row
    //     top-K entry.  (A lower bound of the K-th largest partial maximum; K rounds of one
    //     warp max each - the exact value needed a lane maximum recomputed per round.)
    float theta = -INFINITY;
    {
      float lm = hz[0];
#pragma unroll
      for (int u = 1; u < PPL; ++u) lm = fmaxf(lm, hz[u]);
      unsigned key = fkey(lm);
      for (int c = 0; c < K; ++c) {
        const unsigned wk = warp_max_u32(key);
        theta = wk == 0u ? -INFINITY : fkey_inv(wk);             // (0: fewer than K lanes left)
        const unsigned own = __ballot_sync(0xffffffffu, key == wk);
        if (lane == __ffs(own) - 1) key = 0u;                    // (one lane per round)
      }
    }

#ifdef ONMT_KTRACE
    if (g_ktrace && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && k == 0) {
      unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); g_ktrace[34000 + 1] = t_; }
#endif
    // (3) full lists of the qualifying partials (one more round trip), sorted insertion.  The
    //     qualifying partials are handed out one per lane in (u, lane) order, so every list is
    //     loaded in the same round trip (a lane owning several used to load them one after the
    //     other); beyond 32 of them the rest stay with their owner lanes.
    float lz[KMAX];
    int li[KMAX];
#pragma unroll
    for (int i = 0; i < KMAX; ++i) { lz[i] = -INFINITY; li[i] = 0x7fffffff; }
    unsigned qual = 0;                                           // qualifying partials of this lane
#pragma unroll
    for (int u = 0; u < PPL; ++u) qual |= (hz[u] >= theta && hz[u] != -INFINITY) ? (1u << u) : 0u;
    __shared__ int s_qp[kKMax][32];
    int nq = 0;
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      const unsigned mk = __ballot_sync(0xffffffffu, (qual >> u) & 1u);
      if ((qual >> u) & 1u) {
        const int pos = nq + __popc(mk & ((1u << lane) - 1u));
        if (pos < 32) { s_qp[k][pos] = lane + 32 * u; qual &= ~(1u << u); }
      }
      nq += __popc(mk);
    }
    __syncwarp();
    bool empty_list = true;                                      // (lz / li hold no entry yet)
    auto merge_list = [&](int p) {
      const size_t base = ((size_t)p * ps + (size_t)r * rs) * K;
      float cz[KMAX];
      int ci[KMAX];
#pragma unroll
      for (int c = 0; c < KMAX; ++c) {
        cz[c] = c < K ? __ldcg(&tz[base + c]) : -INFINITY;
        ci[c] = c < K ? __ldcg(&ti[base + c]) : 0x7fffffff;
      }
      if (empty_list) {                                          // a partial's list is sorted: the
#pragma unroll                                                   // lane's first one is its list as is
        for (int c = 0; c < KMAX; ++c) { lz[c] = cz[c]; li[c] = ci[c]; }
        empty_list = false;
        return;
      }
#pragma unroll 1
      for (int c = 0; c < K; ++c) {
        float z = cz[0];
        int id = ci[0];
#pragma unroll
        for (int q = 0; q < KMAX - 1; ++q) { cz[q] = cz[q + 1]; ci[q] = ci[q + 1]; }   // pop the head
        if (!better(z, id, lz[KMAX - 1], li[KMAX - 1])) break;      // (sorted: the rest is worse)
        bool gt[KMAX];                                           // sorted (z desc, id asc) insertion
#pragma unroll
        for (int q = 0; q < KMAX; ++q) gt[q] = better(z, id, lz[q], li[q]);
#pragma unroll
        for (int q = KMAX - 1; q >= 1; --q) {
          const float nz = gt[q - 1] ? lz[q - 1] : z;
          const int ni = gt[q - 1] ? li[q - 1] : id;
          lz[q] = gt[q] ? nz : lz[q];
          li[q] = gt[q] ? ni : li[q];
        }
        lz[0] = gt[0] ? z : lz[0];
        li[0] = gt[0] ? id : li[0];
      }
    };
    if (lane < nq) merge_list(s_qp[k][lane]);
    while (qual) {                                               // (more than 32 qualified)
      const int u = __ffs(qual) - 1;
      qual &= qual - 1;
      merge_list(lane + 32 * u);
    }

#ifdef ONMT_KTRACE
    if (g_ktrace && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && k == 0) {
      unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); g_ktrace[34000 + 2] = t_; }
#endif
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
    if (lane == 0) s_lse[k] = m + logf(sm);
    for (int c = 0; c < K; ++c) {                                // K rounds of warp arg-max over list heads
      // (z desc, id asc): the largest head value, then the smallest id among the lanes holding it
      // (ids are >= 0, 0x7fffffff for an empty slot)
      const unsigned kz = warp_max_u32(fkey(lz[0]));
      const float bz = fkey_inv(kz);
      const int bi = (int)warp_min_u32(fkey(lz[0]) == kz ? (unsigned)li[0] : 0xffffffffu);
      if (lane == 0) { s_z[k][c] = bz; s_id[k][c] = bi; }
      if (pre && lane == c && s_live[k] && bz != -INFINITY) {   // candidate (k, c): prefetch its embedding
        mbar_expect_tx(&s_bar, (uint32_t)E * 4);
        bulk_g2s(gbuf + (size_t)(k * K + c) * emb_f, ga.emb_tgt + (size_t)feed_id(ga, bi) * E, E * 4, &s_bar);
      }
      if (li[0] == bi && lz[0] == bz) {
#pragma unroll
        for (int q = 0; q < KMAX - 1; ++q) { lz[q] = lz[q + 1]; li[q] = li[q + 1]; }
        lz[KMAX - 1] = -INFINITY;
        li[KMAX - 1] = 0x7fffffff;
      }
    }
#ifdef ONMT_KTRACE
    if (g_ktrace && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && k == 0) {
      unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); g_ktrace[34000 + 3] = t_; }
#endif
  }
  __syncthreads();
  if (dn != 0 && dn < t) return;                                 // finished earlier (uniform)
  if (threadIdx.x < K * K && !s_live[threadIdx.x / K]) s_z[threadIdx.x / K][threadIdx.x % K] = -INFINITY;
  if ((pre || rpre) && threadIdx.x == 0) mbar_arrive_local(&s_bar);   // every issuer raised its bytes
  KT(3);
  // ---- selection (parallel ranks): candidate (k, j) = slot k's j-th row best; its raw score
  //      cum_k + z - lse_k in fp64; order (score desc, slot asc, position asc) - the merge of
  //      the slots' sorted lists (R13); the K best survive.
  __shared__ double s_sc[KMAX * KMAX];
  __shared__ int s_valid[KMAX * KMAX];
  __shared__ int s_sel_k[KMAX], s_sel_w[KMAX], s_sel_c[KMAX];
  __shared__ double s_sel_s[KMAX];
  __shared__ float s_sel_lp[KMAX];
  __shared__ int s_nsel;
  const int KK = K * K;
  if (threadIdx.x < KK) {
    const int k = threadIdx.x / K, j = threadIdx.x % K;
    const float z = s_z[k][j];
    const bool ok = s_live[k] && z != -INFINITY;
    s_valid[threadIdx.x] = ok;
    s_sc[threadIdx.x] = ok ? s_cum[k] + ((double)z - (double)s_lse[k]) : -CUDART_INF;
  }
  // (invalid candidates carry score -inf and never outrank a valid one, whose score is finite:
  //  the rank loop needs no validity test and its loads pipeline)
  const int nvalid = __syncthreads_count(threadIdx.x < KK && s_valid[threadIdx.x]);
  KTX(7, threadIdx.x == 0);
  if (threadIdx.x < KK) {
    const int i = threadIdx.x;
    if (s_valid[i]) {
      const double sc = s_sc[i];
      int rank = 0;                                              // (c < i: earlier slot, or same slot earlier position)
#pragma unroll 5
      for (int c = 0; c < KK; ++c) {
        const double o = s_sc[c];
        rank += (o > sc) || (o == sc && c < i);
      }
      if (rank < K) {
        const int k = i / K, j = i % K;
        s_sel_k[rank] = k;
        s_sel_c[rank] = i;
        s_sel_w[rank] = s_id[k][j];
        s_sel_s[rank] = sc;
        s_sel_lp[rank] = (float)((double)s_z[k][j] - (double)s_lse[k]);
      }
      if (rank == 0) s_nsel = nvalid < K ? nvalid : K;
    }
    if (i == 0 && nvalid == 0) s_nsel = 0;
  }
  __syncthreads();
  KTX(8, threadIdx.x == 0);
  const int n_sel = s_nsel;
  const bool stop = [&] {
    bool any_live = false;
    for (int q = 0; q < n_sel; ++q) any_live |= !(s_sel_w[q] == 3 || t == max_len);
    return !any_live || t == max_len || (n_sel > 0 && s_sel_w[0] == 3);
  }();
  if (threadIdx.x < K) {                                         // slot kr of sentence b
    const int kr = threadIdx.x;
    const int r = b * K + kr;
    const bool mine_sel = kr < n_sel;
    const bool mine_live = mine_sel && !(s_sel_w[kr] == 3 || t == max_len);
    s_prow[kr] = mine_live ? b * K + s_sel_k[kr] : r;
    s_y[kr] = mine_live ? s_sel_w[kr] : 0;
    s_go[kr] = mine_live && !stop;
    s_src[kr] = mine_live ? s_sel_c[kr] : 0;
    if (rpre && s_go[kr]) {                                      // my new slot's T[y] row
      mbar_expect_tx(&s_bar2, (uint32_t)G4 * 4);
      bulk_g2s(gbuf + (size_t)K * PR + (size_t)kr * G4, ga.T + (size_t)s_y[kr] * ga.G + 4 * j0, G4 * 4, &s_bar2);
    }
    const size_t hb = (size_t)(t - 1) * (size_t)R + (size_t)r;
    if (slice == 0) {                                            // (the sentence's state: one writer)
      live_out[r] = mine_live;
      cum_out[r] = mine_live ? s_sel_s[kr] : -CUDART_INF;
      bs.prow[r] = s_prow[kr];
      bs.y[r] = s_y[kr];
      bs.hist_parent[hb] = mine_sel ? s_sel_k[kr] : -1;
      bs.hist_token[hb] = mine_sel ? s_sel_w[kr] : 0;
      bs.hist_logp[hb] = mine_sel ? s_sel_lp[kr] : 0.f;
      if (bs.sel_parent) { bs.sel_parent[hb] = mine_sel ? s_sel_k[kr] : -1; bs.sel_score[hb] = mine_sel ? s_sel_s[kr] : -CUDART_INF; }
    }
  }
  // ---- coverage / unknown replacement (S436-448): the new slot q inherits its parent's
  //      cumulative attention plus the parent's step-t attention row; its token's attention
  //      argmax (first maximum: ties -> smallest s) goes to the history
  __shared__ double s_cp[KMAX];
  if ((bs.catt || bs.hist_amax) && slice == 0) {
    __syncthreads();                                             // (selection results visible)
    const int Lb = __ldg(&bs.lens[b]);
    const size_t RS = (size_t)R * bs.S_max;
    if (bs.catt) {
      const float* cin = bs.catt + (size_t)(t & 1) * RS;
      float* cout = bs.catt + (size_t)((t + 1) & 1) * RS;
      for (int i = threadIdx.x; i < n_sel * Lb; i += blockDim.x) {
        const int q = i / Lb, s = i % Lb;
        const size_t pr = (size_t)(b * K + s_sel_k[q]) * bs.S_max + s;
        cout[(size_t)(b * K + q) * bs.S_max + s] = __ldcg(&cin[pr]) + __ldcg(&bs.att[pr]);
      }
    }
    __syncthreads();
    for (int q = warp; q < n_sel; q += nw) {
      const size_t pbase = (size_t)(b * K + s_sel_k[q]) * bs.S_max;
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      double cp = 0.0;
      for (int s = lane; s < Lb; s += 32) {
        const float a = __ldcg(&bs.att[pbase + s]);
        if (a > bv) { bv = a; bi = s; }                          // (s increases along a lane)
        if (bs.catt && bs.beta != 0.0)
          cp += log(fmin((double)__ldcg(&bs.catt[(size_t)((t + 1) & 1) * RS + (size_t)(b * K + q) * bs.S_max + s]), 1.0));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
        cp += __shfl_xor_sync(0xffffffffu, cp, o);
      }
      if (lane == 0) {
        s_cp[q] = bs.beta * cp;
        if (bs.hist_amax) bs.hist_amax[(size_t)(t - 1) * R + b * K + q] = bi;
      }
    }
    __syncthreads();
  }
  KTX(9, threadIdx.x == 0);
  if (threadIdx.x == 0) s_cont = !stop;
  if (threadIdx.x == 0 && slice == 0) {
    // sentence-level banking (final_score = raw / lp + cp, S436-439) into the n-best list
    // (norm desc; an equal norm never displaces an earlier step / lower rank, AMB-19)
    const int nb = bs.nbest > 0 ? bs.nbest : 1;
    const int base = b * nb;
    for (int q = 0; q < n_sel; ++q) {
      if (s_sel_w[q] == 3 || t == max_len) {
        const double norm = s_sel_s[q] / lp + ((bs.catt && bs.beta != 0.0) ? s_cp[q] : 0.0);
        int pos = nb;
        for (int i = nb - 1; i >= 0; --i)
          if (bs.best_t[base + i] == 0 || norm > bs.best_norm[base + i]) pos = i;
          else break;
        if (pos < nb) {
          for (int i = nb - 1; i > pos; --i) {
            bs.best_t[base + i] = bs.best_t[base + i - 1]; bs.best_r[base + i] = bs.best_r[base + i - 1];
            bs.best_raw[base + i] = bs.best_raw[base + i - 1]; bs.best_norm[base + i] = bs.best_norm[base + i - 1];
          }
          bs.best_t[base + pos] = t; bs.best_r[base + pos] = q;
          bs.best_raw[base + pos] = s_sel_s[q]; bs.best_norm[base + pos] = norm;
        }
      }
    }
    if (stop) { bs.done[b] = t; atomicAdd(bs.n_done, 1); }
  }
  __syncthreads();
  KT(4);
  if (rpre && threadIdx.x == 0) mbar_arrive_local(&s_bar2);    // (after the barrier: every T copy issued)
  if (!s_cont) {
    if (pre || rpre) mbar_wait(&s_bar, 0);                       // (no copy may land after exit)
    if (rpre) mbar_wait(&s_bar2, 0);
    return;
  }
  if (rpre) {                                                    // layer 1's cell from shared memory
    mbar_wait(&s_bar, 0);
    mbar_wait(&s_bar2, 0);
    KT(5);
    rsplit_cell_smem(b, K, s_go, s_prow, ga, gbuf, PR, j0, nj);
    KT(6);
    return;
  }
  if (ga.rsplit) {                                               // layer 1's cell instead of a gather
    rsplit_cell<KMAX>(b, K, s_go, s_prow, s_y, ga, gbuf);
    return;
  }
  // ---- gather the next step's inputs of the K rows (x1 = [E_tgt[y]; h~[p]; h_0[p]],
  //      x_l = [.; h_l[p]], c_l[p]); dead slots are not gathered
  if (pre) {
    mbar_wait(&s_bar, 0);
    KT(5);
    const float* pst = gbuf + (size_t)K * K * emb_f;
    const int nseg = 2 + 2 * L;                                  // emb | h~ | (h_l, c_l)
    for (int pr = warp; pr < K * nseg; pr += nw) {               // one warp per (slot, segment)
      const int kr = pr / nseg, seg = pr % nseg;
      if (!s_go[kr]) continue;
      const int r = b * K + kr;
      const int pk = s_prow[kr] - b * K;                         // parent slot
      const float* src;
      int len, cbase;
      XOut xo = ga.x[0];
      float* cdst = nullptr;
      if (seg == 0) { src = gbuf + (size_t)s_src[kr] * emb_f; len = E; cbase = 0; }
      else if (seg == 1) { src = pst + (size_t)pk * st_f; len = H; cbase = E; }
      else {
        const int l = (seg - 2) >> 1;
        src = pst + (size_t)pk * st_f + H + (seg - 2) * H;
        len = H;
        if ((seg - 2) & 1) cdst = ga.cg + ((size_t)l * ga.rows_pad + r) * H;
        else { xo = l == 0 ? ga.x[0] : ga.x[l]; cbase = l == 0 ? E + H : H; }
      }
      for (int j4 = 4 * lane; j4 < len; j4 += 128) {
        const float4 v = *reinterpret_cast<const float4*>(src + j4);
        if (cdst) *reinterpret_cast<float4*>(cdst + j4) = v;
        else store_x4(xo, r, cbase + j4, v);
      }
    }
    KT(6);
    return;
  }
  if (threadIdx.x == 0) { mbar_init(&s_bar, 1); fence_mbar_init(); }   // (fresh phase for the batches)
  __syncthreads();
  const int per_row = E + H * (1 + 2 * L);                       // emb | h~ | h_l, c_l (l < L)
  const bool bulk = gbuf != nullptr && (E & 3) == 0 && (H & 3) == 0;
  const int slot_f = (per_row + 3) & ~3;
  const int spb = bulk ? max(1, min(K, gbuf_floats / slot_f)) : 1;   // slots per staged batch
  int phase = 0;
  for (int k0 = 0; k0 < K; k0 += spb) {
    const int k1 = min(K, k0 + spb);
    if (bulk) {
      // one bulk copy per source row into shared memory (one round trip for the batch)
      if (threadIdx.x == 0) {
        uint32_t bytes = 0;
        for (int kr = k0; kr < k1; ++kr)
          if (s_go[kr]) bytes += (uint32_t)per_row * 4;
        mbar_arrive_expect_tx(&s_bar, bytes);
        for (int kr = k0; kr < k1; ++kr) {
          if (!s_go[kr]) continue;
          const int p = s_prow[kr];
          float* d = gbuf + (size_t)(kr - k0) * slot_f;
          bulk_g2s(d, ga.emb_tgt + (size_t)feed_id(ga, s_y[kr]) * E, E * 4, &s_bar);
          bulk_g2s(d + E, ga.htilde + (size_t)p * H, H * 4, &s_bar);
          for (int l = 0; l < L; ++l) {
            bulk_g2s(d + E + H + 2 * l * H, ga.h + ((size_t)l * ga.rows_pad + p) * H, H * 4, &s_bar);
            bulk_g2s(d + E + H + (2 * l + 1) * H, ga.c + ((size_t)l * ga.rows_pad + p) * H, H * 4, &s_bar);
          }
        }
      }
      mbar_wait(&s_bar, phase & 1);
      ++phase;
      KT(5);
    }
    if (bulk) {
      // segments of each row: [0, E+H) -> x0 cols [0, E+H); h_l -> x0 [E+H, E+2H) or x_l [H, 2H);
      // c_l -> cg[l]; 4 consecutive columns per thread (E, H multiples of 4)
      // one warp per (slot, segment) pair, lanes over 4-column groups
      const int nseg = 1 + 2 * L;
      for (int pr = warp; pr < (k1 - k0) * nseg; pr += nw) {
        const int kr = k0 + pr / nseg, seg = pr % nseg;
        if (!s_go[kr]) continue;
        const int r = b * K + kr;
        const float* src = gbuf + (size_t)(kr - k0) * slot_f;
        const int off = seg == 0 ? 0 : E + H + (seg - 1) * H;
        const int len = seg == 0 ? E + H : H;
        const int l = (seg - 1) >> 1;
        const bool is_c = seg > 0 && ((seg - 1) & 1);
        const XOut xo = seg == 0 || l == 0 ? ga.x[0] : ga.x[l];
        const int cbase = seg == 0 ? 0 : (l == 0 ? E + H : H);
        float* cdst = is_c ? ga.cg + ((size_t)l * ga.rows_pad + r) * H : nullptr;
        for (int j4 = 4 * lane; j4 < len; j4 += 128) {
          const float4 v = *reinterpret_cast<const float4*>(src + off + j4);
          if (is_c) *reinterpret_cast<float4*>(cdst + j4) = v;
          else store_x4(xo, r, cbase + j4, v);
        }
      }
    } else {
      for (int it = threadIdx.x; it < (k1 - k0) * per_row; it += blockDim.x) {
        const int kr = k0 + it / per_row, col = it % per_row;
        if (!s_go[kr]) continue;
        const int r = b * K + kr;
        const int p = s_prow[kr];
        float v;
        if (col < E) v = __ldg(&ga.emb_tgt[(size_t)feed_id(ga, s_y[kr]) * E + col]);
        else if (col < E + H) v = __ldcg(&ga.htilde[(size_t)p * H + col - E]);
        else {
          const int x = col - E - H, l = x / (2 * H), j = x % (2 * H);
          v = __ldcg(&(j < H ? ga.h : ga.c)[((size_t)l * ga.rows_pad + p) * H + (j < H ? j : j - H)]);
        }
        if (col < E + H) {
          store_x(ga.x[0], r, col, v);
        } else {
          const int x = col - E - H, l = x / (2 * H), j = x % (2 * H);
          if (j < H) {
            if (l == 0) store_x(ga.x[0], r, E + H + j, v);
            else store_x(ga.x[l], r, H + j, v);
          } else {
            ga.cg[((size_t)l * ga.rows_pad + r) * H + j - H] = v;
          }
        }
      }
    }
    __syncthreads();                                             // staging buffer reused by the next batch
  }
  KT(6);
}

}  // namespace onmt
