// Copy / pointer generator (PAPER.md P302-304, P316-317 "copy
// mechanism", "dynamic dictionary support for copy/pointer networks"; SPEC S293-301):
//
//   p(w) = g p_vocab(w) + (1 - g) sum_{s : src_ext[s] = w} a_s,   g = sigmoid(w_c . h~ + b_c)
//
// over the extended vocabulary (target vocabulary, then the sentence's source-only ids).  The
// generator kernel already produced LSE and the top-K logits of p_vocab per row (row reduce);
// this kernel turns them into the row's top-K of the extended distribution.  Candidates:
//   * every distinct source id w of the sentence (its copy mass C_w plus, for w < V, its own
//     generator term from a direct dot product W_gen[w] . h~ + b[w]);
//   * the generator's top-K ids that are not source ids, log p = log g + z - LSE.
// This set holds the extended top-K: a non-source id outside the generator top-K is beaten
// by those K entries (p = g p_vocab is monotone in z).  One CTA per hypothesis row; the
// row's K best (log p desc, id asc) replace the row's top-K list with LSE := 0, so the beam
// selection (select_gather_row) ranks extended log-probabilities directly.
#include <math_constants.h>

#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

struct CopyArgs {
  const float* htilde;     // [rows][H] this step's attentional vectors (fp32)
  int H;
  const float* copy_w;     // [H] gate weights, copy_b its bias
  float copy_b;
  const float* att;        // [R][S_max] attention weights of this step
  int S_max;
  const int* src_ext;      // [B][S_max] extended ids (dynamic dictionary)
  const int* lens;         // [B]
  const void* gen_w;       // W_gen rows [V][gen_ld] (bf16 or fp32)
  int gen_ld, gen_bf16;
  const float* gen_b;
  int V, K;
  const int* live;         // this step's live flags [R]
  float* row_lse;          // in: LSE of p_vocab; out: 0
  float* row_z;            // in: top-K logits; out: top-K extended log-probs
  int* row_i;              // in: their ids; out: extended ids
  StepCtl ctl;
};

__global__ void __launch_bounds__(256) copy_rows_kernel(CopyArgs a) {
  pdl_trigger();
  pdl_wait();
  if (all_done(a.ctl)) return;
  const int r = blockIdx.x, b = r / a.K;
  if (a.live && !a.live[r]) return;
  extern __shared__ __align__(16) uint8_t cp_raw[];
  const int S = a.S_max, H = a.H, KC = a.K;
  double* s_c = reinterpret_cast<double*>(cp_raw);               // [S] copy mass of a first occurrence
  double* s_lp = s_c + S;                                        // [S + K] candidate log p
  float* s_h = reinterpret_cast<float*>(s_lp + S + KC);         // [H]
  float* s_z = s_h + H;                                          // [S] generator logit of source ids < V
  int* s_first = reinterpret_cast<int*>(s_z + S);                // [S] first occurrence of its id
  int* s_id = s_first + S;                                       // [S + K] candidate ids
  __shared__ double s_red[8];
  __shared__ double s_g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = a.lens[b];
  const int* ext = a.src_ext + (size_t)b * S;
  const float* att = a.att + (size_t)r * S;
  // ---- h~ and the gate g = sigmoid(w_c . h~ + b_c)
  double part = 0.0;
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float hv = a.htilde[(size_t)r * H + j];
    s_h[j] = hv;
    part += (double)a.copy_w[j] * (double)hv;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) s_red[warp] = part;
  // ---- source positions: first occurrences and their copy mass sum_{s': ext = w} a_s'
  for (int s = threadIdx.x; s < L; s += blockDim.x) {
    const int w = ext[s];
    int first = 1;
    for (int q = 0; q < s && first; ++q) first = ext[q] != w;
    double c = 0.0;
    if (first)
      for (int q = s; q < L; ++q)
        if (ext[q] == w) c += (double)att[q];                    // (fixed position order)
    s_first[s] = first;
    s_c[s] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = a.copy_b;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) d += s_red[w];
    s_g = 1.0 / (1.0 + exp(-d));
  }
  // ---- generator logits of the source ids inside the target vocabulary (warp per position)
  for (int s = warp; s < L; s += blockDim.x >> 5) {
    const int w = ext[s];
    if (!s_first[s] || w >= a.V) continue;
    float acc = 0.f;
    if (a.gen_bf16) {
      const __nv_bfloat16* row = reinterpret_cast<const __nv_bfloat16*>(a.gen_w) + (size_t)w * a.gen_ld;
      for (int j = lane; j < H; j += 32) acc = fmaf(__bfloat162float(row[j]), s_h[j], acc);
    } else {
      const float* row = reinterpret_cast<const float*>(a.gen_w) + (size_t)w * a.gen_ld;
      for (int j = lane; j < H; j += 32) acc = fmaf(row[j], s_h[j], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) s_z[s] = acc + a.gen_b[w];
  }
  __syncthreads();
  // ---- candidates: distinct source ids, then the generator's top-K ids that are not source ids
  const double g = s_g, lse = (double)a.row_lse[r];
  for (int s = threadIdx.x; s < L; s += blockDim.x) {
    const int w = ext[s];
    double lp = -CUDART_INF;
    if (s_first[s]) {
      const double pv = w < a.V ? g * exp((double)s_z[s] - lse) : 0.0;
      lp = log(pv + (1.0 - g) * s_c[s]);
    }
    s_lp[s] = lp;
    s_id[s] = s_first[s] ? w : 0x7fffffff;
  }
  if (threadIdx.x < KC) {
    const int k = threadIdx.x;
    const float z = a.row_z[(size_t)r * KC + k];
    const int w = a.row_i[(size_t)r * KC + k];
    bool in_src = false;
    for (int q = 0; q < L && !in_src; ++q) in_src = ext[q] == w;
    const bool ok = !in_src && z != -INFINITY && w >= 0 && w < a.V;
    s_lp[S + k] = ok ? log(g) + (double)z - lse : -CUDART_INF;
    s_id[S + k] = ok ? w : 0x7fffffff;
  }
  __syncthreads();
  // ---- the row's K best (log p desc, id asc): every candidate counts the better ones
  auto cand = [&](int i) { return i < L ? i : S + (i - L); };   // candidate i -> its slot
  const int n = L + KC;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int ci = cand(i);
    const double lp = s_lp[ci];
    const int id = s_id[ci];
    if (lp == -CUDART_INF) continue;
    int rank = 0;
    for (int q = 0; q < n && rank < KC; ++q) {
      const int cq = cand(q);
      const double o = s_lp[cq];
      rank += (o > lp) || (o == lp && s_id[cq] < id);
    }
    if (rank < KC) {
      a.row_z[(size_t)r * KC + rank] = (float)lp;
      a.row_i[(size_t)r * KC + rank] = id;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nv = 0;                                                  // ranks without a candidate
    for (int i = 0; i < n; ++i) nv += s_lp[cand(i)] != -CUDART_INF;
    for (int k = nv; k < KC; ++k) { a.row_z[(size_t)r * KC + k] = -INFINITY; a.row_i[(size_t)r * KC + k] = 0x7fffffff; }
    a.row_lse[r] = 0.f;
  }
}

cudaError_t launch_copy_rows(const CopyArgs& a, int R, cudaStream_t st) {
  const size_t smem = (size_t)(2 * a.S_max + a.K) * 8 + (size_t)a.H * 4 + (size_t)a.S_max * 4 +
                      (size_t)(2 * a.S_max + a.K) * 4;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(copy_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(copy_rows_kernel, dim3(R), dim3(256), smem, st, a);
}

}  // namespace onmt
