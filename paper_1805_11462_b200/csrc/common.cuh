// Shared device-side types of the onmt B200 library (kernels + runtime).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace onmt {

// Programmatic dependent launch (PDL): every decode-step kernel lets its successor launch
// early and waits for its predecessor's memory before touching any input.  Every CTA calls
// pdl_wait() before exiting (even on early-exit paths) so completion stays transitive.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Optional per-CTA phase timestamps for microbenchmarks (tools/ubench, -DONMT_KTRACE):
// thread 0 of CTA (x, y) writes %globaltimer into g_ktrace[(y * gridDim.x + x) * 12 + i].
#ifdef ONMT_KTRACE
__device__ unsigned long long* g_ktrace;
#define KT(i)                                                                                   \
  do {                                                                                          \
    if (threadIdx.x == 0 && g_ktrace) {                                                         \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                     \
      g_ktrace[(blockIdx.y * gridDim.x + blockIdx.x) * 12 + (i)] = t_;                          \
    }                                                                                           \
  } while (0)
#define KTX(i, cond)                                                                            \
  do {                                                                                          \
    if ((cond) && g_ktrace) {                                                                   \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                     \
      g_ktrace[(blockIdx.y * gridDim.x + blockIdx.x) * 12 + (i)] = t_;                          \
    }                                                                                           \
  } while (0)
#else
#define KT(i) do {} while (0)
#define KTX(i, cond) do {} while (0)
#endif

constexpr int kKMax = 16;     // ONMT_K_MAX
constexpr int kBK = 64;       // K block (64 bf16 = 128 B = one swizzle row)
constexpr int kTileM = 128;   // weight rows per tcgen05 tile (TMEM lanes)
constexpr int kVTile = 128;   // vocabulary rows per generator partial

// Destination of an activation operand: either fp32 [rows_pad x k_pad] (fp32 models,
// SIMT GEMM) or two bf16 planes hi/lo [2 x rows_pad x k_pad] (bf16 models, tcgen05
// GEMM; x = hi + lo with hi = bf16(x), lo = bf16(x - hi); DESIGN.md §6 H4).
struct XOut {
  float* f32;
  __nv_bfloat16* hl;
  int rows_pad;
  int k_pad;
};

// W_out folded into attention: the context accumulates the projected
// values W_out[:, :H] m_s, the top cell layer left W_out[:, H:2H] h_t in n_wt tile shares
// wpart [n_wt][rows_pad][H], and the combine writes h~ = tanh(sum) to htilde and xg.
struct AttFold {
  const float* wpart;           // nullptr: plain attention (context -> xo)
  int n_wt;
  int rows_pad;
  float* htilde;
  XOut xg;
  int pref;                     // (set by the launcher) shares prefetched into shared memory
  int hp_floats;                // (set by the launcher) size of that prefetch region
  float* att_out;               // [B*K][S_max] normalised attention weights (coverage / unk), or nullptr
  int push;                     // (set by the launcher) push combine: its receive buffer fits shared memory
};

__device__ __forceinline__ void store_x(const XOut& x, int r, int c, float v) {
  size_t i = (size_t)r * x.k_pad + c;
  if (x.hl) {
    __nv_bfloat16 hi = __float2bfloat16_rn(v);
    float lo = v - __bfloat162float(hi);
    x.hl[i] = hi;
    x.hl[(size_t)x.rows_pad * x.k_pad + i] = __float2bfloat16_rn(lo);
  } else {
    x.f32[i] = v;
  }
}

// 4 consecutive columns (c multiple of 4, row starts 8-byte aligned in the bf16 planes:
// k_pad is a multiple of 64)
__device__ __forceinline__ void store_x4(const XOut& x, int r, int c, float4 v) {
  size_t i = (size_t)r * x.k_pad + c;
  if (x.hl) {
    const __nv_bfloat16 h0 = __float2bfloat16_rn(v.x), h1 = __float2bfloat16_rn(v.y), h2 = __float2bfloat16_rn(v.z),
                        h3 = __float2bfloat16_rn(v.w);
    __nv_bfloat162 hi01(h0, h1), hi23(h2, h3);
    __nv_bfloat162 lo01(__float2bfloat16_rn(v.x - __bfloat162float(h0)), __float2bfloat16_rn(v.y - __bfloat162float(h1)));
    __nv_bfloat162 lo23(__float2bfloat16_rn(v.z - __bfloat162float(h2)), __float2bfloat16_rn(v.w - __bfloat162float(h3)));
    uint2 hu, lu;
    hu.x = *reinterpret_cast<uint32_t*>(&hi01); hu.y = *reinterpret_cast<uint32_t*>(&hi23);
    lu.x = *reinterpret_cast<uint32_t*>(&lo01); lu.y = *reinterpret_cast<uint32_t*>(&lo23);
    *reinterpret_cast<uint2*>(x.hl + i) = hu;
    *reinterpret_cast<uint2*>(x.hl + (size_t)x.rows_pad * x.k_pad + i) = lu;
  } else {
    *reinterpret_cast<float4*>(x.f32 + i) = v;
  }
}

// Early-exit control: every decode-step kernel returns at once when all B sentences
// have stopped (n_done written by the beam merge kernel).
struct StepCtl {
  const int* n_done;
  int B;
};
__device__ __forceinline__ bool all_done(const StepCtl& c) {
  return c.n_done != nullptr && *(volatile const int*)c.n_done >= c.B;
}

// (z desc, id asc) ordering used by every top-k in the library (R13).
__device__ __forceinline__ bool better(float za, int ia, float zb, int ib) {
  return za > zb || (za == zb && ia < ib);
}

// Generator partial outputs per (vocabulary tile, row): running max and sum of
// exp(z - max) over the tile, and the tile's top-k (z, id) in (z desc, id asc) order.
struct GenOut {
  float2* ms;      // [n_vt][rows_pad]
  float* tz;       // [n_vt][rows_pad][K]
  int* ti;         // [n_vt][rows_pad][K]
  const float* bias;  // [V]
  int V;
  int K;
  int rows_valid;
  int rows_pad;
  const int* gold;    // teacher-forced scoring (optional): gold id of each row, or -1
  float* zgold;       // [rows] the gold logit, written by the tile that holds the id
};

// Scan one tile column (n <= 128 logits of one row): online max / sum-exp plus an
// unrolled register top-KMAX insertion (ids scanned in increasing order).
template <int KMAX>
__device__ __forceinline__ void scan_tile_column(const float* vals, int stride, int vbase, const GenOut& g,
                                                 float& mx, float& sm, float (&tz)[KMAX], int (&ti)[KMAX]) {
  mx = -INFINITY;
  sm = 0.f;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) { tz[i] = -INFINITY; ti[i] = 0x7fffffff; }
  int n = g.V - vbase;
  if (n > kVTile) n = kVTile;
  for (int v = 0; v < n; ++v) {
    const int id = vbase + v;
    const float z = vals[v * stride] + g.bias[id];
    if (z > mx) {
      sm = sm * expf(mx - z) + 1.f;
      mx = z;
    } else {
      sm += expf(z - mx);
    }
    if (better(z, id, tz[KMAX - 1], ti[KMAX - 1])) {
      float cz = z;
      int ci = id;
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        if (better(cz, ci, tz[i], ti[i])) {
          float tzz = tz[i]; int tii = ti[i];
          tz[i] = cz; ti[i] = ci;
          cz = tzz; ci = tii;
        }
      }
    }
  }
}

template <int KMAX>
__device__ __forceinline__ void write_gen_partial(const GenOut& g, int vt, int r, float mx, float sm,
                                                  const float (&tz)[KMAX], const int (&ti)[KMAX]) {
  g.ms[(size_t)vt * g.rows_pad + r] = make_float2(mx, sm);
  size_t base = ((size_t)vt * g.rows_pad + r) * g.K;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    if (i < g.K) { g.tz[base + i] = tz[i]; g.ti[base + i] = ti[i]; }
  }
}


// Gate tiles of the generator step kernel: n_gt tiles of 128 rows of the
// gate weight matrix (tensor map tmWg), tile g over K blocks [q * gkbh, (q + 1) * gkbh) of the
// generator's activation operand, q = g / gt_per_q, written to gout[q][row][g % gt_per_q * 128 + m]
// (row stride gld floats).  n_gt = 0: none.
struct GateTiles {
  const CUtensorMap* tmWg;
  int n_gt, gt_per_q, gkbh, gld;
  float* gout;
};

// Vocabulary-parallel generator: the generator of rank r
// runs CTAs [ci0, ci0 + C) of a Ct-CTA vocabulary split and stores its partials into EVERY
// rank's exchange buffer (peer pointers over NVLink), then raises its flag there with the step
// epoch (*seq << 16 | t); each rank's beam step waits for all Ct x groups flags before it
// merges the Ct partials of a row - the same partials everywhere, hence the same selection.
struct VpOut {
  int world;                       // exchange buffers written (0: off)
  int ranks;                       // ranks of the vocabulary split (== world; tests emulate ranks with world 1)
  float2* ms[8];                   // [rows_pad][Ct] of rank w (this step's parity)
  float* tz[8];                    // [rows_pad][Ct][K]
  int* ti[8];
  unsigned long long* flag[8];     // [groups][Ct] of rank w (this step's parity)
  const unsigned long long* seq;   // call sequence number (device; identical on every rank)
};
struct VpWait {
  const unsigned long long* flags; // this rank's flags (this step's parity), nullptr: off
  int n;                           // groups x Ct
  const unsigned long long* seq;
};
__device__ __forceinline__ unsigned long long vp_epoch(const unsigned long long* seq, int t) {
  return (*(volatile const unsigned long long*)seq << 16) | (unsigned long long)t;
}

// Destinations of a decoder cell's h output (operand buffers and column offsets).
struct CellDst {
  XOut x[2];
  int col[2];
  int n;
};

// Device beam state (DESIGN.md §5 layout); histories are [max_len][B*K].
struct BeamState {
  double* cum;        // [2][B*K] cumulative raw log-prob of live slots (step t uses buffer t & 1)
  int* live;          // [2][B*K]
  int* y;             // [B*K] token fed at the next step
  int* prow;          // [B*K] row (b*K + parent slot) whose state slot r continues
  int* done;          // [B] 0 = running, else the step after which the sentence stopped
  int* n_done;        // [1]
  int* best_t;        // [B] banked best entry: step (1-based), 0 = none
  int* best_r;        // [B]
  double* best_raw;   // [B]
  double* best_norm;  // [B]
  int* hist_parent;   // [max_len][B*K]
  int* hist_token;    // [max_len][B*K]
  float* hist_logp;   // [max_len][B*K]
  double* sel_score;  // [max_len][B*K] (trace)
  int* sel_parent;    // [max_len][B*K] (trace; -1 = none)
  // coverage penalty / n-best / unknown replacement (S422-448)
  const float* att;   // [B*K][S_max] attention weights of the current step (nullptr: off)
  float* catt;        // [2][B*K][S_max] cumulative attention (step t reads buffer t & 1), or nullptr
  int* hist_amax;     // [max_len][B*K] attention argmax of each history entry, or nullptr
  const int* lens;    // [B] source lengths
  int S_max;
  double beta;        // coverage penalty weight (0: off)
  int nbest;          // bank entries kept per sentence: best_* are [B][nbest] (norm desc, t asc, r asc)
};

// Operands of the parent gather (A5).
struct GatherArgs {
  const float* emb_tgt;
  int E, H, L;
  const float* htilde;
  const float* h;      // [L][rows_pad][H]
  const float* c;      // [L][rows_pad][H]
  float* cg;           // [L][rows_pad][H]
  int rows_pad;
  XOut x[8];           // x[0] = layer-0 operand; x[l] = layer-l operand
  int v_map;           // copy models: an emitted extended id >= v_map is fed back as <unk> (0: off)
  // recurrent-split step: instead of gathering operands, the beam step runs
  // layer 1's cell for every new slot r (parent p, token y):
  //   gates = T[y] + P[0][p] + P[1][p] + bias[0]   (T = E_tgt W_emb^T, P[0] = W_feed h~, P[1] = W_hh h_1)
  //   c_1 = f * c_1[p] + i * g, h_1 = o * tanh(c_1)  -> c1_out[r], xh1[0..1] (operand columns col_h1)
  // and gathers layer l >= 2's recurrent gate term P[l][p] -> gb[l-2][r] and c_l[p] -> cg[l-1][r]
  // (its cell kernel adds W_ih h_{l-1} and the bias)
  int rsplit;
  const float* T;      // [V][G]
  const float* P;      // [L+1][rows_pad][G] gate tiles of the generator (row stride G)
  int G;               // gate row stride (4H rounded to 128)
  const float4* bias[8];
  float* gb;           // [L-1][rows_pad][G]
  float* c1_out;       // layer-1 cell state [rows_pad][H]
  XOut xh1[2];
  int col_h1[2];
};
// the embedding row fed back for an emitted (possibly extended) id
__device__ __forceinline__ int feed_id(const GatherArgs& ga, int y) { return (ga.v_map && y >= ga.v_map) ? 1 : y; }


// Software barrier among n co-resident CTAs (thread 0 of each calls it).  One 32-bit word:
// bits 0-15 count arrivals, bits 16-31 the generation.  The last arriver resets the count
// and bumps the generation with a single atomic, so consecutive episodes may use a
// different n (grids of different shapes sharing a counter).  Every participant must be
// resident (callers guarantee grid <= #SMs at one CTA per SM, or a cluster).
// Every cross-CTA spin is bounded: the host plans grids whose CTAs (clusters) are all
// co-resident (occupancy-checked), so a wait longer than kSpinTimeoutNs means that promise
// was broken (e.g. another context holding SMs) - the kernel traps (the call then fails with
// a CUDA error) instead of hanging the GPU.
constexpr unsigned long long kSpinTimeoutNs = 4000000000ull;
__device__ __forceinline__ unsigned long long spin_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void spin_check(unsigned long long t0, unsigned int& it) {
  if ((++it & 1023u) == 0u && spin_clock() - t0 > kSpinTimeoutNs) __trap();
}

__device__ __forceinline__ void cta_group_barrier(unsigned int* b, unsigned int n) {
  __threadfence();
  const unsigned int old = atomicAdd(b, 1u);
  if ((old & 0xffffu) == n - 1u) {
    atomicAdd(b, 0x10000u - n);
  } else {
    const unsigned int gen = old >> 16;
    const unsigned long long t0 = spin_clock();
    unsigned int it = 0;
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(b) : "memory");
      if ((v >> 16) != gen) break;
      spin_check(t0, it);
    }
  }
  __threadfence();
}

// launch with the programmatic-stream-serialization attribute (captured as a programmatic
// edge inside CUDA graphs)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace onmt
