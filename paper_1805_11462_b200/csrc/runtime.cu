// Host runtime + C-ABI of the onmt B200 library (include/onmt.h).
//
//   loader      MNMT parse -> config inference -> bf16 rounding -> gate-row interleave
//               (row 4j+g holds gate g of unit j) -> padded device matrices + TMA maps
//   encoder     A1 gather, A2 hoisted input projection (tcgen05), A3 recurrence
//               (per step: recurrent GEMM + fused cell), A4 memory bank + init states
//   decoder     per step: gates GEMM + cell per layer, q GEMM, attention, W_out GEMM +
//               tanh, fused generator/log-softmax/top-k, beam merge, parent gather -
//               all enqueued on one stream, no host round-trip per step (optionally
//               replayed as a CUDA graph)
//   C-ABI       argument validation, status codes, thread-local error string
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/onmt.h"
#include "common.cuh"

namespace onmt {
// kernels / launchers defined in the other translation units
cudaError_t tc_gemm_partial(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                            int n_valid, int k_blocks, int splits, float* out, StepCtl ctl, cudaStream_t st,
                            bool groups_from_valid = false);
cudaError_t tc_gemm_gen(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                        int k_blocks, const GenOut& g, StepCtl ctl, cudaStream_t st);
cudaError_t tc_gen_persistent(const CUtensorMap& tmW, const CUtensorMap& tmX, int n_vt, int n_rows_pad, int n_group,
                              int k_blocks, int num_sms, int cs, const GenOut& g, StepCtl ctl, cudaStream_t st);
int gen_persistent_parts(int n_vt, int n_groups, int num_sms, int cs);
bool gen_persistent_fits(int n_group);
bool gen_step_wide_plan(int n_vt, int n_group, int groups, int num_sms);
int gen_step_parts(int n_vt, int n_group, int groups, int num_sms);
cudaError_t gen_step(const CUtensorMap& tmW, const CUtensorMap& tmX, int n_vt, int n_rows_pad, int n_group,
                     int k_blocks, int num_sms, const GenOut& g, float* row_lse, float* row_z, int* row_i, int t,
                     unsigned int* thr, StepCtl ctl, cudaStream_t st, const GateTiles& gt,
                     const VpOut* vp = nullptr, int vp_rank = 0, int vp_C = 0);
void launch_vp_seq(unsigned long long* seq, cudaStream_t st);
int gen_step_gate_capacity(int n_vt, int n_group, int groups, int num_sms);
extern unsigned long long* g_gen_dbg;

cudaError_t simt_gemm_partial(const void* W, bool w_bf16, int m_pad, int k_pad, const float* X, int n_rows_pad,
                              int n_valid, int splits, float* out, StepCtl ctl, cudaStream_t st);
int simt_effective_splits(int k_pad, int splits);
cudaError_t tc_gemm_cell(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                         int n_valid, int k_blocks, const float* bias, const float* cg, float* c_out, float* h_out,
                         int H, CellDst dst, float* scratch, unsigned int* counters, int num_sms, StepCtl ctl,
                         cudaStream_t st, const __nv_bfloat16* woh = nullptr, float* woh_part = nullptr,
                         const float* gb = nullptr, int gb_ld = 0);
bool tc_cell_fold_fits(int m_pad, int n_rows_pad, int n_group, int k_blocks, int H, int num_sms, bool gb = false);
bool tc_cell_fits(int m_pad, int n_rows_pad, int n_group, int k_blocks, int H, int num_sms, bool gb);
struct EncRecDir {
  const float* Z;
  int z_ld;
  const float4* bias;
  XOut xrec[2];
  float* h_st;
  float* c_st;
  int st_ld;
  XOut xnext;
  int next_col;
  float* mem;
  int mem_ld, mem_col;
  int backward;
};
struct EncRecArgs {
  EncRecDir dir[2];
  int T, S, Hd, B, N, S_max, kb;
  const int* lens;
  unsigned int* bar;
  unsigned long long* trace;
};
int enc_rec_splits(int kb, int N, int D, int T, int num_sms);
struct EncClDir {
  const float* Z;
  int z_ld;
  const float4* bias;
  float* h_st;
  float* c_st;
  int st_ld;
  XOut xnext;
  int next_col;
  float* mem;
  int mem_ld, mem_col;
  int backward;
};
struct EncClArgs {
  EncClDir dir[2];
  int T, Hd, B, N, S_max, kb;
  const int* lens;
  unsigned long long* trace;
};
int enc_cl_fits(int T, int kb, int N, int D, int num_sms);
cudaError_t launch_enc_cl(const CUtensorMap* tmW, const EncClArgs& a, int D, cudaStream_t st);
struct EncWaveLayer {
  int T, S, kb, kb_in;
  int cta0;
  const float* Z;
  int z_ld;
  const float4* bias;
  XOut xrec[2];
  float* h_st;
  float* c_st;
  int st_ld;
  XOut xnext;
  float* mem;
  int mem_ld;
};
struct EncWaveArgs {
  EncWaveLayer layer[4];
  int L, Hd, B, N, S_max;
  const int* lens;
  unsigned long long* cnt;
};
int enc_wave_splits(int L, const int* kb, int N, int T, int num_sms);
cudaError_t launch_enc_wave(const CUtensorMap* tw, const CUtensorMap (*tx)[2], const EncWaveArgs& a, int grid, int S,
                            cudaStream_t st);
struct CopyArgs {
  const float* htilde;
  int H;
  const float* copy_w;
  float copy_b;
  const float* att;
  int S_max;
  const int* src_ext;
  const int* lens;
  const void* gen_w;
  int gen_ld, gen_bf16;
  const float* gen_b;
  int V, K;
  const int* live;
  float* row_lse;
  float* row_z;
  int* row_i;
  StepCtl ctl;
};
cudaError_t launch_copy_rows(const CopyArgs& a, int R, cudaStream_t st);
void launch_row_topk(const float2* ms, const float* tz, const int* ti, int n_parts, int ps, int rs, int B, int K, int t,
                     const BeamState& bs, float* row_lse, float* row_z, int* row_i, StepCtl ctl, cudaStream_t st);
void launch_select_gather(int B, int K, int t, int max_len, double lp, const BeamState& bs, const GatherArgs& ga,
                          const float* row_lse, const float* row_z, const int* row_i, StepCtl ctl, cudaStream_t st);
cudaError_t launch_enc_rec(const CUtensorMap* tmW, const CUtensorMap* tmX0, const CUtensorMap* tmX1,
                           const EncRecArgs& a, int D, cudaStream_t st);
cudaError_t tc_gemm_tanh(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                         int n_valid, int k_blocks, int H, float* htilde, XOut xg, float* scratch,
                         unsigned int* counters, int num_sms, StepCtl ctl, cudaStream_t st);
size_t fused_scratch_floats(int m_pad, int n_rows_pad, int n_group, int k_blocks, int num_sms);
cudaError_t simt_gen_partials(const float* logits, int v_pad, const GenOut& g, StepCtl ctl, cudaStream_t st);

void launch_embed_gather(const float* emb, int E, const int* ids, const int* lens, int B, int S_max, XOut x,
                         cudaStream_t st);
void launch_enc_cell(const float* Z, int z_ld, const float* P, int splits, int p_rows_pad, int p_ld,
                     const float* bias, int Hd, int B, const int* lens, int S_max, int t, int backward, float* h_st,
                     float* c_st, int st_ld, XOut xrec, XOut xnext, int next_col, float* mem, int mem_ld,
                     int mem_col, cudaStream_t st);
void launch_dec_cell(const float* P, int splits, int p_rows_pad, int p_ld, const float* bias, const float* cg,
                     float* c_out, float* h_out, int H, int R, CellDst dst, StepCtl ctl, cudaStream_t st);
cudaError_t launch_attention(const float* htop, const float* keys, int key_ld, const float* mem, int val_ld,
                             const int* lens, int B, int S_max, int H, int K, XOut xo, const int* done, int num_sms,
                             StepCtl ctl, cudaStream_t st, AttFold fo);
void launch_attn_out(const float* P, int splits, int p_rows_pad, int p_ld, float* htilde, int H, int R, XOut xg,
                     StepCtl ctl, cudaStream_t st);
void launch_init_decode(const BeamState& bs, int B, int K, const float* enc_h, const float* enc_c, int L, int H,
                        float* dec_h, float* dec_c, int dec_rows_pad, float* htilde, cudaStream_t st);
void launch_gather(const BeamState& bs, const GatherArgs& g, int R, int K, StepCtl ctl, cudaStream_t st);
void launch_beam_merge(const float2* ms, const float* tz, const int* ti, int n_parts, int ps, int rs, int B, int K,
                       int t, int max_len, double lp, const BeamState& bs, const GatherArgs& ga, float* row_lse,
                       float* row_z, int* row_i, StepCtl ctl, cudaStream_t st, int nslice = 1,
                       const VpWait* vw = nullptr);
void launch_finalize(const BeamState& bs, int B, int K, int max_len, int* hyps, int* lens, float* scores, float* raw,
                     float* tlogp, int* unk_pos, cudaStream_t st);
void launch_row_reduce(const float2* ms, const float* tz, const int* ti, int n_vt, int ps, int rs, int R, int K,
                       float* lse, float* oz, int* oi, cudaStream_t st);

void launch_teacher_gather(const int* tgt, int T_max, int t, int B, const GatherArgs& g, cudaStream_t st);
void launch_score_reduce(const float2* ms, int n_vt, int rows_pad, const float* zgold, const int* gold, int B,
                         int T_max, float* out, cudaStream_t st);
void launch_score_row(const float* logits, int v_pad, const float* bias, int V, const int* gold, int B, int T_max,
                      int t, float* out, cudaStream_t st);

static thread_local std::string g_err;

struct Error {
  onmt_status s;
  std::string msg;
};
#define ONMT_CUDA(call)                                                                              \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      throw Error{e_ == cudaErrorMemoryAllocation ? ONMT_E_OOM : ONMT_E_CUDA,                        \
                  std::string(#call) + ": " + cudaGetErrorString(e_)};                               \
  } while (0)

static inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// NVTX range for the host-side phases (C-ABI calls, and the enqueue of encode / decode /
// finalize - inside a graph capture these mark when the graph was built, replays show as
// the enclosing API range)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ TMA descriptors
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ONMT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error{ONMT_E_CUDA, "cuTensorMapEncodeTiled not available"};
    fn = (PFN_encodeTiled_t)p;
  }
  return fn;
}
// bf16 [rows x k_pad] row-major, box {64 (=128 B), box_rows}, 128-byte swizzle.
static CUtensorMap make_tmap(const void* base, int k_pad, int rows, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)k_pad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)k_pad * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error{ONMT_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return m;
}

// ------------------------------------------------------------------ device buffers
static uint64_t g_alloc_gen = 0;   // bumped on every device (re)allocation: invalidates cached graphs

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    ONMT_CUDA(cudaMalloc(&p, n));
    bytes = n;
    ++g_alloc_gen;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

static float bf16_round_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// GEMM weight operand: [m_pad x k_pad] (bf16 for bf16 models, fp32 otherwise).
struct Mat {
  int m = 0, k = 0, m_pad = 0, k_pad = 0;
  bool bf16 = false;
  DevBuf w;
  CUtensorMap tmap;
  void upload(const std::vector<float>& host, int m_, int k_, bool bf) {  // host already padded
    m = m_; k = k_; m_pad = round_up(m_, kTileM); k_pad = round_up(k_, kBK); bf16 = bf;
    if (bf) {
      std::vector<__nv_bfloat16> hb(host.size());
      for (size_t i = 0; i < host.size(); ++i) hb[i] = __float2bfloat16_rn(host[i]);
      w.ensure(hb.size() * 2);
      ONMT_CUDA(cudaMemcpy(w.p, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
      tmap = make_tmap(w.p, k_pad, m_pad, kTileM);
    } else {
      w.ensure(host.size() * 4);
      ONMT_CUDA(cudaMemcpy(w.p, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
    }
  }
};

struct RowPlan {
  int rows_pad, n_group;
};
static RowPlan plan_rows(int n) {
  int p = round_up(std::max(n, 1), 16);
  if (p <= 256) return {p, p};
  int g = (p + 255) / 256;
  int grp = round_up((p + g - 1) / g, 16);
  return {grp * g, grp};
}

// Activation operand [rows_pad x k_pad]: fp32 copy and (bf16 models) hi/lo planes.
struct Act {
  int rows = 0, rows_pad = 0, n_group = 0, k = 0, k_pad = 0;
  bool bf16 = false;
  DevBuf f32, hl;
  CUtensorMap tmap;           // box {64, n_group}
  int rg_ng = 0;              // box rows of rg_tmap (0: not built for the current buffers)
  CUtensorMap rg_tmap;        // box {64, rg_ng}: single-split decoder gate GEMMs re-grouped (§6.4)
  void ensure(int rows_, int k_, bool bf) {
    RowPlan rp = plan_rows(rows_);
    int kp = round_up(k_, kBK);
    if (rp.rows_pad == rows_pad && kp == k_pad && bf == bf16 && f32.p) { rows = rows_; return; }
    rg_ng = 0;
    rows = rows_; rows_pad = rp.rows_pad; n_group = rp.n_group; k = k_; k_pad = kp; bf16 = bf;
    f32.ensure((size_t)rows_pad * k_pad * 4);
    ONMT_CUDA(cudaMemset(f32.p, 0, (size_t)rows_pad * k_pad * 4));
    if (bf) {
      hl.ensure((size_t)2 * rows_pad * k_pad * 2);
      ONMT_CUDA(cudaMemset(hl.p, 0, (size_t)2 * rows_pad * k_pad * 2));
      tmap = make_tmap(hl.p, k_pad, 2 * rows_pad, n_group);
    }
  }
  XOut xo(bool use_tc) const {
    XOut x;
    x.f32 = use_tc ? nullptr : f32.as<float>();
    x.hl = use_tc ? hl.as<__nv_bfloat16>() : nullptr;
    x.rows_pad = rows_pad;
    x.k_pad = k_pad;
    return x;
  }
};

struct EvPair {
  cudaEvent_t a, b;
};
// CUDA-event pairs around a kernel family.  Pairs recorded by direct launches return to the
// free list after drain(); pairs baked into a cached graph stay owned by the graph and are
// re-queued after every replay.
struct EventPairs {
  std::vector<EvPair> all, free_;
  std::vector<std::pair<EvPair, bool>> pending;
  double acc_ms = 0;
  int64_t count = 0;
  ~EventPairs() {
    for (auto& p : all) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  }
  EvPair acquire() {
    if (free_.empty()) {
      EvPair p;
      ONMT_CUDA(cudaEventCreate(&p.a));
      ONMT_CUDA(cudaEventCreate(&p.b));
      all.push_back(p);
      free_.push_back(p);
    }
    EvPair p = free_.back();
    free_.pop_back();
    return p;
  }
  void release(const std::vector<EvPair>& v) { free_.insert(free_.end(), v.begin(), v.end()); }
  void drain() {
    for (auto& pp : pending) {
      float ms = 0;
      ONMT_CUDA(cudaEventElapsedTime(&ms, pp.first.a, pp.first.b));
      acc_ms += ms;
      ++count;
      if (pp.second) free_.push_back(pp.first);
    }
    pending.clear();
  }
};

// Event record usable both on a plain stream and inside stream capture (external node).
static void ev_record(cudaEvent_t e, cudaStream_t s, bool capturing) {
  if (capturing) ONMT_CUDA(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
  else ONMT_CUDA(cudaEventRecord(e, s));
}

struct GraphCache {
  cudaGraphExec_t exec = nullptr;
  std::vector<int64_t> key;
  int64_t kernels = 0;
  uint64_t last_use = 0;
  std::vector<std::pair<std::string, EvPair>> ev_nodes;   // profiling events baked into the graph
};
constexpr int kGraphCacheEntries = 8;   // distinct (shape, pointer set) graphs kept instantiated

}  // namespace onmt

using namespace onmt;

struct onmt_model {
  int device = 0;
  onmt_precision prec = ONMT_PREC_FP32;
  int L = 0, E = 0, H = 0, Hd = 0, Vs = 0, Vt = 0, D = 1;
  bool bidir = false, general = false;
  bool use_tc = false;       // tcgen05 GEMM backend (bf16 models)
  int profile = 0;             // 0 off, 1 generator launches only, 2 every kernel family
  bool fused = true;           // split-K GEMM with the reduction and the cell / tanh epilogue fused in
                               // (one launch per layer instead of GEMM + consumer kernel)
  bool gen_step = true;        // K-outer persistent generator (gen_step.cu)
  bool regroup = true;         // unfused single-split gate GEMMs in smaller row groups (§6.4)
  bool fold_wout = true;       // W_out folded into the top cell layer + attention (no W_out launch)
  bool enc_persistent = true;  // encoder recurrence of a layer as one persistent kernel (enc_rec.cu)
  bool enc_cluster = true;     // ... as one cluster per direction with the state on chip (enc_cl.cu)
  bool fold_cur = false;       // ... for the call being enqueued (fold_on)
  bool use_graph = true;
  bool rsplit = true;          // recurrent-split decode step where it applies
  int test_gen_world = 0;      // onmt_test_gen: emulate this many vocabulary-parallel ranks (sequential launches)
  bool rs_cur = false;         // ... for the call being enqueued
  int num_sms = 148;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  int64_t launches = 0;

  // weights
  DevBuf emb_src, emb_tgt;                   // fp32 [V x E]
  std::vector<std::unique_ptr<Mat>> enc_wih, enc_whh;  // [l*D + d]
  std::vector<std::unique_ptr<Mat>> enc_wcat;          // [l] (D == 1, bf16): [W_ih | W_hh] for the wavefront encoder
  bool enc_wavefront = true;                           // unidirectional stacked encoder as a layer wavefront
  std::vector<std::unique_ptr<DevBuf>> enc_bias;
  std::vector<std::unique_ptr<Mat>> dec_w;
  std::vector<std::unique_ptr<DevBuf>> dec_bias;
  Mat attn_win, attn_win_t, attn_wout, gen_w;
  DevBuf gen_b;
  Mat attn_woc;                              // W_out[:, :H] (value projection, folded W_out)
  bool copy = false;                         // copy / pointer generator (copy.w, copy.b present)
  DevBuf copy_w;                             // [H] fp32 (bf16-rounded in bf16 mode)
  float copy_b = 0.f;
  DevBuf woh_t;                              // W_out[:, H:2H] bf16 per 32-unit tile, swizzled (gemm_fused.cu)
  // recurrent-split step (bf16 models with L >= 2)
  Mat wg;                                    // gate-tile weights [(L+1) blocks of 4H rows][H]: W_feed (dec.l0.w_ih
                                             // input-feed columns), then W_hh of layers 1..L, gate-interleaved
  std::vector<std::unique_ptr<Mat>> dec_wih; // [L]: layer l >= 1's W_ih alone (K = H); [0] unused
  DevBuf emb_proj;                           // T = E_tgt W_emb^T  [V rows][4H rounded to 128] fp32

  // encoder workspace
  DevBuf d_ids, d_lens;
  Act enc_in0, enc_mid[2], enc_rec[2], enc_rec2[2];   // enc_rec2: 2nd parity (persistent recurrence)
  DevBuf er_bar;                             // step barriers of the persistent encoder recurrence
  Act wave_rec[4][2];                        // wavefront encoder: per-layer recurrent-operand parity buffers
  DevBuf wave_cnt;                           // wavefront encoder: per-layer finished-CTA counters
  DevBuf enc_z[2], enc_p, mem, enc_h, enc_c, keys, vals;
  Act mem_x;                                 // memory bank as a GEMM operand (keys / values GEMMs)
  // decoder workspace
  std::vector<std::unique_ptr<Act>> xdec;    // [L]
  Act xo, xg;
  DevBuf dec_p, st_h, st_c, st_cg, htilde, logits;
  DevBuf f_scratch, f_count;                 // fused GEMM partial tiles + per-tile arrival counters
  DevBuf g_thr;                              // generator: shared per-row top-K thresholds [2][rows_pad] + slots [2][rows_pad][16]
  DevBuf woh_part;                           // folded W_out: top-layer shares W_out[:, units] h [tiles][rows_pad][H]
  DevBuf pgate, gbias;                       // recurrent split: gate tiles [L+1][rows_pad][G], gate biases [L-1][rows_pad][G]
  Act xr[8];                                 // recurrent split: layer l >= 1's operand [h_{l-1}] (K = H)
  DevBuf g_ms, g_tz, g_ti;
  DevBuf row_lse, row_z, row_i;
  DevBuf b_cum, b_live, b_y, b_prow, b_done, b_ndone, b_bt, b_br, b_braw, b_bnorm;
  DevBuf h_par, h_tok, h_lp, s_score, s_par;
  DevBuf b_att, b_catt, h_amax;              // coverage / unknown replacement state
  DevBuf d_ext;                              // copy models: the call's extended source ids [B][S_max]
  DevBuf o_hyps, o_lens, o_scores, o_raw, o_tlogp, o_unk;

  std::map<std::string, EventPairs> evs;   // per kernel family ("gen", "step", "encode", ...)
  bool capturing = false;
  std::vector<GraphCache> graphs;            // LRU cache of instantiated whole-call graphs
  uint64_t graph_clock = 0;
  int64_t graph_captures = 0;                // captures since load (corpus runs: should stop growing)
  onmt_plan_info plan{};                     // how the last call ran (onmt_last_plan)
  // vocabulary-parallel generator: this rank's exchange
  // buffer (peers store partials + flags into it over NVLink) and the mapped buffers of every rank
  struct Vp {
    int world = 0, rank = 0;
    DevBuf own, seq;
    void* peer[8] = {};
    bool ipc[8] = {};
    int rows_cap = 0;
    size_t parity_bytes = 0;
  } vp;
  static constexpr int kVpCt = 256, kVpK = 16, kVpG = 4;     // partials per row, beam, row groups (caps)
  GraphCache* cap_graph = nullptr;           // the graph being captured (profiling event nodes)
  // teacher-forced scoring workspace
  Act xs_all;                                // generator operand of every (step, sentence) row
  DevBuf s_tgt, s_gold, s_zgold, s_out, s_ms, s_tz, s_ti;

  ~onmt_model() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    for (int w = 0; w < 8; ++w)
      if (vp.ipc[w] && vp.peer[w]) cudaIpcCloseMemHandle(vp.peer[w]);
    if (own_stream) cudaStreamDestroy(own_stream);
  }
};

namespace onmt {

static void count(onmt_model* m, int n = 1) { m->launches += n; }

// vocabulary-parallel exchange buffer, per parity: ms [rows_cap][Ct] float2 | tz [rows_cap][Ct][K]
// | ti [rows_cap][Ct][K] | flags [groups][Ct] u64 (strides of the call's Ct / K inside the caps)
struct VpOffsets {
  size_t ms, tz, ti, flag;
};
static VpOffsets vp_offsets(const onmt_model* m, int parity) {
  const size_t rc = (size_t)m->vp.rows_cap, Ct = onmt_model::kVpCt, Kc = onmt_model::kVpK;
  VpOffsets o;
  o.ms = (size_t)parity * m->vp.parity_bytes;
  o.tz = o.ms + rc * Ct * 8;
  o.ti = o.tz + rc * Ct * Kc * 4;
  o.flag = o.ti + rc * Ct * Kc * 4;
  return o;
}
static size_t vp_parity_bytes(int rows_cap) {
  const size_t rc = (size_t)rows_cap, Ct = onmt_model::kVpCt, Kc = onmt_model::kVpK;
  return ((rc * Ct * 8 + 2 * rc * Ct * Kc * 4 + (size_t)onmt_model::kVpG * Ct * 8) + 255) / 256 * 256;
}
// generator CTAs per row group on each rank (partials per row = world x this <= kVpCt)
static int vp_ctas(const onmt_model* m, int groups) {
  return std::max(1, std::min(m->num_sms / std::max(groups, 1), onmt_model::kVpCt / std::max(m->vp.world, 1)));
}

static int auto_splits(onmt_model* m, const Mat& W, int n_groups) {
  int ctas = (W.m_pad / kTileM) * n_groups;
  int s = std::max(1, m->num_sms / std::max(ctas, 1));
  int kb = W.k_pad / kBK;
  return std::min(std::min(s, kb), 16);
}

// P[split][n][m] partial sums of W * X^T; returns the number of splits written.
static int gemm(onmt_model* m, const Mat& W, const Act& X, int n_valid, int splits, float* out, StepCtl ctl) {
  if (W.k_pad != X.k_pad)
    throw Error{ONMT_E_INVALID_ARG, "internal: K mismatch (W " + std::to_string(W.m) + "x" + std::to_string(W.k_pad) +
                                        ", X " + std::to_string(X.rows) + "x" + std::to_string(X.k_pad) + ")"};
  if (splits <= 0) splits = auto_splits(m, W, X.rows_pad / X.n_group);
  if (m->use_tc) {
    int kb = W.k_pad / kBK;
    int kbps = (kb + splits - 1) / splits;
    int eff = (kb + kbps - 1) / kbps;
    ONMT_CUDA(tc_gemm_partial(W.tmap, X.tmap, W.m_pad, X.rows_pad, X.n_group, n_valid, kb, eff, out, ctl, m->stream));
    count(m);
    return eff;
  }
  int eff = simt_effective_splits(W.k_pad, splits);
  ONMT_CUDA(simt_gemm_partial(W.w.p, W.bf16, W.m_pad, W.k_pad, X.f32.as<float>(), X.rows_pad, n_valid, eff, out, ctl,
                              m->stream));
  count(m);
  return eff;
}

// ---- per-kernel-family CUDA-event timing (profile mode); inside stream capture the events
// become external event-record nodes of the cached graph
static bool prof_on(onmt_model* m, const char* name) {
  return m->profile >= 2 || (m->profile == 1 && std::strcmp(name, "gen") == 0);
}
static EvPair prof_begin(onmt_model* m, const char* name) {
  EvPair ev{};
  if (!prof_on(m, name)) return ev;
  ev = m->evs[name].acquire();
  ev_record(ev.a, m->stream, m->capturing);
  return ev;
}
static void prof_end(onmt_model* m, const char* name, const EvPair& ev) {
  if (!prof_on(m, name)) return;
  ev_record(ev.b, m->stream, m->capturing);
  if (m->capturing) m->cap_graph->ev_nodes.push_back({name, ev});
  else m->evs[name].pending.push_back({ev, true});
}

// does the decode step run the K-outer generator (gen_step.cu) for row groups of n_group?
static bool gen_step_chosen(onmt_model* m, int n_group, int groups) {
  const int n_vt = (m->Vt + kVTile - 1) / kVTile;
  if (!(m->use_tc && m->gen_step && gen_step_parts(n_vt, n_group, groups, m->num_sms) > 0)) return false;
  // the one-buffer plan of wide row groups measured slower than the tile-outer generator (c4:
  // 123.6 vs 118 us per step): only where the latter does not fit (e.g. 256 rows)
  return !(gen_step_wide_plan(n_vt, n_group, groups, m->num_sms) && gen_persistent_fits(n_group));
}
static bool use_gen_step(onmt_model* m, const Act& X) { return gen_step_chosen(m, X.n_group, X.rows_pad / X.n_group); }
static int gen_parts(onmt_model* m, const Act& X) {
  const int n_vt = (m->Vt + kVTile - 1) / kVTile;
  if (use_gen_step(m, X)) return gen_step_parts(n_vt, X.n_group, X.rows_pad / X.n_group, m->num_sms);
  return m->use_tc ? gen_persistent_parts(n_vt, X.rows_pad / X.n_group, m->num_sms, 1) : n_vt;
}

static void gen(onmt_model* m, const Act& X, const GenOut& g, StepCtl ctl) {
  EvPair ev = prof_begin(m, "gen");
  if (m->use_tc) {
    ONMT_CUDA(tc_gen_persistent(m->gen_w.tmap, X.tmap, m->gen_w.m_pad / kTileM, X.rows_pad, X.n_group,
                                m->gen_w.k_pad / kBK, m->num_sms, 1, g, ctl, m->stream));
    count(m);
  } else {
    m->logits.ensure((size_t)X.rows_pad * m->gen_w.m_pad * 4);
    ONMT_CUDA(simt_gemm_partial(m->gen_w.w.p, m->gen_w.bf16, m->gen_w.m_pad, m->gen_w.k_pad, X.f32.as<float>(),
                                X.rows_pad, g.rows_valid, 1, m->logits.as<float>(), ctl, m->stream));
    ONMT_CUDA(simt_gen_partials(m->logits.as<float>(), m->gen_w.m_pad, g, ctl, m->stream));
    count(m, 2);
  }
  prof_end(m, "gen", ev);
}

// ------------------------------------------------------------------ loader
struct HostTensor {
  std::vector<uint64_t> dims;
  std::vector<float> v;
};

static std::map<std::string, HostTensor> read_mnmt(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error{ONMT_E_IO, std::string("cannot open ") + path};
  std::vector<char> data((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  size_t off = 0;
  auto need = [&](size_t n) {
    if (off + n > data.size()) throw Error{ONMT_E_FORMAT, "truncated MNMT file"};
  };
  auto u32 = [&]() { need(4); uint32_t v; std::memcpy(&v, data.data() + off, 4); off += 4; return v; };
  auto u64 = [&]() { need(8); uint64_t v; std::memcpy(&v, data.data() + off, 8); off += 8; return v; };
  need(4);
  if (std::memcmp(data.data(), "MNMT", 4) != 0) throw Error{ONMT_E_FORMAT, "bad magic"};
  off = 4;
  if (u32() != 1) throw Error{ONMT_E_FORMAT, "unsupported MNMT version"};
  std::map<std::string, HostTensor> out;
  while (off < data.size()) {
    uint32_t nlen = u32();
    need(nlen);
    std::string name(data.data() + off, nlen);
    off += nlen;
    uint32_t rank = u32();
    if (rank > 8) throw Error{ONMT_E_FORMAT, "rank too large for " + name};
    HostTensor t;
    uint64_t n = 1;
    for (uint32_t i = 0; i < rank; ++i) { t.dims.push_back(u64()); n *= t.dims.back(); }
    if (u32() != 0) throw Error{ONMT_E_FORMAT, "unsupported dtype tag for " + name};
    need(n * 4);
    t.v.resize(n);
    std::memcpy(t.v.data(), data.data() + off, n * 4);
    off += n * 4;
    if (out.count(name)) throw Error{ONMT_E_FORMAT, "duplicate tensor " + name};
    out[name] = std::move(t);
  }
  return out;
}

static const HostTensor& get(std::map<std::string, HostTensor>& t, const std::string& n, std::vector<uint64_t> dims,
                             std::vector<std::string>& seen) {
  auto it = t.find(n);
  if (it == t.end()) throw Error{ONMT_E_FORMAT, "missing tensor " + n};
  if (it->second.dims != dims) throw Error{ONMT_E_FORMAT, "bad shape for " + n};
  seen.push_back(n);
  return it->second;
}

// Interleaved gate rows: row 4j+g <- row g*Hn+j of the concatenation [A | B] (columns).
static std::vector<float> gate_interleave(const HostTensor& A, const HostTensor* Bm, int Hn, int& K) {
  int ka = (int)A.dims[1], kb = Bm ? (int)Bm->dims[1] : 0;
  K = ka + kb;
  int mp = round_up(4 * Hn, kTileM), kp = round_up(K, kBK);
  std::vector<float> h((size_t)mp * kp, 0.f);
  for (int g = 0; g < 4; ++g)
    for (int j = 0; j < Hn; ++j) {
      float* dst = h.data() + (size_t)(4 * j + g) * kp;
      const float* a = A.v.data() + (size_t)(g * Hn + j) * ka;
      std::copy(a, a + ka, dst);
      if (Bm) {
        const float* b = Bm->v.data() + (size_t)(g * Hn + j) * kb;
        std::copy(b, b + kb, dst + ka);
      }
    }
  return h;
}
static std::vector<float> gate_bias(const HostTensor& bi, const HostTensor& bh, int Hn) {
  std::vector<float> b(4 * Hn);
  for (int g = 0; g < 4; ++g)
    for (int j = 0; j < Hn; ++j) b[4 * j + g] = bi.v[g * Hn + j] + bh.v[g * Hn + j];
  return b;
}
static std::vector<float> plain_pad(const HostTensor& A) {
  int mm = (int)A.dims[0], kk = (int)A.dims[1];
  int mp = round_up(mm, kTileM), kp = round_up(kk, kBK);
  std::vector<float> h((size_t)mp * kp, 0.f);
  for (int i = 0; i < mm; ++i) std::copy(A.v.data() + (size_t)i * kk, A.v.data() + (size_t)(i + 1) * kk, h.data() + (size_t)i * kp);
  return h;
}
static void upload_f32(DevBuf& d, const std::vector<float>& h) {
  d.ensure(h.size() * 4);
  ONMT_CUDA(cudaMemcpy(d.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
}

// Recurrent-split step weights.  The layer-1 gates of step t+1 are
//   W_emb E_tgt[y] + W_feed h~_t[p] + W_hh1 h_1,t[p] + b_1
// and (W x)[p] = W (x[p]): everything but the embedding term is computed for all step-t rows
// BEFORE the beam step picks the parents p - by gate tiles of the generator kernel, whose
// activation operand becomes [h~ | h_1 | ... | h_L] - and the embedding term is a row of the
// table T = E_tgt W_emb^T (computed here once, one tcgen05 GEMM over the vocabulary).
// Layers l >= 2 keep only W_ih h_{l-1} on the critical path; W_hh h_l comes from gate tiles.
static int gemm(onmt_model* m, const Mat& W, const Act& X, int n_valid, int splits, float* out, StepCtl ctl);
static void build_rsplit(onmt_model* m, std::map<std::string, HostTensor>& t) {
  const int H = m->H, E = m->E, L = m->L;
  const int G = round_up(4 * H, kTileM), kpH = round_up(H, kBK);
  // gate-tile weights: block q = 0: W_feed = dec.l0.w_ih[:, E:E+H]; q = l (1..L): dec.l{l-1}.w_hh
  std::vector<float> wg((size_t)(L + 1) * G * kpH, 0.f);
  for (int q = 0; q <= L; ++q) {
    const HostTensor& src = q == 0 ? t.at("dec.l0.w_ih") : t.at("dec.l" + std::to_string(q - 1) + ".w_hh");
    const int ld = (int)src.dims[1], c0 = q == 0 ? E : 0;
    for (int g = 0; g < 4; ++g)
      for (int j = 0; j < H; ++j) {
        const float* a = src.v.data() + (size_t)(g * H + j) * ld + c0;
        std::copy(a, a + H, wg.data() + ((size_t)q * G + 4 * j + g) * kpH);
      }
  }
  m->wg.upload(wg, (L + 1) * G, kpH, true);
  // W_ih of layers >= 2 alone (K = H)
  m->dec_wih.clear();
  m->dec_wih.push_back(nullptr);
  for (int l = 1; l < L; ++l) {
    int K;
    auto hw = gate_interleave(t.at("dec.l" + std::to_string(l) + ".w_ih"), nullptr, H, K);
    auto w = std::make_unique<Mat>();
    w->upload(hw, 4 * H, K, true);
    m->dec_wih.push_back(std::move(w));
  }
  // T = E_tgt W_emb^T: W_emb = dec.l0.w_ih[:, 0:E] (gate-interleaved), E_tgt as a bf16 operand
  // (the model's weights are bf16, so its lo plane is zero and the products are exact)
  {
    HostTensor we;
    const HostTensor& w0 = t.at("dec.l0.w_ih");
    we.dims = {(uint64_t)4 * H, (uint64_t)E};
    we.v.resize((size_t)4 * H * E);
    for (int r = 0; r < 4 * H; ++r)
      std::copy(w0.v.data() + (size_t)r * (E + H), w0.v.data() + (size_t)r * (E + H) + E, we.v.data() + (size_t)r * E);
    int K = 0;
    const std::vector<float> hw = gate_interleave(we, nullptr, H, K);   // (sets K before upload reads it)
    Mat W;
    W.upload(hw, 4 * H, K, true);
    Act X;
    X.ensure(m->Vt, E, true);
    const HostTensor& et = t.at("dec.emb");
    std::vector<__nv_bfloat16> hl((size_t)2 * X.rows_pad * X.k_pad, __float2bfloat16_rn(0.f));
    for (int v = 0; v < m->Vt; ++v)
      for (int k = 0; k < E; ++k) hl[(size_t)v * X.k_pad + k] = __float2bfloat16_rn(et.v[(size_t)v * E + k]);
    ONMT_CUDA(cudaMemcpy(X.hl.p, hl.data(), hl.size() * 2, cudaMemcpyHostToDevice));
    m->emb_proj.ensure((size_t)X.rows_pad * G * 4);
    gemm(m, W, X, m->Vt, 1, m->emb_proj.as<float>(), StepCtl{nullptr, 0});
    ONMT_CUDA(cudaStreamSynchronize(m->stream));
  }
}

static void load_model(onmt_model* m, const char* path) {
  auto t = read_mnmt(path);
  auto has = [&](const std::string& n) { return t.count(n) > 0; };
  if (!has("enc.emb") || !has("dec.emb") || !has("dec.l0.w_hh") || !has("enc.l0.fwd.w_hh") || !has("gen.w"))
    throw Error{ONMT_E_FORMAT, "missing core tensors"};
  if (t["enc.emb"].dims.size() != 2 || t["dec.l0.w_hh"].dims.size() != 2 || t["enc.l0.fwd.w_hh"].dims.size() != 2 ||
      t["gen.w"].dims.size() != 2)
    throw Error{ONMT_E_FORMAT, "bad rank"};
  m->Vs = (int)t["enc.emb"].dims[0];
  m->E = (int)t["enc.emb"].dims[1];
  m->H = (int)t["dec.l0.w_hh"].dims[1];
  m->Hd = (int)t["enc.l0.fwd.w_hh"].dims[1];
  m->Vt = (int)t["gen.w"].dims[0];
  m->bidir = has("enc.l0.bwd.w_ih");
  m->D = m->bidir ? 2 : 1;
  m->general = has("attn.w_in");
  m->L = 0;
  while (has("dec.l" + std::to_string(m->L) + ".w_ih")) ++m->L;
  if (m->L < 1 || m->L > 8) throw Error{ONMT_E_FORMAT, "decoder layer count must be 1..8"};
  if (m->Hd * m->D != m->H) throw Error{ONMT_E_FORMAT, "encoder width [fwd;bwd] must equal decoder width"};
  if (m->Vt < ONMT_K_MAX || m->Vs < 1) throw Error{ONMT_E_FORMAT, "vocabulary too small"};
  const bool bf = m->prec == ONMT_PREC_BF16;
  if (bf)
    for (auto& kv : t)
      for (auto& x : kv.second.v) x = bf16_round_host(x);
  std::vector<std::string> seen;
  const uint64_t E = m->E, H = m->H, Hd = m->Hd, Vs = m->Vs, Vt = m->Vt;
  const auto& es = get(t, "enc.emb", {Vs, E}, seen);
  upload_f32(m->emb_src, es.v);
  const char* dn[2] = {"fwd", "bwd"};
  for (int l = 0; l < m->L; ++l)
    for (int d = 0; d < m->D; ++d) {
      std::string p = "enc.l" + std::to_string(l) + "." + dn[d] + ".";
      uint64_t in = l == 0 ? E : (uint64_t)m->D * Hd;
      const auto& wih = get(t, p + "w_ih", {4 * Hd, in}, seen);
      const auto& whh = get(t, p + "w_hh", {4 * Hd, Hd}, seen);
      const auto& bih = get(t, p + "b_ih", {4 * Hd}, seen);
      const auto& bhh = get(t, p + "b_hh", {4 * Hd}, seen);
      int Ka, Kb;
      auto ha = gate_interleave(wih, nullptr, (int)Hd, Ka);
      auto hb = gate_interleave(whh, nullptr, (int)Hd, Kb);
      auto a = std::make_unique<Mat>();
      a->upload(ha, 4 * (int)Hd, Ka, bf);
      auto b = std::make_unique<Mat>();
      b->upload(hb, 4 * (int)Hd, Kb, bf);
      auto bb = std::make_unique<DevBuf>();
      upload_f32(*bb, gate_bias(bih, bhh, (int)Hd));
      m->enc_wih.push_back(std::move(a));
      m->enc_whh.push_back(std::move(b));
      m->enc_bias.push_back(std::move(bb));
      if (bf && m->D == 1) {
        // wavefront encoder (enc_wave.cu): layer l >= 1 reduces [h_{l-1,t} ; h_{l,t-1}] against
        // [W_ih | W_hh], each part padded to whole 64-column K blocks, gate rows interleaved
        std::unique_ptr<Mat> wc;
        if (l >= 1) {
          const int kin = round_up((int)in, kBK), kown = round_up((int)Hd, kBK);
          const int mp = round_up(4 * (int)Hd, kTileM);
          std::vector<float> h((size_t)mp * (kin + kown), 0.f);
          for (int g = 0; g < 4; ++g)
            for (uint64_t j = 0; j < Hd; ++j) {
              float* dst = h.data() + (size_t)(4 * j + g) * (kin + kown);
              const float* wa = wih.v.data() + (size_t)(g * Hd + j) * in;
              const float* wb = whh.v.data() + (size_t)(g * Hd + j) * Hd;
              std::copy(wa, wa + in, dst);
              std::copy(wb, wb + Hd, dst + kin);
            }
          wc = std::make_unique<Mat>();
          wc->upload(h, 4 * (int)Hd, kin + kown, bf);
        }
        m->enc_wcat.push_back(std::move(wc));
      }
    }
  const auto& et = get(t, "dec.emb", {Vt, E}, seen);
  upload_f32(m->emb_tgt, et.v);
  for (int l = 0; l < m->L; ++l) {
    std::string p = "dec.l" + std::to_string(l) + ".";
    uint64_t in = l == 0 ? E + H : H;
    const auto& wih = get(t, p + "w_ih", {4 * H, in}, seen);
    const auto& whh = get(t, p + "w_hh", {4 * H, H}, seen);
    const auto& bih = get(t, p + "b_ih", {4 * H}, seen);
    const auto& bhh = get(t, p + "b_hh", {4 * H}, seen);
    int K;
    auto hw = gate_interleave(wih, &whh, (int)H, K);
    auto w = std::make_unique<Mat>();
    w->upload(hw, 4 * (int)H, K, bf);
    auto bb = std::make_unique<DevBuf>();
    upload_f32(*bb, gate_bias(bih, bhh, (int)H));
    m->dec_w.push_back(std::move(w));
    m->dec_bias.push_back(std::move(bb));
  }
  if (bf && m->L >= 2 && m->rsplit) build_rsplit(m, t);
  if (m->general) {
    const auto& wi = get(t, "attn.w_in", {H, H}, seen);
    m->attn_win.upload(plain_pad(wi), (int)H, (int)H, bf);
    HostTensor wt;                                  // W_in^T: keys k_s = W_in^T m_s (DESIGN.md §6 K4)
    wt.dims = {H, H};
    wt.v.resize(H * H);
    for (uint64_t i = 0; i < H; ++i)
      for (uint64_t j = 0; j < H; ++j) wt.v[i * H + j] = wi.v[j * H + i];
    m->attn_win_t.upload(plain_pad(wt), (int)H, (int)H, bf);
  }
  const auto& wo = get(t, "attn.w_out", {H, 2 * H}, seen);
  m->attn_wout.upload(plain_pad(wo), (int)H, 2 * (int)H, bf);
  if (bf) {
    // folded W_out: W_oc = W_out[:, :H] projects the memory bank once per
    // batch (values); W_oh^T = W_out[:, H:2H]^T rows by unit, in the top layer's 32-unit tiles
    HostTensor woc;
    woc.dims = {H, H};
    woc.v.resize(H * H);
    for (uint64_t i = 0; i < H; ++i)
      for (uint64_t j = 0; j < H; ++j) woc.v[i * H + j] = wo.v[i * 2 * H + j];
    m->attn_woc.upload(plain_pad(woc), (int)H, (int)H, bf);
    // W_out[:, H:2H] per top-layer tile of 32 units: [fold_mo(H) outputs][32 units] bf16 with the
    // 64-byte swizzle applied (gemm_fused.cu fold_sw64: the shared-memory image of the fold MMA's
    // A operand, loaded by one bulk copy)
    const size_t tiles = (size_t)m->dec_w[m->L - 1]->m_pad / 4 / 32;
    const size_t mo = (H + 127) / 128 * 128, tb = mo * 64;
    std::vector<__nv_bfloat16> wt(tiles * tb / 2, __float2bfloat16_rn(0.f));
    for (size_t t = 0; t < tiles; ++t)
      for (uint64_t o = 0; o < mo; ++o)
        for (int ul = 0; ul < 32; ++ul) {
          const uint64_t j = t * 32 + ul;
          const size_t off = o * 64 + ((((ul >> 3) ^ (o >> 1)) & 3) << 4) + ((ul & 7) << 1);
          wt[(t * tb + off) / 2] = __float2bfloat16_rn(o < H && j < H ? wo.v[o * 2 * H + H + j] : 0.f);
        }
    m->woh_t.ensure(wt.size() * 2);
    ONMT_CUDA(cudaMemcpy(m->woh_t.p, wt.data(), wt.size() * 2, cudaMemcpyHostToDevice));
  }
  const auto& gw = get(t, "gen.w", {Vt, H}, seen);
  m->gen_w.upload(plain_pad(gw), (int)Vt, (int)H, bf);
  const auto& gb = get(t, "gen.b", {Vt}, seen);
  upload_f32(m->gen_b, gb.v);
  if (t.count("copy.w")) {                          // copy / pointer generator (SPEC S293-301)
    const auto& cw = get(t, "copy.w", {1, H}, seen);
    const auto& cb = get(t, "copy.b", {1}, seen);
    std::vector<float> w = cw.v;
    float bv = cb.v[0];
    if (bf) {                                       // (every tensor of a bf16 model is bf16-rounded)
      for (auto& x : w) x = __bfloat162float(__float2bfloat16_rn(x));
      bv = __bfloat162float(__float2bfloat16_rn(bv));
    }
    upload_f32(m->copy_w, w);
    m->copy_b = bv;
    m->copy = true;
  }
  if (seen.size() != t.size()) throw Error{ONMT_E_FORMAT, "unexpected extra tensors in file"};
  ONMT_CUDA(cudaDeviceSynchronize());
}

// W_out folded away: bf16 models on the fused cell-GEMM path whose top
// layer kernel fits the extra W_out share
static bool fold_on(onmt_model* m, int rows) {
  if (!(m->use_tc && m->fused && m->fold_wout && m->attn_woc.m > 0)) return false;
  const Mat& W = *m->dec_w[m->L - 1];
  const RowPlan rp = plan_rows(rows);
  return tc_cell_fold_fits(W.m_pad, rp.rows_pad, rp.n_group, W.k_pad / kBK, m->H, m->num_sms);
}

// recurrent split: layer l >= 2's GEMM (K = H) splits the hypothesis rows into groups of ns
// instead of splitting K: every CTA owns a whole 128-row x ns-column output tile (no split-K
// exchange through L2), m_tiles x rows_pad / ns <= #SMs
static int rs_nsplit(onmt_model* m, int rows_pad) {
  const int m_tiles = round_up(4 * m->H, kTileM) / kTileM;
  for (int ns = 32; ns <= 256; ns += 16)
    if (rows_pad % ns == 0 && m_tiles * (rows_pad / ns) <= m->num_sms) return ns;
  return 0;
}

// recurrent-split step for a plain translation of R rows: bf16 models with
// the folded W_out, L >= 2, whose gate tiles fit the generator's smaller-share CTAs and whose
// layer kernels (with per-row gate biases) fit
static bool rsplit_on(onmt_model* m, int B, int K, bool att) {
  if (!(m->rsplit && m->use_tc && m->fused && m->gen_step && m->fold_cur && m->L >= 2 && m->wg.m > 0 && !att))
    return false;
  const int H = m->H, R = B * K;
  if ((H & 3) != 0 || (size_t)2 * K * H * 4 > 120 * 1024) return false;       // beam step staging
  const RowPlan rp = plan_rows(R);
  const int groups = rp.rows_pad / rp.n_group;
  if (!gen_step_chosen(m, rp.n_group, groups)) return false;   // (the gate tiles run in gen_step)
  const int n_vt = (m->Vt + kVTile - 1) / kVTile;
  const int G = round_up(4 * H, kTileM);
  const int n_gt = (m->L + 1) * (G / kTileM);
  if (gen_step_gate_capacity(n_vt, rp.n_group, groups, m->num_sms) < n_gt) return false;
  const int ns = rs_nsplit(m, rp.rows_pad);
  if (ns == 0) return false;
  for (int l = 1; l < m->L; ++l) {
    const Mat& W = *m->dec_wih[l];
    const bool ok = l + 1 == m->L
                        ? tc_cell_fold_fits(W.m_pad, rp.rows_pad, ns, W.k_pad / kBK, H, m->num_sms, true)
                        : tc_cell_fits(W.m_pad, rp.rows_pad, ns, W.k_pad / kBK, H, m->num_sms, true);
    if (!ok) return false;
  }
  return true;
}

// ------------------------------------------------------------------ encoder
// splits of the wavefront encoder for this batch (0 = not used): unidirectional bf16 models
// with 2..4 layers whose layers all fit the persistent kernel's shared memory
static int wave_splits(onmt_model* m, int B) {
  if (!(m->use_tc && m->enc_persistent && m->enc_wavefront && m->D == 1 && m->L >= 2 && m->L <= 4 &&
        (int)m->enc_wcat.size() == m->L))
    return 0;
  const RowPlan rp = plan_rows(B);
  if (rp.n_group != rp.rows_pad) return 0;
  int kb[4];
  kb[0] = m->enc_whh[0]->k_pad / kBK;
  for (int l = 1; l < m->L; ++l) kb[l] = m->enc_wcat[l]->k_pad / kBK;
  return enc_wave_splits(m->L, kb, rp.rows_pad, m->enc_whh[0]->m_pad / kTileM, m->num_sms);
}

static void prepare_encoder(onmt_model* m, int B, int S_max) {
  const int rows = B * S_max, H = m->H, Hd = m->Hd, D = m->D;
  m->enc_in0.ensure(rows, m->E, m->prec == ONMT_PREC_BF16);
  if (m->L > 1) { m->enc_mid[0].ensure(rows, H, m->prec == ONMT_PREC_BF16); m->enc_mid[1].ensure(rows, H, m->prec == ONMT_PREC_BF16); }
  for (int d = 0; d < D; ++d) m->enc_rec[d].ensure(B, Hd, m->prec == ONMT_PREC_BF16);
  if (wave_splits(m, B) > 0) {
    for (int l = 0; l < m->L; ++l)
      for (int p = 0; p < 2; ++p) m->wave_rec[l][p].ensure(B, Hd, true);
    m->wave_cnt.ensure(4 * 16 * 8);
  }
  if (m->use_tc && m->enc_persistent) {
    for (int d = 0; d < D; ++d) m->enc_rec2[d].ensure(B, Hd, true);
    if (!m->er_bar.p) {
      m->er_bar.ensure(64 * 4);
      ONMT_CUDA(cudaMemset(m->er_bar.p, 0, 64 * 4));
    }
  }
  const int zrows = std::max(m->enc_in0.rows_pad, m->L > 1 ? m->enc_mid[0].rows_pad : 0);
  const int zld = m->enc_wih[0]->m_pad;
  for (int d = 0; d < D; ++d) m->enc_z[d].ensure((size_t)zrows * zld * 4);
  m->enc_p.ensure((size_t)16 * m->enc_rec[0].rows_pad * m->enc_whh[0]->m_pad * 4);
  m->mem.ensure((size_t)rows * H * 4);
  if (m->general || m->fold_cur) m->mem_x.ensure(rows, H, m->prec == ONMT_PREC_BF16);
  if (m->fold_cur) m->vals.ensure((size_t)m->mem_x.rows_pad * m->attn_woc.m_pad * 4);
  m->enc_h.ensure((size_t)m->L * B * H * 4);
  m->enc_c.ensure((size_t)m->L * B * H * 4);
  if (m->general) m->keys.ensure((size_t)m->mem_x.rows_pad * m->attn_win_t.m_pad * 4);
}

static void enqueue_encoder(onmt_model* m, const int* d_ids, const int* d_lens, int B, int S_max) {
  Nvtx nv("onmt.encode");
  const bool bf = m->use_tc;
  const int rows = B * S_max, H = m->H, Hd = m->Hd, D = m->D;
  StepCtl none{nullptr, 0};
  const int zld = m->enc_wih[0]->m_pad;
  EvPair pe = prof_begin(m, "encode");
  ONMT_CUDA(cudaMemsetAsync(m->mem.p, 0, (size_t)rows * H * 4, m->stream));

  launch_embed_gather(m->emb_src.as<float>(), m->E, d_ids, d_lens, B, S_max, m->enc_in0.xo(bf), m->stream);
  count(m);
  const int WS = wave_splits(m, B);
  if (WS > 0) {
    // unidirectional stack as one wavefront launch (enc_wave.cu): layer 0's input projection
    // is hoisted as usual, every other layer reduces [h_{l-1,t} ; h_{l,t-1}] per step
    gemm(m, *m->enc_wih[0], m->enc_in0, rows, 1, m->enc_z[0].as<float>(), none);
    EncWaveArgs wa{};
    CUtensorMap tw[4], tx[4][2];
    int cta = 0;
    const int T = m->enc_whh[0]->m_pad / kTileM;
    for (int l = 0; l < m->L; ++l) {
      EncWaveLayer& ly = wa.layer[l];
      const Mat& W = l == 0 ? *m->enc_whh[0] : *m->enc_wcat[l];
      ly.T = T;
      ly.S = WS;
      ly.kb = W.k_pad / kBK;
      ly.kb_in = l == 0 ? 0 : round_up(H, kBK) / kBK;
      ly.cta0 = cta;
      cta += T * WS;
      ly.Z = l == 0 ? m->enc_z[0].as<float>() : nullptr;
      ly.z_ld = zld;
      ly.bias = m->enc_bias[l]->as<float4>();
      ly.xrec[0] = m->wave_rec[l][0].xo(true);
      ly.xrec[1] = m->wave_rec[l][1].xo(true);
      ly.h_st = m->enc_h.as<float>() + (size_t)l * B * H;
      ly.c_st = m->enc_c.as<float>() + (size_t)l * B * H;
      ly.st_ld = H;
      const bool top = l + 1 == m->L;
      if (top && (m->general || m->fold_cur)) ly.xnext = m->mem_x.xo(true);
      ly.mem = top ? m->mem.as<float>() : nullptr;
      ly.mem_ld = H;
      tw[l] = W.tmap;
      tx[l][0] = m->wave_rec[l][0].tmap;
      tx[l][1] = m->wave_rec[l][1].tmap;
    }
    wa.L = m->L; wa.Hd = Hd; wa.B = B; wa.N = m->wave_rec[0][0].rows_pad; wa.S_max = S_max;
    wa.lens = d_lens;
    wa.cnt = m->wave_cnt.as<unsigned long long>();
    ONMT_CUDA(launch_enc_wave(tw, tx, wa, cta, WS, m->stream));
    count(m);
  }
  const Act* xin = &m->enc_in0;
  for (int l = 0; l < (WS > 0 ? 0 : m->L); ++l) {
    const Act* xnext = l + 1 < m->L ? &m->enc_mid[l % 2] : nullptr;
    for (int d = 0; d < D; ++d)
      gemm(m, *m->enc_wih[l * D + d], *xin, rows, 1, m->enc_z[d].as<float>(), none);
    {
      const Mat& w0 = *m->enc_whh[l * D];
      const Act& r0 = m->enc_rec[0];
      const int T = w0.m_pad / kTileM, kb = w0.k_pad / kBK;
      if (m->use_tc && m->enc_persistent && m->enc_cluster && r0.n_group == r0.rows_pad &&
          enc_cl_fits(T, kb, r0.rows_pad, D, m->num_sms)) {
        // the whole recurrence of this layer, one cluster per direction, state on chip (enc_cl.cu)
        EncClArgs ca{};
        CUtensorMap tw[2];
        for (int d = 0; d < D; ++d) {
          EncClDir& dr = ca.dir[d];
          dr.Z = m->enc_z[d].as<float>();
          dr.z_ld = zld;
          dr.bias = m->enc_bias[l * D + d]->as<float4>();
          dr.h_st = m->enc_h.as<float>() + (size_t)l * B * H + d * Hd;
          dr.c_st = m->enc_c.as<float>() + (size_t)l * B * H + d * Hd;
          dr.st_ld = H;
          if (xnext) dr.xnext = xnext->xo(bf);
          else if (m->general || m->fold_cur) dr.xnext = m->mem_x.xo(bf);
          dr.next_col = d * Hd;
          dr.mem = l + 1 == m->L ? m->mem.as<float>() : nullptr;
          dr.mem_ld = H;
          dr.mem_col = d * Hd;
          dr.backward = d == 1;
          tw[d] = m->enc_whh[l * D + d]->tmap;
        }
        ca.T = T; ca.Hd = Hd; ca.B = B; ca.N = r0.rows_pad; ca.S_max = S_max; ca.kb = kb;
        ca.lens = d_lens;
        static unsigned long long* ec_trace = nullptr;            // (debug: ONMT_ENC_TRACE, no graph)
        const bool trc = std::getenv("ONMT_ENC_TRACE") && !m->capturing;
        if (trc && !ec_trace) cudaMalloc(&ec_trace, 64 * 8 * 8);
        ca.trace = trc ? ec_trace : nullptr;
        ONMT_CUDA(launch_enc_cl(tw, ca, D, m->stream));
        count(m);
        if (trc) {
          std::vector<unsigned long long> h(64 * 8);
          ONMT_CUDA(cudaStreamSynchronize(m->stream));
          ONMT_CUDA(cudaMemcpy(h.data(), ec_trace, h.size() * 8, cudaMemcpyDeviceToHost));
          for (int t = 8; t < 12; ++t)
            std::fprintf(stderr, "enc_cl l%d t%d: h wait + mma issue %lld  mma done %lld  staged+z %lld  cell+sync %lld  "
                         "to next step %lld ns\n", l, t,
                         (long long)(h[t * 8 + 1] - h[t * 8 + 0]), (long long)(h[t * 8 + 2] - h[t * 8 + 0]),
                         (long long)(h[t * 8 + 3] - h[t * 8 + 2]), (long long)(h[t * 8 + 5] - h[t * 8 + 3]),
                         (long long)(h[(t + 1) * 8 + 0] - h[t * 8 + 5]));
        }
        xin = xnext;
        continue;
      }
      const int S = (m->use_tc && m->enc_persistent && r0.n_group == r0.rows_pad)
                        ? enc_rec_splits(kb, r0.rows_pad, D, T, m->num_sms) : 0;
      if (S > 0) {
        // the whole recurrence of this layer (both directions) in one launch (enc_rec.cu)
        EncRecArgs ea{};
        CUtensorMap tw[2], tx0[2], tx1[2];
        for (int d = 0; d < D; ++d) {
          EncRecDir& dr = ea.dir[d];
          dr.Z = m->enc_z[d].as<float>();
          dr.z_ld = zld;
          dr.bias = m->enc_bias[l * D + d]->as<float4>();
          dr.xrec[0] = m->enc_rec[d].xo(bf);
          dr.xrec[1] = m->enc_rec2[d].xo(bf);
          dr.h_st = m->enc_h.as<float>() + (size_t)l * B * H + d * Hd;
          dr.c_st = m->enc_c.as<float>() + (size_t)l * B * H + d * Hd;
          dr.st_ld = H;
          if (xnext) dr.xnext = xnext->xo(bf);
          else if (m->general || m->fold_cur) dr.xnext = m->mem_x.xo(bf);
          dr.next_col = d * Hd;
          dr.mem = l + 1 == m->L ? m->mem.as<float>() : nullptr;
          dr.mem_ld = H;
          dr.mem_col = d * Hd;
          dr.backward = d == 1;
          tw[d] = m->enc_whh[l * D + d]->tmap;
          tx0[d] = m->enc_rec[d].tmap;
          tx1[d] = m->enc_rec2[d].tmap;
        }
        ea.T = T; ea.S = S; ea.Hd = Hd; ea.B = B; ea.N = r0.rows_pad; ea.S_max = S_max; ea.kb = kb;
        ea.lens = d_lens;
        ea.bar = m->er_bar.as<unsigned int>();
        static unsigned long long* er_trace = nullptr;            // (debug: ONMT_ENC_TRACE, no graph)
        const bool trc = std::getenv("ONMT_ENC_TRACE") && !m->capturing;
        if (trc && !er_trace) cudaMalloc(&er_trace, 64 * 8 * 8);
        ea.trace = trc ? er_trace : nullptr;
        ONMT_CUDA(launch_enc_rec(tw, tx0, tx1, ea, D, m->stream));
        count(m);
        if (trc) {
          std::vector<unsigned long long> h(64 * 8);
          ONMT_CUDA(cudaStreamSynchronize(m->stream));
          ONMT_CUDA(cudaMemcpy(h.data(), er_trace, h.size() * 8, cudaMemcpyDeviceToHost));
          for (int t = 8; t < 12; ++t)
            std::fprintf(stderr, "enc_rec l%d t%d: bar %lld  mma_done %lld  exch %lld  zwait %lld  math %lld  stores %lld  next %lld ns\n", l, t,
                         (long long)(h[t * 8 + 1] - h[t * 8 + 0]), (long long)(h[t * 8 + 3] - h[t * 8 + 1]),
                         (long long)(h[t * 8 + 6] - h[t * 8 + 3]), (long long)(h[t * 8 + 4] - h[t * 8 + 6]),
                         (long long)(h[t * 8 + 2] - h[t * 8 + 4]), (long long)(h[t * 8 + 7] - h[t * 8 + 2]),
                         (long long)(h[(t + 1) * 8 + 0] - h[t * 8 + 5]));
        }
        xin = xnext;
        continue;
      }
    }
    for (int t = 0; t < S_max; ++t)
      for (int d = 0; d < D; ++d) {
        const Mat& whh = *m->enc_whh[l * D + d];
        int splits = 0;
        const float* P = nullptr;
        if (t > 0) {
          splits = gemm(m, whh, m->enc_rec[d], B, 0, m->enc_p.as<float>(), none);
          P = m->enc_p.as<float>();
        }
        XOut xn{};
        if (xnext) xn = xnext->xo(bf);
        else if (m->general || m->fold_cur) xn = m->mem_x.xo(bf);   // top layer: memory as a GEMM operand
        launch_enc_cell(m->enc_z[d].as<float>(), zld, P, splits, m->enc_rec[d].rows_pad, whh.m_pad,
                        m->enc_bias[l * D + d]->as<float>(), Hd, B, d_lens, S_max, t, d == 1,
                        m->enc_h.as<float>() + (size_t)l * B * H + d * Hd,
                        m->enc_c.as<float>() + (size_t)l * B * H + d * Hd, H, m->enc_rec[d].xo(bf), xn, d * Hd,
                        l + 1 == m->L ? m->mem.as<float>() : nullptr, H, d * Hd, m->stream);
        count(m);
      }
    xin = xnext;
  }
  if (m->general)    // keys k_s = W_in^T m_s for every source position (hoisted 'general' query GEMM)
    gemm(m, m->attn_win_t, m->mem_x, rows, 1, m->keys.as<float>(), none);
  if (m->fold_cur)   // values W_out[:, :H] m_s (folded W_out: the step's context arrives projected)
    gemm(m, m->attn_woc, m->mem_x, rows, 1, m->vals.as<float>(), none);
  prof_end(m, "encode", pe);
  ONMT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ decoder
struct DecodeOut {
  int* hyps;            // [B][nbest][max_len]
  int* lens;            // [B][nbest]
  float* scores;
  float* raw;
  float* tlogp;
  int* unk_pos = nullptr;   // [B][nbest][max_len] source position replacing an <unk>, else -1
};

// Decoding customisations (SPEC S421-424): coverage penalty beta,
// n-best list size, attention-based unknown replacement.  Defaults = the plain path.
struct DecodeOpts {
  double beta = 0.0;
  int nbest = 1;
  bool unk = false;
  const int* src_ext = nullptr;   // copy models: device [B][S_max] extended source ids
  bool att() const { return beta != 0.0 || unk || src_ext; }
};

static BeamState beam_state(onmt_model* m, bool trace, const DecodeOpts& op = DecodeOpts{}, const int* d_lens = nullptr,
                            int S_max = 0) {
  BeamState bs{};
  bs.nbest = op.nbest;
  bs.beta = op.beta;
  if (op.att()) {
    bs.att = m->b_att.as<float>();
    bs.catt = op.beta != 0.0 ? m->b_catt.as<float>() : nullptr;
    bs.hist_amax = op.unk ? m->h_amax.as<int>() : nullptr;
    bs.lens = d_lens;
    bs.S_max = S_max;
  }
  bs.cum = m->b_cum.as<double>();
  bs.live = m->b_live.as<int>();
  bs.y = m->b_y.as<int>();
  bs.prow = m->b_prow.as<int>();
  bs.done = m->b_done.as<int>();
  bs.n_done = m->b_ndone.as<int>();
  bs.best_t = m->b_bt.as<int>();
  bs.best_r = m->b_br.as<int>();
  bs.best_raw = m->b_braw.as<double>();
  bs.best_norm = m->b_bnorm.as<double>();
  bs.hist_parent = m->h_par.as<int>();
  bs.hist_token = m->h_tok.as<int>();
  bs.hist_logp = m->h_lp.as<float>();
  bs.sel_score = trace ? m->s_score.as<double>() : nullptr;
  bs.sel_parent = trace ? m->s_par.as<int>() : nullptr;
  return bs;
}

static void prepare_decoder(onmt_model* m, int B, int S_max, int K, int max_len, bool trace,
                            const DecodeOpts& op = DecodeOpts{}) {
  const bool bfm = m->prec == ONMT_PREC_BF16;
  const int R = B * K, H = m->H, E = m->E, L = m->L;
  while ((int)m->xdec.size() < L) m->xdec.push_back(std::make_unique<Act>());
  m->xdec[0]->ensure(R, E + 2 * H, bfm);
  for (int l = 1; l < L; ++l) m->xdec[l]->ensure(R, 2 * H, bfm);
  m->xo.ensure(R, 2 * H, bfm);
  const int kpH = round_up(H, kBK), G = round_up(4 * H, kTileM);
  m->xg.ensure(R, m->rs_cur ? (L + 1) * kpH : H, bfm);          // recurrent split: [h~ | h_1 | .. | h_L]
  const int rp = m->xg.rows_pad;
  if (m->rs_cur) {
    m->pgate.ensure((size_t)(L + 1) * rp * G * 4);
    m->gbias.ensure((size_t)std::max(L - 1, 1) * rp * G * 4);
    for (int l = 1; l < L; ++l) m->xr[l].ensure(R, H, true);
  }
  size_t pm = (size_t)m->dec_w[0]->m_pad;
  m->dec_p.ensure((size_t)16 * rp * pm * 4);
  m->st_h.ensure((size_t)L * rp * H * 4);
  m->st_c.ensure((size_t)L * rp * H * 4);
  m->st_cg.ensure((size_t)L * rp * H * 4);
  m->htilde.ensure((size_t)rp * H * 4);
  if (m->fold_cur) m->woh_part.ensure((size_t)(m->dec_w[L - 1]->m_pad / kTileM) * rp * H * 4);
  const int n_vt = gen_parts(m, m->xg);
  m->g_ms.ensure((size_t)n_vt * rp * 8);
  m->g_tz.ensure((size_t)n_vt * rp * K * 4);
  m->g_ti.ensure((size_t)n_vt * rp * K * 4);
  m->row_lse.ensure((size_t)R * 4);
  m->row_z.ensure((size_t)R * K * 4);
  m->row_i.ensure((size_t)R * K * 4);
  m->b_cum.ensure((size_t)2 * R * 8);     // double-buffered by step parity
  m->b_live.ensure((size_t)2 * R * 4);
  m->b_y.ensure((size_t)R * 4);
  m->b_prow.ensure((size_t)R * 4);
  m->b_done.ensure((size_t)B * 4);
  m->b_ndone.ensure(4);
  m->b_bt.ensure((size_t)B * op.nbest * 4);
  m->b_br.ensure((size_t)B * op.nbest * 4);
  m->b_braw.ensure((size_t)B * op.nbest * 8);
  m->b_bnorm.ensure((size_t)B * op.nbest * 8);
  if (op.att()) {
    m->b_att.ensure((size_t)R * S_max * 4);
    if (op.beta != 0.0) m->b_catt.ensure((size_t)2 * R * S_max * 4);
    if (op.unk) m->h_amax.ensure((size_t)max_len * R * 4);
  }
  m->h_par.ensure((size_t)max_len * R * 4);
  m->h_tok.ensure((size_t)max_len * R * 4);
  m->h_lp.ensure((size_t)max_len * R * 4);
  if (trace) {
    m->s_score.ensure((size_t)max_len * R * 8);
    m->s_par.ensure((size_t)max_len * R * 4);
    ONMT_CUDA(cudaMemsetAsync(m->s_par.p, 0xff, (size_t)max_len * R * 4, m->stream));
    ONMT_CUDA(cudaMemsetAsync(m->h_tok.p, 0, (size_t)max_len * R * 4, m->stream));
    std::vector<double> ninf((size_t)max_len * R, -INFINITY);
    ONMT_CUDA(cudaMemcpyAsync(m->s_score.p, ninf.data(), ninf.size() * 8, cudaMemcpyHostToDevice, m->stream));
    ONMT_CUDA(cudaStreamSynchronize(m->stream));
  }
  if (!m->use_tc) m->logits.ensure((size_t)m->xg.rows_pad * m->gen_w.m_pad * 4);
  if (m->use_tc) {
    size_t fs = fused_scratch_floats(m->attn_wout.m_pad, m->xo.rows_pad, m->xo.n_group, m->attn_wout.k_pad / kBK,
                                     m->num_sms);
    for (int l = 0; l < L; ++l)
      fs = std::max(fs, fused_scratch_floats(m->dec_w[l]->m_pad, m->xdec[l]->rows_pad, m->xdec[l]->n_group,
                                             m->dec_w[l]->k_pad / kBK, m->num_sms));
    if (m->rs_cur)
      for (int l = 1; l < L; ++l)
        fs = std::max(fs, fused_scratch_floats(m->dec_wih[l]->m_pad, m->xr[l].rows_pad, rs_nsplit(m, m->xr[l].rows_pad),
                                               m->dec_wih[l]->k_pad / kBK, m->num_sms));
    m->f_scratch.ensure(std::max<size_t>(fs, 1) * 4);
    if (m->g_thr.bytes < (size_t)2 * m->xg.rows_pad * 17 * 4) {
      m->g_thr.ensure((size_t)2 * m->xg.rows_pad * 17 * 4);
      ONMT_CUDA(cudaMemset(m->g_thr.p, 0, m->g_thr.bytes));
    }
    const size_t nc = (size_t)(L + 1) * 2048 * 4;
    if (m->f_count.bytes < nc) {
      m->f_count.ensure(nc);
      ONMT_CUDA(cudaMemset(m->f_count.p, 0, nc));
    }
  }
}

// Attention (+ h~ = tanh(W_out [c; h]), folded or by the W_out kernel) on the top layer's h.
static void enqueue_attention(onmt_model* m, const int* d_lens, int B, int S_max, int K, const int* done,
                              XOut xg_dst, StepCtl ctl, float* att_out) {
  const bool bf = m->use_tc;
  const int R = B * K, H = m->H, L = m->L;
  const int rp = m->xg.rows_pad;
  float* hh = m->st_h.as<float>();
  float* P = m->dec_p.as<float>();
  const float* htop = hh + (size_t)(L - 1) * rp * H;
  {
    EvPair pa = prof_begin(m, "attention");
    const float* keys = m->general ? m->keys.as<float>() : m->mem.as<float>();
    const int key_ld = m->general ? m->attn_win_t.m_pad : H;
    AttFold fo{};
    fo.att_out = att_out;
    if (m->fold_cur) {
      fo.wpart = m->woh_part.as<float>();
      fo.n_wt = m->dec_w[L - 1]->m_pad / kTileM;
      fo.rows_pad = rp;
      fo.htilde = m->htilde.as<float>();
      fo.xg = xg_dst;
    }
    ONMT_CUDA(launch_attention(htop, keys, key_ld, m->fold_cur ? m->vals.as<float>() : m->mem.as<float>(),
                               m->fold_cur ? m->attn_woc.m_pad : H, d_lens, B, S_max, H, K, m->xo.xo(bf), done,
                               m->num_sms, ctl, m->stream, fo));
    count(m);
    prof_end(m, "attention", pa);
  }
  if (m->fold_cur) return;                                   // h~ written by the attention combine
  cudaError_t fe = cudaErrorInvalidConfiguration;
  if (m->use_tc && m->fused) {
    EvPair pg = prof_begin(m, "gemm");
    fe = tc_gemm_tanh(m->attn_wout.tmap, m->xo.tmap, m->attn_wout.m_pad, m->xo.rows_pad, m->xo.n_group, R,
                      m->attn_wout.k_pad / kBK, H, m->htilde.as<float>(), xg_dst, m->f_scratch.as<float>(),
                      m->f_count.as<unsigned int>() + (size_t)L * 2048, m->num_sms, ctl, m->stream);
    prof_end(m, "gemm", pg);
    if (fe != cudaErrorInvalidConfiguration) {
      ONMT_CUDA(fe);
      count(m);
    }
  }
  if (fe == cudaErrorInvalidConfiguration) {
    EvPair pg = prof_begin(m, "gemm");
    int s = gemm(m, m->attn_wout, m->xo, R, 0, P, ctl);
    prof_end(m, "gemm", pg);
    EvPair po = prof_begin(m, "attn_out");
    launch_attn_out(P, s, m->xo.rows_pad, m->attn_wout.m_pad, m->htilde.as<float>(), H, R, xg_dst, ctl,
                    m->stream);
    count(m);
    prof_end(m, "attn_out", po);
  }
}

// One decoder step up to h~ (A5 inputs already gathered): the L LSTM layers, attention and
// h~ = tanh(W_out [c; h]); h~ goes to m->htilde (input feed) and to the generator operand
// xg_dst.  Used by translation (per-layer path) and by teacher-forced scoring.
static void enqueue_dec_layers(onmt_model* m, const int* d_lens, int B, int S_max, int K, const int* done,
                               XOut xg_dst, StepCtl ctl, float* att_out = nullptr) {
  const bool bf = m->use_tc;
  const int R = B * K, H = m->H, L = m->L;
  const int rp = m->xg.rows_pad;
  float* hh = m->st_h.as<float>();
  float* cc = m->st_c.as<float>();
  float* cg = m->st_cg.as<float>();
  float* P = m->dec_p.as<float>();
  for (int l = 0; l < L; ++l) {
    const Mat& W = *m->dec_w[l];
    CellDst dst{};
    if (l + 1 < L) {
      dst.x[0] = m->xdec[l + 1]->xo(bf); dst.col[0] = 0; dst.n = 1;
    } else {
      dst.x[0] = m->xo.xo(bf); dst.col[0] = H; dst.n = 1;
    }
    if (m->rs_cur) {                    // recurrent split, step 1: h_l also feeds the gate tiles
      dst.x[1] = m->xg.xo(bf); dst.col[1] = (l + 1) * round_up(H, kBK); dst.n = 2;
    }
    if (m->use_tc && m->fused) {
      // gates GEMM + split-K cluster reduction + LSTM cell in one kernel
      EvPair pg = prof_begin(m, "gemm");
      const Act& X = *m->xdec[l];
      const bool fold_l = m->fold_cur && l + 1 == L;        // top layer also leaves its W_out share
      cudaError_t e = tc_gemm_cell(W.tmap, X.tmap, W.m_pad, X.rows_pad, X.n_group, R, W.k_pad / kBK,
                                   m->dec_bias[l]->as<float>(), cg + (size_t)l * rp * H, cc + (size_t)l * rp * H,
                                   hh + (size_t)l * rp * H, H, dst, m->f_scratch.as<float>(),
                                   m->f_count.as<unsigned int>() + (size_t)l * 2048, m->num_sms, ctl, m->stream,
                                   fold_l ? m->woh_t.as<__nv_bfloat16>() : nullptr,
                                   fold_l ? m->woh_part.as<float>() : nullptr);
      if (fold_l && e == cudaErrorInvalidConfiguration) throw Error{ONMT_E_CUDA, "internal: folded W_out does not fit"};
      prof_end(m, "gemm", pg);
      if (e != cudaErrorInvalidConfiguration) {   // (no cluster shape fits: unfused path below)
        ONMT_CUDA(e);
        count(m);
        continue;
      }
    }
    EvPair pg = prof_begin(m, "gemm");
    int s;
    Act& X = *m->xdec[l];
    const int per = std::max(1, m->num_sms / (W.m_pad / kTileM));
    const int ng = std::min(X.n_group, std::max(16, round_up((R + per - 1) / per, 16)));
    if (m->use_tc && m->regroup && W.k_pad == X.k_pad && ng < X.n_group &&
        auto_splits(m, W, X.rows_pad / X.n_group) == 1) {
      // one K split: row groups as small as the SM count allows (c4: 4 x 160 rows x 32 weight
      // tiles = 128 CTAs instead of 3 x 224 = 96; the per-CTA work scales with the rows)
      if (X.rg_ng != ng) { X.rg_tmap = make_tmap(X.hl.p, X.k_pad, 2 * X.rows_pad, ng); X.rg_ng = ng; }
      ONMT_CUDA(tc_gemm_partial(W.tmap, X.rg_tmap, W.m_pad, X.rows_pad, ng, R, W.k_pad / kBK, 1, P, ctl, m->stream,
                                true));
      count(m);
      s = 1;
    } else {
      s = gemm(m, W, X, R, 0, P, ctl);
    }
    prof_end(m, "gemm", pg);
    EvPair pc = prof_begin(m, "cell");
    launch_dec_cell(P, s, m->xdec[l]->rows_pad, W.m_pad, m->dec_bias[l]->as<float>(), cg + (size_t)l * rp * H,
                    cc + (size_t)l * rp * H, hh + (size_t)l * rp * H, H, R, dst, ctl, m->stream);
    count(m);
    prof_end(m, "cell", pc);
  }
  enqueue_attention(m, d_lens, B, S_max, K, done, xg_dst, ctl, att_out);
}

// Recurrent-split step, steps t >= 2: layer 1 already ran in the previous
// beam step; layers l >= 2 reduce only W_ih h_{l-1} (K = H) and add the gathered recurrent term
// (gb) in the cell epilogue; the top layer leaves its folded W_out share; then attention.
static void enqueue_rs_layers(onmt_model* m, const int* d_lens, int B, int S_max, int K, const int* done, StepCtl ctl) {
  const int R = B * K, H = m->H, L = m->L;
  const int rp = m->xg.rows_pad, kpH = round_up(H, kBK), G = round_up(4 * H, kTileM);
  float* hh = m->st_h.as<float>();
  float* cc = m->st_c.as<float>();
  float* cg = m->st_cg.as<float>();
  const int ns = rs_nsplit(m, rp);
  for (int l = 1; l < L; ++l) {
    const Mat& W = *m->dec_wih[l];
    const Act& X = m->xr[l];
    const CUtensorMap tx = make_tmap(X.hl.p, X.k_pad, 2 * X.rows_pad, ns);   // box: ns hypothesis rows
    CellDst dst{};
    if (l + 1 < L) {
      dst.x[0] = m->xr[l + 1].xo(true); dst.col[0] = 0;
      dst.x[1] = m->xg.xo(true); dst.col[1] = (l + 1) * kpH; dst.n = 2;
    } else {
      dst.x[0] = m->xg.xo(true); dst.col[0] = L * kpH; dst.n = 1;
    }
    const bool top = l + 1 == L;
    EvPair pg = prof_begin(m, "gemm");
    ONMT_CUDA(tc_gemm_cell(W.tmap, tx, W.m_pad, X.rows_pad, ns, R, W.k_pad / kBK, m->dec_bias[l]->as<float>(),
                           cg + (size_t)l * rp * H, cc + (size_t)l * rp * H, hh + (size_t)l * rp * H, H, dst,
                           m->f_scratch.as<float>(), m->f_count.as<unsigned int>() + (size_t)l * 2048, m->num_sms, ctl,
                           m->stream, top ? m->woh_t.as<__nv_bfloat16>() : nullptr,
                           top ? m->woh_part.as<float>() : nullptr, m->gbias.as<float>() + (size_t)(l - 1) * rp * G, G));
    prof_end(m, "gemm", pg);
    count(m);
  }
  enqueue_attention(m, d_lens, B, S_max, K, done, m->xg.xo(true), ctl, nullptr);
}

static void enqueue_decoder(onmt_model* m, const int* d_lens, int B, int S_max, int K, int max_len, float alpha,
                            bool trace, const DecodeOut& out, const DecodeOpts& op) {
  Nvtx nv("onmt.decode");
  const bool bf = m->use_tc;
  const int R = B * K, H = m->H, E = m->E, L = m->L;
  const int rp = m->xg.rows_pad;
  const int groups = rp / m->xg.n_group;
  const int vpC = m->vp.world > 0 ? vp_ctas(m, groups) : 0;        // vocabulary-parallel: CTAs per group here
  const int n_vt = m->vp.world > 0 ? m->vp.world * vpC : gen_parts(m, m->xg);
  BeamState bs = beam_state(m, trace, op, d_lens, S_max);
  if ((op.beta != 0.0 || op.unk) && n_vt > 256)
    throw Error{ONMT_E_UNSUPPORTED, "coverage / unk replacement need the one-CTA-per-sentence beam step (<= 256 generator partials)"};
  float* hh = m->st_h.as<float>();
  float* cc = m->st_c.as<float>();
  float* cg = m->st_cg.as<float>();
  launch_init_decode(bs, B, K, m->enc_h.as<float>(), m->enc_c.as<float>(), L, H, hh, cc, rp, m->htilde.as<float>(),
                     m->stream);
  count(m);
  StepCtl ctl{bs.n_done, B};
  GatherArgs ga{};
  ga.emb_tgt = m->emb_tgt.as<float>();
  ga.E = E; ga.H = H; ga.L = L;
  ga.htilde = m->htilde.as<float>();
  ga.h = hh; ga.c = cc; ga.cg = cg; ga.rows_pad = rp;
  for (int l = 0; l < L; ++l) ga.x[l] = m->xdec[l]->xo(bf);
  ga.v_map = op.src_ext ? m->Vt : 0;
  launch_gather(bs, ga, R, K, StepCtl{nullptr, 0}, m->stream);
  count(m);
  GenOut g;
  g.ms = m->g_ms.as<float2>();
  g.tz = m->g_tz.as<float>();
  g.ti = m->g_ti.as<int>();
  g.bias = m->gen_b.as<float>();
  g.V = m->Vt;
  g.K = K;
  g.rows_valid = R;
  g.rows_pad = rp;
  // copy models: generator row top-K -> extended top-K (copy.cu) -> selection + gather
  auto merge_copy = [&](int n_parts, int ps, int rs, int t, double lp) {
    launch_row_topk(g.ms, g.tz, g.ti, n_parts, ps, rs, B, K, t, bs, m->row_lse.as<float>(), m->row_z.as<float>(),
                    m->row_i.as<int>(), ctl, m->stream);
    CopyArgs ca{};
    ca.htilde = m->htilde.as<float>();
    ca.H = H;
    ca.copy_w = m->copy_w.as<float>();
    ca.copy_b = m->copy_b;
    ca.att = m->b_att.as<float>();
    ca.S_max = S_max;
    ca.src_ext = op.src_ext;
    ca.lens = d_lens;
    ca.gen_w = m->gen_w.w.p;
    ca.gen_ld = m->gen_w.k_pad;
    ca.gen_bf16 = m->gen_w.bf16;
    ca.gen_b = m->gen_b.as<float>();
    ca.V = m->Vt;
    ca.K = K;
    ca.live = bs.live + (size_t)(t & 1) * R;
    ca.row_lse = m->row_lse.as<float>();
    ca.row_z = m->row_z.as<float>();
    ca.row_i = m->row_i.as<int>();
    ca.ctl = ctl;
    ONMT_CUDA(launch_copy_rows(ca, R, m->stream));
    launch_select_gather(B, K, t, max_len, lp, bs, ga, m->row_lse.as<float>(), m->row_z.as<float>(),
                         m->row_i.as<int>(), ctl, m->stream);
    count(m, 3);
  };
  // recurrent split: the beam step runs layer 1's cell for the next step (GatherArgs::rsplit)
  // and the generator computes the gate tiles; step 1 starts from the gathered initial state
  GatherArgs gam = ga;
  GateTiles gt{};
  if (m->rs_cur) {
    const int kpH = round_up(H, kBK), G = round_up(4 * H, kTileM);
    gam.rsplit = 1;
    gam.T = m->emb_proj.as<float>();
    gam.P = m->pgate.as<float>();
    gam.G = G;
    for (int l = 0; l < L; ++l) gam.bias[l] = m->dec_bias[l]->as<float4>();
    gam.gb = m->gbias.as<float>();
    gam.c1_out = cc;
    gam.xh1[0] = m->xr[1].xo(true); gam.col_h1[0] = 0;
    gam.xh1[1] = m->xg.xo(true); gam.col_h1[1] = kpH;
    gt = GateTiles{&m->wg.tmap, (L + 1) * (G / kTileM), G / kTileM, kpH / kBK, G, m->pgate.as<float>()};
  }
  if (m->vp.world > 0) {                                        // this call's flag epochs
    launch_vp_seq(m->vp.seq.as<unsigned long long>(), m->stream);
    count(m);
  }
  for (int t = 1; t <= max_len; ++t) {
    EvPair ev = prof_begin(m, "step");
    // vocabulary-parallel: this step's parity of every rank's exchange buffer
    VpOut vo{};
    VpWait vw{};
    GenOut gs = g;
    if (m->vp.world > 0) {
      const VpOffsets o = vp_offsets(m, t & 1);
      vo.world = m->vp.world;
      vo.ranks = m->vp.world;
      for (int w = 0; w < m->vp.world; ++w) {
        char* base = static_cast<char*>(m->vp.peer[w]);
        vo.ms[w] = reinterpret_cast<float2*>(base + o.ms);
        vo.tz[w] = reinterpret_cast<float*>(base + o.tz);
        vo.ti[w] = reinterpret_cast<int*>(base + o.ti);
        vo.flag[w] = reinterpret_cast<unsigned long long*>(base + o.flag);
      }
      vo.seq = m->vp.seq.as<unsigned long long>();
      char* own = m->vp.own.as<char>();
      gs.ms = reinterpret_cast<float2*>(own + o.ms);
      gs.tz = reinterpret_cast<float*>(own + o.tz);
      gs.ti = reinterpret_cast<int*>(own + o.ti);
      vw = VpWait{reinterpret_cast<const unsigned long long*>(own + o.flag), groups * n_vt, vo.seq};
    }
    if (m->rs_cur && t > 1)
      enqueue_rs_layers(m, d_lens, B, S_max, K, bs.done, ctl);
    else
      enqueue_dec_layers(m, d_lens, B, S_max, K, bs.done, m->xg.xo(bf), ctl, op.att() ? m->b_att.as<float>() : nullptr);
    const double lp = std::pow((5.0 + t) / 6.0, (double)alpha);
    if (use_gen_step(m, m->xg)) {
      // K-outer generator (phase A of gen_step.cu), partials [row][C]; then row reduce + beam step
      EvPair pgs = prof_begin(m, "gen");
      ONMT_CUDA(gen_step(m->gen_w.tmap, m->xg.tmap, (m->Vt + kVTile - 1) / kVTile, m->xg.rows_pad, m->xg.n_group,
                           m->gen_w.k_pad / kBK, m->num_sms, gs, m->row_lse.as<float>(), m->row_z.as<float>(),
                           m->row_i.as<int>(), t, m->g_thr.as<unsigned int>(), ctl, m->stream,
                           t < max_len ? gt : GateTiles{}, m->vp.world > 0 ? &vo : nullptr, m->vp.rank, vpC));
      count(m);
      prof_end(m, "gen", pgs);
      EvPair pm = prof_begin(m, "merge");
      if (op.src_ext) {
        merge_copy(n_vt, 1, n_vt, t, lp);
      } else {
        // recurrent split: a few CTAs per sentence share layer 1's cell (each selects redundantly)
        static const int nsl_env = std::getenv("ONMT_BEAM_NSLICE") ? std::atoi(std::getenv("ONMT_BEAM_NSLICE")) : 0;
        const int nsl = m->rs_cur ? (nsl_env > 0 ? nsl_env : std::max(1, std::min(4, m->num_sms / std::max(B, 1)))) : 1;
        launch_beam_merge(gs.ms, gs.tz, gs.ti, n_vt, 1, n_vt, B, K, t, max_len, lp, bs, m->rs_cur ? gam : ga,
                          m->row_lse.as<float>(), m->row_z.as<float>(), m->row_i.as<int>(), ctl, m->stream, nsl,
                          m->vp.world > 0 ? &vw : nullptr);
        count(m, n_vt <= 256 ? 1 : 2);
      }
      prof_end(m, "merge", pm);
    } else {
      gen(m, m->xg, g, ctl);
      EvPair pm = prof_begin(m, "merge");
      if (op.src_ext) {
        merge_copy(n_vt, rp, 1, t, lp);
      } else {
        launch_beam_merge(g.ms, g.tz, g.ti, n_vt, rp, 1, B, K, t, max_len, lp, bs, ga, m->row_lse.as<float>(),
                          m->row_z.as<float>(), m->row_i.as<int>(), ctl, m->stream);
        count(m, n_vt <= 256 ? 1 : 2);
      }
      prof_end(m, "merge", pm);
    }
    prof_end(m, "step", ev);
  }
  {
    Nvtx nf("onmt.finalize");
    launch_finalize(bs, B, K, max_len, out.hyps, out.lens, out.scores, out.raw, out.tlogp, out.unk_pos, m->stream);
  }
  count(m);
  ONMT_CUDA(cudaGetLastError());
}

// Replay the whole call as one cached CUDA graph (LRU over kGraphCacheEntries shapes /
// pointer sets): the first call of a key captures `enqueue` and instantiates it, later calls
// are one cudaGraphLaunch.  A corpus whose batches differ in S_max reuses the graphs of its
// (bucketed, translate_impl) S_max values instead of re-capturing every batch.
template <typename F>
static void replay_graph(onmt_model* m, const std::vector<int64_t>& key, F&& enqueue) {
  GraphCache* gc = nullptr;
  for (auto& g : m->graphs)
    if (g.exec && g.key == key) gc = &g;
  if (!gc) {
    if ((int)m->graphs.size() < kGraphCacheEntries) {
      m->graphs.emplace_back();
      gc = &m->graphs.back();
    } else {                                            // evict the least recently used graph
      gc = &m->graphs[0];
      for (auto& g : m->graphs)
        if (g.last_use < gc->last_use) gc = &g;
    }
    if (gc->exec) {
      ONMT_CUDA(cudaStreamSynchronize(m->stream));
      ONMT_CUDA(cudaGraphExecDestroy(gc->exec));
      gc->exec = nullptr;
      for (auto& pe : gc->ev_nodes) m->evs[pe.first].release({pe.second});
      gc->ev_nodes.clear();
    }
    cudaGraph_t graph;
    const int64_t before = m->launches;
    ONMT_CUDA(cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal));
    m->capturing = true;
    m->cap_graph = gc;
    try {
      enqueue();
    } catch (...) {
      m->capturing = false;
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(m->stream, &junk);
      if (junk) cudaGraphDestroy(junk);
      throw;
    }
    m->capturing = false;
    ONMT_CUDA(cudaStreamEndCapture(m->stream, &graph));
    ONMT_CUDA(cudaGraphInstantiate(&gc->exec, graph, 0));
    ONMT_CUDA(cudaGraphDestroy(graph));
    gc->kernels = m->launches - before;
    m->launches = before;
    gc->key = key;
    ++m->graph_captures;
  }
  gc->last_use = ++m->graph_clock;
  ONMT_CUDA(cudaGraphLaunch(gc->exec, m->stream));
  m->launches += gc->kernels;
  for (auto& pe : gc->ev_nodes) m->evs[pe.first].pending.push_back({pe.second, false});
}

// Teacher-forced scoring: encoder, then T_max decoder steps fed with
// the gold tokens (A5 with parent = self), then ONE generator pass over every (step,
// sentence) row - a tensor-core GEMM of [T_max*B x H] by [H x V] with the log-softmax and
// the gold-logit gather fused (tc_gemm_kernel MODE_GEN) - and log p = z_gold - LSE.
// fp32 models run the generator per step (SIMT logits + score_row_kernel).
static void enqueue_score(onmt_model* m, const int* d_ids, const int* d_lens, int B, int S_max, int T_max) {
  const bool bf = m->use_tc;
  const int H = m->H, L = m->L;
  const int rp = m->xg.rows_pad;
  enqueue_encoder(m, d_ids, d_lens, B, S_max);
  BeamState bs = beam_state(m, false);
  float* hh = m->st_h.as<float>();
  float* cc = m->st_c.as<float>();
  launch_init_decode(bs, B, 1, m->enc_h.as<float>(), m->enc_c.as<float>(), L, H, hh, cc, rp, m->htilde.as<float>(),
                     m->stream);
  count(m);
  GatherArgs ga{};
  ga.emb_tgt = m->emb_tgt.as<float>();
  ga.E = m->E; ga.H = H; ga.L = L;
  ga.htilde = m->htilde.as<float>();
  ga.h = hh; ga.c = cc; ga.cg = m->st_cg.as<float>(); ga.rows_pad = rp;
  for (int l = 0; l < L; ++l) ga.x[l] = m->xdec[l]->xo(bf);
  const StepCtl none{nullptr, 0};
  for (int t = 1; t <= T_max; ++t) {
    launch_teacher_gather(m->s_tgt.as<int>(), T_max, t, B, ga, m->stream);
    count(m);
    XOut dst = m->xg.xo(bf);
    if (bf) {                                  // rows (t-1)*B .. of the all-steps operand
      dst = m->xs_all.xo(true);
      dst.hl += (size_t)(t - 1) * B * dst.k_pad;
    }
    enqueue_dec_layers(m, d_lens, B, S_max, 1, nullptr, dst, none);
    if (!bf) {
      ONMT_CUDA(simt_gemm_partial(m->gen_w.w.p, m->gen_w.bf16, m->gen_w.m_pad, m->gen_w.k_pad, m->xg.f32.as<float>(),
                                  m->xg.rows_pad, B, 1, m->logits.as<float>(), none, m->stream));
      launch_score_row(m->logits.as<float>(), m->gen_w.m_pad, m->gen_b.as<float>(), m->Vt, m->s_gold.as<int>(), B,
                       T_max, t, m->s_out.as<float>(), m->stream);
      count(m, 2);
    }
  }
  if (bf) {
    const Act& X = m->xs_all;
    GenOut g{};
    g.ms = m->s_ms.as<float2>();
    g.tz = m->s_tz.as<float>();
    g.ti = m->s_ti.as<int>();
    g.bias = m->gen_b.as<float>();
    g.V = m->Vt;
    g.K = 1;
    g.rows_valid = T_max * B;
    g.rows_pad = X.rows_pad;
    g.gold = m->s_gold.as<int>();
    g.zgold = m->s_zgold.as<float>();
    EvPair pg = prof_begin(m, "gen");
    ONMT_CUDA(tc_gemm_gen(m->gen_w.tmap, X.tmap, m->gen_w.m_pad, X.rows_pad, X.n_group, m->gen_w.k_pad / kBK, g, none,
                          m->stream));
    prof_end(m, "gen", pg);
    launch_score_reduce(g.ms, m->gen_w.m_pad / kTileM, X.rows_pad, g.zgold, g.gold, B, T_max, m->s_out.as<float>(),
                        m->stream);
    count(m, 2);
  }
  ONMT_CUDA(cudaGetLastError());
}

static void run_score(onmt_model* m, const int* d_ids, const int* d_lens, int B, int S_max, int T_max) {
  m->fold_cur = fold_on(m, B);
  m->rs_cur = false;
  prepare_encoder(m, B, S_max);
  prepare_decoder(m, B, S_max, 1, T_max, false);
  const bool bf = m->use_tc;
  if (bf) {
    m->xs_all.ensure(T_max * B, m->H, true);
    const size_t n_vt = m->gen_w.m_pad / kTileM, rp = m->xs_all.rows_pad;
    m->s_ms.ensure(n_vt * rp * 8);
    m->s_tz.ensure(n_vt * rp * 4);
    m->s_ti.ensure(n_vt * rp * 4);
    m->s_zgold.ensure(rp * 4);
  }
  if (!m->use_graph) {
    enqueue_score(m, d_ids, d_lens, B, S_max, T_max);
    return;
  }
  std::vector<int64_t> key = {-1, B, S_max, T_max, m->profile, m->use_tc, m->fused, m->gen_step, m->regroup, m->fold_cur,
                              m->enc_persistent, m->enc_wavefront, m->enc_cluster, (int64_t)g_alloc_gen,
                              (int64_t)(intptr_t)d_ids,
                              (int64_t)(intptr_t)d_lens, (int64_t)(intptr_t)m->stream};
  replay_graph(m, key, [&]() { enqueue_score(m, d_ids, d_lens, B, S_max, T_max); });
}

// The whole translation (encoder, decoder init, every decode step, finalize) as one CUDA
// graph, cached per shape / pointer set: one cudaGraphLaunch per call, no host round trip.
static void run_translate(onmt_model* m, const int* d_ids, const int* d_lens, int B, int S_max, int K, int max_len,
                          float alpha, bool trace, const DecodeOut& out, const DecodeOpts& op = DecodeOpts{}) {
  m->fold_cur = fold_on(m, B * K);
  m->rs_cur = m->vp.world > 0 ? false : rsplit_on(m, B, K, op.att() || op.src_ext);
  if (m->vp.world > 0) {
    const RowPlan rp = plan_rows(B * K);
    if (!m->use_tc || !m->gen_step || op.att() || op.src_ext || K > onmt_model::kVpK ||
        rp.rows_pad > m->vp.rows_cap || rp.rows_pad / rp.n_group > onmt_model::kVpG)
      throw Error{ONMT_E_UNSUPPORTED, "vocabulary-parallel decoding: bf16 plain translate with rows <= the exchange "
                                      "capacity, beam <= 16 and <= 4 row groups"};
  }
  prepare_encoder(m, B, S_max);
  prepare_decoder(m, B, S_max, K, max_len, trace, op);
  m->plan.rsplit = m->rs_cur;
  m->plan.fold = m->fold_cur;
  m->plan.gen_parts = m->vp.world > 0 ? m->vp.world * vp_ctas(m, m->xg.rows_pad / m->xg.n_group) : gen_parts(m, m->xg);
  m->plan.gate_tiles = m->rs_cur ? (m->L + 1) * (round_up(4 * m->H, kTileM) / kTileM) : 0;
  m->plan.groups = m->xg.rows_pad / m->xg.n_group;
  auto enqueue = [&]() {
    enqueue_encoder(m, d_ids, d_lens, B, S_max);
    enqueue_decoder(m, d_lens, B, S_max, K, max_len, alpha, trace, out, op);
  };
  if (!m->use_graph) {
    enqueue();
    return;
  }
  std::vector<int64_t> key = {B, S_max, K, max_len, (int64_t)(alpha * 1e6), trace, m->profile, m->use_tc, m->fused,
                              m->gen_step, m->regroup, m->fold_cur, m->enc_persistent, m->enc_wavefront, m->enc_cluster, m->rs_cur,
                              m->vp.world,
                              m->vp.rank,
                              (int64_t)g_alloc_gen, (int64_t)(intptr_t)d_ids, (int64_t)(intptr_t)d_lens,
                              (int64_t)(intptr_t)m->stream, (int64_t)(intptr_t)out.hyps, (int64_t)(intptr_t)out.lens,
                              (int64_t)(intptr_t)out.scores, (int64_t)(intptr_t)out.raw, (int64_t)(intptr_t)out.tlogp,
                              (int64_t)(intptr_t)out.unk_pos, (int64_t)(op.beta * 1e9), op.nbest, op.unk,
                              (int64_t)(intptr_t)op.src_ext};
  replay_graph(m, key, enqueue);
}

}  // namespace onmt

// ====================================================================== C-ABI
#define ONMT_API_BEGIN try {
#define ONMT_API_END                              \
  }                                               \
  catch (const Error& e) {                        \
    g_err = e.msg;                                \
    return e.s;                                   \
  }                                               \
  catch (const std::bad_alloc&) {                 \
    g_err = "host out of memory";                 \
    return ONMT_E_OOM;                            \
  }                                               \
  catch (const std::exception& e) {               \
    g_err = e.what();                             \
    return ONMT_E_INVALID_ARG;                    \
  }

static onmt_status fail(onmt_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

extern "C" {

const char* onmt_last_error(void) { return g_err.c_str(); }

onmt_status onmt_load_weights(const char* path, int32_t device, onmt_precision prec, onmt_model** out) {
  if (out) *out = nullptr;
  if (!path || !out) return fail(ONMT_E_INVALID_ARG, "null path or out");
  if (prec != ONMT_PREC_FP32 && prec != ONMT_PREC_BF16) return fail(ONMT_E_INVALID_ARG, "bad precision");
  g_err.clear();
  ONMT_API_BEGIN
  int ndev = 0;
  ONMT_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ONMT_E_INVALID_ARG, "bad device index");
  ONMT_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  ONMT_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(ONMT_E_UNSUPPORTED, "requires an sm_100 (B200) device");
  std::unique_ptr<onmt_model> m(new onmt_model());
  m->device = device;
  m->prec = prec;
  m->use_tc = prec == ONMT_PREC_BF16;
  m->num_sms = prop.multiProcessorCount;
  if (const char* ev = std::getenv("ONMT_NUM_SMS")) {   // size every grid for a part of the GPU
    const int n = std::atoi(ev);
    if (n >= 8 && n < m->num_sms) m->num_sms = n;
  }
  if (const char* ev = std::getenv("ONMT_USE_GRAPH")) m->use_graph = std::atoi(ev) != 0;   // ncu runs use 0
  if (const char* ev = std::getenv("ONMT_FUSED_GEMM")) m->fused = std::atoi(ev) != 0;
  if (const char* ev = std::getenv("ONMT_GEN_STEP")) m->gen_step = std::atoi(ev) != 0;
  if (const char* ev = std::getenv("ONMT_REGROUP")) m->regroup = std::atoi(ev) != 0;
  if (const char* ev = std::getenv("ONMT_FOLD_WOUT")) m->fold_wout = std::atoi(ev) != 0;
  if (const char* ev = std::getenv("ONMT_ENC_PERSISTENT")) m->enc_persistent = std::atoi(ev) != 0;
  if (const char* ev = std::getenv("ONMT_ENC_WAVE")) m->enc_wavefront = std::atoi(ev) != 0;
  if (const char* ev = std::getenv("ONMT_ENC_CLUSTER")) m->enc_cluster = std::atoi(ev) != 0;
  if (const char* ev = std::getenv("ONMT_RSPLIT")) m->rsplit = std::atoi(ev) != 0;

  ONMT_CUDA(cudaStreamCreateWithFlags(&m->own_stream, cudaStreamNonBlocking));
  m->stream = m->own_stream;
  load_model(m.get(), path);
  *out = m.release();
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_model_get_info(const onmt_model* m, onmt_model_info* o) {
  if (!m || !o) return fail(ONMT_E_INVALID_ARG, "null argument");
  o->layers = m->L; o->emb = m->E; o->hidden = m->H; o->v_src = m->Vs; o->v_tgt = m->Vt;
  o->bidir = m->bidir; o->attn_general = m->general; o->precision = m->prec;
  return ONMT_OK;
}

onmt_status onmt_set_stream(onmt_model* m, void* s) {
  if (!m) return fail(ONMT_E_INVALID_ARG, "null model");
  m->stream = s ? (cudaStream_t)s : m->own_stream;
  return ONMT_OK;
}

onmt_status onmt_set_option(onmt_model* m, const char* name, int64_t v) {
  if (!m || !name) return fail(ONMT_E_INVALID_ARG, "null argument");
  std::string n(name);
  if (n == "gemm_backend") {
    if (v != 0 && v != 1) return fail(ONMT_E_INVALID_ARG, "gemm_backend must be 0 or 1");
    m->use_tc = (v == 0) && m->prec == ONMT_PREC_BF16;
  } else if (n == "profile") {
    if (v < 0 || v > 2) return fail(ONMT_E_INVALID_ARG, "profile must be 0, 1 or 2");
    m->profile = (int)v;
  } else if (n == "fused_gemm") {
    m->fused = v != 0;
  } else if (n == "gen_step") {
    m->gen_step = v != 0;
  } else if (n == "regroup") {
    m->regroup = v != 0;
  } else if (n == "fold_wout") {
    m->fold_wout = v != 0;
  } else if (n == "enc_persistent") {
    m->enc_persistent = v != 0;
  } else if (n == "enc_wavefront") {
    m->enc_wavefront = v != 0;
  } else if (n == "enc_cluster") {
    m->enc_cluster = v != 0;
  } else if (n == "use_graph") {
    m->use_graph = v != 0;
  } else if (n == "rsplit") {
    m->rsplit = v != 0;
  } else if (n == "test_gen_world") {
    if (v < 0 || v > 8) return fail(ONMT_E_INVALID_ARG, "test_gen_world must be in [0, 8]");
    m->test_gen_world = (int)v;
  } else {
    return fail(ONMT_E_INVALID_ARG, "unknown option " + n);
  }
  return ONMT_OK;
}

static onmt_status validate(onmt_model* m, const int32_t* ids, const int32_t* lens, int32_t B, int32_t S_max,
                            bool check_ids) {
  if (!m) return fail(ONMT_E_INVALID_ARG, "null model");
  if (B < 0) return fail(ONMT_E_INVALID_ARG, "B < 0");
  if (B == 0) return ONMT_OK;
  if (S_max < 1) return fail(ONMT_E_INVALID_ARG, "S_max < 1");
  if (S_max > 2048) return fail(ONMT_E_UNSUPPORTED, "S_max > 2048");
  if (!lens || (check_ids && !ids)) return fail(ONMT_E_INVALID_ARG, "null source pointer");
  for (int b = 0; b < B; ++b) {
    if (lens[b] < 1) return fail(ONMT_E_EMPTY_SOURCE, "empty source sentence " + std::to_string(b));
    if (lens[b] > S_max) return fail(ONMT_E_INVALID_ARG, "src_len > S_max");
  }
  if (check_ids)
    for (int b = 0; b < B; ++b)
      for (int s = 0; s < lens[b]; ++s) {
        int v = ids[(size_t)b * S_max + s];
        if (v < 0 || v >= m->Vs) return fail(ONMT_E_ID_RANGE, "source id out of range");
      }
  return ONMT_OK;
}

// Host-API calls pad the source to a bucket of 8 positions: padded positions are never read
// (packed encoder, length-masked attention), so the result is the same up to the attention's
// chunking of the source, and a corpus whose batches differ in S_max replays a handful of
// cached graphs (replay_graph) instead of capturing one per batch.
static int bucket_smax(int S_max) { return std::min(round_up(S_max, 8), 2048); }

// ids [B x S_max] (host) -> device [B x S_dev] with pads zeroed (S_dev >= S_max)
static void upload_src(onmt_model* m, const int32_t* ids, const int32_t* lens, int B, int S_max, int S_dev) {
  m->d_ids.ensure((size_t)B * S_dev * 4);
  m->d_lens.ensure((size_t)B * 4);
  // ids at padded positions are ignored by contract; sanitize them so gathers stay in range
  std::vector<int32_t> clean((size_t)B * S_dev, 0);
  for (int b = 0; b < B; ++b)
    for (int s = 0; s < lens[b]; ++s) clean[(size_t)b * S_dev + s] = ids[(size_t)b * S_max + s];
  ONMT_CUDA(cudaMemcpyAsync(m->d_ids.p, clean.data(), clean.size() * 4, cudaMemcpyHostToDevice, m->stream));
  ONMT_CUDA(cudaMemcpyAsync(m->d_lens.p, lens, (size_t)B * 4, cudaMemcpyHostToDevice, m->stream));
}

onmt_status onmt_encode(onmt_model* m, const int32_t* ids, const int32_t* lens, int32_t B, int32_t S_max,
                        float* out_memory, float* out_h, float* out_c) {
  onmt_status s = validate(m, ids, lens, B, S_max, true);
  if (s != ONMT_OK || B == 0) return s;
  ONMT_API_BEGIN
  ONMT_CUDA(cudaSetDevice(m->device));
  upload_src(m, ids, lens, B, S_max, S_max);
  m->fold_cur = false;
  m->rs_cur = false;
  prepare_encoder(m, B, S_max);
  enqueue_encoder(m, m->d_ids.as<int>(), m->d_lens.as<int>(), B, S_max);
  if (out_memory)
    ONMT_CUDA(cudaMemcpyAsync(out_memory, m->mem.p, (size_t)B * S_max * m->H * 4, cudaMemcpyDeviceToHost, m->stream));
  if (out_h) ONMT_CUDA(cudaMemcpyAsync(out_h, m->enc_h.p, (size_t)m->L * B * m->H * 4, cudaMemcpyDeviceToHost, m->stream));
  if (out_c) ONMT_CUDA(cudaMemcpyAsync(out_c, m->enc_c.p, (size_t)m->L * B * m->H * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaStreamSynchronize(m->stream));
  return ONMT_OK;
  ONMT_API_END
}

static onmt_status check_decode_args(int32_t beam, int32_t max_len, float alpha) {
  if (beam < 1) return fail(ONMT_E_INVALID_ARG, "beam < 1");
  if (beam > ONMT_K_MAX) return fail(ONMT_E_UNSUPPORTED, "beam > ONMT_K_MAX");
  if (max_len < 1) return fail(ONMT_E_INVALID_ARG, "max_len < 1");
  if (!(alpha >= 0.f)) return fail(ONMT_E_INVALID_ARG, "length_penalty must be >= 0");
  return ONMT_OK;
}

static onmt_status translate_impl(onmt_model* m, const int32_t* ids, const int32_t* lens, int32_t B, int32_t S_max,
                                  int32_t beam, int32_t max_len, float alpha, int32_t* hyps, int32_t* olens,
                                  float* scores, float* raw, float* tlogp, int32_t* sel_parent, int32_t* sel_token,
                                  double* sel_score, DecodeOpts op = DecodeOpts{}, int32_t* unk_pos = nullptr,
                                  const int32_t* src_ext = nullptr) {
  onmt_status s = validate(m, ids, lens, B, S_max, true);
  if (s != ONMT_OK) return s;
  if (m && m->copy != (src_ext != nullptr))
    return fail(ONMT_E_INVALID_ARG, m->copy ? "a copy model needs the extended source ids (onmt_translate_copy)"
                                            : "src_ext given for a model without a copy generator");
  if (src_ext)
    for (int b = 0; b < B; ++b)
      for (int t = 0; t < lens[b]; ++t) {
        const int v = src_ext[(size_t)b * S_max + t];
        if (v < 0 || v >= m->Vt + S_max) return fail(ONMT_E_ID_RANGE, "extended source id out of range");
      }
  s = check_decode_args(beam, max_len, alpha);
  if (s != ONMT_OK) return s;
  if (B == 0) return ONMT_OK;
  if (!hyps || !olens || !scores) return fail(ONMT_E_INVALID_ARG, "null output pointer");
  const bool trace = sel_parent || sel_token || sel_score;
  ONMT_API_BEGIN
  Nvtx nv("onmt_translate");
  ONMT_CUDA(cudaSetDevice(m->device));
  const int S_dev = bucket_smax(S_max);
  upload_src(m, ids, lens, B, S_max, S_dev);
  if (src_ext) {                                     // pads -> 0 (never read)
    std::vector<int32_t> e((size_t)B * S_dev, 0);
    for (int b = 0; b < B; ++b)
      for (int t = 0; t < lens[b]; ++t) e[(size_t)b * S_dev + t] = src_ext[(size_t)b * S_max + t];
    m->d_ext.ensure(e.size() * 4);
    ONMT_CUDA(cudaMemcpyAsync(m->d_ext.p, e.data(), e.size() * 4, cudaMemcpyHostToDevice, m->stream));
    ONMT_CUDA(cudaStreamSynchronize(m->stream));
    op.src_ext = m->d_ext.as<int>();
  }
  const size_t nb = (size_t)op.nbest;
  m->o_hyps.ensure((size_t)B * nb * max_len * 4);
  m->o_lens.ensure((size_t)B * nb * 4);
  m->o_scores.ensure((size_t)B * nb * 4);
  m->o_raw.ensure((size_t)B * nb * 4);
  m->o_tlogp.ensure((size_t)B * nb * max_len * 4);
  if (unk_pos) m->o_unk.ensure((size_t)B * nb * max_len * 4);
  DecodeOut o{m->o_hyps.as<int>(), m->o_lens.as<int>(), m->o_scores.as<float>(), m->o_raw.as<float>(),
              m->o_tlogp.as<float>(), unk_pos ? m->o_unk.as<int>() : nullptr};
  run_translate(m, m->d_ids.as<int>(), m->d_lens.as<int>(), B, S_dev, beam, max_len, alpha, trace, o, op);
  ONMT_CUDA(cudaMemcpyAsync(hyps, o.hyps, (size_t)B * nb * max_len * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaMemcpyAsync(olens, o.lens, (size_t)B * nb * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaMemcpyAsync(scores, o.scores, (size_t)B * nb * 4, cudaMemcpyDeviceToHost, m->stream));
  if (raw) ONMT_CUDA(cudaMemcpyAsync(raw, o.raw, (size_t)B * nb * 4, cudaMemcpyDeviceToHost, m->stream));
  if (tlogp) ONMT_CUDA(cudaMemcpyAsync(tlogp, o.tlogp, (size_t)B * nb * max_len * 4, cudaMemcpyDeviceToHost, m->stream));
  if (unk_pos)
    ONMT_CUDA(cudaMemcpyAsync(unk_pos, o.unk_pos, (size_t)B * nb * max_len * 4, cudaMemcpyDeviceToHost, m->stream));
  const size_t n = (size_t)max_len * B * beam;
  if (sel_parent) ONMT_CUDA(cudaMemcpyAsync(sel_parent, m->s_par.p, n * 4, cudaMemcpyDeviceToHost, m->stream));
  if (sel_token) ONMT_CUDA(cudaMemcpyAsync(sel_token, m->h_tok.p, n * 4, cudaMemcpyDeviceToHost, m->stream));
  if (sel_score) ONMT_CUDA(cudaMemcpyAsync(sel_score, m->s_score.p, n * 8, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaStreamSynchronize(m->stream));
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_translate(onmt_model* m, const int32_t* ids, const int32_t* lens, int32_t B, int32_t S_max,
                           int32_t beam, int32_t max_len, float alpha, int32_t* hyps, int32_t* olens, float* scores,
                           float* raw, float* tlogp) {
  return translate_impl(m, ids, lens, B, S_max, beam, max_len, alpha, hyps, olens, scores, raw, tlogp, nullptr,
                        nullptr, nullptr);
}

onmt_status onmt_translate_ex(onmt_model* m, const int32_t* ids, const int32_t* lens, int32_t B, int32_t S_max,
                              const onmt_decode_opts* opts, int32_t* hyps, int32_t* olens, float* scores, float* raw,
                              float* tlogp, int32_t* unk_pos) {
  if (!opts) return fail(ONMT_E_INVALID_ARG, "null options");
  if (opts->n_best < 1 || opts->n_best > opts->beam) return fail(ONMT_E_INVALID_ARG, "n_best must be in [1, beam]");
  if (!(opts->coverage_penalty >= 0.f)) return fail(ONMT_E_INVALID_ARG, "coverage_penalty must be >= 0");
  if (unk_pos && !opts->replace_unk) return fail(ONMT_E_INVALID_ARG, "unk_pos needs replace_unk");
  DecodeOpts op;
  op.beta = opts->coverage_penalty;
  op.nbest = opts->n_best;
  op.unk = opts->replace_unk != 0;
  return translate_impl(m, ids, lens, B, S_max, opts->beam, opts->max_len, opts->length_penalty, hyps, olens, scores,
                        raw, tlogp, nullptr, nullptr, nullptr, op, unk_pos);
}

onmt_status onmt_translate_copy(onmt_model* m, const int32_t* ids, const int32_t* lens, const int32_t* src_ext,
                                int32_t B, int32_t S_max, const onmt_decode_opts* opts, int32_t* hyps, int32_t* olens,
                                float* scores, float* raw, float* tlogp) {
  if (!opts) return fail(ONMT_E_INVALID_ARG, "null options");
  if (!src_ext && B > 0) return fail(ONMT_E_INVALID_ARG, "null src_ext");
  if (m && !m->copy) return fail(ONMT_E_UNSUPPORTED, "the model has no copy generator (copy.w / copy.b)");
  if (opts->n_best != 1 || opts->coverage_penalty != 0.f || opts->replace_unk)
    return fail(ONMT_E_UNSUPPORTED, "copy decoding supports n_best = 1, no coverage penalty, no unk replacement");
  return translate_impl(m, ids, lens, B, S_max, opts->beam, opts->max_len, opts->length_penalty, hyps, olens, scores,
                        raw, tlogp, nullptr, nullptr, nullptr, DecodeOpts{}, nullptr, B > 0 ? src_ext : nullptr);
}

onmt_status onmt_translate_trace(onmt_model* m, const int32_t* ids, const int32_t* lens, int32_t B, int32_t S_max,
                                 int32_t beam, int32_t max_len, float alpha, int32_t* hyps, int32_t* olens,
                                 float* scores, float* raw, float* tlogp, int32_t* sel_parent, int32_t* sel_token,
                                 double* sel_score) {
  if (!sel_parent || !sel_token || !sel_score) return fail(ONMT_E_INVALID_ARG, "null trace pointer");
  return translate_impl(m, ids, lens, B, S_max, beam, max_len, alpha, hyps, olens, scores, raw, tlogp, sel_parent,
                        sel_token, sel_score);
}

onmt_status onmt_score(onmt_model* m, const int32_t* ids, const int32_t* lens, int32_t B, int32_t S_max,
                       const int32_t* tgt, const int32_t* tgt_lens, int32_t T_max, float* out_token_logp,
                       double* out_nll) {
  onmt_status s = validate(m, ids, lens, B, S_max, true);
  if (s != ONMT_OK) return s;
  if (B == 0) return ONMT_OK;
  if (T_max < 1) return fail(ONMT_E_INVALID_ARG, "T_max < 1");
  if (m->copy) return fail(ONMT_E_UNSUPPORTED, "teacher-forced scoring of copy models is not built");
  if (!tgt || !tgt_lens || !out_token_logp) return fail(ONMT_E_INVALID_ARG, "null target / output pointer");
  for (int b = 0; b < B; ++b) {
    if (tgt_lens[b] < 1) return fail(ONMT_E_EMPTY_SOURCE, "empty target sentence " + std::to_string(b));
    if (tgt_lens[b] > T_max) return fail(ONMT_E_INVALID_ARG, "tgt_len > T_max");
    for (int t = 0; t < tgt_lens[b]; ++t) {
      const int v = tgt[(size_t)b * T_max + t];
      if (v < 0 || v >= m->Vt) return fail(ONMT_E_ID_RANGE, "target id out of range");
    }
  }
  ONMT_API_BEGIN
  ONMT_CUDA(cudaSetDevice(m->device));
  const int S_dev = bucket_smax(S_max);
  upload_src(m, ids, lens, B, S_max, S_dev);
  std::vector<int32_t> clean((size_t)B * T_max, 0), gold((size_t)T_max * B, -1);
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < tgt_lens[b]; ++t) {
      clean[(size_t)b * T_max + t] = tgt[(size_t)b * T_max + t];
      gold[(size_t)t * B + b] = tgt[(size_t)b * T_max + t];
    }
  m->s_tgt.ensure(clean.size() * 4);
  m->s_gold.ensure(gold.size() * 4);
  m->s_out.ensure((size_t)B * T_max * 4);
  ONMT_CUDA(cudaMemcpyAsync(m->s_tgt.p, clean.data(), clean.size() * 4, cudaMemcpyHostToDevice, m->stream));
  ONMT_CUDA(cudaMemcpyAsync(m->s_gold.p, gold.data(), gold.size() * 4, cudaMemcpyHostToDevice, m->stream));
  run_score(m, m->d_ids.as<int>(), m->d_lens.as<int>(), B, S_dev, T_max);
  ONMT_CUDA(cudaMemcpyAsync(out_token_logp, m->s_out.p, (size_t)B * T_max * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaStreamSynchronize(m->stream));
  if (out_nll)
    for (int b = 0; b < B; ++b) {
      double acc = 0.0;
      for (int t = 0; t < tgt_lens[b]; ++t) acc -= (double)out_token_logp[(size_t)b * T_max + t];
      out_nll[b] = acc;
    }
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_translate_dev(onmt_model* m, const int32_t* d_ids, const int32_t* d_lens, const int32_t* lens_host,
                               int32_t B, int32_t S_max, int32_t beam, int32_t max_len, float alpha, int32_t* d_hyps,
                               int32_t* d_olens, float* d_scores, float* d_raw, float* d_tlogp) {
  if (!m) return fail(ONMT_E_INVALID_ARG, "null model");
  if (B < 0) return fail(ONMT_E_INVALID_ARG, "B < 0");
  onmt_status s = check_decode_args(beam, max_len, alpha);
  if (s != ONMT_OK) return s;
  if (B == 0) return ONMT_OK;
  if (S_max < 1) return fail(ONMT_E_INVALID_ARG, "S_max < 1");
  if (S_max > 2048) return fail(ONMT_E_UNSUPPORTED, "S_max > 2048");
  if (lens_host) {
    s = validate(m, nullptr, lens_host, B, S_max, false);
    if (s != ONMT_OK) return s;
  }
  if (!d_ids || !d_lens || !d_hyps || !d_olens || !d_scores) return fail(ONMT_E_INVALID_ARG, "null device pointer");
  if (m->copy) return fail(ONMT_E_UNSUPPORTED, "copy models decode through onmt_translate_copy");
  ONMT_API_BEGIN
  Nvtx nv("onmt_translate_dev");
  ONMT_CUDA(cudaSetDevice(m->device));
  m->o_raw.ensure((size_t)B * 4);
  m->o_tlogp.ensure((size_t)B * max_len * 4);
  DecodeOut o{d_hyps, d_olens, d_scores, d_raw ? d_raw : m->o_raw.as<float>(),
              d_tlogp ? d_tlogp : m->o_tlogp.as<float>()};
  run_translate(m, d_ids, d_lens, B, S_max, beam, max_len, alpha, false, o);
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_get_kernel_time(onmt_model* m, const char* name, int32_t reset, double* total_ms, int64_t* launches) {
  if (!m || !name || !total_ms || !launches) return fail(ONMT_E_INVALID_ARG, "null argument");
  ONMT_API_BEGIN
  std::string n(name);
  static const char* known[] = {"gen", "step", "encode", "gemm", "cell", "attention", "attn_out", "merge"};
  bool ok = false;
  for (const char* k : known) ok |= n == k;
  if (!ok) return fail(ONMT_E_INVALID_ARG, "unknown kernel family " + n);
  EventPairs* e = &m->evs[n];
  ONMT_CUDA(cudaStreamSynchronize(m->stream));
  e->drain();
  *total_ms = e->acc_ms;
  *launches = e->count;
  if (reset) { e->acc_ms = 0; e->count = 0; }
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_kernel_launches(onmt_model* m, int32_t reset, int64_t* launches) {
  if (!m || !launches) return fail(ONMT_E_INVALID_ARG, "null argument");
  *launches = m->launches;
  if (reset) m->launches = 0;
  return ONMT_OK;
}

onmt_status onmt_vp_handle(onmt_model* m, int32_t max_rows, void* handle_out) {
  if (!m || !handle_out || max_rows < 1) return fail(ONMT_E_INVALID_ARG, "bad argument");
  ONMT_API_BEGIN
  ONMT_CUDA(cudaSetDevice(m->device));
  const int rc = plan_rows(max_rows).rows_pad;
  if (m->vp.world > 0) return fail(ONMT_E_INVALID_ARG, "close the vocabulary-parallel group first");
  m->vp.rows_cap = rc;
  m->vp.parity_bytes = vp_parity_bytes(rc);
  m->vp.own.ensure(2 * m->vp.parity_bytes);
  ONMT_CUDA(cudaMemset(m->vp.own.p, 0, 2 * m->vp.parity_bytes));   // flags 0: no epoch is 0
  m->vp.seq.ensure(8);
  ONMT_CUDA(cudaMemset(m->vp.seq.p, 0, 8));
  cudaIpcMemHandle_t h;
  ONMT_CUDA(cudaIpcGetMemHandle(&h, m->vp.own.p));
  std::memcpy(handle_out, &h, sizeof(h));
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_vp_open(onmt_model* m, int32_t world, int32_t rank, const void* handles) {
  if (!m || world < 1 || world > 8 || rank < 0 || rank >= world || (world > 1 && !handles))
    return fail(ONMT_E_INVALID_ARG, "bad world / rank / handles");
  if (!m->vp.own.p) return fail(ONMT_E_INVALID_ARG, "onmt_vp_handle first");
  if (m->prec != ONMT_PREC_BF16) return fail(ONMT_E_UNSUPPORTED, "vocabulary-parallel decoding needs a bf16 model");
  ONMT_API_BEGIN
  ONMT_CUDA(cudaSetDevice(m->device));
  for (int w = 0; w < world; ++w) {
    if (w == rank) {
      m->vp.peer[w] = m->vp.own.p;
      m->vp.ipc[w] = false;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)w * sizeof(h), sizeof(h));
    void* p = nullptr;
    ONMT_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    m->vp.peer[w] = p;
    m->vp.ipc[w] = true;
  }
  m->vp.world = world;
  m->vp.rank = rank;
  ++g_alloc_gen;                                    // (cached graphs hold the old pointers)
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_vp_close(onmt_model* m) {
  if (!m) return fail(ONMT_E_INVALID_ARG, "null model");
  ONMT_API_BEGIN
  ONMT_CUDA(cudaSetDevice(m->device));
  ONMT_CUDA(cudaStreamSynchronize(m->stream));
  for (int w = 0; w < m->vp.world; ++w)
    if (m->vp.ipc[w]) ONMT_CUDA(cudaIpcCloseMemHandle(m->vp.peer[w]));
  for (int w = 0; w < 8; ++w) { m->vp.peer[w] = nullptr; m->vp.ipc[w] = false; }
  m->vp.world = 0;
  ++g_alloc_gen;
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_last_plan(const onmt_model* m, onmt_plan_info* out) {
  if (!m || !out) return fail(ONMT_E_INVALID_ARG, "null argument");
  *out = m->plan;
  return ONMT_OK;
}

onmt_status onmt_graph_captures(onmt_model* m, int64_t* captures) {
  if (!m || !captures) return fail(ONMT_E_INVALID_ARG, "null argument");
  *captures = m->graph_captures;
  return ONMT_OK;
}

void onmt_free(onmt_model* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  cudaStreamSynchronize(m->stream);
  delete m;
}

onmt_status onmt_test_gemm(onmt_model* m, const float* W, const float* X, int32_t M, int32_t N, int32_t K,
                           int32_t splits, float* out) {
  if (!m || !W || !X || !out || M < 1 || N < 1 || K < 1 || splits < 0) return fail(ONMT_E_INVALID_ARG, "bad args");
  ONMT_API_BEGIN
  ONMT_CUDA(cudaSetDevice(m->device));
  const bool bfm = m->prec == ONMT_PREC_BF16;
  Mat w;
  int mp = round_up(M, kTileM), kp = round_up(K, kBK);
  std::vector<float> hw((size_t)mp * kp, 0.f);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < K; ++k) hw[(size_t)i * kp + k] = bfm ? bf16_round_host(W[(size_t)i * K + k]) : W[(size_t)i * K + k];
  w.upload(hw, M, K, bfm);
  Act x;
  x.ensure(N, K, bfm);
  std::vector<float> hx((size_t)x.rows_pad * kp, 0.f);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) hx[(size_t)n * kp + k] = X[(size_t)n * K + k];
  ONMT_CUDA(cudaMemcpy(x.f32.p, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
  if (bfm) {
    std::vector<__nv_bfloat16> hl(2 * hx.size());
    for (size_t i = 0; i < hx.size(); ++i) {
      __nv_bfloat16 hi = __float2bfloat16_rn(hx[i]);
      hl[i] = hi;
      hl[hx.size() + i] = __float2bfloat16_rn(hx[i] - __bfloat162float(hi));
    }
    ONMT_CUDA(cudaMemcpy(x.hl.p, hl.data(), hl.size() * 2, cudaMemcpyHostToDevice));
  }
  DevBuf P;
  P.ensure((size_t)16 * x.rows_pad * w.m_pad * 4);
  int eff = gemm(m, w, x, N, splits == 0 ? 0 : std::min(splits, 16), P.as<float>(), StepCtl{nullptr, 0});
  std::vector<float> hp((size_t)eff * x.rows_pad * w.m_pad);
  ONMT_CUDA(cudaMemcpyAsync(hp.data(), P.p, hp.size() * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaStreamSynchronize(m->stream));
  for (int n = 0; n < N; ++n)
    for (int i = 0; i < M; ++i) {
      float s = 0.f;
      for (int z = 0; z < eff; ++z) s += hp[((size_t)z * x.rows_pad + n) * w.m_pad + i];
      out[(size_t)n * M + i] = s;
    }
  return ONMT_OK;
  ONMT_API_END
}

onmt_status onmt_test_gen(onmt_model* m, const float* htilde, int32_t R, int32_t k, float* lse, float* top_z,
                          int32_t* top_id) {
  if (!m || !htilde || !lse || !top_z || !top_id || R < 1 || k < 1 || k > ONMT_K_MAX)
    return fail(ONMT_E_INVALID_ARG, "bad args");
  ONMT_API_BEGIN
  ONMT_CUDA(cudaSetDevice(m->device));
  const bool bfm = m->prec == ONMT_PREC_BF16;
  Act x;
  x.ensure(R, m->H, bfm);
  std::vector<float> hx((size_t)x.rows_pad * x.k_pad, 0.f);
  for (int r = 0; r < R; ++r)
    for (int j = 0; j < m->H; ++j) hx[(size_t)r * x.k_pad + j] = htilde[(size_t)r * m->H + j];
  ONMT_CUDA(cudaMemcpy(x.f32.p, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
  if (bfm) {
    std::vector<__nv_bfloat16> hl(2 * hx.size());
    for (size_t i = 0; i < hx.size(); ++i) {
      __nv_bfloat16 hi = __float2bfloat16_rn(hx[i]);
      hl[i] = hi;
      hl[hx.size() + i] = __float2bfloat16_rn(hx[i] - __bfloat162float(hi));
    }
    ONMT_CUDA(cudaMemcpy(x.hl.p, hl.data(), hl.size() * 2, cudaMemcpyHostToDevice));
  }
  const int n_vt = std::max(gen_parts(m, x), (m->Vt + kVTile - 1) / kVTile);
  const int n_parts = gen_parts(m, x);
  DevBuf ms, tz, ti, dl, dz, di;
  ms.ensure((size_t)n_vt * x.rows_pad * 8);
  tz.ensure((size_t)n_vt * x.rows_pad * k * 4);
  ti.ensure((size_t)n_vt * x.rows_pad * k * 4);
  dl.ensure((size_t)R * 4);
  dz.ensure((size_t)R * k * 4);
  di.ensure((size_t)R * k * 4);
  GenOut g{ms.as<float2>(), tz.as<float>(), ti.as<int>(), m->gen_b.as<float>(), m->Vt, k, R, x.rows_pad};
  DevBuf dbg;
  const bool trace_gen = std::getenv("ONMT_GEN_TRACE") != nullptr;
  if (trace_gen) {
    dbg.ensure(256 * 8);
    ONMT_CUDA(cudaMemset(dbg.p, 0, 256 * 8));
    g_gen_dbg = dbg.as<unsigned long long>();
  }
  const bool gs = use_gen_step(m, x);
  if (gs) {
    if (m->g_thr.bytes < (size_t)2 * x.rows_pad * 17 * 4) m->g_thr.ensure((size_t)2 * x.rows_pad * 17 * 4);
    ONMT_CUDA(cudaMemset(m->g_thr.p, 0, m->g_thr.bytes));
    const int W = m->test_gen_world;
    if (W > 1) {
      // the vocabulary-parallel split, its W ranks emulated by W launches one after another on this
      // GPU (no launch waits on another): rank r runs CTAs [r C / W, (r + 1) C / W) of the C-CTA
      // split and stores its partial columns through the exchange pointers (here: one buffer)
      if (n_parts % W != 0 || W > 8) return fail(ONMT_E_INVALID_ARG, "test_gen_world must divide the partial count");
      DevBuf flags, seq;
      flags.ensure((size_t)(x.rows_pad / x.n_group) * n_parts * 8);
      ONMT_CUDA(cudaMemset(flags.p, 0, flags.bytes));
      seq.ensure(8);
      ONMT_CUDA(cudaMemset(seq.p, 0, 8));
      VpOut vo{};
      vo.world = 1;
      vo.ranks = W;
      vo.ms[0] = g.ms; vo.tz[0] = g.tz; vo.ti[0] = g.ti;
      vo.flag[0] = flags.as<unsigned long long>();
      vo.seq = seq.as<unsigned long long>();
      for (int r = 0; r < W; ++r) {
        ONMT_CUDA(gen_step(m->gen_w.tmap, x.tmap, (m->Vt + kVTile - 1) / kVTile, x.rows_pad, x.n_group,
                           m->gen_w.k_pad / kBK, m->num_sms, g, dl.as<float>(), dz.as<float>(), di.as<int>(), 0,
                           m->g_thr.as<unsigned int>(), StepCtl{nullptr, 0}, m->stream, GateTiles{}, &vo, r,
                           n_parts / W));
      }
      // (emulation: every launch wrote column block r of the same Ct = C partials)
      vo.world = 0;
    } else {
      ONMT_CUDA(gen_step(m->gen_w.tmap, x.tmap, (m->Vt + kVTile - 1) / kVTile, x.rows_pad, x.n_group,
                         m->gen_w.k_pad / kBK, m->num_sms, g, dl.as<float>(), dz.as<float>(), di.as<int>(), 0,
                         m->g_thr.as<unsigned int>(), StepCtl{nullptr, 0}, m->stream, GateTiles{}));
    }
  } else {
    gen(m, x, g, StepCtl{nullptr, 0});
  }
  g_gen_dbg = nullptr;
  if (trace_gen) {
    std::vector<unsigned long long> h(256);
    ONMT_CUDA(cudaStreamSynchronize(m->stream));
    ONMT_CUDA(cudaMemcpy(h.data(), dbg.p, 256 * 8, cudaMemcpyDeviceToHost));
    const unsigned long long t0 = h[200];
    auto rel = [&](unsigned long long v) { return v ? (long long)(v - t0) : -1LL; };
    std::fprintf(stderr, "gen trace CTA0: tiles=%llu stages=%llu total=%lld ns\n", h[202], h[203], rel(h[201]));
    for (int i = 0; i < 32; ++i) std::fprintf(stderr, "  kb%02d tma_issue=%lld mma_start=%lld\n", i, rel(h[i]), rel(h[64 + i]));
    for (int p = 0; p < 4; ++p)
      std::fprintf(stderr, "  gu%d: start=%lld sum=%lld cand=%lld merge=%lld end=%lld\n", p, rel(h[210 + 8 * p]),
                   rel(h[211 + 8 * p]), rel(h[212 + 8 * p]), rel(h[213 + 8 * p]), rel(h[214 + 8 * p]));
    for (int j = 0; j < 4; ++j)
      std::fprintf(stderr, "  tile%d mma_done=%lld epi_start=%lld scan0=%lld end0=%lld scan1=%lld end1=%lld\n", j,
                   rel(h[128 + j]), rel(h[144 + j]), rel(h[160 + 2 * j]), rel(h[176 + 2 * j]), rel(h[161 + 2 * j]),
                   rel(h[177 + 2 * j]));
  }
  // partials: [row][part] from the step generator, [part][row] from the others
  launch_row_reduce(g.ms, g.tz, g.ti, n_parts, gs ? 1 : x.rows_pad, gs ? n_parts : 1, R, k, dl.as<float>(),
                    dz.as<float>(), di.as<int>(), m->stream);
  ONMT_CUDA(cudaGetLastError());
  ONMT_CUDA(cudaMemcpyAsync(lse, dl.p, (size_t)R * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaMemcpyAsync(top_z, dz.p, (size_t)R * k * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaMemcpyAsync(top_id, di.p, (size_t)R * k * 4, cudaMemcpyDeviceToHost, m->stream));
  ONMT_CUDA(cudaStreamSynchronize(m->stream));
  return ONMT_OK;
  ONMT_API_END
}

}  // extern "C"
