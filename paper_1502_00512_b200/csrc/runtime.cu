// libdesklm_cuda.so runtime: the C ABI of include/desklm_cuda.h.
//
// Owns all device memory of one model on one GPU and sequences the kernels
// of one truncated-BPTT window (backprop.hpp:76-222), the rmsprop update
// (rmsprop.hpp:113-133), the forward scorers (eval.hpp:84-222) and the
// offset-stream epoch schedule (trainer.hpp:350-410).  There is no CPU
// compute path: every number is produced by a kernel in gemm_tc.cu,
// gemm_simt.cu or kernels.cu.
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/desklm_cuda.h"
#include "comm.cuh"
#include "kernels.cuh"

using namespace dl;

namespace {
thread_local std::string g_err;

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  DL_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
}

struct PhaseTimer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  size_t used = 0;
  std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> open;
};
}  // namespace

struct dl_ctx {
  int device = 0;
  int64_t V = 0, H = 0;
  int act = 0, precision = DL_FP32;
  cudaStream_t st = nullptr;
  std::string err;
  std::atomic<uint64_t> launches{0};

  // parameters (fp32 masters, bf16 shadows for the tensor-core path)
  float *w_in = nullptr, *w_rec = nullptr, *w_out = nullptr;
  bf16 *w_rec_bf = nullptr, *w_out_bf = nullptr;
  // second W_out shadow: a forked update writes it while the dh GEMM still
  // reads w_out_bf; swap_shadow() flips them (par tracks the flip parity)
  bf16* w_out_bf_next = nullptr;
  int par = 0;
  // optimiser
  float *m_rec = nullptr, *m_in = nullptr, *m_out = nullptr;
  double rho = 0.9995, eps = 1e-6;
  // gradients of the last window
  float *g_rec = nullptr, *g_out = nullptr, *g_in_rows = nullptr;
  uint32_t* g_in_words = nullptr;
  int* g_in_n = nullptr;
  int* nonfinite = nullptr;
  bool have_grads = false;
  // bf16 mode: dW_out as bf16 + row sums of squares from the GEMM epilogue
  // (DL_G16=0 keeps the fp32 gradient); g16_valid = the last window used it
  bf16* g_out_bf = nullptr;
  double* rowsq = nullptr;
  int rowsq_n = 0;
  bool g16 = true, g16_valid = false;
  // data parallel, bf16 mode, finite clip: dW_out is produced and summed over
  // ranks in bf16 (unclipped), then clip + the dense update in one kernel
  bool dp16 = false;
  float dp16_clip = 1.f;
  cudaStream_t st2 = nullptr;  // side stream (W_out update during backward)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_sort_fork = nullptr, ev_sort_join = nullptr;  // W_in id sort on st2
  cudaEvent_t ev_hfinal = nullptr;  // forward recurrence done (h_final readable)
  // data-parallel + vocabulary-parallel: dh partials ready / dh reduce-scattered
  cudaEvent_t ev_dh = nullptr, ev_rs = nullptr;

  // window workspace
  int64_t capT = 0, capB = 0;
  float* htape = nullptr;  // (T+1) x B x H
  bf16* htape_bf = nullptr;
  uint32_t *x_d = nullptr, *y_d = nullptr;
  uint8_t* w_d = nullptr;
  void* S = nullptr;  // logits / dS: fp32 or bf16 [TB x V]
  // bf16 mode: dS formed on the fly in the dh GEMM's operand path
  // (GemmDesc::xf) -- the dh GEMM stores it here for dW_out; the softmax
  // rows kernel then only computes lse / loss and the transform constants
  bf16* dS = nullptr;
  float *xf_lse = nullptr, *xf_sc = nullptr;
  const uint32_t* xf_tgt = nullptr;  // the target columns of this window's output rows
  // DL_XF=1 turns it on: bit-identical to the in-place softmax kernel but
  // slower at C3 (dh 1.27 vs 0.34 ms: the SFU-bound transform sits on the
  // MMA's critical path, plus a cross-CTA handshake per k-block)
  bool xf = false;
  // DL_TF32X3: the fp32 mode's GEMMs as 3xTF32 on the tensor cores
  // (gemm_tc.cu) instead of the fp32 FMA kernel (gemm_simt.cu)
  bool tf32x3 = false;
  int dp_chunks = 4;  // dense DP: dW_out GEMM + allreduce in V chunks (DL_DP_CHUNKS)
  float *xpose_a = nullptr, *xpose_b = nullptr;  // K-major copies of MN-major operands
  size_t xpose_a_cap = 0, xpose_b_cap = 0;
  bool xf_on = false;                // this window's dS is formed in the dh GEMM
  // bf16 trainer: shifted-exponential softmax (kernels.cu k_pfac_rows) --
  // the logits GEMM stores E = e^(s - shift), dS = diag(pf_sigma) E'; no
  // pass over the logits after the GEMM.  DL_PFAC=0 keeps the in-place
  // softmax rows kernel.  pf_on: this window used it (dh / dW_out follow).
  bool pfac = true;
  bool pf_on = false;
  bool rec_fused = false;  // this window's W_rec step ran in the dW_rec reduction
  bool in_decayed = false;  // this window's m_in decay ran on the side stream (run_window)
  float *pf_shift = nullptr, *pf_sigma = nullptr, *pf_resid = nullptr;
  const uint32_t* pf_tgt = nullptr;  // this window's output-row targets
  bf16* pf_hs = nullptr;     // diag(sigma) Hs in bf16 [MO x H] (dW_out's B operand)
  int* pf_repaired = nullptr;  // rows recomputed with the row maximum as shift (device counter)
  float2* part = nullptr;
  int part_tiles = 0;
  float* tgt_logit = nullptr;
  double* loss_row = nullptr;
  double* logp_row = nullptr;
  float* dh_out = nullptr;
  float* dpre = nullptr;
  cudaEvent_t score_ev[2] = {nullptr, nullptr};  // dl_score's two host slots
  bf16* dpre_bf = nullptr;
  float* splitws = nullptr;
  size_t splitws_elems = 0;
  EmbedWs ews{};
  double* d_loss = nullptr;
  unsigned long long* d_pos = nullptr;
  unsigned long long* d_skipped = nullptr;
  float* h0_d = nullptr;  // B x H staging for the trainer

  // pinned staging for the host-buffer API
  void* pinned = nullptr;
  size_t pinned_bytes = 0;

  // trainer
  uint32_t* ids = nullptr;
  int64_t L = 0;
  int noffset = 0, minibatch = 0, unroll = 0;
  double clip = 1.0;
  uint32_t bos = 1;
  int64_t* cursors = nullptr;  // rank-local [noffset*minibatch]
  float* hidden = nullptr;     // rank-local [noffset*minibatch x H]
  int64_t* win_counter = nullptr;
  cudaGraphExec_t graph = nullptr;
  cudaGraphExec_t graphs[2] = {nullptr, nullptr};  // indexed by shadow parity
  int graph_par0 = -1;
  double graph_eta = NAN;
  uint64_t graph_launches = 0;
  bool use_graph = true;
  // dl_train_window as one CUDA graph per (T, B, scale, clip, eta): the
  // window's H2D / D2H copies are graph nodes whose host side is re-pointed
  // at each call's buffers (cudaGraphExecMemcpyNodeSetParams1D)
  struct TwGraph {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t e = nullptr;
    cudaGraphNode_t nx = nullptr, ny = nullptr, nw = nullptr, nh0 = nullptr, nhf = nullptr;
    int64_t T = 0, B = 0;
    double scale = 0, eta = 0;
    float clip = 0;
    bool fuse = false;
    uint8_t* pin = nullptr;  // staging: x, y, w, h0, h_final, results
    uint64_t launches = 0;
  } tw;
  // recurrence steps as one cluster kernel each (rec_tc.cu); DL_REC_CLUSTER=0
  // falls back to split-K GEMM + reduction kernels (both are sm_100a CUDA)
  bool rec_cluster = true;
  bool h0_bf_ready = false;  // window_build already wrote htape_bf[0] (trainer path)
  // DL_FORK_OUT=1: run the dense W_out update concurrently with the dh GEMM
  // (measured neutral on B200: both contend for L2/HBM bandwidth)
  bool fork_out = false;
  bool logits_pair = true;  // DL_LOGITS_2CTA=0: single-CTA tiles for the logits GEMM
  // trainer path: the dense W_out rmsprop runs inside the dW_out GEMM's
  // epilogue (gemm_tc.cu epilogue_rms); DL_FUSE_OUT=0 keeps the separate
  // kernel.  fuse_cap: -1 unknown, else whether the device can run it.
  bool fuse_out = true;
  bool fork_late = false;  // DL_FORK_LATE=1 (run_window late_eta)
  int fuse_cap = -1;
  unsigned* rms_cnt = nullptr;  // [ceil(Vo / 256)] per-M-block arrival counters

  // DP
  Comm* comm = nullptr;  // NcclComm (production) or LocalComm (single-device tests)
  // vocabulary-sharded output layer: this rank owns W_out
  // rows [v0, v0 + Vo); W_in / W_rec and the recurrence are replicated
  bool vshard = false;
  // dpv: data-parallel streams (each rank its own B) AND a vocabulary-
  // parallel output layer over the gathered global window: hidden states,
  // targets and weights are all-gathered, each rank scores every row of the
  // global window against its W_out block, dh is reduce-scattered back.
  // No V x H gradient crosses the links and the dense W_out update is
  // sharded.  (vshard is set too: W_out rows are sharded.)
  bool dpv = false;
  bf16* hs_all_bf = nullptr;  // dpv: [G*TB x H] gathered hidden states (bf16 mode)
  float* hs_all = nullptr;    // dpv: [G*TB x H] (fp32 mode)
  uint32_t* y_all = nullptr;  // dpv: [G*TB] gathered targets
  uint8_t* w_all = nullptr;   // dpv: [G*TB] gathered weights
  float* dh_all = nullptr;    // dpv: [G*TB x H] partial dh over the local W_out block
  int64_t Vo = 0, v0 = 0;
  uint32_t* tgt_loc = nullptr;  // [TB] target column inside this rank's block, or ~0
  double* lse_loc = nullptr;    // [TB] this rank's log-sum-exp over its block
  double* lse_all = nullptr;    // [G x TB] gathered
  int nranks = 1, rank = 0;
  uint32_t* x_all = nullptr;  // [G][T][B] gathered window ids
  float* dpre_all = nullptr;  // [G][T][B][H] gathered dpre
  double* win_loss = nullptr;  // [loss, positions(u64)] of one window
  unsigned* bar_counter = nullptr;  // grid barrier of the persistent recurrence
  unsigned long long* win_pos = nullptr;

  // NCE output layer (LossMode::kNce, trainer.hpp:53): noise model tables
  // (host: alias sampler; device: ln(k q)), the bptt / trainer rng whose
  // draws pick the noise words (host, std::mt19937_64 as the reference), and
  // one window's records
  int loss_mode = 1;  // 0 NCE, 1 exact softmax (LossMode order)
  int nce_k = 0;
  std::vector<double> nz_prob;
  std::vector<uint32_t> nz_alias;
  double* ln_kq_d = nullptr;
  std::mt19937_64 rng{0};
  bool out_sparse = false;  // the last window's dW_out is sparse rows (g_out compact)
  int64_t nce_cap = 0, nce_P = 0, nce_N = 0;
  uint32_t *rec_word_d = nullptr, *rec_row_d = nullptr, *proc_r_d = nullptr;
  float *score_d = nullptr, *ds_d = nullptr, *nce_scale = nullptr;
  double* loss_pos_d = nullptr;
  uint32_t *sort_keys_in = nullptr, *sort_vals_in = nullptr, *sort_keys_out = nullptr,
           *sort_vals_out = nullptr;
  int *sort_head = nullptr, *sort_slot = nullptr;
  void* sort_temp = nullptr;
  size_t sort_temp_bytes = 0;
  EmbedWs nce_ws{};
  uint32_t* g_out_words = nullptr;  // [Vo] words of the compact sparse rows
  int* g_out_n = nullptr;
  double* nz_prob_d = nullptr;    // alias tables on the device (draws from raw outputs)
  uint32_t* nz_alias_d = nullptr;
  unsigned long long* raw_d = nullptr;  // [2 k P] raw mt19937_64 outputs of the window
  uint32_t* pos_of_d = nullptr;   // [TB] unmasked positions in t-major order
  int* first_d = nullptr;         // [T + 1]
  int64_t raw_cap = 0, pos_cap = 0;
  void* raw_pin[2] = {nullptr, nullptr};  // double-buffered host staging of raw outputs
  cudaEvent_t raw_ev[2] = {nullptr, nullptr};
  int raw_slot = 0;
  int raw_last = 0;  // slot of the last prepared window's draws
  // dl_window / dl_train_window in NCE mode draw the NEXT window's noise
  // while the device runs this one (nce_predraw): pre_n outputs of the
  // generator following rng's state, in raw_pin[pre_slot]; rng_ahead
  // continues after them.  rng itself stays at the consumed point.
  std::mt19937_64 rng_ahead{0};
  int64_t pre_n = 0;
  int pre_slot = 0;
  int64_t pre_used = 0;  // outputs of the queue the last prepared window took
  // a caller that sets the generator's state before every window (the C++
  // Traits drop-in: BpttOptions::rng) would have every queue dropped unused:
  // no pre-drawing until a window comes without a dl_set_rng_state first
  bool rng_set = false, predraw_off = false;
  bool nce_pending = false;       // records of the prepared window not built yet
  double nce_wait_s = 0.0, nce_gen_s = 0.0, nce_res_s = 0.0, nce_copy_s = 0.0;  // (DL_DEBUG)
  std::vector<uint32_t> h_ids;  // trainer: host copy of the stream (NCE draws)
  // NCE under data parallel ranks: every rank runs the (cheap, sparse) NCE
  // output layer over the whole global window -- the gathered targets, mask
  // and hidden states laid out t-major over the global streams r*B + b --
  // with the shared generator's draws, so the loss, the sparse W_out rows
  // and their update are identical on every rank; each keeps its own dh rows
  uint32_t *ng_y = nullptr, *ng_y_rb = nullptr;
  uint8_t *ng_w = nullptr, *ng_w_rb = nullptr;
  float *ng_hs = nullptr, *ng_hs_rb = nullptr, *ng_dh = nullptr;

  // profiling
  bool profiling = false;
  std::map<std::string, std::pair<double, int64_t>> prof;  // name -> (ms sum, count)
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
};

namespace {

int fail(dl_ctx* c, int code, const std::string& m) {
  g_err = m;
  if (c) c->err = m;
  return code;
}

template <class F>
int guarded(dl_ctx* c, F&& f) {
  try {
    if (c) DL_CUDA(cudaSetDevice(c->device));
    f();
    return DL_OK;
  } catch (const Error& e) {
    return fail(c, e.code, e.what());
  } catch (const std::exception& e) {
    return fail(c, DL_EDEVICE, e.what());
  }
}

// Ranks that split the minibatch (data parallel).  A vocabulary-sharded
// group runs the same streams on every rank.
int64_t dp_ranks(const dl_ctx* c) { return c->vshard && !c->dpv ? 1 : c->nranks; }
int dp_rank(const dl_ctx* c) { return c->vshard && !c->dpv ? 0 : c->rank; }
// rows the output layer processes per window, as a multiple of T*B
int64_t out_ranks(const dl_ctx* c) { return c->dpv ? c->nranks : 1; }

void drop_graphs(dl_ctx* c) {
  for (int v = 0; v < 2; ++v)
    if (c->graphs[v]) {
      cudaGraphExecDestroy(c->graphs[v]);
      c->graphs[v] = nullptr;
    }
  c->graph = nullptr;
  if (c->tw.e) cudaGraphExecDestroy(c->tw.e);
  if (c->tw.g) cudaGraphDestroy(c->tw.g);
  if (c->tw.pin) cudaFreeHost(c->tw.pin);
  c->tw = dl_ctx::TwGraph{};
}

// ---------------------------------------------------------------- timing
cudaEvent_t ev_get(dl_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    DL_CUDA(cudaEventCreate(&e));
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

struct Phase {
  dl_ctx* c;
  std::string name;
  cudaEvent_t a = nullptr, b = nullptr;
  Phase(dl_ctx* c_, const char* n) : c(c_), name(n) {
    if (c->profiling) {
      a = ev_get(c);
      b = ev_get(c);
      DL_CUDA(cudaEventRecord(a, c->st));
    }
  }
  ~Phase() {
    if (c->profiling) {
      cudaEventRecord(b, c->st);
      c->pending.push_back({name, {a, b}});
    }
  }
};

void prof_collect(dl_ctx* c) {
  if (!c->profiling) return;
  DL_CUDA(cudaStreamSynchronize(c->st));
  for (auto& p : c->pending) {
    float ms = 0.f;
    DL_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
    auto& slot = c->prof[p.first];
    slot.first += ms;
    slot.second += 1;
  }
  c->pending.clear();
  c->ev_used = 0;
}

// ----------------------------------------------------------- allocation
// A workspace is about to be freed and reallocated: the per-window CUDA
// graphs of dl_trainer_run hold its old pointers, so finish the work in
// flight and drop them (they are re-captured on the next dl_trainer_run).
// Never inside a capture (presize() sizes everything before capturing).
void invalidate_workspace(dl_ctx* c) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  DL_CUDA(cudaStreamIsCapturing(c->st, &cs));
  DL_REQUIRE(cs == cudaStreamCaptureStatusNone, DL_EDEVICE,
             "internal: workspace reallocation during graph capture");
  DL_CUDA(cudaStreamSynchronize(c->st));
  if (c->st2) DL_CUDA(cudaStreamSynchronize(c->st2));
  drop_graphs(c);
}

void ensure_window(dl_ctx* c, int64_t T, int64_t B) {
  if (T <= c->capT && B <= c->capB && c->htape) return;
  invalidate_workspace(c);
  const int64_t nT = std::max(T, c->capT), nB = std::max(B, c->capB);
  const int64_t TB = nT * nB, H = c->H, V = c->V;
  auto fr = [](auto*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  fr(c->htape); fr(c->htape_bf); fr(c->x_d); fr(c->y_d); fr(c->w_d); fr(c->S); fr(c->part);
  fr(c->tgt_logit); fr(c->loss_row); fr(c->logp_row); fr(c->dh_out); fr(c->dpre); fr(c->dpre_bf);
  fr(c->g_in_rows); fr(c->g_in_words); fr(c->ews.seg_start); fr(c->ews.order_pos); fr(c->h0_d);
  fr(c->x_all); fr(c->dpre_all);
  fr(c->hs_all_bf); fr(c->hs_all); fr(c->y_all); fr(c->w_all); fr(c->dh_all);
  fr(c->dS); fr(c->xf_lse); fr(c->xf_sc); fr(c->xpose_a); fr(c->xpose_b);
  fr(c->pf_shift); fr(c->pf_sigma); fr(c->pf_resid); fr(c->pf_hs);
  fr(c->ng_y); fr(c->ng_y_rb); fr(c->ng_w); fr(c->ng_w_rb); fr(c->ng_hs); fr(c->ng_hs_rb);
  fr(c->ng_dh);
  c->xpose_a_cap = c->xpose_b_cap = 0;
  c->capT = nT;
  c->capB = nB;
  const int64_t G = dp_ranks(c);  // W_in gradient rows cover the gathered window
  c->htape = dalloc<float>((nT + 1) * nB * H);
  c->x_d = dalloc<uint32_t>(TB);
  c->y_d = dalloc<uint32_t>(TB);
  c->w_d = dalloc<uint8_t>(TB);
  const int64_t MO = out_ranks(c) * TB;  // output-layer rows
  c->loss_row = dalloc<double>(MO);
  c->logp_row = dalloc<double>(MO);
  if (c->dpv) {
    if (c->precision == DL_BF16) c->hs_all_bf = dalloc<bf16>(MO * H);
    else c->hs_all = dalloc<float>(MO * H);
    c->y_all = dalloc<uint32_t>(MO);
    c->w_all = dalloc<uint8_t>(MO);
    c->dh_all = dalloc<float>(MO * H);
  }
  c->dh_out = dalloc<float>(TB * H);
  c->dpre = dalloc<float>(TB * H);
  c->g_in_rows = dalloc<float>(G * TB * H);
  c->g_in_words = dalloc<uint32_t>(G * TB);
  c->ews.seg_start = dalloc<int>(2 * G * TB + 2);
  c->ews.order_pos = dalloc<int>(G * TB);
  c->ews.cap = G * TB;
  c->h0_d = dalloc<float>(nB * H);
  if (G > 1 || c->comm) {  // (a one-rank communicator gathers too)
    c->x_all = dalloc<uint32_t>(G * TB);
    c->dpre_all = dalloc<float>(G * TB * H);
  }
  if (c->comm && !c->vshard && c->loss_mode == 0) {
    c->ng_y = dalloc<uint32_t>(G * TB);
    c->ng_y_rb = dalloc<uint32_t>(G * TB);
    c->ng_w = dalloc<uint8_t>(G * TB);
    c->ng_w_rb = dalloc<uint8_t>(G * TB);
    c->ng_hs = dalloc<float>(G * TB * H);
    c->ng_hs_rb = dalloc<float>(G * TB * H);
    c->ng_dh = dalloc<float>(G * TB * H);
  }
  const int64_t Vo = c->Vo;  // output rows held by this context
  (void)V;
  if (c->precision == DL_BF16) {
    c->htape_bf = dalloc<bf16>((nT + 1) * nB * H);
    c->dpre_bf = dalloc<bf16>(TB * H);
    c->S = dalloc<bf16>(MO * Vo);
    if (c->xf && tc_pair_tiles((int)MO, (int)c->H)) {
      c->dS = dalloc<bf16>(MO * Vo);
      c->xf_lse = dalloc<float>(MO);
      c->xf_sc = dalloc<float>(MO);
    }
    c->part_tiles = tc_n_tiles((int)Vo);
    c->part = dalloc<float2>((size_t)c->part_tiles * MO);
    c->tgt_logit = dalloc<float>(MO);
    if (c->pfac) {
      c->pf_shift = dalloc<float>(MO);
      c->pf_sigma = dalloc<float>(MO);
      c->pf_resid = dalloc<float>(MO);
      c->pf_hs = dalloc<bf16>(MO * H);
    }
  } else {
    c->S = dalloc<float>(MO * Vo);
    if (c->tf32x3) {
      // the window's MN-major fp32 operands, made K-major for 3xTF32:
      // A -- dS^T [Vo x MO] (dW_out), dpre^T [H x TB] (dW_rec);
      // B -- W_out^T [H x Vo] (dh), Hs^T [H x MO] (dW_out), W_rec^T (recurrence)
      auto r4 = [](int64_t x) { return (x + 3) / 4 * 4; };
      c->xpose_a_cap = (size_t)std::max(Vo * r4(MO), H * r4(TB));
      c->xpose_b_cap = (size_t)std::max({H * r4(Vo), H * r4(MO), H * r4(H)});
      c->xpose_a = dalloc<float>(c->xpose_a_cap);
      c->xpose_b = dalloc<float>(c->xpose_b_cap);
    }
  }
  fr(c->tgt_loc); fr(c->lse_loc); fr(c->lse_all);
  if (c->vshard) {
    c->tgt_loc = dalloc<uint32_t>(MO);
    c->lse_loc = dalloc<double>(MO);
    c->lse_all = dalloc<double>((int64_t)c->nranks * MO);
    if (!c->tgt_logit) c->tgt_logit = dalloc<float>(MO);
  }
}

void ensure_splitws(dl_ctx* c, size_t elems) {
  if (elems <= c->splitws_elems) return;
  invalidate_workspace(c);
  if (c->splitws) cudaFree(c->splitws);
  c->splitws = dalloc<float>(elems);
  c->splitws_elems = elems;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void* ensure_pinned(dl_ctx* c, size_t bytes) {
  if (bytes <= c->pinned_bytes) return c->pinned;
  if (c->pinned) cudaFreeHost(c->pinned);
  DL_CUDA(cudaMallocHost(&c->pinned, bytes));
  c->pinned_bytes = bytes;
  return c->pinned;
}

// ---------------------------------------------------------------- GEMMs
bool tc(dl_ctx* c) { return c->precision == DL_BF16; }

int pick_splits(dl_ctx* c, int M, int N, int K, int max_splits = 32) {
  const int bn = tc(c) ? (N >= 256 ? 256 : (N >= 128 ? 128 : 64)) : 128;
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  int s = std::max(1, std::min(max_splits, kNumSMs / std::max(1, tiles)));
  if (tc(c)) s = tc_splits(K, s);
  else if (c->tf32x3) s = tf32_splits(K, s);  // (valid for the SIMT kernel too)
  else s = std::max(1, std::min(s, (K + 63) / 64));
  return s;
}

// fp32 mode on the tensor cores: 3xTF32 (gemm_tc.cu), whose tcgen05
// kind::tf32 MMAs read K-major operands only -- an MN-major operand is
// transposed into the context's scratch first (xpose_a / xpose_b, sized by
// ensure_window for the window's GEMMs)
void gemm(dl_ctx* c, GemmDesc g) {
  c->launches++;
  if (tc(c)) {
    gemm_tc(g, c->st);
    return;
  }
  auto fits = [](int64_t rows, int64_t cols, size_t cap) {
    return (size_t)rows * (size_t)((cols + 3) / 4 * 4) <= cap;
  };
  if (c->tf32x3 && (g.a_major == K_MAJOR || fits(g.M, g.K, c->xpose_a_cap)) &&
      (g.b_major == K_MAJOR || fits(g.N, g.K, c->xpose_b_cap))) {
    if (g.a_major == MN_MAJOR) {
      const int64_t ld = (g.K + 3) / 4 * 4;
      transpose_f32(static_cast<const float*>(g.A), g.K, g.M, g.lda, c->xpose_a, ld, c->st);
      g.A = c->xpose_a;
      g.lda = ld;
      g.a_major = K_MAJOR;
      c->launches++;
    }
    if (g.b_major == MN_MAJOR) {
      const int64_t ld = (g.K + 3) / 4 * 4;
      transpose_f32(static_cast<const float*>(g.B), g.K, g.N, g.ldb, c->xpose_b, ld, c->st);
      g.B = c->xpose_b;
      g.ldb = ld;
      g.b_major = K_MAJOR;
      c->launches++;
    }
    if (tf32x3_ok(g)) {
      gemm_tf32x3(g, c->st);
      return;
    }
  }
  gemm_f32(g, c->st);
}

GemmDesc desc(int M, int N, int K, int am, const void* A, int64_t lda, int bm, const void* B,
              int64_t ldb, float* C, int64_t ldc) {
  GemmDesc g{};
  g.M = M; g.N = N; g.K = K;
  g.a_major = am; g.b_major = bm;
  g.A = A; g.B = B; g.lda = lda; g.ldb = ldb;
  g.C = C; g.ldc = ldc;
  g.k_splits = 1;
  g.split_stride = 0;
  return g;
}

void refresh_shadows(dl_ctx* c) {
  if (!tc(c)) return;
  f32_to_bf16(c->w_rec, c->w_rec_bf, c->H * c->H, c->st);
  f32_to_bf16(c->w_out, c->w_out_bf, c->Vo * c->H, c->st);
  c->launches += 2;
}

// ------------------------------------------------ forward recurrence step
// h_{t+1} = act(h_t . W_rec^T + W_in[x_t]) for Bn rows (backprop.hpp:102-112)
void rec_step_fwd(dl_ctx* c, int64_t Bn, const float* h_prev, const bf16* h_prev_bf,
                  const uint32_t* x, float* h_next, bf16* h_next_bf) {
  const int64_t H = c->H;
  if (tc(c) && c->rec_cluster) {
    rec_step_tc(0, (int)Bn, (int)H, c->act, h_prev_bf, c->w_rec_bf, c->w_in, x, nullptr, nullptr,
                h_next, h_next_bf, c->st);
    c->launches++;
    return;
  }
  const int s = pick_splits(c, (int)Bn, (int)H, (int)H);
  ensure_splitws(c, (size_t)s * Bn * H);
  GemmDesc g = tc(c) ? desc((int)Bn, (int)H, (int)H, K_MAJOR, h_prev_bf, H, K_MAJOR, c->w_rec_bf,
                            H, c->splitws, H)
                     : desc((int)Bn, (int)H, (int)H, K_MAJOR, h_prev, H, K_MAJOR, c->w_rec, H,
                            c->splitws, H);
  g.k_splits = s;
  g.split_stride = Bn * H;
  gemm(c, g);
  rec_fwd(c->splitws, s, Bn * H, Bn, H, c->w_in, x, c->act, h_next, h_next_bf, c->st);
  c->launches++;
}

// logits over M rows of `hs` with per-row targets; writes loss_row /
// logp_row; with grads leaves dS in c->S.
void output_layer(dl_ctx* c, int64_t M, const float* hs, const bf16* hs_bf, const uint32_t* tgt,
                  const uint8_t* wts, double scale, bool grads, double* loss_row,
                  double* logp_row) {
  const int64_t V = c->Vo, H = c->H;  // this context's vocabulary rows
  // Vocabulary-sharded: logits over the local block, the
  // per-row block lse gathered from every rank (G x M doubles) and the target
  // logit summed from its owner -- the only exchange of the forward pass.
  const bool vs = c->vshard && c->comm;
  if (vs) {
    shard_targets(tgt, M, c->v0, V, c->tgt_loc, c->st);
    c->launches++;
    tgt = c->tgt_loc;
  }
  if (tc(c)) {
    // shifted-exponential softmax (kernels.cu k_pfac_rows): the shift is
    // the row's target logit, summed from its owner when the vocabulary is
    // sharded (each rank's E is then relative to the same shift, until a
    // rank repairs a row with its own block maximum -- the block lse
    // exchange carries that)
    c->pf_on = grads && c->pfac && c->pf_shift != nullptr && !c->xf;
    float nats = 40.f;
    if (const char* e = std::getenv("DL_PFAC_REPAIR_NATS")) nats = (float)std::atof(e);
    if (c->pf_on) {
      Phase p(c, "softmax");
      target_shift(hs_bf, c->w_out_bf, H, M, tgt, V, c->pf_shift, c->st);
      c->pf_tgt = tgt;
      c->launches++;
      if (vs) c->comm->allreduce_sum(c->pf_shift, (size_t)M, DType::F32, c->st);
    }
    GemmDesc g = desc((int)M, (int)V, (int)H, K_MAJOR, hs_bf, H, K_MAJOR, c->w_out_bf, H, nullptr, 0);
    g.logits = 1;
    g.S = grads ? static_cast<bf16*>(c->S) : nullptr;
    g.shift = c->pf_on ? c->pf_shift : nullptr;
    g.part_n = c->part_tiles;
    g.lds = V;
    g.part = c->part;
    g.tgt = tgt;
    g.tgt_logit = c->tgt_logit;
    g.raster = 0;
    // with the 8-warp epilogue the logits GEMM gains most from CTA pairs
    // (C3: 0.352 vs 0.404 ms single-CTA)
    g.no_pair = c->logits_pair ? 0 : 1;
    if (vs) DL_CUDA(cudaMemsetAsync(c->tgt_logit, 0, M * sizeof(float), c->st));
    {
      Phase p(c, "logits");
      gemm(c, g);
    }
    if (vs) {
      Phase p(c, "vocab_exchange");
      if (c->pf_on)
        pfac_lse(static_cast<bf16*>(c->S), M, V, c->part, c->part_tiles, wts, c->pf_shift,
                 c->lse_loc, nats, c->pf_repaired, c->st);
      else
        block_lse_bf16(c->part, c->part_tiles, M, c->lse_loc, c->st);
      c->launches++;
      c->comm->allgather(c->lse_loc, c->lse_all, (size_t)M, DType::F64, c->st);
      c->comm->allreduce_sum(c->tgt_logit, (size_t)M, DType::F32, c->st);
    }
    Phase p(c, "softmax");
    // dS on the fly in the dh GEMM (pair tiles over the whole output-row
    // block): only the rows' lse / loss here
    c->xf_on = !c->pf_on && grads && c->dS != nullptr && tc_pair_tiles((int)M, (int)H);
    if (c->pf_on) {
      // (the gathered window of the vocabulary-parallel layout has its
      // hidden states in bf16 only)
      pfac_rows(static_cast<bf16*>(c->S), M, V, H, c->part, c->part_tiles, c->tgt_logit, tgt, wts,
                scale, loss_row, logp_row, c->pf_shift, c->pf_sigma, c->pf_resid,
                c->dpv ? nullptr : hs, c->pf_hs, hs_bf, nats, c->pf_repaired, c->st,
                vs ? c->lse_all : nullptr, c->nranks);
    } else if (c->xf_on) {
      c->xf_tgt = tgt;
      lse_rows_bf16(M, c->part, c->part_tiles, c->tgt_logit, wts, scale, loss_row, logp_row,
                    c->xf_lse, c->xf_sc, c->st, vs ? c->lse_all : nullptr, c->nranks);
    } else {
      softmax_rows_bf16(grads ? static_cast<bf16*>(c->S) : nullptr, M, V, c->part,
                        c->part_tiles, c->tgt_logit, tgt, wts, scale, grads ? 1 : 0, loss_row,
                        logp_row, c->st, vs ? c->lse_all : nullptr, c->nranks);
    }
    c->launches++;
  } else {
    c->xf_on = false;
    GemmDesc g = desc((int)M, (int)V, (int)H, K_MAJOR, hs, H, K_MAJOR, c->w_out, H,
                      static_cast<float*>(c->S), V);
    {
      Phase p(c, "logits");
      gemm(c, g);
    }
    if (vs) {
      Phase p(c, "vocab_exchange");
      block_lse_f32(static_cast<float*>(c->S), M, V, tgt, c->lse_loc, c->tgt_logit, c->st);
      c->launches++;
      c->comm->allgather(c->lse_loc, c->lse_all, (size_t)M, DType::F64, c->st);
      c->comm->allreduce_sum(c->tgt_logit, (size_t)M, DType::F32, c->st);
    }
    Phase p(c, "softmax");
    softmax_rows_f32(static_cast<float*>(c->S), M, V, tgt, wts, scale, grads ? 1 : 0, loss_row,
                     logp_row, c->st, vs ? c->lse_all : nullptr, c->nranks, c->tgt_logit);
    c->launches++;
  }
}

// ------------------------------------------------------------------ NCE
// NoiseModel (nce.hpp:41-66) + AliasSampler (rng.hpp:54-89), host side.
void nce_build(dl_ctx* c, const double* counts, int64_t V, int k, double floor,
               bool dist = false) {
  std::vector<double> lnkq, prob;
  std::vector<uint32_t> alias;
  if (dist) noise_tables_q(counts, V, k, lnkq, prob, alias);
  else noise_tables(counts, V, k, floor, lnkq, prob, alias);
  c->nce_k = k;
  if (!c->ln_kq_d) c->ln_kq_d = dalloc<double>(V);
  if (!c->nz_prob_d) c->nz_prob_d = dalloc<double>(V);
  if (!c->nz_alias_d) c->nz_alias_d = dalloc<uint32_t>(V);
  DL_CUDA(cudaMemcpy(c->ln_kq_d, lnkq.data(), V * 8, cudaMemcpyHostToDevice));
  DL_CUDA(cudaMemcpy(c->nz_prob_d, prob.data(), V * 8, cudaMemcpyHostToDevice));
  DL_CUDA(cudaMemcpy(c->nz_alias_d, alias.data(), V * 4, cudaMemcpyHostToDevice));
  c->nz_prob = std::move(prob);
  c->nz_alias = std::move(alias);
}

void nce_reserve(dl_ctx* c, int64_t N) {
  if (N <= c->nce_cap) return;
  auto fr = [](auto*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  fr(c->rec_word_d); fr(c->rec_row_d); fr(c->proc_r_d); fr(c->score_d); fr(c->ds_d);
  fr(c->nce_scale); fr(c->loss_pos_d); fr(c->sort_keys_in); fr(c->sort_vals_in);
  fr(c->sort_keys_out); fr(c->sort_vals_out); fr(c->sort_head); fr(c->sort_slot);
  fr(c->sort_temp); fr(c->nce_ws.seg_start); fr(c->nce_ws.order_pos);
  c->rec_word_d = dalloc<uint32_t>(N);
  c->rec_row_d = dalloc<uint32_t>(N);
  c->proc_r_d = dalloc<uint32_t>(N);
  c->score_d = dalloc<float>(N);
  c->ds_d = dalloc<float>(N);
  c->nce_scale = dalloc<float>(N);
  c->loss_pos_d = dalloc<double>(N);
  c->sort_keys_in = dalloc<uint32_t>(N);
  c->sort_vals_in = dalloc<uint32_t>(N);
  c->sort_keys_out = dalloc<uint32_t>(N);
  c->sort_vals_out = dalloc<uint32_t>(N);
  c->sort_head = dalloc<int>(N);
  c->sort_slot = dalloc<int>(N);
  c->sort_temp_bytes = nce_sort_temp_bytes(N);
  c->sort_temp = dalloc<uint8_t>(c->sort_temp_bytes);
  c->nce_ws.seg_start = dalloc<int>(2 * N + 2);
  c->nce_ws.order_pos = dalloc<int>(N);
  c->nce_ws.cap = N;
  c->nce_cap = N;
}

// The window's noise draws (backprop.hpp:126-156 order: t, b, then sample;
// masked positions draw nothing): the host advances the trainer's
// mt19937_64 by exactly the reference's 2 outputs per draw and ships the raw
// outputs; the device turns them into words with the alias tables and
// builds the records (nce.cu k_nce_records) once the window's targets and
// mask are on the device (run_window).  The staging is double-buffered so
// the host can draw the next window while the device runs this one.
// predraw: the caller runs nce_predraw after launching the window (else
// any pre-drawn outputs are dropped: rng is at the consumed point anyway).
void nce_prepare(dl_ctx* c, int64_t T, int64_t B, const uint8_t* weights, bool predraw = false) {
  DL_REQUIRE(c->nce_k > 0 && !c->nz_prob.empty(), 1,
             "bptt: NCE mode needs noise model and rng (dl_set_noise)");
  const int K1 = c->nce_k + 1;
  int64_t P = 0;
  for (int64_t i = 0; i < T * B; ++i) P += weights[i] ? 1 : 0;
  const int64_t N = P * K1, ND = 2 * P * c->nce_k;  // raw outputs
  const auto r0 = std::chrono::steady_clock::now();
  // (for the window's maximum, every position unmasked: no reallocation --
  // a device-synchronising cudaFree -- as the masked count varies)
  nce_reserve(c, std::max<int64_t>(T * B * K1, 1));
  c->nce_res_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - r0).count();
  if (ND > c->raw_cap || !c->pos_of_d || c->capT * c->capB > c->raw_cap / 2 ||
      c->pos_cap < T * B) {
    const int64_t cap = std::max<int64_t>({ND, 2 * c->capT * c->capB * c->nce_k, 2});
    c->pre_n = 0;  // (any pre-drawn outputs live in the buffers freed here)
    for (int i = 0; i < 2; ++i) {
      if (c->raw_ev[i]) DL_CUDA(cudaEventSynchronize(c->raw_ev[i]));
      if (c->raw_pin[i]) cudaFreeHost(c->raw_pin[i]);
      DL_CUDA(cudaMallocHost(&c->raw_pin[i], cap * 8));
      if (!c->raw_ev[i])
        DL_CUDA(cudaEventCreateWithFlags(&c->raw_ev[i], cudaEventDisableTiming));
    }
    if (c->raw_d) cudaFree(c->raw_d);
    if (c->pos_of_d) cudaFree(c->pos_of_d);
    if (c->first_d) cudaFree(c->first_d);
    c->raw_d = dalloc<unsigned long long>(cap);
    c->pos_cap = std::max<int64_t>(c->capT * c->capB, T * B);
    c->pos_of_d = dalloc<uint32_t>(c->pos_cap);
    c->first_d = dalloc<int>(std::max(c->capT, T) + 1);
    c->raw_cap = cap;
  }
  if (predraw) {
    if (!c->rng_set) c->predraw_off = false;
    c->rng_set = false;
  }
  if (c->pre_used > 0) {  // (a window that failed after taking its draws)
    c->rng.discard(c->pre_used);
    c->pre_n = 0;
  }
  c->pre_used = 0;
  int slot;
  unsigned long long* raw;
  const auto t0 = std::chrono::steady_clock::now();
  auto t1 = t0;
  if (predraw && c->pre_n > 0 && c->pre_n >= ND) {
    // drawn during the previous call (nce_predraw): the same outputs rng
    // would give now; rng advances past them in nce_predraw
    slot = c->pre_slot;
    raw = static_cast<unsigned long long*>(c->raw_pin[slot]);
    c->pre_used = ND;
    t1 = std::chrono::steady_clock::now();
  } else {
    c->pre_n = 0;
    slot = c->raw_slot;
    DL_CUDA(cudaEventSynchronize(c->raw_ev[slot]));  // its previous upload is done
    t1 = std::chrono::steady_clock::now();
    raw = static_cast<unsigned long long*>(c->raw_pin[slot]);
    for (int64_t i = 0; i < ND; ++i) raw[i] = c->rng();
  }
  c->raw_slot = slot ^ 1;
  c->raw_last = slot;
  const auto t2 = std::chrono::steady_clock::now();
  c->nce_wait_s += std::chrono::duration<double>(t1 - t0).count();
  c->nce_gen_s += std::chrono::duration<double>(t2 - t1).count();
  if (ND > 0)
    DL_CUDA(cudaMemcpyAsync(c->raw_d, raw, ND * 8, cudaMemcpyHostToDevice, c->st));
  DL_CUDA(cudaEventRecord(c->raw_ev[slot], c->st));
  c->nce_copy_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
  c->nce_P = P;
  c->nce_N = N;
  c->nce_pending = true;
}

// After the window prepared by nce_prepare has been launched: rng moves to
// the consumed point, then the outputs a next window of the same shape can
// take at most (every position unmasked) are drawn into the other staging
// slot while the device works -- what is left of the queue first, then
// rng_ahead.  The sequence of outputs is the generator's either way.
void nce_predraw(dl_ctx* c, int64_t T, int64_t B) {
  const int64_t cap_n = 2 * T * B * c->nce_k;
  const int cur = c->raw_last, nxt = cur ^ 1;
  int64_t have = 0;
  unsigned long long* dst = static_cast<unsigned long long*>(c->raw_pin[nxt]);
  if (cap_n > c->raw_cap || c->predraw_off) {
    if (c->pre_used > 0) c->rng.discard(c->pre_used);
    c->pre_n = 0;
    c->pre_used = 0;
    return;
  }
  DL_CUDA(cudaEventSynchronize(c->raw_ev[nxt]));  // its last upload (two windows back)
  if (c->pre_used > 0) {
    c->rng.discard(c->pre_used);
    have = c->pre_n - c->pre_used;
    if (have > 0)
      std::memcpy(dst, static_cast<unsigned long long*>(c->raw_pin[cur]) + c->pre_used, have * 8);
  } else {
    c->rng_ahead = c->rng;
  }
  for (; have < cap_n; ++have) dst[have] = c->rng_ahead();
  c->pre_n = have;
  c->pre_slot = nxt;
  c->pre_used = 0;
}

// One window with device-resident inputs (x_d, y_d, w_d, htape[0]).
// Accumulates loss into d_loss and scored positions into d_pos.
// fork_out_eta > 0: apply the dense W_out rmsprop with that eta on the side
// stream as soon as dW_out is final (caller joins ev_join).
// fuse_eta > 0: the dense W_out rmsprop with that eta runs inside the dW_out
// GEMM's epilogue (fuse_ok); dh then runs first, as it reads this window's
// W_out shadow, which the fused update overwrites in place.
void run_window(dl_ctx* c, int64_t T, int64_t B, double scale, float clip, bool grads,
                double fork_out_eta = 0.0, double fuse_eta = 0.0, double late_eta = 0.0) {
  // V: input vocabulary (W_in rows); Vo: output rows held here (V / G when
  // the softmax is vocabulary-sharded)
  const int64_t H = c->H, V = c->V, Vo = c->Vo, TB = T * B, BH = B * H;
  cudaStream_t st = c->st;
  // dp: dense dW_out summed over ranks; dprec: the recurrence side (W_rec,
  // W_in) is data parallel; vs: replicated streams, vocabulary-sharded
  // output (dh summed); dpv: data-parallel streams with a vocabulary-
  // parallel output layer over the gathered window (dh reduce-scattered)
  const bool dp = c->comm != nullptr && !c->vshard;
  const bool dpv = c->comm != nullptr && c->dpv;
  const bool dprec = dp || dpv;
  const bool vs = c->comm != nullptr && c->vshard && !dpv;
  const int64_t MO = dpv ? c->nranks * TB : TB;  // output-layer rows
  c->pf_on = false;  // (set by output_layer for this window)
  c->rec_fused = false;
  if (grads && !dprec) {
    // the W_in gradient's id sort depends on x only: run it on the side
    // stream under the forward recurrence (which leaves SMs free) (joined before embed_rows)
    DL_CUDA(cudaEventRecord(c->ev_sort_fork, st));
    DL_CUDA(cudaStreamWaitEvent(c->st2, c->ev_sort_fork, 0));
    embed_sort(c->x_d, T, B, 1, V, c->ews, c->g_in_words, c->g_in_n, c->st2);
    c->launches++;
    if (fuse_eta > 0.0 && std::isfinite(clip)) {
      // this window's update cannot be rejected (a finite clip maps every
      // gradient element to a finite value): every W_in accumulator's decay
      // (rmsprop.hpp:84) runs here too, instead of after the backward pass
      rms_decay(c->m_in, c->V, c->rho, nullptr, c->st2);
      c->launches++;
      c->in_decayed = true;
    }
    DL_CUDA(cudaEventRecord(c->ev_sort_join, c->st2));
  }
  if (tc(c) && !c->h0_bf_ready) {
    f32_to_bf16(c->htape, c->htape_bf, BH, st);
    c->launches++;
  }
  {
    Phase p(c, "recurrence_fwd");
    const bool persist = tc(c) && c->rec_cluster &&
                         rec_window_tc(0, (int)T, (int)B, (int)H, c->act, c->htape_bf, (T + 1) * B,
                                       c->w_rec_bf, c->w_in, c->x_d, nullptr, nullptr, c->htape,
                                       c->htape_bf, c->bar_counter, st);
    if (persist) {
      c->launches++;
    } else {
      for (int64_t t = 0; t < T; ++t)
        rec_step_fwd(c, B, c->htape + t * BH, tc(c) ? c->htape_bf + t * BH : nullptr,
                     c->x_d + t * B, c->htape + (t + 1) * BH,
                     tc(c) ? c->htape_bf + (t + 1) * BH : nullptr);
    }
  }
  DL_CUDA(cudaEventRecord(c->ev_hfinal, st));  // h_T final (window_call's D2H)
  const float* Hs = c->htape + BH;
  const bf16* Hs_bf = tc(c) ? c->htape_bf + BH : nullptr;
  const uint32_t* yo = c->y_d;
  const uint8_t* wo = c->w_d;
  if (dpv) {
    // gather the global window's hidden states, targets and weights
    // (rank-blocked rows r*TB + t*B + b): every rank scores all of them
    // against its W_out block
    Phase p(c, "vocab_exchange");
    if (tc(c)) {
      c->comm->allgather(Hs_bf, c->hs_all_bf, (size_t)(TB * H), DType::BF16, st);
      Hs_bf = c->hs_all_bf;
    } else {
      c->comm->allgather(Hs, c->hs_all, (size_t)(TB * H), DType::F32, st);
      Hs = c->hs_all;
    }
    c->comm->allgather(c->y_d, c->y_all, (size_t)TB, DType::U32, st);
    c->comm->allgather(c->w_d, c->w_all, (size_t)TB, DType::U8, st);
    yo = c->y_all;
    wo = c->w_all;
  }
  const bool nce = c->loss_mode == 0;
  // NCE with data-parallel ranks: the output layer runs over the global
  // window (t-major over the global streams r*B + b) on every rank
  const bool nce_dp = nce && dp;
  const int64_t Bn = nce_dp ? c->nranks * B : B;  // streams of the NCE window
  const float* Hn = Hs;
  if (nce_dp) {
    Phase p(c, "nce_gather");
    DL_REQUIRE(c->ng_hs != nullptr, DL_EDEVICE, "internal: NCE gather buffers");
    const int G = c->nranks;
    c->comm->allgather(c->y_d, c->ng_y_rb, (size_t)TB, DType::U32, st);
    c->comm->allgather(c->w_d, c->ng_w_rb, (size_t)TB, DType::U8, st);
    c->comm->allgather(Hs, c->ng_hs_rb, (size_t)(TB * H), DType::F32, st);
    // rank-blocked [r][t][b] -> t-major [t][r][b]
    for (int r = 0; r < G; ++r) {
      DL_CUDA(cudaMemcpy2DAsync(c->ng_y + r * B, Bn * 4, c->ng_y_rb + r * TB, B * 4, B * 4, T,
                                cudaMemcpyDeviceToDevice, st));
      DL_CUDA(cudaMemcpy2DAsync(c->ng_w + r * B, Bn, c->ng_w_rb + r * TB, B, B, T,
                                cudaMemcpyDeviceToDevice, st));
      DL_CUDA(cudaMemcpy2DAsync(c->ng_hs + r * B * H, Bn * H * 4, c->ng_hs_rb + r * TB * H,
                                B * H * 4, B * H * 4, T, cudaMemcpyDeviceToDevice, st));
    }
    Hn = c->ng_hs;
  }
  if (nce) {
    // NCE loss over the window's records (backprop.hpp:126-156)
    Phase p(c, "nce_loss");
    const int K1 = c->nce_k + 1;
    DL_REQUIRE(c->nce_pending, 1, "NCE window without prepared draws");
    nce_records(nce_dp ? c->ng_w : c->w_d, nce_dp ? c->ng_y : c->y_d, T, Bn, c->nce_P, K1,
                c->raw_d, c->nz_prob_d, c->nz_alias_d, V, c->pos_of_d, c->first_d,
                c->rec_word_d, c->rec_row_d, c->proc_r_d, st);
    c->nce_pending = false;
    c->launches += 2;
    nce_scores(Hn, c->w_out, H, c->rec_word_d, c->rec_row_d, c->nce_N, c->score_d, st,
               tc(c) ? c->w_out_bf : nullptr);
    c->launches++;
    nce_loss(c->score_d, c->rec_word_d, c->ln_kq_d, c->nce_P, K1, scale, c->loss_pos_d, c->ds_d,
             st);
    sum_rows(c->loss_pos_d, nullptr, c->nce_P, c->d_loss, c->d_pos, st);
    c->launches += 3;
  } else {
    output_layer(c, MO, Hs, Hs_bf, yo, wo, scale, grads, c->loss_row, nullptr);
  }
  if (nce) {
  } else if (dp) {
    // the window's loss is the sum over all ranks' streams
    DL_CUDA(cudaMemsetAsync(c->win_loss, 0, 16, st));
    sum_rows(c->loss_row, c->w_d, TB, c->win_loss, c->win_pos, st);
    c->comm->allreduce_sum(c->win_loss, 1, DType::F64, st);
    c->comm->allreduce_sum(c->win_pos, 1, DType::U64, st);
    accum_loss(c->d_loss, c->win_loss, c->d_pos, c->win_pos, st);
    c->launches += 2;
  } else {
    // (dpv: the gathered rows are the global window on every rank)
    sum_rows(c->loss_row, wo, MO, c->d_loss, c->d_pos, st);
    c->launches++;
  }
  if (!grads) return;

  DL_CUDA(cudaMemsetAsync(c->nonfinite, 0, sizeof(int), st));
  c->out_sparse = nce;
  const bool fused = fuse_eta > 0.0 && !nce;
  // late fork: dh, then dW_out, then the dense update on the side stream
  // (in place: dh has consumed this window's shadow), overlapping the
  // latency-bound backward recurrence, dW_rec and the W_in rows
  const bool late = late_eta > 0.0;
  // dW_out = dS^T . Hs  [V x H], clipped (rnn.hpp:256 matmul_tn_add; rnn.hpp:158-159)
  auto dw_out = [&] {
    Phase p(c, "dw_out");
    if (fused) {
      // + the dense rmsprop of every row (rmsprop.hpp:94-107) in the epilogue
      GemmDesc g = desc((int)Vo, (int)H, (int)MO, MN_MAJOR, c->xf_on ? c->dS : c->S, Vo,
                        MN_MAJOR, c->pf_on ? c->pf_hs : Hs_bf, H, nullptr, H);
      g.raster = 1;
      g.clip = clip;
      g.rowsq = c->rowsq;
      g.rms = 1;
      g.rms_w = c->w_out;
      g.rms_wb = c->w_out_bf;
      g.rms_m = c->m_out;
      g.rms_cnt = c->rms_cnt;
      g.rho = c->rho;
      g.eps = c->eps;
      g.eta = fuse_eta;
      DL_CUDA(cudaMemsetAsync(c->rms_cnt, 0, ((Vo + 255) / 256) * sizeof(unsigned), st));
      c->g16_valid = false;
      c->dp16 = false;
      static const bool tracing = std::getenv("DL_GEMM_TRACE") != nullptr;
      static unsigned long long* trace = nullptr;
      if (tracing && !c->profiling) {
        if (!trace) DL_CUDA(cudaMalloc(&trace, (3 * 64 * 4 + 148 * 8 * 32) * 8));
        DL_CUDA(cudaMemsetAsync(trace, 0, (3 * 64 * 4 + 148 * 8 * 32) * 8, st));
        g.trace = trace;
        g.trace_warps = std::getenv("DL_GEMM_TRACE_WARPS") != nullptr;
      }
      gemm(c, g);
      if (g.trace) {
        // per-tile epilogue phases of three pairs (diagnostics)
        static unsigned long long h[3 * 64 * 4 + 148 * 8 * 32];
        DL_CUDA(cudaStreamSynchronize(st));
        DL_CUDA(cudaMemcpy(h, g.trace, sizeof h, cudaMemcpyDeviceToHost));
        {
          // arrival time of every epilogue warp per round: within each M
          // block (8 pairs = 16 CTAs x 8 warps), the spread and who is last
          const unsigned long long* a = h + 3 * 64 * 4;
          double spread = 0;
          int ns = 0;
          std::vector<int> last_w(8, 0), last_c(144, 0);
          for (int it = 1; it < 26; ++it)
            for (int b = 0; b < 9; ++b) {
              unsigned long long mn = ~0ull, mx = 0;
              int aw = -1, ac = -1;
              for (int cta = b * 16; cta < b * 16 + 16; ++cta)
                for (int w = 0; w < 8; ++w) {
                  const unsigned long long v = a[(cta * 8 + w) * 32 + it];
                  if (!v) continue;
                  mn = std::min(mn, v);
                  if (v > mx) { mx = v; aw = w; ac = cta; }
                }
              if (aw >= 0) { spread += (double)(mx - mn); ++ns; last_w[aw]++; last_c[ac]++; }
            }
          fprintf(stderr, "[desklm] fused dW_out: mean arrival spread within an M block %.0f ns; "
                  "last warp (2..9):", ns ? spread / ns : 0.0);
          for (int w = 0; w < 8; ++w) fprintf(stderr, " %d", last_w[w]);
          fprintf(stderr, "; last CTA parity even/odd: ");
          int ev = 0, od = 0;
          for (int cta = 0; cta < 144; ++cta) (cta % 2 ? od : ev) += last_c[cta];
          fprintf(stderr, "%d/%d\n", ev, od);
        }
        for (int p = 0; p < 3; ++p) {
          double a = 0, b = 0, cc = 0, per = 0;
          int n = 0;
          for (int i = 1; i + 1 < 64; ++i) {
            const unsigned long long* r = h + (p * 64 + i) * 4;
            const unsigned long long* q = h + (p * 64 + i + 1) * 4;
            if (!r[0] || !r[3] || !q[0]) break;
            a += (double)(r[1] - r[0]);
            b += (double)(r[2] - r[1]);
            cc += (double)(r[3] - r[2]);
            per += (double)(q[0] - r[0]);
            ++n;
          }
          if (n)
            fprintf(stderr, "[desklm] fused dW_out pair-slot %d: pass1 %.0f  sync %.0f  pass2 %.0f  "
                    "tile period %.0f ns (%d tiles)\n", p, a / n, b / n, cc / n, per / n, n);
        }
      }
      return;
    }
    GemmDesc g = tc(c) ? desc((int)Vo, (int)H, (int)MO, MN_MAJOR, c->xf_on ? c->dS : c->S, Vo,
                              MN_MAJOR, c->pf_on ? c->pf_hs : Hs_bf, H, c->g_out, H)
                       : desc((int)Vo, (int)H, (int)MO, MN_MAJOR, c->S, Vo, MN_MAJOR, Hs, H,
                              c->g_out, H);
    g.raster = 1;
    g.do_clip = dp ? 0 : 1;
    g.clip = clip;
    g.nonfinite = c->nonfinite;
    // throughput mode: bf16 clipped dW_out + row sums of squares (halves the
    // gradient's HBM traffic); needs a finite clip (no non-finite check) and
    // no allreduce between the GEMM and the update
    c->g16_valid = tc(c) && c->g16 && !dp && std::isfinite(clip);
    c->dp16 = tc(c) && dp && std::isfinite(clip) && (H % 8) == 0;
    c->dp16_clip = clip;
    if (c->g16_valid) {
      g.Cb = c->g_out_bf;
      g.rowsq = c->rowsq;
    } else if (c->dp16) {
      // per-rank partial, unclipped (the sum is clipped): bf16, no row sums
      g.Cb = c->g_out_bf;
      g.clip = INFINITY;
    }
    if (!dp) {
      gemm(c, g);
      return;
    }
    // data parallel: dW_out in V chunks, each summed over
    // the ranks on the communication stream as soon as its GEMM is done --
    // the allreduce of chunk i overlaps the GEMM of chunk i+1, the last one
    // overlaps dh and the backward recurrence (joined before the update);
    // the fp32 sum is clipped after the reduction
    const int64_t nch = std::min<int64_t>(c->dp_chunks, std::max<int64_t>(1, Vo / 256));
    for (int64_t k = 0; k < nch; ++k) {
      const int64_t v0 = (Vo * k / nch) / 256 * 256;
      const int64_t v1 = k + 1 == nch ? Vo : (Vo * (k + 1) / nch) / 256 * 256;
      GemmDesc gk = g;
      gk.M = (int)(v1 - v0);
      gk.A = tc(c) ? (const void*)(static_cast<const bf16*>(gk.A) + v0)
                   : (const void*)(static_cast<const float*>(gk.A) + v0);
      gk.C = c->g_out + v0 * H;
      if (gk.Cb) gk.Cb = c->g_out_bf + v0 * H;
      gemm(c, gk);
      DL_CUDA(cudaEventRecord(c->ev_fork, st));
      DL_CUDA(cudaStreamWaitEvent(c->st2, c->ev_fork, 0));
      if (c->dp16) {
        c->comm->allreduce_sum(c->g_out_bf + v0 * H, (size_t)((v1 - v0) * H), DType::BF16,
                               c->st2);
      } else {
        c->comm->allreduce_sum(c->g_out + v0 * H, (size_t)((v1 - v0) * H), DType::F32, c->st2);
        reduce_splits(c->g_out + v0 * H, 1, 0, (v1 - v0) * H, c->g_out + v0 * H, clip, 1,
                      c->nonfinite, c->st2);
        c->launches++;
      }
    }
  };
  if (nce) {
    // score_backward of every record: dh[t][b] = sum ds * W_out[w]
    // (rnn.hpp:251-255); masked positions contribute nothing
    Phase p(c, "nce_dh");
    float* dhn = nce_dp ? c->ng_dh : c->dh_out;
    DL_CUDA(cudaMemsetAsync(dhn, 0, T * Bn * H * sizeof(float), st));
    nce_dh(c->w_out, H, c->rec_word_d, c->rec_row_d, c->ds_d, c->nce_P, c->nce_k + 1, dhn, st,
           tc(c) ? c->w_out_bf : nullptr);
    c->launches++;
    if (nce_dp)  // this rank's rows of the global window
      DL_CUDA(cudaMemcpy2DAsync(c->dh_out, B * H * 4, c->ng_dh + c->rank * B * H, Bn * H * 4,
                                B * H * 4, T, cudaMemcpyDeviceToDevice, st));
  }
  // With a finite clip bound every clipped component is finite (clip1 maps
  // NaN to -c), so rmsprop_update's all-finite check (rmsprop.hpp:116)
  // cannot fail and the dense W_out update -- HBM-bound -- may start as soon
  // as dW_out is final, on the side stream, concurrently with the
  // tensor-bound dh GEMM below.  It writes the fp32 master and the *other*
  // bf16 shadow, so dh keeps reading this window's W_out; the caller joins
  // ev_join and flips the shadows (swap_shadow).
  auto fork_update = [&](double eta, bf16* shadow) {
    DL_CUDA(cudaEventRecord(c->ev_fork, st));
    DL_CUDA(cudaStreamWaitEvent(c->st2, c->ev_fork, 0));
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->profiling) {
      a = ev_get(c);
      b = ev_get(c);
      DL_CUDA(cudaEventRecord(a, c->st2));
    }
    if (c->g16_valid)
      rms_dense_g16(c->w_out, shadow, c->m_out, c->g_out_bf, c->rowsq, c->rowsq_n, Vo, H, c->rho,
                    c->eps, eta, c->st2);
    else
      rms_rows(c->w_out, shadow, c->m_out, c->g_out, nullptr, nullptr, Vo, H, c->rho, c->eps,
               eta, 1, nullptr, c->st2);
    c->launches++;
    if (c->profiling) {
      DL_CUDA(cudaEventRecord(b, c->st2));
      c->pending.push_back({"rmsprop_out", {a, b}});
    }
    DL_CUDA(cudaEventRecord(c->ev_join, c->st2));
  };
  // (dW_out reads the dS the dh GEMM stores when it is formed there; with
  // the vocabulary-parallel layer the dh reduce-scatter runs under dW_out)
  const bool dw_after_dh = fused || late || c->xf_on || dpv;
  auto after_dw = [&] {
    if (fork_out_eta > 0.0) fork_update(fork_out_eta, c->w_out_bf_next);
  };
  if (!dw_after_dh && !nce) {
    dw_out();
    after_dw();
  }
  // dh_out = dS . W_out   [TB x H]  (rnn.hpp:257 matmul_nn)
  auto dh = [&] {
    Phase p(c, "dh");
    float* dst = dpv ? c->dh_all : c->dh_out;
    const int s = pick_splits(c, (int)MO, (int)H, (int)Vo, 8);
    GemmDesc g = tc(c) ? desc((int)MO, (int)H, (int)Vo, K_MAJOR, c->S, Vo, MN_MAJOR, c->w_out_bf,
                              H, dst, H)
                       : desc((int)MO, (int)H, (int)Vo, K_MAJOR, c->S, Vo, MN_MAJOR, c->w_out, H,
                              dst, H);
    g.raster = 0;
    if (c->pf_on) {
      g.row_scale = c->pf_sigma;  // dS = diag(sigma) E' (+ the target column's residual)
      g.row_resid = c->pf_resid;
      g.resid_idx = c->pf_tgt;
      g.resid_w = c->w_out_bf;
    }
    if (c->xf_on) {
      // the A tiles are logits: dS = scale (p - 1[y]) is formed in shared
      // memory (backprop.hpp:179-186) and stored to c->dS for dW_out
      g.xf = 1;
      g.xf_lse = c->xf_lse;
      g.xf_sc = c->xf_sc;
      g.xf_tgt = c->xf_tgt;
      g.xf_out = c->dS;
    }
    if (s > 1) {
      ensure_splitws(c, (size_t)s * MO * H);
      g.C = c->splitws;
      g.k_splits = s;
      g.split_stride = MO * H;
      gemm(c, g);
      reduce_splits(c->splitws, s, MO * H, MO * H, dst, 0.f, 0, nullptr, st);
      c->launches++;
    } else {
      gemm(c, g);
    }
  };
  if (!nce) dh();
  if (dpv && !nce) {
    // every rank's partial dh over the global window, summed over ranks and
    // scattered (this rank keeps its own TB rows) on the side stream while
    // dW_out runs; the backward recurrence joins it.  (Against the fused
    // dW_out's co-resident CTAs the collective only delays some of them: it
    // never waits on them, so the spin-waits resolve once it finishes.)
    DL_CUDA(cudaEventRecord(c->ev_dh, st));
    DL_CUDA(cudaStreamWaitEvent(c->st2, c->ev_dh, 0));
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->profiling) {
      a = ev_get(c);
      b = ev_get(c);
      DL_CUDA(cudaEventRecord(a, c->st2));
    }
    c->comm->reduce_scatter_sum(c->dh_all, c->dh_out, (size_t)(TB * H), DType::F32, c->st2);
    if (c->profiling) {
      DL_CUDA(cudaEventRecord(b, c->st2));
      c->pending.push_back({"vocab_exchange", {a, b}});
    }
    DL_CUDA(cudaEventRecord(c->ev_rs, c->st2));
  }
  if (dw_after_dh && !nce) {
    dw_out();
    after_dw();
  }
  if (late) fork_update(late_eta, c->w_out_bf);
  if (vs) {
    // each rank contracted its vocabulary block: dh_out = sum over ranks.
    // After this the backward recurrence, dW_rec and the W_in rows are
    // replicated computations on identical inputs.
    Phase p(c, "vocab_exchange");
    c->comm->allreduce_sum(c->dh_out, (size_t)(TB * H), DType::F32, st);
  } else if (dpv && !nce) {
    DL_CUDA(cudaStreamWaitEvent(st, c->ev_rs, 0));
  } else if (dpv) {
    Phase p(c, "vocab_exchange");
    c->comm->reduce_scatter_sum(c->dh_all, c->dh_out, (size_t)(TB * H), DType::F32, st);
  }
  // backward recurrence (backprop.hpp:197-219)
  {
    Phase p(c, "recurrence_bwd");
    const bool persist = tc(c) && c->rec_cluster &&
                         rec_window_tc(1, (int)T, (int)B, (int)H, c->act, c->dpre_bf, T * B,
                                       c->w_rec_bf, nullptr, nullptr, c->dh_out, c->htape,
                                       c->dpre, c->dpre_bf, c->bar_counter, st);
    if (persist) c->launches++;
    for (int64_t t = persist ? -1 : T - 1; t >= 0; --t) {
      float* dp_t = c->dpre + t * BH;
      bf16* dpb_t = tc(c) ? c->dpre_bf + t * BH : nullptr;
      int s = 0;
      if (t < T - 1 && tc(c) && c->rec_cluster) {
        rec_step_tc(1, (int)B, (int)H, c->act, c->dpre_bf + (t + 1) * BH, c->w_rec_bf, nullptr,
                    nullptr, c->dh_out + t * BH, c->htape + (t + 1) * BH, dp_t, dpb_t, st);
        c->launches++;
        continue;
      }
      if (t < T - 1) {
        s = pick_splits(c, (int)B, (int)H, (int)H);
        ensure_splitws(c, (size_t)s * BH);
        GemmDesc g = tc(c) ? desc((int)B, (int)H, (int)H, K_MAJOR, c->dpre_bf + (t + 1) * BH, H,
                                  MN_MAJOR, c->w_rec_bf, H, c->splitws, H)
                           : desc((int)B, (int)H, (int)H, K_MAJOR, c->dpre + (t + 1) * BH, H,
                                  MN_MAJOR, c->w_rec, H, c->splitws, H);
        g.k_splits = s;
        g.split_stride = BH;
        gemm(c, g);
      }
      rec_bwd(c->splitws, s, BH, BH, c->dh_out + t * BH, c->htape + (t + 1) * BH, c->act, dp_t,
              dpb_t, st);
      c->launches++;
    }
  }
  // dW_rec = sum_t dpre_t^T . h_t  [H x H] (backprop.hpp:214)
  {
    Phase p(c, "dw_rec");
    const int s = pick_splits(c, (int)H, (int)H, (int)TB, 16);
    ensure_splitws(c, (size_t)s * H * H);
    GemmDesc g = tc(c) ? desc((int)H, (int)H, (int)TB, MN_MAJOR, c->dpre_bf, H, MN_MAJOR,
                              c->htape_bf, H, c->splitws, H)
                       : desc((int)H, (int)H, (int)TB, MN_MAJOR, c->dpre, H, MN_MAJOR, c->htape, H,
                              c->splitws, H);
    g.k_splits = s;
    g.split_stride = H * H;
    gemm(c, g);
    // with the W_out update fused (a finite clip: nothing can be rejected)
    // the W_rec rmsprop step rides on the reduction pass (run_rmsprop skips it)
    c->rec_fused = fuse_eta > 0.0 && !dprec && tc(c) && std::isfinite(clip) && (H * H) % 4 == 0;
    if (c->rec_fused)
      reduce_rms_rec(c->splitws, s, H * H, H * H, c->g_rec, clip, c->w_rec, c->w_rec_bf, c->m_rec,
                     c->rho, c->eps, fuse_eta, st);
    else
      reduce_splits(c->splitws, s, H * H, H * H, c->g_rec, clip, dprec ? 0 : 1, c->nonfinite, st);
    c->launches++;
  }
  if (dprec) {
    // dW_rec: allreduce + clip.  W_in: allgather every rank's (ids, dpre) so
    // all ranks run the identical segmented sum over the global window in
    // the reference's order (t descending, global stream ascending).
    const int G = c->nranks;
    DL_CUDA(cudaEventRecord(c->ev_fork, st));
    DL_CUDA(cudaStreamWaitEvent(c->st2, c->ev_fork, 0));
    c->comm->allreduce_sum(c->g_rec, (size_t)(H * H), DType::F32, c->st2);
    reduce_splits(c->g_rec, 1, 0, H * H, c->g_rec, clip, 1, c->nonfinite, c->st2);
    c->comm->allgather(c->x_d, c->x_all, (size_t)TB, DType::U32, c->st2);
    c->comm->allgather(c->dpre, c->dpre_all, (size_t)(TB * H), DType::F32, c->st2);
    DL_CUDA(cudaEventRecord(c->ev_join, c->st2));
    DL_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));
    c->launches++;
    Phase p(c, "embed_grad");
    embed_grads(c->x_all, T, B, G, V, c->dpre_all, H, clip, c->ews, c->g_in_rows, c->g_in_words,
                c->g_in_n, c->nonfinite, st);
    c->launches += 3;
  } else {
    // W_in rows (rnn.hpp:218-222) -- deterministic segmented sum, clipped;
    // the id sort was forked at the start of the window
    DL_CUDA(cudaStreamWaitEvent(st, c->ev_sort_join, 0));
    Phase p(c, "embed_grad");
    embed_rows(TB, c->dpre, H, clip, c->ews, c->g_in_rows, c->g_in_n, c->nonfinite, st);
    c->launches += 2;
  }
  if (nce) {
    // sparse W_out rows: records by word in processing order, sum of
    // ds * h[t+1][b], clipped (SparseRowGrads, rnn.hpp:89-127, 155-162)
    Phase p(c, "nce_out_rows");
    NceRecs R{c->rec_word_d, c->rec_row_d, c->proc_r_d, c->ds_d, c->sort_keys_in,
              c->sort_vals_in, c->sort_keys_out, c->sort_vals_out, c->sort_head,
              c->sort_slot, c->sort_temp, c->sort_temp_bytes};
    nce_out_rows(R, c->nce_N, Vo, Hn, H, clip, c->nce_ws, c->nce_scale, c->g_out,
                 c->g_out_words, c->g_out_n, c->nonfinite, st);
    c->launches += 8;
  }
  // a non-finite dW_out block on one rank must skip the update everywhere
  // (only reachable with an infinite clip bound)
  if ((vs || dpv) && !std::isfinite(clip)) {
    if (fork_out_eta > 0.0) DL_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));
    c->comm->allreduce_sum(c->nonfinite, 1, DType::U32, st);
  }
  c->have_grads = true;
}

// rmsprop_update (rmsprop.hpp:113-133).  skip_out: the dense W_out part was
// already issued on the side stream by run_window (fork_out_eta).
void run_rmsprop(dl_ctx* c, double eta, int64_t TB, bool skip_out = false, bool count = true) {
  Phase p(c, "rmsprop");
  cudaStream_t st = c->st;
  if (!(skip_out && c->rec_fused))  // (else applied by the dW_rec reduction, run_window)
    rms_rec(c->w_rec, tc(c) ? c->w_rec_bf : nullptr, c->m_rec, c->g_rec, c->H * c->H, c->rho,
            c->eps, eta, c->nonfinite, st);
  if (c->in_decayed) {
    c->in_decayed = false;
    c->launches--;
  } else {
    rms_decay(c->m_in, c->V, c->rho, c->nonfinite, st);
  }
  rms_rows(c->w_in, nullptr, c->m_in, c->g_in_rows, c->g_in_words, c->g_in_n, TB, c->H, c->rho,
           c->eps, eta, 0, c->nonfinite, st);
  if (!skip_out && c->out_sparse) {
    // NCE: per-word-averaged sparse update of W_out (rmsprop.hpp:77-92, :129)
    rms_decay(c->m_out, c->Vo, c->rho, c->nonfinite, st);
    rms_rows(c->w_out, tc(c) ? c->w_out_bf : nullptr, c->m_out, c->g_out, c->g_out_words,
             c->g_out_n, c->Vo, c->H, c->rho, c->eps, eta, 0, c->nonfinite, st);
    c->launches += 2;
  } else if (!skip_out && c->dp16)
    rms_dense_g16c(c->w_out, c->w_out_bf, c->m_out, c->g_out_bf, c->Vo, c->H, c->dp16_clip,
                   c->rho, c->eps, eta, st);
  else if (!skip_out && c->g16_valid)
    rms_dense_g16(c->w_out, c->w_out_bf, c->m_out, c->g_out_bf, c->rowsq, c->rowsq_n, c->Vo, c->H,
                  c->rho, c->eps, eta, st);
  else if (!skip_out)
    rms_rows(c->w_out, tc(c) ? c->w_out_bf : nullptr, c->m_out, c->g_out, nullptr, nullptr, c->Vo,
             c->H, c->rho, c->eps, eta, 1, c->nonfinite, st);
  if (count) count_skip(c->nonfinite, c->d_skipped, st);
  c->launches += count ? 4 : 3;
}

float act0(int act) { return act == 0 ? 0.5f : 0.0f; }

// (Re)allocates the output-layer state for this context's Vo vocabulary
// rows: W_out and its shadows, m_out, dW_out (+ bf16 copy and row sums of
// squares), all zeroed.  Window buffers sized by Vo are dropped too.
void alloc_output(dl_ctx* c) {
  auto fr = [](auto*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  fr(c->w_out); fr(c->m_out); fr(c->g_out); fr(c->w_out_bf); fr(c->w_out_bf_next);
  fr(c->g_out_bf); fr(c->rowsq); fr(c->rms_cnt); fr(c->g_out_words); fr(c->g_out_n);
  const int64_t Vo = c->Vo, H = c->H;
  c->w_out = dalloc<float>(Vo * H);
  c->m_out = dalloc<float>(Vo);
  c->g_out = dalloc<float>(Vo * H);
  c->g_out_words = dalloc<uint32_t>(Vo);
  c->g_out_n = dalloc<int>(1);
  DL_CUDA(cudaMemsetAsync(c->w_out, 0, Vo * H * 4, c->st));
  DL_CUDA(cudaMemsetAsync(c->m_out, 0, Vo * 4, c->st));
  if (c->precision == DL_BF16) {
    c->w_out_bf = dalloc<bf16>(Vo * H);
    c->w_out_bf_next = dalloc<bf16>(Vo * H);
    c->g_out_bf = dalloc<bf16>(Vo * H);
    c->rowsq_n = tc_n_tiles((int)H);
    // (the fused dW_out epilogue writes 2 partials per 128-column tile)
    c->rowsq = dalloc<double>((size_t)std::max<int64_t>(c->rowsq_n, 2 * ((H + 127) / 128)) * Vo);
    c->rms_cnt = dalloc<unsigned>((Vo + 255) / 256);
  }
  c->fuse_cap = -1;
  c->capT = c->capB = 0;  // window buffers re-size on the next call
  fr(c->htape);
  c->have_grads = false;
  drop_graphs(c);
}

// Back to the full output layer (W_out zeroed: set the parameters again).
void reset_vshard(dl_ctx* c) {
  if (!c->vshard) return;
  c->vshard = false;
  c->dpv = false;
  c->Vo = c->V;
  c->v0 = 0;
  alloc_output(c);
  refresh_shadows(c);
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char* dl_last_error(const dl_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }
const char* dl_version(void) { return "desklm-b200 0.1 (sm_100a)"; }

int dl_create(dl_ctx** out, int device, int64_t V, int64_t H, int act, int precision) {
  if (!out) return fail(nullptr, DL_EINVAL, "dl_create: null out");
  *out = nullptr;
  if (V < 1 || H < 1) return fail(nullptr, DL_EINVAL, "RnnParams: V,H >= 1");
  if (act != DL_SIGMOID && act != DL_TANH) return fail(nullptr, DL_EINVAL, "bad activation");
  if (precision != DL_FP32 && precision != DL_BF16 && precision != DL_TF32X3)
    return fail(nullptr, DL_EINVAL, "bad precision");
  if (precision == DL_BF16 && ((H % 8) != 0 || (V % 8) != 0))
    return fail(nullptr, DL_EINVAL, "bf16 tensor-core mode needs V and H multiples of 8 (TMA)");
  dl_ctx* c = new dl_ctx();
  c->device = device;
  c->V = V;
  c->H = H;
  c->act = act;
  c->precision = precision;
  if (const char* e = std::getenv("DL_REC_CLUSTER")) c->rec_cluster = std::atoi(e) != 0;
  if (const char* e = std::getenv("DL_FORK_OUT")) c->fork_out = std::atoi(e) != 0;
  if (const char* e = std::getenv("DL_LOGITS_2CTA")) c->logits_pair = std::atoi(e) != 0;
  if (const char* e = std::getenv("DL_G16")) c->g16 = std::atoi(e) != 0;
  if (const char* e = std::getenv("DL_FUSE_OUT")) c->fuse_out = std::atoi(e) != 0;
  if (const char* e = std::getenv("DL_FORK_LATE")) c->fork_late = std::atoi(e) != 0;
  if (const char* e = std::getenv("DL_XF")) c->xf = std::atoi(e) != 0;
  if (const char* e = std::getenv("DL_PFAC")) c->pfac = std::atoi(e) != 0;
  c->tf32x3 = precision == DL_TF32X3;
  if (const char* e = std::getenv("DL_DP_CHUNKS")) c->dp_chunks = std::max(1, std::atoi(e));
  const int rc = guarded(c, [&] {
    int n = 0;
    DL_CUDA(cudaGetDeviceCount(&n));
    DL_REQUIRE(device >= 0 && device < n, DL_EINVAL, "dl_create: no such device");
    cudaDeviceProp prop;
    DL_CUDA(cudaGetDeviceProperties(&prop, device));
    DL_REQUIRE(prop.major == 10, DL_EDEVICE,
               "libdesklm_cuda is built for sm_100a (B200); device is sm_" +
                   std::to_string(prop.major * 10 + prop.minor));
    // main stream at the highest priority so the tensor-core GEMMs claim SMs
    // first; the side stream (bandwidth-bound W_out update) fills in
    int prio_lo = 0, prio_hi = 0;
    DL_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    DL_CUDA(cudaStreamCreateWithPriority(&c->st, cudaStreamNonBlocking, prio_hi));
    DL_CUDA(cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, prio_lo));
    DL_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    DL_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    DL_CUDA(cudaEventCreateWithFlags(&c->ev_sort_fork, cudaEventDisableTiming));
    DL_CUDA(cudaEventCreateWithFlags(&c->ev_sort_join, cudaEventDisableTiming));
    DL_CUDA(cudaEventCreateWithFlags(&c->ev_hfinal, cudaEventDisableTiming));
    DL_CUDA(cudaEventCreateWithFlags(&c->ev_dh, cudaEventDisableTiming));
    DL_CUDA(cudaEventCreateWithFlags(&c->ev_rs, cudaEventDisableTiming));
    c->w_in = dalloc<float>(V * H);
    c->w_rec = dalloc<float>(H * H);
    c->m_rec = dalloc<float>(H * H);
    c->m_in = dalloc<float>(V);
    c->g_rec = dalloc<float>(H * H);
    c->Vo = V;
    c->v0 = 0;
    alloc_output(c);
    c->g_in_n = dalloc<int>(1);
    // loss, positions and the non-finite flag side by side: a window's
    // results come back in one 24-byte copy
    c->d_loss = dalloc<double>(4);
    c->d_pos = reinterpret_cast<unsigned long long*>(c->d_loss + 1);
    c->nonfinite = reinterpret_cast<int*>(c->d_loss + 2);
    c->pf_repaired = reinterpret_cast<int*>(c->d_loss + 3);
    DL_CUDA(cudaMemsetAsync(c->d_loss + 3, 0, 8, c->st));
    c->d_skipped = dalloc<unsigned long long>(1);
    c->bar_counter = dalloc<unsigned>(256);  // rec_tc.cu kRecCounters
    c->win_loss = dalloc<double>(2);
    c->win_pos = reinterpret_cast<unsigned long long*>(c->win_loss + 1);
    c->win_counter = dalloc<int64_t>(1);
    if (precision == DL_BF16) c->w_rec_bf = dalloc<bf16>(H * H);
    DL_CUDA(cudaMemsetAsync(c->w_in, 0, V * H * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->w_rec, 0, H * H * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->m_rec, 0, H * H * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->m_in, 0, V * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->nonfinite, 0, 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->g_in_n, 0, 4, c->st));
    refresh_shadows(c);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
  if (rc != DL_OK) {
    g_err = c->err;
    dl_destroy(c);
    return rc;
  }
  *out = c;
  return DL_OK;
}

int dl_destroy(dl_ctx* c) {
  if (!c) return DL_OK;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  if (c->pf_repaired && std::getenv("DL_DEBUG")) {
    int n[2] = {0, 0};
    if (cudaMemcpy(n, c->pf_repaired, 8, cudaMemcpyDeviceToHost) == cudaSuccess)
      fprintf(stderr, "[desklm] shifted-exponential softmax: %d row(s) rescaled, %d with redone tiles\n",
              n[0], n[1]);
  }
  drop_graphs(c);
  delete c->comm;
  void* ptrs[] = {c->w_in, c->w_rec, c->w_out, c->w_rec_bf, c->w_out_bf, c->w_out_bf_next, c->m_rec, c->m_in,
                  c->m_out, c->g_rec, c->g_out, c->g_in_rows, c->g_in_words, c->g_in_n,
                  c->htape, c->htape_bf, c->x_d, c->y_d, c->w_d, c->S, c->part,
                  c->tgt_logit, c->loss_row, c->logp_row, c->dh_out, c->dpre, c->dpre_bf,
                  c->splitws, c->ews.seg_start, c->ews.order_pos, c->d_loss,
                  c->d_skipped, c->h0_d, c->ids, c->cursors, c->hidden, c->win_counter,
                  c->win_loss, c->x_all, c->dpre_all, c->bar_counter, c->g_out_bf,
                  c->hs_all_bf, c->hs_all, c->y_all, c->w_all, c->dh_all,
                  c->ln_kq_d, c->rec_word_d, c->rec_row_d, c->proc_r_d, c->score_d, c->ds_d,
                  c->nce_scale, c->loss_pos_d, c->sort_keys_in, c->sort_vals_in,
                  c->sort_keys_out, c->sort_vals_out, c->sort_head, c->sort_slot, c->sort_temp,
                  c->nce_ws.seg_start, c->nce_ws.order_pos, c->g_out_words, c->g_out_n,
                  c->nz_prob_d, c->nz_alias_d, c->raw_d, c->pos_of_d, c->first_d,
                  c->rowsq, c->tgt_loc, c->lse_loc, c->lse_all, c->rms_cnt, c->dS, c->xf_lse,
                  c->xf_sc, c->xpose_a, c->xpose_b, c->ng_y, c->ng_y_rb, c->ng_w, c->ng_w_rb,
                  c->ng_hs, c->ng_hs_rb, c->ng_dh};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  for (auto e : c->score_ev)
    if (e) cudaEventDestroy(e);
  if (c->ev_sort_fork) cudaEventDestroy(c->ev_sort_fork);
  if (c->ev_sort_join) cudaEventDestroy(c->ev_sort_join);
  if (c->ev_hfinal) cudaEventDestroy(c->ev_hfinal);
  if (c->ev_dh) cudaEventDestroy(c->ev_dh);
  if (c->ev_rs) cudaEventDestroy(c->ev_rs);
  for (int i = 0; i < 2; ++i) {
    if (c->raw_pin[i]) cudaFreeHost(c->raw_pin[i]);
    if (c->raw_ev[i]) cudaEventDestroy(c->raw_ev[i]);
  }
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
  return DL_OK;
}

int dl_set_params(dl_ctx* c, const float* w_in, const float* w_rec, const float* w_out) {
  if (!c || !w_in || !w_rec || !w_out) return fail(c, DL_EINVAL, "dl_set_params: null argument");
  return guarded(c, [&] {
    DL_CUDA(cudaMemcpyAsync(c->w_in, w_in, c->V * c->H * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaMemcpyAsync(c->w_rec, w_rec, c->H * c->H * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaMemcpyAsync(c->w_out, w_out + c->v0 * c->H, c->Vo * c->H * 4,
                            cudaMemcpyHostToDevice, c->st));
    refresh_shadows(c);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_get_params(dl_ctx* c, float* w_in, float* w_rec, float* w_out) {
  if (!c) return fail(c, DL_EINVAL, "dl_get_params: null ctx");
  return guarded(c, [&] {
    if (w_in) DL_CUDA(cudaMemcpyAsync(w_in, c->w_in, c->V * c->H * 4, cudaMemcpyDeviceToHost, c->st));
    if (w_rec) DL_CUDA(cudaMemcpyAsync(w_rec, c->w_rec, c->H * c->H * 4, cudaMemcpyDeviceToHost, c->st));
    if (w_out)
      DL_CUDA(cudaMemcpyAsync(w_out + c->v0 * c->H, c->w_out, c->Vo * c->H * 4,
                              cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_set_opt(dl_ctx* c, const float* m_rec, const float* m_in, const float* m_out, double rho,
               double eps) {
  if (!c) return fail(c, DL_EINVAL, "dl_set_opt: null ctx");
  if (!(rho > 0.0 && rho < 1.0)) return fail(c, DL_EINVAL, "rmsprop: rho must be in (0,1)");
  if (!(eps > 0.0)) return fail(c, DL_EINVAL, "rmsprop: eps must be > 0");
  return guarded(c, [&] {
    c->rho = rho;
    c->eps = eps;
    if (m_rec) DL_CUDA(cudaMemcpyAsync(c->m_rec, m_rec, c->H * c->H * 4, cudaMemcpyHostToDevice, c->st));
    if (m_in) DL_CUDA(cudaMemcpyAsync(c->m_in, m_in, c->V * 4, cudaMemcpyHostToDevice, c->st));
    if (m_out)
      DL_CUDA(cudaMemcpyAsync(c->m_out, m_out + c->v0, c->Vo * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
    drop_graphs(c);
  });
}

int dl_get_opt(dl_ctx* c, float* m_rec, float* m_in, float* m_out) {
  if (!c) return fail(c, DL_EINVAL, "dl_get_opt: null ctx");
  return guarded(c, [&] {
    if (m_rec) DL_CUDA(cudaMemcpyAsync(m_rec, c->m_rec, c->H * c->H * 4, cudaMemcpyDeviceToHost, c->st));
    if (m_in) DL_CUDA(cudaMemcpyAsync(m_in, c->m_in, c->V * 4, cudaMemcpyDeviceToHost, c->st));
    if (m_out)
      DL_CUDA(cudaMemcpyAsync(m_out + c->v0, c->m_out, c->Vo * 4, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

namespace {
bool fuse_ok(dl_ctx* c, double clip);
}

namespace {
// dl_window / dl_train_window: validate, stage the window's host arrays
// through pinned memory, run the window (+ the update when eta > 0), read
// back loss, positions, h_final and the update's verdict.
// dl_train_window's window (bptt_run + rmsprop_update) replayed from one
// CUDA graph: the ~20 kernel launches, events and copies of a window cost
// ~370 us of host time per call (measured at V = 1,000, H = 128, where the
// device work is tiny), which a synchronous per-window API exposes.  The
// graph holds the H2D copies of the window (from its own page-locked
// staging), the device work, the results' D2H and h_final's D2H on the side
// stream; per call the copies' host ends are re-pointed at the caller's
// page-locked buffers (pageable ones go through the staging), then one
// launch and one synchronize.
void presize(dl_ctx* c, int64_t T, int64_t B);

bool tw_graph_ok(dl_ctx* c) {
  static const bool on = [] {
    const char* e = std::getenv("DL_TW_GRAPH");
    if (e && std::atoi(e) == 0) return false;
    return std::getenv("DL_GEMM_TRACE") == nullptr && std::getenv("DL_REC_TRACE") == nullptr;
  }();
  return on && c->use_graph && !c->profiling && c->comm == nullptr && c->loss_mode != 0;
}

void train_window_graph(dl_ctx* c, int64_t T, int64_t B, const uint32_t* inputs,
                        const uint32_t* targets, const uint8_t* weights, const float* h0,
                        float* h_final, double loss_scale, float clip, double eta, double* loss,
                        uint64_t* positions, int* applied) {
  const int64_t TB = T * B, BH = B * c->H;
  const bool fuse = fuse_ok(c, clip);
  // staging layout: x | y | w | h0 | h_final | results
  const size_t o_y = TB * 4, o_w = 2 * TB * 4, o_h0 = ((TB * 9 + 15) / 16) * 16,
               o_hf = o_h0 + BH * 4, o_res = o_hf + BH * 4, bytes = o_res + 64;
  auto& g = c->tw;
  if (!g.e || g.T != T || g.B != B || g.scale != loss_scale || g.clip != clip || g.eta != eta ||
      g.fuse != fuse) {
    drop_graphs(c);  // (also any trainer graph: they share the window buffers)
    presize(c, T, B);  // (no allocation inside the capture)
    DL_CUDA(cudaMallocHost(&g.pin, bytes));
    uint8_t* pin = g.pin;
    const uint64_t before = c->launches.load();
    DL_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    try {
      DL_CUDA(cudaMemcpyAsync(c->x_d, pin, TB * 4, cudaMemcpyHostToDevice, c->st));
      DL_CUDA(cudaMemcpyAsync(c->y_d, pin + o_y, TB * 4, cudaMemcpyHostToDevice, c->st));
      DL_CUDA(cudaMemcpyAsync(c->w_d, pin + o_w, TB, cudaMemcpyHostToDevice, c->st));
      DL_CUDA(cudaMemcpyAsync(c->htape, pin + o_h0, BH * 4, cudaMemcpyHostToDevice, c->st));
      DL_CUDA(cudaMemsetAsync(c->d_loss, 0, 16, c->st));
      run_window(c, T, B, loss_scale, clip, true, 0.0, fuse ? eta : 0.0);
      run_rmsprop(c, eta, TB * dp_ranks(c), /*skip_out=*/fuse);
      DL_CUDA(cudaMemcpyAsync(pin + o_res, c->d_loss, 20, cudaMemcpyDeviceToHost, c->st));
      DL_CUDA(cudaStreamWaitEvent(c->st2, c->ev_hfinal, 0));
      DL_CUDA(cudaMemcpyAsync(pin + o_hf, c->htape + T * BH, BH * 4, cudaMemcpyDeviceToHost,
                              c->st2));
      DL_CUDA(cudaEventRecord(c->ev_join, c->st2));
      DL_CUDA(cudaStreamWaitEvent(c->st, c->ev_join, 0));
    } catch (...) {
      cudaGraph_t junk;
      cudaStreamEndCapture(c->st, &junk);
      if (junk) cudaGraphDestroy(junk);
      throw;
    }
    DL_CUDA(cudaStreamEndCapture(c->st, &g.g));
    g.launches = c->launches.load() - before;
    c->launches -= g.launches;  // counted when replayed
    // the copy nodes whose host ends move per call
    size_t nn = 0;
    DL_CUDA(cudaGraphGetNodes(g.g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    DL_CUDA(cudaGraphGetNodes(g.g, nodes.data(), &nn));
    for (cudaGraphNode_t n : nodes) {
      cudaGraphNodeType ty;
      DL_CUDA(cudaGraphNodeGetType(n, &ty));
      if (ty != cudaGraphNodeTypeMemcpy) continue;
      cudaMemcpy3DParms mp{};
      DL_CUDA(cudaGraphMemcpyNodeGetParams(n, &mp));
      const void* hp = mp.kind == cudaMemcpyHostToDevice ? mp.srcPtr.ptr : mp.dstPtr.ptr;
      if (hp == pin) g.nx = n;
      else if (hp == pin + o_y) g.ny = n;
      else if (hp == pin + o_w) g.nw = n;
      else if (hp == pin + o_h0) g.nh0 = n;
      else if (hp == pin + o_hf) g.nhf = n;
    }
    DL_REQUIRE(g.nx && g.ny && g.nw && g.nh0 && g.nhf, DL_EDEVICE,
               "internal: train-window graph copy nodes not found");
    DL_CUDA(cudaGraphInstantiate(&g.e, g.g, 0));
    g.T = T; g.B = B; g.scale = loss_scale; g.clip = clip; g.eta = eta; g.fuse = fuse;
  }
  uint8_t* pin = g.pin;
  auto h2d = [&](cudaGraphNode_t n, void* dst, const void* src, size_t nb, size_t off) {
    if (!is_pinned(src)) {
      std::memcpy(pin + off, src, nb);
      src = pin + off;
    }
    DL_CUDA(cudaGraphExecMemcpyNodeSetParams1D(g.e, n, dst, src, nb, cudaMemcpyHostToDevice));
  };
  h2d(g.nx, c->x_d, inputs, TB * 4, 0);
  h2d(g.ny, c->y_d, targets, TB * 4, o_y);
  h2d(g.nw, c->w_d, weights, TB, o_w);
  h2d(g.nh0, c->htape, h0, BH * 4, o_h0);
  const bool hf_direct = h_final && is_pinned(h_final);
  DL_CUDA(cudaGraphExecMemcpyNodeSetParams1D(g.e, g.nhf, hf_direct ? (void*)h_final : pin + o_hf,
                                             c->htape + T * BH, BH * 4, cudaMemcpyDeviceToHost));
  DL_CUDA(cudaGraphLaunch(g.e, c->st));
  c->launches += g.launches;
  DL_CUDA(cudaStreamSynchronize(c->st));
  if (h_final && !hf_direct) std::memcpy(h_final, pin + o_hf, BH * 4);
  struct { double l; unsigned long long p; int bad; int pad; } res;
  std::memcpy(&res, pin + o_res, 20);
  if (loss) *loss = res.l;
  if (positions) *positions = res.p;
  if (applied) *applied = res.bad ? 0 : 1;
  c->capT = std::max(c->capT, T);
}

int window_call(dl_ctx* c, const char* who, int64_t T, int64_t B, const uint32_t* inputs,
                const uint32_t* targets, const uint8_t* weights, const float* h0,
                float* h_final, double loss_scale, float clip, bool grads, double eta,
                double* loss, uint64_t* positions, int* applied) {
  if (!c) return fail(c, DL_EINVAL, std::string(who) + ": null ctx");
  if (T < 1 || B < 1) return fail(c, DL_EINVAL, "bptt: empty window");
  if (!inputs || !targets || !weights || !h0) return fail(c, DL_EINVAL, "bptt: null window arrays");
  if (eta > 0.0 || applied) {
    if (!(eta > 0.0)) return fail(c, DL_EINVAL, "config: eta must be > 0");
  }
  for (int64_t i = 0; i < T * B; ++i)
    if (inputs[i] >= (uint64_t)c->V || targets[i] >= (uint64_t)c->V)
      return fail(c, DL_EINVAL, "bptt: word id out of range");
  if (c->loss_mode == 0 && c->comm)
    return fail(c, DL_EINVAL, "NCE mode: multi-rank windows are not supported");
  return guarded(c, [&] {
    ensure_window(c, T, B);
    if (eta > 0.0 && tw_graph_ok(c)) {
      train_window_graph(c, T, B, inputs, targets, weights, h0, h_final, loss_scale, clip, eta,
                         loss, positions, applied);
      return;
    }
    if (c->loss_mode == 0) nce_prepare(c, T, B, weights, /*predraw=*/true);
    const int64_t TB = T * B, BH = B * c->H;
    // H2D of the window: page-locked caller buffers are copied from directly,
    // pageable ones through one pinned staging buffer
    const size_t bytes = TB * 4 * 2 + TB + BH * 4 + 64;
    uint8_t* pin = static_cast<uint8_t*>(ensure_pinned(c, std::max<size_t>(bytes, BH * 4 + 64)));
    auto h2d = [&](void* dst, const void* src, size_t n, size_t off) {
      if (!is_pinned(src)) {
        std::memcpy(pin + off, src, n);
        src = pin + off;
      }
      DL_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, c->st));
    };
    h2d(c->x_d, inputs, TB * 4, 0);
    h2d(c->y_d, targets, TB * 4, TB * 4);
    h2d(c->w_d, weights, TB, TB * 8);
    h2d(c->htape, h0, BH * 4, ((TB * 9 + 15) / 16) * 16);
    DL_CUDA(cudaMemsetAsync(c->d_loss, 0, 8, c->st));
    DL_CUDA(cudaMemsetAsync(c->d_pos, 0, 8, c->st));
    if (eta > 0.0) {
      // Trainer::run_epoch's bptt_run + update (trainer.hpp:391-397)
      const bool fuse = c->loss_mode != 0 && fuse_ok(c, clip);
      run_window(c, T, B, loss_scale, clip, true, 0.0, fuse ? eta : 0.0);
      run_rmsprop(c, eta, TB * dp_ranks(c), /*skip_out=*/fuse);
    } else {
      run_window(c, T, B, loss_scale, clip, grads);
    }
    // (NCE: the next window's draws on the host while the device runs this
    // one; before the D2H below, which blocks until the window is done)
    if (c->loss_mode == 0) nce_predraw(c, T, B);
    // loss, positions, non-finite flag: adjacent on the device (dl_create)
    struct { double l; unsigned long long p; int bad; int pad; } res{};
    static_assert(sizeof(res) == 24, "result block layout");
    DL_CUDA(cudaMemcpyAsync(&res, c->d_loss, eta > 0.0 ? 20 : 16, cudaMemcpyDeviceToHost, c->st));
    // h_final is final after the forward recurrence: its D2H runs on the
    // side stream, under the rest of the window
    if (h_final) {
      DL_CUDA(cudaStreamWaitEvent(c->st2, c->ev_hfinal, 0));
      DL_CUDA(cudaMemcpyAsync(h_final, c->htape + T * BH, BH * 4, cudaMemcpyDeviceToHost,
                              c->st2));
    }
    DL_CUDA(cudaStreamSynchronize(c->st));
    DL_CUDA(cudaStreamSynchronize(c->st2));
    prof_collect(c);
    if (loss) *loss = res.l;
    if (positions) *positions = res.p;
    if (applied) *applied = res.bad ? 0 : 1;
    c->capT = std::max(c->capT, T);
  });
}
}  // namespace

int dl_window(dl_ctx* c, int64_t T, int64_t B, const uint32_t* inputs, const uint32_t* targets,
              const uint8_t* weights, const float* h0, float* h_final, double loss_scale,
              float clip, int compute_grads, double* loss, uint64_t* positions) {
  return window_call(c, "dl_window", T, B, inputs, targets, weights, h0, h_final, loss_scale,
                     clip, compute_grads != 0, 0.0, loss, positions, nullptr);
}

int dl_train_window(dl_ctx* c, int64_t T, int64_t B, const uint32_t* inputs,
                    const uint32_t* targets, const uint8_t* weights, const float* h0,
                    float* h_final, double loss_scale, float clip, double eta, double* loss,
                    uint64_t* positions, int* applied) {
  if (!(eta > 0.0)) return fail(c, DL_EINVAL, "config: eta must be > 0");
  return window_call(c, "dl_train_window", T, B, inputs, targets, weights, h0, h_final,
                     loss_scale, clip, true, eta, loss, positions, applied);
}

int dl_get_grads(dl_ctx* c, float* g_in_dense, float* g_rec, float* g_out) {
  if (!c) return fail(c, DL_EINVAL, "dl_get_grads: null ctx");
  if (!c->have_grads) return fail(c, DL_EINVAL, "dl_get_grads: no gradients computed yet");
  return guarded(c, [&] {
    if (g_in_dense) {
      float* dense = dalloc<float>(c->V * c->H);
      DL_CUDA(cudaMemsetAsync(dense, 0, c->V * c->H * 4, c->st));
      embed_dense(c->g_in_rows, c->g_in_words, c->g_in_n, c->capT * c->capB, c->H, dense, c->st);
      DL_CUDA(cudaMemcpyAsync(g_in_dense, dense, c->V * c->H * 4, cudaMemcpyDeviceToHost, c->st));
      DL_CUDA(cudaStreamSynchronize(c->st));
      cudaFree(dense);
    }
    if (g_rec) DL_CUDA(cudaMemcpyAsync(g_rec, c->g_rec, c->H * c->H * 4, cudaMemcpyDeviceToHost, c->st));
    if (g_out && c->out_sparse) {
      // NCE: the sparse rows scattered into the dense layout (to_dense)
      float* dense = dalloc<float>(c->Vo * c->H);
      DL_CUDA(cudaMemsetAsync(dense, 0, c->Vo * c->H * 4, c->st));
      embed_dense(c->g_out, c->g_out_words, c->g_out_n, c->Vo, c->H, dense, c->st);
      DL_CUDA(cudaMemcpyAsync(g_out + c->v0 * c->H, dense, c->Vo * c->H * 4,
                              cudaMemcpyDeviceToHost, c->st));
      DL_CUDA(cudaStreamSynchronize(c->st));
      cudaFree(dense);
    } else if (g_out && (c->g16_valid || c->dp16)) {
      // bf16 gradient of the throughput path, widened on the host (the
      // data-parallel one is the unclipped rank sum: clipped here as the
      // update kernel does, rnn.hpp:131-134)
      std::vector<uint16_t> tmp((size_t)(c->Vo * c->H));
      DL_CUDA(cudaMemcpyAsync(tmp.data(), c->g_out_bf, tmp.size() * 2, cudaMemcpyDeviceToHost,
                              c->st));
      DL_CUDA(cudaStreamSynchronize(c->st));
      float* dst = g_out + c->v0 * c->H;
      for (size_t i = 0; i < tmp.size(); ++i) {
        const uint32_t u = (uint32_t)tmp[i] << 16;
        std::memcpy(&dst[i], &u, 4);
        if (c->dp16) dst[i] = std::min(c->dp16_clip, std::max(-c->dp16_clip, dst[i]));
      }
    } else if (g_out) {
      DL_CUDA(cudaMemcpyAsync(g_out + c->v0 * c->H, c->g_out, c->Vo * c->H * 4,
                              cudaMemcpyDeviceToHost, c->st));
    }
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_set_grads(dl_ctx* c, int64_t n_in_rows, const uint32_t* in_words, const float* in_rows,
                 const float* g_rec, const float* g_out) {
  if (!c || !g_rec || !g_out || (n_in_rows > 0 && (!in_words || !in_rows)))
    return fail(c, DL_EINVAL, "dl_set_grads: null argument");
  if (n_in_rows < 0) return fail(c, DL_EINVAL, "dl_set_grads: bad row count");
  for (int64_t i = 0; i < n_in_rows; ++i)
    if (in_words[i] >= (uint64_t)c->V) return fail(c, DL_EINVAL, "dl_set_grads: word out of range");
  return guarded(c, [&] {
    if (n_in_rows > c->capT * c->capB) ensure_window(c, n_in_rows, 1);
    const int n = (int)n_in_rows;
    DL_CUDA(cudaMemcpyAsync(c->g_in_n, &n, 4, cudaMemcpyHostToDevice, c->st));
    if (n_in_rows > 0) {
      DL_CUDA(cudaMemcpyAsync(c->g_in_words, in_words, n_in_rows * 4, cudaMemcpyHostToDevice, c->st));
      DL_CUDA(cudaMemcpyAsync(c->g_in_rows, in_rows, n_in_rows * c->H * 4, cudaMemcpyHostToDevice, c->st));
    }
    DL_CUDA(cudaMemcpyAsync(c->g_rec, g_rec, c->H * c->H * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaMemcpyAsync(c->g_out, g_out + c->v0 * c->H, c->Vo * c->H * 4,
                            cudaMemcpyHostToDevice, c->st));
    // finite check of the injected gradients (rmsprop.hpp:116 / rnn.hpp:165-171)
    int bad = 0;
    auto fin = [&](const float* p, int64_t k) {
      for (int64_t i = 0; i < k; ++i)
        if (!std::isfinite(p[i])) return false;
      return true;
    };
    bad = !(fin(g_rec, c->H * c->H) && fin(g_out, c->V * c->H) &&
            (n_in_rows == 0 || fin(in_rows, n_in_rows * c->H)));
    DL_CUDA(cudaMemcpyAsync(c->nonfinite, &bad, 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
    c->have_grads = true;
    c->g16_valid = false;  // injected gradients are fp32
    c->dp16 = false;
  });
}

int dl_rmsprop(dl_ctx* c, double eta, int* applied) {
  if (!c) return fail(c, DL_EINVAL, "dl_rmsprop: null ctx");
  if (!c->have_grads) return fail(c, DL_EINVAL, "dl_rmsprop: no gradients computed yet");
  return guarded(c, [&] {
    run_rmsprop(c, eta, c->capT * c->capB * dp_ranks(c));
    int bad = 0;
    DL_CUDA(cudaMemcpyAsync(&bad, c->nonfinite, 4, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
    prof_collect(c);
    if (applied) *applied = bad ? 0 : 1;
  });
}

int dl_score(dl_ctx* c, int64_t S, int64_t steps, const uint32_t* in, const int64_t* tgt,
             const float* h0, float* h_final, double* logp, double* total_logprob,
             uint64_t* predicted) {
  if (!c) return fail(c, DL_EINVAL, "dl_score: null ctx");
  if (S < 1 || steps < 0) return fail(c, DL_EINVAL, "dl_score: bad shape");
  for (int64_t i = 0; i < S * steps; ++i) {
    if (in[i] >= (uint64_t)c->V) return fail(c, DL_EDATA, "score: id out of vocabulary range");
    if (tgt[i] >= c->V) return fail(c, DL_EDATA, "score: id out of vocabulary range");
  }
  return guarded(c, [&] {
    const int64_t H = c->H, SH = S * H;
    // bank several steps per logits GEMM (eval.hpp:45 kScoreBank idea)
    // (16,384 rows per logits GEMM: 2 GB of bf16 logits at V = 64,000 --
    // fewer host synchronisations per scored word)
    int64_t bank = std::max<int64_t>(1, std::min<int64_t>(steps, 16384 / S));
    if (bank < 1) bank = 1;
    ensure_window(c, bank, S);
    std::vector<double> lp(S * steps, NAN);
    // two page-locked slots (ids, targets, mask, log-probs per bank): the
    // host prepares bank j + 1 and scatters bank j - 1's log-probs while the
    // device runs bank j -- no synchronisation inside the walk
    const int64_t BS = bank * S;
    const size_t slot_bytes = ((BS * 4 + 15) / 16) * 16 * 2 + ((BS + 15) / 16) * 16 + BS * 8;
    uint8_t* pin = static_cast<uint8_t*>(ensure_pinned(c, 2 * slot_bytes + 64));
    auto slot_x = [&](int k) { return reinterpret_cast<uint32_t*>(pin + k * slot_bytes); };
    auto slot_y = [&](int k) {
      return reinterpret_cast<uint32_t*>(pin + k * slot_bytes + ((BS * 4 + 15) / 16) * 16);
    };
    auto slot_w = [&](int k) { return pin + k * slot_bytes + ((BS * 4 + 15) / 16) * 16 * 2; };
    auto slot_lp = [&](int k) {
      return reinterpret_cast<double*>(pin + k * slot_bytes + ((BS * 4 + 15) / 16) * 16 * 2 +
                                       ((BS + 15) / 16) * 16);
    };
    for (int k = 0; k < 2; ++k)
      if (!c->score_ev[k]) DL_CUDA(cudaEventCreateWithFlags(&c->score_ev[k], cudaEventDisableTiming));
    int64_t pend_j0[2] = {-1, -1}, pend_nb[2] = {0, 0};
    auto drain = [&](int k) {  // bank in slot k done: scatter its log-probs
      if (pend_j0[k] < 0) return;
      DL_CUDA(cudaEventSynchronize(c->score_ev[k]));
      const uint8_t* wk = slot_w(k);
      const double* lk = slot_lp(k);
      for (int64_t i = 0; i < pend_nb[k] * S; ++i)
        if (wk[i]) lp[pend_j0[k] * S + i] = lk[i];
      pend_j0[k] = -1;
    };
    // initial state
    if (h0) DL_CUDA(cudaMemcpyAsync(c->htape, h0, SH * 4, cudaMemcpyHostToDevice, c->st));
    else fill_f32(c->htape, act0(c->act), SH, c->st);
    int k = 0;
    for (int64_t j0 = 0; j0 < steps; j0 += bank, k ^= 1) {
      const int64_t nb = std::min(bank, steps - j0);
      drain(k);  // (its bank two back: long finished while this one was prepared)
      uint32_t* xk = slot_x(k);
      uint32_t* yk = slot_y(k);
      uint8_t* wk = slot_w(k);
      std::memcpy(xk, in + j0 * S, nb * S * 4);
      bool any = false;
      for (int64_t i = 0; i < nb * S; ++i) {
        const int64_t t = tgt[j0 * S + i];
        yk[i] = t >= 0 ? (uint32_t)t : 0u;
        wk[i] = t >= 0 ? 1 : 0;
        any |= t >= 0;
      }
      DL_CUDA(cudaMemcpyAsync(c->x_d, xk, nb * S * 4, cudaMemcpyHostToDevice, c->st));
      DL_CUDA(cudaMemcpyAsync(c->y_d, yk, nb * S * 4, cudaMemcpyHostToDevice, c->st));
      DL_CUDA(cudaMemcpyAsync(c->w_d, wk, nb * S, cudaMemcpyHostToDevice, c->st));
      if (tc(c)) f32_to_bf16(c->htape, c->htape_bf, SH, c->st);
      {
        Phase p(c, "recurrence_fwd");
        for (int64_t t = 0; t < nb; ++t)
          rec_step_fwd(c, S, c->htape + t * SH, tc(c) ? c->htape_bf + t * SH : nullptr,
                       c->x_d + t * S, c->htape + (t + 1) * SH,
                       tc(c) ? c->htape_bf + (t + 1) * SH : nullptr);
      }
      if (any)
        output_layer(c, nb * S, c->htape + SH, tc(c) ? c->htape_bf + SH : nullptr, c->y_d, c->w_d,
                     1.0, false, nullptr, c->logp_row);
      // carry the last state to slot 0 for the next bank
      DL_CUDA(cudaMemcpyAsync(c->htape, c->htape + nb * SH, SH * 4, cudaMemcpyDeviceToDevice, c->st));
      if (any) {
        DL_CUDA(cudaMemcpyAsync(slot_lp(k), c->logp_row, nb * S * 8, cudaMemcpyDeviceToHost, c->st));
        DL_CUDA(cudaEventRecord(c->score_ev[k], c->st));
        pend_j0[k] = j0;
        pend_nb[k] = nb;
      }
    }
    drain(0);
    drain(1);
    if (h_final) DL_CUDA(cudaMemcpyAsync(h_final, c->htape, SH * 4, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
    prof_collect(c);
    double tot = 0.0;
    uint64_t pred = 0;
    for (int64_t i = 0; i < S * steps; ++i)
      if (tgt[i] >= 0) {
        tot += lp[i];
        ++pred;
      }
    if (logp) std::memcpy(logp, lp.data(), sizeof(double) * S * steps);
    if (total_logprob) *total_logprob = tot;
    if (predicted) *predicted = pred;
  });
}

int dl_sharded_perplexity(dl_ctx* c, const uint32_t* ids, int64_t n, int shards, uint32_t bos,
                          double* total_logprob, uint64_t* predicted, double* perplexity) {
  if (!c) return fail(c, DL_EINVAL, "dl_sharded_perplexity: null ctx");
  if (n < 2) return fail(c, DL_EINVAL, "sharded perplexity: stream too short");
  if (shards < 1) return fail(c, DL_EINVAL, "sharded perplexity: shards must be >= 1");
  // eval.hpp:160-195: S = min(shards, n/2) slices begin = s*n/S walked cold
  const int64_t S = std::min<int64_t>(shards, n / 2);
  std::vector<int64_t> begin(S + 1);
  for (int64_t s = 0; s <= S; ++s) begin[s] = s * n / S;
  int64_t max_len = 0;
  for (int64_t s = 0; s < S; ++s) max_len = std::max(max_len, begin[s + 1] - begin[s]);
  const int64_t steps = std::max<int64_t>(0, max_len - 1);
  std::vector<uint32_t> in(S * steps);
  std::vector<int64_t> tg(S * steps);
  for (int64_t j = 0; j < steps; ++j)
    for (int64_t s = 0; s < S; ++s) {
      const int64_t len = begin[s + 1] - begin[s];
      if (j + 1 < len) {
        const uint32_t x = ids[begin[s] + j], y = ids[begin[s] + j + 1];
        if (x >= (uint64_t)c->V || y >= (uint64_t)c->V)
          return fail(c, DL_EDATA, "sharded perplexity: id out of vocabulary range");
        in[j * S + s] = x;
        tg[j * S + s] = y == bos ? -1 : (int64_t)y;
      } else {
        in[j * S + s] = 0;
        tg[j * S + s] = -1;
      }
    }
  double tot = 0.0;
  uint64_t pred = 0;
  const int rc = dl_score(c, S, steps, in.data(), tg.data(), nullptr, nullptr, nullptr, &tot, &pred);
  if (rc != DL_OK) return rc;
  if (pred == 0) return fail(c, DL_EINVAL, "sharded perplexity: no predicted tokens");
  if (total_logprob) *total_logprob = tot;
  if (predicted) *predicted = pred;
  if (perplexity) *perplexity = std::exp(-tot / (double)pred);
  return DL_OK;
}

int dl_rnn_perplexity(dl_ctx* c, const uint32_t* ids, int64_t n, uint32_t bos,
                      double* total_logprob, uint64_t* predicted, double* perplexity) {
  if (!c) return fail(c, DL_EINVAL, "dl_rnn_perplexity: null ctx");
  if (n < 2) return fail(c, DL_EINVAL, "rnn perplexity: stream too short");
  // eval.hpp:123-137: one stream, every token is input; non-bos targets scored
  std::vector<int64_t> tg(n - 1);
  for (int64_t i = 0; i + 1 < n; ++i) {
    if (ids[i] >= (uint64_t)c->V || ids[i + 1] >= (uint64_t)c->V)
      return fail(c, DL_EDATA, "rnn perplexity: id out of vocabulary range");
    tg[i] = ids[i + 1] == bos ? -1 : (int64_t)ids[i + 1];
  }
  double tot = 0.0;
  uint64_t pred = 0;
  const int rc = dl_score(c, 1, n - 1, ids, tg.data(), nullptr, nullptr, nullptr, &tot, &pred);
  if (rc != DL_OK) return rc;
  if (pred == 0) return fail(c, DL_EINVAL, "rnn perplexity: no predicted tokens");
  if (total_logprob) *total_logprob = tot;
  if (predicted) *predicted = pred;
  if (perplexity) *perplexity = std::exp(-tot / (double)pred);
  return DL_OK;
}

// ln_z_samples (eval.hpp:805-857): one pass over the stream with the state
// carried across sentences; after reading ids[i] with i % stride == 0 the
// state's log partition function ln Z = lse_w(s_w) is recorded, stride =
// max(1, n / count), until count states are taken.  The recurrence runs in
// banks on the device; the sampled states come back to the host and go
// through the logits GEMM + block log-sum-exp in chunks.
int dl_ln_z_samples(dl_ctx* c, const uint32_t* ids, int64_t n, int64_t count, double* out,
                    int64_t* n_out) {
  if (!c) return fail(c, DL_EINVAL, "dl_ln_z_samples: null ctx");
  if (!ids || n < 1 || count < 1) return fail(c, DL_EINVAL, "ln Z samples: empty stream or zero count");
  if (c->vshard) return fail(c, DL_EINVAL, "ln Z samples: not on a vocabulary-sharded context");
  const int64_t stride = std::max<int64_t>(1, n / count);
  std::vector<int64_t> pos;
  int64_t steps = 0;
  for (int64_t i = 0; i < n && (int64_t)pos.size() < count; ++i) {
    if (ids[i] >= (uint64_t)c->V) return fail(c, DL_EDATA, "ln Z samples: id out of vocabulary range");
    steps = i + 1;
    if (i % stride == 0) pos.push_back(i);
  }
  return guarded(c, [&] {
    const int64_t H = c->H, V = c->Vo;
    const int64_t bank = std::min<int64_t>(steps, 4096);
    ensure_window(c, bank, 1);
    cudaStream_t st = c->st;
    fill_f32(c->htape, act0(c->act), H, st);
    std::vector<float> states(pos.size() * H);
    size_t k = 0;
    for (int64_t j0 = 0; j0 < steps; j0 += bank) {
      const int64_t nb = std::min(bank, steps - j0);
      DL_CUDA(cudaMemcpyAsync(c->x_d, ids + j0, nb * 4, cudaMemcpyHostToDevice, st));
      if (tc(c)) f32_to_bf16(c->htape, c->htape_bf, H, st);
      for (int64_t t = 0; t < nb; ++t)
        rec_step_fwd(c, 1, c->htape + t * H, tc(c) ? c->htape_bf + t * H : nullptr, c->x_d + t,
                     c->htape + (t + 1) * H, tc(c) ? c->htape_bf + (t + 1) * H : nullptr);
      while (k < pos.size() && pos[k] < j0 + nb) {
        DL_CUDA(cudaMemcpyAsync(states.data() + k * H, c->htape + (pos[k] - j0 + 1) * H, H * 4,
                                cudaMemcpyDeviceToHost, st));
        ++k;
      }
      DL_CUDA(cudaMemcpyAsync(c->htape, c->htape + nb * H, H * 4, cudaMemcpyDeviceToDevice, st));
      DL_CUDA(cudaStreamSynchronize(st));
    }
    // ln Z of the sampled states, `bank` rows at a time (softmax_scores_t +
    // lse_column, eval.hpp:829-837)
    const int64_t ns = (int64_t)pos.size();
    DL_CUDA(cudaMemsetAsync(c->y_d, 0xff, bank * 4, st));  // no target column
    for (int64_t r0 = 0; r0 < ns; r0 += bank) {
      const int64_t M = std::min(bank, ns - r0);
      DL_CUDA(cudaMemcpyAsync(c->htape, states.data() + r0 * H, M * H * 4, cudaMemcpyHostToDevice,
                              st));
      if (tc(c)) {
        f32_to_bf16(c->htape, c->htape_bf, M * H, st);
        GemmDesc g = desc((int)M, (int)V, (int)H, K_MAJOR, c->htape_bf, H, K_MAJOR, c->w_out_bf, H,
                          nullptr, 0);
        g.logits = 1;
        g.S = nullptr;
        g.lds = V;
        g.part = c->part;
        g.part_n = c->part_tiles;
        g.tgt = c->y_d;
        g.tgt_logit = c->tgt_logit;
        g.no_pair = c->logits_pair ? 0 : 1;
        gemm(c, g);
        block_lse_bf16(c->part, c->part_tiles, M, c->loss_row, st);
      } else {
        GemmDesc g = desc((int)M, (int)V, (int)H, K_MAJOR, c->htape, H, K_MAJOR, c->w_out, H,
                          static_cast<float*>(c->S), V);
        gemm(c, g);
        block_lse_f32(static_cast<float*>(c->S), M, V, c->y_d, c->loss_row, c->dh_out, st);
      }
      c->launches += 2;
      DL_CUDA(cudaMemcpyAsync(out + r0, c->loss_row, M * 8, cudaMemcpyDeviceToHost, st));
      DL_CUDA(cudaStreamSynchronize(st));
    }
    if (n_out) *n_out = ns;
  });
}

// RnnHitScorer::score over a single stream (eval.hpp:476-510): after each
// input id, the raw scores float(dot_acc(h, W_out[w])) of up to K candidate
// words (cand[j*K + k], -1 = none) -- the NCE score kernel's 8-lane double
// dot product, bit-identical to the reference's Adapter::score.
int dl_score_candidates(dl_ctx* c, const uint32_t* in, int64_t steps, int64_t K,
                        const int64_t* cand, float* out) {
  if (!c) return fail(c, DL_EINVAL, "dl_score_candidates: null ctx");
  if (!in || steps < 1 || K < 1 || !cand || !out)
    return fail(c, DL_EINVAL, "dl_score_candidates: bad arguments");
  if (c->vshard) return fail(c, DL_EINVAL, "dl_score_candidates: not on a vocabulary-sharded context");
  for (int64_t i = 0; i < steps; ++i)
    if (in[i] >= (uint64_t)c->V) return fail(c, DL_EDATA, "hit rate: id out of vocabulary range");
  for (int64_t i = 0; i < steps * K; ++i)
    if (cand[i] >= c->V) return fail(c, DL_EDATA, "hit rate: candidate out of vocabulary range");
  return guarded(c, [&] {
    const int64_t H = c->H;
    const int64_t bank = std::min<int64_t>(steps, 4096);
    ensure_window(c, bank, 1);
    cudaStream_t st = c->st;
    uint32_t* rw = dalloc<uint32_t>(bank * K);
    uint32_t* rr = dalloc<uint32_t>(bank * K);
    float* sc = dalloc<float>(bank * K);
    std::vector<uint32_t> hw, hr;
    std::vector<int64_t> slot;
    std::vector<float> hs;
    fill_f32(c->htape, act0(c->act), H, st);
    for (int64_t j0 = 0; j0 < steps; j0 += bank) {
      const int64_t nb = std::min(bank, steps - j0);
      DL_CUDA(cudaMemcpyAsync(c->x_d, in + j0, nb * 4, cudaMemcpyHostToDevice, st));
      if (tc(c)) f32_to_bf16(c->htape, c->htape_bf, H, st);
      for (int64_t t = 0; t < nb; ++t)
        rec_step_fwd(c, 1, c->htape + t * H, tc(c) ? c->htape_bf + t * H : nullptr, c->x_d + t,
                     c->htape + (t + 1) * H, tc(c) ? c->htape_bf + (t + 1) * H : nullptr);
      hw.clear();
      hr.clear();
      slot.clear();
      for (int64_t t = 0; t < nb; ++t)
        for (int64_t k = 0; k < K; ++k) {
          const int64_t w = cand[(j0 + t) * K + k];
          if (w < 0) continue;
          hw.push_back((uint32_t)w);
          hr.push_back((uint32_t)(t + 1));  // htape row of the state after in[j0+t]
          slot.push_back((j0 + t) * K + k);
        }
      const int64_t N = (int64_t)hw.size();
      if (N > 0) {
        DL_CUDA(cudaMemcpyAsync(rw, hw.data(), N * 4, cudaMemcpyHostToDevice, st));
        DL_CUDA(cudaMemcpyAsync(rr, hr.data(), N * 4, cudaMemcpyHostToDevice, st));
        nce_scores(c->htape, c->w_out, H, rw, rr, N, sc, st);
        c->launches++;
        hs.resize(N);
        DL_CUDA(cudaMemcpyAsync(hs.data(), sc, N * 4, cudaMemcpyDeviceToHost, st));
      }
      DL_CUDA(cudaMemcpyAsync(c->htape, c->htape + nb * H, H * 4, cudaMemcpyDeviceToDevice, st));
      DL_CUDA(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < N; ++i) out[slot[i]] = hs[i];
    }
    cudaFree(rw);
    cudaFree(rr);
    cudaFree(sc);
  });
}

// RnnParams::init_uniform (rnn.hpp:79-83): one std::mt19937_64(seed), w_in
// then w_rec then w_out, each element float(lo + (hi - lo) * u) with
// u = (rng() >> 11) * 2^-53 (rng.hpp:37-44).  Pure host code; bit-exact.
int dl_init_uniform(int64_t V, int64_t H, uint64_t seed, double range, float* w_in,
                    float* w_rec, float* w_out) {
  if (V < 1 || H < 1) return fail(nullptr, DL_EINVAL, "RnnParams: V,H >= 1");
  if (!w_in || !w_rec || !w_out) return fail(nullptr, DL_EINVAL, "dl_init_uniform: null output");
  std::mt19937_64 rng(seed);
  const double lo = -range, hi = range;
  auto fill = [&](float* p, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
      p[i] = static_cast<float>(lo + (hi - lo) * (static_cast<double>(rng() >> 11) * 0x1.0p-53));
  };
  fill(w_in, V * H);
  fill(w_rec, H * H);
  fill(w_out, V * H);
  return DL_OK;
}

// ------------------------------------------------------------- trainer
// trainer.hpp:194-195 (cursor_i = floor(i*L/N)) for this rank's slice of
// every group: with G ranks the global minibatch is G*minibatch and rank r
// owns global streams g*G*minibatch + r*minibatch + b.  Pure host code.
int dl_rank_cursors(int64_t L, int noffset, int minibatch, int nranks, int rank,
                    int64_t* out) {
  if (L < 1 || noffset < 1 || minibatch < 1 || nranks < 1 || rank < 0 || rank >= nranks || !out)
    return fail(nullptr, DL_EINVAL, "dl_rank_cursors: bad arguments");
  const int64_t Bg = (int64_t)minibatch * nranks;
  const int64_t Nglob = (int64_t)noffset * Bg;
  for (int64_t g = 0; g < noffset; ++g)
    for (int64_t b = 0; b < minibatch; ++b) {
      const int64_t s = g * Bg + (int64_t)rank * minibatch + b;
      out[g * minibatch + b] = s * L / Nglob;
    }
  return DL_OK;
}

int dl_trainer_init(dl_ctx* c, const uint32_t* ids, int64_t L, int noffset, int minibatch,
                    int unroll, double clip, uint32_t bos) {
  if (!c) return fail(c, DL_EINVAL, "dl_trainer_init: null ctx");
  if (noffset < 1 || minibatch < 1 || unroll < 1)
    return fail(c, DL_EINVAL, "config: noffset, minibatch, unroll must be >= 1");
  if (!(clip > 0.0)) return fail(c, DL_EINVAL, "config: clip must be > 0");
  const int64_t Nglob = (int64_t)noffset * minibatch * dp_ranks(c);
  if (L < Nglob) return fail(c, DL_EINVAL, "trainer: training stream shorter than the stream count");
  for (int64_t i = 0; i < L; ++i)
    if (ids[i] >= (uint64_t)c->V) return fail(c, DL_EDATA, "trainer: id out of vocabulary range");
  return guarded(c, [&] {
    if (c->ids) cudaFree(c->ids);
    if (c->cursors) cudaFree(c->cursors);
    if (c->hidden) cudaFree(c->hidden);
    c->L = L;
    c->noffset = noffset;
    c->minibatch = minibatch;
    c->unroll = unroll;
    c->clip = clip;
    c->bos = bos;
    c->ids = dalloc<uint32_t>(L);
    DL_CUDA(cudaMemcpyAsync(c->ids, ids, L * 4, cudaMemcpyHostToDevice, c->st));
    // NCE windows draw their noise on the host from the window's targets:
    // the host keeps the stream too (any mode may be selected later)
    c->h_ids.assign(ids, ids + L);
    const int64_t Nl = (int64_t)noffset * minibatch;
    c->cursors = dalloc<int64_t>(Nl);
    c->hidden = dalloc<float>(Nl * c->H);
    std::vector<int64_t> cur(Nl);
    dl_rank_cursors(L, noffset, minibatch, (int)dp_ranks(c), dp_rank(c), cur.data());
    DL_CUDA(cudaMemcpyAsync(c->cursors, cur.data(), Nl * 8, cudaMemcpyHostToDevice, c->st));
    fill_f32(c->hidden, act0(c->act), Nl * c->H, c->st);
    ensure_window(c, unroll, minibatch);
    DL_CUDA(cudaStreamSynchronize(c->st));
    drop_graphs(c);
  });
}

int dl_trainer_get_state(dl_ctx* c, int64_t* cursors, float* hidden) {
  if (!c || !c->cursors) return fail(c, DL_EINVAL, "trainer not initialised");
  return guarded(c, [&] {
    const int64_t Nl = (int64_t)c->noffset * c->minibatch;
    if (cursors) DL_CUDA(cudaMemcpyAsync(cursors, c->cursors, Nl * 8, cudaMemcpyDeviceToHost, c->st));
    if (hidden) DL_CUDA(cudaMemcpyAsync(hidden, c->hidden, Nl * c->H * 4, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_trainer_set_state(dl_ctx* c, const int64_t* cursors, const float* hidden) {
  if (!c || !c->cursors) return fail(c, DL_EINVAL, "trainer not initialised");
  const int64_t Nl = (int64_t)c->noffset * c->minibatch;
  if (cursors)
    for (int64_t i = 0; i < Nl; ++i)
      if (cursors[i] < 0 || cursors[i] >= c->L)
        return fail(c, DL_EDATA, "trainer checkpoint: cursor out of range");
  return guarded(c, [&] {
    if (cursors) DL_CUDA(cudaMemcpyAsync(c->cursors, cursors, Nl * 8, cudaMemcpyHostToDevice, c->st));
    if (hidden) DL_CUDA(cudaMemcpyAsync(c->hidden, hidden, Nl * c->H * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

namespace {
// The dense W_out update can run inside the dW_out epilogue when it cannot be
// rejected (finite clip: every clipped component is finite), no dW_out
// allreduce sits between the GEMM and the update (single GPU or vocabulary
// shards) and the pair kernel has the whole device to itself.
bool fuse_ok(dl_ctx* c, double clip) {
  if (!(c->fuse_out && tc(c) && std::isfinite((float)clip))) return false;
  if (c->comm && (!c->vshard || c->comm->shares_device())) return false;
  if (c->fuse_cap < 0) c->fuse_cap = tc_rms_fusable((int)c->Vo, (int)c->H) ? 1 : 0;
  return c->fuse_cap == 1;
}

bool late_ok(dl_ctx* c) {
  return c->fork_late && tc(c) && std::isfinite((float)c->clip) && c->comm == nullptr;
}

bool fork_ok(dl_ctx* c) {
  return c->fork_out && tc(c) && c->w_out_bf_next && std::isfinite((float)c->clip) &&
         c->comm == nullptr;
}

void swap_shadow(dl_ctx* c) {
  std::swap(c->w_out_bf, c->w_out_bf_next);
  c->par ^= 1;
}

// Size the split-K workspace for a T x B window before graph capture
// (no allocation may happen inside a capture).
void presize(dl_ctx* c, int64_t T, int64_t B) {
  const int64_t H = c->H, Vo = c->Vo, TB = T * B;
  size_t need = (size_t)pick_splits(c, (int)B, (int)H, (int)H) * B * H;
  const int64_t MO = out_ranks(c) * TB;
  const int sdh = pick_splits(c, (int)MO, (int)H, (int)Vo, 8);
  if (sdh > 1) need = std::max(need, (size_t)sdh * MO * H);
  need = std::max(need, (size_t)pick_splits(c, (int)H, (int)H, (int)TB, 16) * H * H);
  ensure_splitws(c, need);
}

// One device-resident window of the epoch schedule (trainer.hpp:376-405).
void trainer_window(dl_ctx* c, double eta) {
  const int64_t B = c->minibatch, T = c->unroll, H = c->H;
  const double scale = 1.0 / (double)(B * dp_ranks(c) * T);
  window_build(c->ids, c->L, c->cursors, c->hidden, c->win_counter, c->noffset, B, T, H, c->bos,
               c->x_d, c->y_d, c->w_d, c->htape, c->st, tc(c) ? c->htape_bf : nullptr);
  c->launches++;
  c->h0_bf_ready = tc(c);
  // the dense W_out update overlaps the dh GEMM when it cannot be rejected
  // (finite clip, see run_window), a second bf16 shadow exists and no
  // allreduce is pending
  const bool sm = c->loss_mode != 0;  // (the W_out update placements are softmax-only)
  const bool fuse = sm && fuse_ok(c, c->clip);
  const bool late = sm && !fuse && late_ok(c);
  const bool fork = sm && !fuse && !late && fork_ok(c);
  run_window(c, T, B, scale, (float)c->clip, true, fork ? eta : 0.0, fuse ? eta : 0.0,
             late ? eta : 0.0);
  c->h0_bf_ready = false;
  run_rmsprop(c, eta, T * B * dp_ranks(c), /*skip_out=*/fork || fuse || late, /*count=*/false);
  window_finish(c->cursors, c->hidden, c->htape + T * B * H, c->win_counter, c->noffset, B, T, H,
                c->L, act0(c->act), c->st, c->nonfinite, c->d_skipped);
  c->launches += 2;
  if (fork || late) DL_CUDA(cudaStreamWaitEvent(c->st, c->ev_join, 0));
  if (fork) swap_shadow(c);
}
}  // namespace

int dl_trainer_run(dl_ctx* c, int64_t first, int64_t count, double eta, double* loss_sum,
                   uint64_t* skipped) {
  if (!c || !c->ids) return fail(c, DL_EINVAL, "trainer not initialised");
  if (!(eta > 0.0)) return fail(c, DL_EINVAL, "config: eta must be > 0");
  return guarded(c, [&] {
    DL_CUDA(cudaMemcpyAsync(c->win_counter, &first, 8, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaMemsetAsync(c->d_loss, 0, 8, c->st));
    DL_CUDA(cudaMemsetAsync(c->d_pos, 0, 8, c->st));
    DL_CUDA(cudaMemsetAsync(c->d_skipped, 0, 8, c->st));
    const bool nce = c->loss_mode == 0;
    DL_REQUIRE(!nce || c->comm == nullptr || !c->vshard, 1,
               "NCE mode: not with a vocabulary-sharded output layer");
    const bool graphs = c->use_graph && !c->profiling && c->comm == nullptr && !nce;
    presize(c, c->unroll, c->minibatch);
    if (nce) {
      // the noise draws depend on the window's targets / mask, which the
      // device builds from the resident stream: the host mirrors the same
      // schedule (cursors, window counter; trainer.hpp:374-406) to draw
      // them, window by window, in the reference's order
      // With data-parallel ranks the draws cover the global window (every
      // rank's streams, in the reference's (t, global stream, sample) order)
      // and every rank makes all of them: the generator stays identical
      // across ranks, as the reference's single Trainer::rng_.
      const int64_t B = c->minibatch, T = c->unroll, Nl = (int64_t)c->noffset * B;
      const int64_t G = c->comm ? c->nranks : 1, BG = G * B;
      ensure_window(c, T, B);
      std::vector<int64_t> cur(G * Nl);  // [rank][group * B + b]
      if (G > 1 || c->comm) {
        int64_t* cur_all = dalloc<int64_t>(G * Nl);
        c->comm->allgather(c->cursors, cur_all, (size_t)Nl, DType::U64, c->st);
        DL_CUDA(cudaMemcpyAsync(cur.data(), cur_all, G * Nl * 8, cudaMemcpyDeviceToHost, c->st));
        DL_CUDA(cudaStreamSynchronize(c->st));
        cudaFree(cur_all);
      } else {
        DL_CUDA(cudaMemcpyAsync(cur.data(), c->cursors, Nl * 8, cudaMemcpyDeviceToHost, c->st));
        DL_CUDA(cudaStreamSynchronize(c->st));
      }
      std::vector<uint32_t> y(T * BG);
      std::vector<uint8_t> w(T * BG);
      const int64_t L = c->L;
      double host_draw_s = 0.0, host_enqueue_s = 0.0;
      const auto run0 = std::chrono::steady_clock::now();
      for (int64_t i = 0; i < count; ++i) {
        const int64_t s0 = ((first + i) % c->noffset) * B;
        for (int64_t t = 0; t < T; ++t)
          for (int64_t r = 0; r < G; ++r)
            for (int64_t b = 0; b < B; ++b) {
              const int64_t pos = cur[r * Nl + s0 + b] + t;
              const int64_t k = t * BG + r * B + b;
              y[k] = c->h_ids[(pos + 1) % L];
              w[k] = y[k] == c->bos ? 0 : 1;
            }
        const auto h0 = std::chrono::steady_clock::now();
        nce_prepare(c, T, BG, w.data());
        const auto h1 = std::chrono::steady_clock::now();
        trainer_window(c, eta);
        const auto h2 = std::chrono::steady_clock::now();
        host_draw_s += std::chrono::duration<double>(h1 - h0).count();
        host_enqueue_s += std::chrono::duration<double>(h2 - h1).count();
        for (int64_t r = 0; r < G; ++r)
          for (int64_t b = 0; b < B; ++b) {
            int64_t v = cur[r * Nl + s0 + b] + T;
            if (v >= L) v -= L;
            cur[r * Nl + s0 + b] = v;
          }
      }
      if (std::getenv("DL_DEBUG"))
        fprintf(stderr, "[desklm] NCE trainer: %lld windows, host draws %.3f ms/window, "
                "enqueue %.3f ms/window, wall %.3f ms/window (slot wait %.3f, rng %.3f, reserve "
                "%.3f, copy %.3f ms total)\n",
                (long long)count,
                1e3 * host_draw_s / std::max<int64_t>(count, 1),
                1e3 * host_enqueue_s / std::max<int64_t>(count, 1),
                1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - run0)
                          .count() / std::max<int64_t>(count, 1),
                1e3 * c->nce_wait_s, 1e3 * c->nce_gen_s, 1e3 * c->nce_res_s, 1e3 * c->nce_copy_s);
    } else if (graphs) {
      // one graph per W_out-shadow parity (the forked update writes the
      // other shadow, so consecutive windows alternate between two graphs)
      const int nvar = !fuse_ok(c, c->clip) && !late_ok(c) && fork_ok(c) ? 2 : 1;
      if (!c->graph || c->graph_eta != eta) {
        drop_graphs(c);
        c->graph_par0 = c->par;
        for (int v = 0; v < nvar; ++v) {
          cudaGraph_t gph;
          const uint64_t before = c->launches.load();
          DL_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
          try {
            trainer_window(c, eta);  // host side flips the shadows when forking
          } catch (...) {
            cudaStreamEndCapture(c->st, &gph);
            throw;
          }
          DL_CUDA(cudaStreamEndCapture(c->st, &gph));
          DL_CUDA(cudaGraphInstantiate(&c->graphs[(c->graph_par0 + v) & 1], gph, 0));
          cudaGraphDestroy(gph);
          c->graph_launches = c->launches.load() - before;
          c->launches -= c->graph_launches;  // counted when replayed
        }
        if (nvar == 2 && c->par != c->graph_par0) swap_shadow(c);  // (never: 2 flips)
        c->graph = c->graphs[c->graph_par0];
        c->graph_eta = eta;
      }
      for (int64_t i = 0; i < count; ++i) {
        DL_CUDA(cudaGraphLaunch(nvar == 2 ? c->graphs[c->par] : c->graph, c->st));
        if (nvar == 2) swap_shadow(c);
        c->launches += c->graph_launches;
      }
    } else {
      for (int64_t i = 0; i < count; ++i) trainer_window(c, eta);
    }
    double l = 0.0;
    unsigned long long sk = 0;
    DL_CUDA(cudaMemcpyAsync(&l, c->d_loss, 8, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaMemcpyAsync(&sk, c->d_skipped, 8, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
    prof_collect(c);
    if (loss_sum) *loss_sum += l;
    if (skipped) *skipped += sk;
  });
}

// ---------------------------------------------------------------- comm
int dl_comm_unique_id(uint8_t id[128]) {
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return fail(nullptr, DL_EDEVICE, "ncclGetUniqueId failed");
  std::memcpy(id, &u, 128);
  return DL_OK;
}

int dl_comm_init(dl_ctx* c, const uint8_t id[128], int nranks, int rank) {
  if (!c) return fail(c, DL_EINVAL, "dl_comm_init: null ctx");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, DL_EINVAL, "dl_comm_init: bad rank");
  return guarded(c, [&] {
    reset_vshard(c);
    c->nranks = nranks;
    c->rank = rank;
    c->capT = c->capB = 0;  // window buffers are re-sized for the gathered window
    drop_graphs(c);
    delete c->comm;
    c->comm = nullptr;
    // (a one-rank communicator is real too: it runs the multi-rank code
    // paths -- collectives, gathered windows, sharded output -- on one GPU)
    c->comm = new NcclComm(id, nranks, rank);
  });
}

// In-process groups: G contexts on one device behave as G ranks (one host
// thread per context).  Used to run the multi-rank code paths -- data
// parallel and vocabulary sharded -- on a single GPU.
int dl_local_group_create(int G, void** group) {
  if (G < 1 || G > 16 || !group) return fail(nullptr, DL_EINVAL, "dl_local_group_create: 1..16");
  *group = new LocalGroup(G);
  return DL_OK;
}

int dl_local_group_destroy(void* group) {
  delete static_cast<LocalGroup*>(group);
  return DL_OK;
}

int dl_comm_init_local(dl_ctx* c, void* group, int rank) {
  if (!c || !group) return fail(c, DL_EINVAL, "dl_comm_init_local: null argument");
  LocalGroup* g = static_cast<LocalGroup*>(group);
  if (rank < 0 || rank >= g->G) return fail(c, DL_EINVAL, "dl_comm_init_local: bad rank");
  return guarded(c, [&] {
    reset_vshard(c);
    c->nranks = g->G;
    c->rank = rank;
    c->capT = c->capB = 0;
    drop_graphs(c);
    delete c->comm;
    c->comm = g->G > 1 ? new LocalComm(g, rank) : nullptr;
  });
}

int dl_set_loss_mode(dl_ctx* c, int mode) {
  if (!c) return fail(c, DL_EINVAL, "dl_set_loss_mode: null ctx");
  if (mode != 0 && mode != 1) return fail(c, DL_EINVAL, "dl_set_loss_mode: 0 (NCE) or 1 (softmax)");
  c->loss_mode = mode;
  c->have_grads = false;
  drop_graphs(c);
  if (c->comm) c->capT = c->capB = 0;  // (re)size the NCE gather buffers
  return DL_OK;
}

int dl_set_noise(dl_ctx* c, const double* counts, int64_t V, int k, double floor) {
  if (!c || !counts) return fail(c, DL_EINVAL, "dl_set_noise: null argument");
  if (V != c->V) return fail(c, DL_EINVAL, "NoiseModel: vocabulary size mismatch");
  if (k < 1) return fail(c, DL_EINVAL, "NoiseModel: k must be >= 1");
  if (!(floor > 0.0)) return fail(c, DL_EINVAL, "config: noise_floor must be > 0");
  return guarded(c, [&] { nce_build(c, counts, V, k, floor); });
}

int dl_set_noise_dist(dl_ctx* c, const double* q, int64_t V, int k) {
  if (!c || !q) return fail(c, DL_EINVAL, "dl_set_noise_dist: null argument");
  if (V != c->V) return fail(c, DL_EINVAL, "NoiseModel: vocabulary size mismatch");
  if (k < 1) return fail(c, DL_EINVAL, "NoiseModel: k must be >= 1");
  return guarded(c, [&] { nce_build(c, q, V, k, 0.0, true); });
}

int dl_set_rng_state(dl_ctx* c, const uint64_t state[313]) {
  if (!c || !state) return fail(c, DL_EINVAL, "dl_set_rng_state: null argument");
  std::stringstream ss;
  for (int i = 0; i < 313; ++i) ss << state[i] << ' ';
  ss >> c->rng;
  if (!ss) return fail(c, DL_EINVAL, "dl_set_rng_state: bad state");
  if (c->pre_n > 0) c->predraw_off = true;  // (that queue was drawn for nothing)
  c->pre_n = 0;
  c->rng_set = true;
  drop_graphs(c);
  return DL_OK;
}

int dl_get_rng_state(const dl_ctx* c, uint64_t state[313]) {
  if (!c || !state) return fail(nullptr, DL_EINVAL, "dl_get_rng_state: null argument");
  std::stringstream ss;
  ss << c->rng;
  for (int i = 0; i < 313; ++i) ss >> state[i];
  return DL_OK;
}

int dl_rng_seed_state(uint64_t seed, uint64_t state[313]) {
  if (!state) return fail(nullptr, DL_EINVAL, "dl_rng_seed_state: null argument");
  std::stringstream ss;
  ss << std::mt19937_64(seed);
  for (int i = 0; i < 313; ++i) ss >> state[i];
  return DL_OK;
}

int dl_set_vocab_shard(dl_ctx* c, int on) {
  if (!c) return fail(c, DL_EINVAL, "dl_set_vocab_shard: null ctx");
  if (on) {
    if (!c->comm)
      return fail(c, DL_EINVAL, "dl_set_vocab_shard: needs a communicator (dl_comm_init)");
    if (c->V % c->nranks != 0)
      return fail(c, DL_EINVAL, "dl_set_vocab_shard: V must be a multiple of the rank count");
    if (c->precision == DL_BF16 && ((c->V / c->nranks) % 8) != 0)
      return fail(c, DL_EINVAL, "dl_set_vocab_shard: bf16 mode needs V/G a multiple of 8 (TMA)");
  }
  if (on != 0 && on != 1 && on != 2)
    return fail(c, DL_EINVAL, "dl_set_vocab_shard: mode must be 0, 1 or 2");
  return guarded(c, [&] {
    if (!on) {
      reset_vshard(c);
      return;
    }
    c->vshard = true;
    c->dpv = on == 2;
    c->capT = c->capB = 0;  // window buffers re-size for the gathered rows
    c->Vo = c->V / c->nranks;
    c->v0 = (int64_t)c->rank * c->Vo;
    alloc_output(c);
    refresh_shadows(c);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

// Test hook for the data-parallel W_in gradient: G rank-blocked windows
// x_all [G][T][B], dpre_all [G][T][B][H] -> clipped dense g_in [V x H],
// summed per word in the reference's processing order over the global
// window (t descending, global stream r*B+b ascending).
int dl_test_embed(dl_ctx* c, int G, int64_t T, int64_t B, const uint32_t* x_all,
                  const float* dpre_all, float clip, float* g_in_dense) {
  if (!c || G < 1 || T < 1 || B < 1) return fail(c, DL_EINVAL, "dl_test_embed: bad shape");
  return guarded(c, [&] {
    const int64_t n = G * T * B, H = c->H;
    uint32_t* x = dalloc<uint32_t>(n);
    float* d = dalloc<float>(n * H);
    float* rows = dalloc<float>(n * H);
    uint32_t* words = dalloc<uint32_t>(n);
    int* nr = dalloc<int>(1);
    EmbedWs ws{dalloc<int>(2 * n + 2), dalloc<int>(n), n};
    float* dense = dalloc<float>(c->V * H);
    DL_CUDA(cudaMemcpyAsync(x, x_all, n * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaMemcpyAsync(d, dpre_all, n * H * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaMemsetAsync(dense, 0, c->V * H * 4, c->st));
    embed_grads(x, T, B, G, c->V, d, H, clip, ws, rows, words, nr, nullptr, c->st);
    embed_dense(rows, words, nr, n, H, dense, c->st);
    DL_CUDA(cudaMemcpyAsync(g_in_dense, dense, c->V * H * 4, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
    for (void* p : {(void*)x, (void*)d, (void*)rows, (void*)words, (void*)nr, (void*)ws.seg_start,
                    (void*)ws.order_pos, (void*)dense})
      cudaFree(p);
  });
}

// Test hook: C[M x N] = A . B^T through the context's GEMM engine, with A
// stored K-major [M x K] or MN-major [K x M] (likewise B), fp32 host arrays
// (rounded to bf16 on the device in DL_BF16 mode).  With tgt != NULL the
// logits epilogue runs instead and C receives per-row (lse, target logit).
int dl_test_gemm(dl_ctx* c, int M, int N, int K, int a_major, int b_major, const float* A,
                 const float* B, float* Cout, int splits, const uint32_t* tgt) {
  if (!c || M < 1 || N < 1 || K < 1) return fail(c, DL_EINVAL, "dl_test_gemm: bad shape");
  return guarded(c, [&] {
    const int64_t na = (int64_t)M * K, nb = (int64_t)N * K;
    float *a32 = dalloc<float>(na), *b32 = dalloc<float>(nb);
    DL_CUDA(cudaMemcpyAsync(a32, A, na * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaMemcpyAsync(b32, B, nb * 4, cudaMemcpyHostToDevice, c->st));
    bf16 *a16 = nullptr, *b16 = nullptr;
    if (tc(c)) {
      a16 = dalloc<bf16>(na);
      b16 = dalloc<bf16>(nb);
      f32_to_bf16(a32, a16, na, c->st);
      f32_to_bf16(b32, b16, nb, c->st);
    }
    const int64_t lda = a_major == K_MAJOR ? K : M, ldb = b_major == K_MAJOR ? K : N;
    const void* Ap = tc(c) ? (const void*)a16 : (const void*)a32;
    const void* Bp = tc(c) ? (const void*)b16 : (const void*)b32;
    if (tgt && tc(c)) {
      const int nt = tc_n_tiles(N);
      float2* part = dalloc<float2>((int64_t)nt * M);
      float* tl = dalloc<float>(M);
      uint32_t* tg = dalloc<uint32_t>(M);
      bf16* S = dalloc<bf16>((int64_t)M * N);
      double* lse = dalloc<double>(M);
      DL_CUDA(cudaMemcpyAsync(tg, tgt, M * 4, cudaMemcpyHostToDevice, c->st));
      GemmDesc g = desc(M, N, K, a_major, Ap, lda, b_major, Bp, ldb, nullptr, 0);
      g.logits = 1;
      g.S = S;
      g.lds = N;
      g.part = part;
      g.part_n = nt;
      g.tgt = tg;
      g.tgt_logit = tl;
      gemm(c, g);
      // logp = s_y - lse per row via the softmax-rows kernel (grads off)
      softmax_rows_bf16(nullptr, M, N, part, nt, tl, tg, nullptr, 1.0, 0, nullptr, lse, c->st);
      std::vector<double> lp(M);
      std::vector<float> t(M);
      DL_CUDA(cudaMemcpyAsync(lp.data(), lse, M * 8, cudaMemcpyDeviceToHost, c->st));
      DL_CUDA(cudaMemcpyAsync(t.data(), tl, M * 4, cudaMemcpyDeviceToHost, c->st));
      std::vector<uint16_t> sb((size_t)M * N);
      DL_CUDA(cudaMemcpyAsync(sb.data(), S, (size_t)M * N * 2, cudaMemcpyDeviceToHost, c->st));
      DL_CUDA(cudaStreamSynchronize(c->st));
      // Cout: [M x N] bf16 logits widened, then M logp, then M target logits
      for (int64_t i = 0; i < (int64_t)M * N; ++i) {
        uint32_t u = (uint32_t)sb[i] << 16;
        std::memcpy(&Cout[i], &u, 4);
      }
      for (int i = 0; i < M; ++i) {
        Cout[(int64_t)M * N + i] = (float)lp[i];
        Cout[(int64_t)M * N + M + i] = t[i];
      }
      cudaFree(part); cudaFree(tl); cudaFree(tg); cudaFree(S); cudaFree(lse);
    } else {
      const int s = tc(c)        ? tc_splits(K, std::max(1, splits))
                    : c->tf32x3 ? tf32_splits(K, std::max(1, splits))
                                : std::max(1, splits);
      float* out = dalloc<float>((int64_t)s * M * N);
      float* red = dalloc<float>((int64_t)M * N);
      GemmDesc g = desc(M, N, K, a_major, Ap, lda, b_major, Bp, ldb, out, N);
      g.k_splits = s;
      g.split_stride = (int64_t)M * N;
      // (fp32 / 3xTF32: transpose scratch for this shape)
      float *sa = c->xpose_a, *sb = c->xpose_b;
      const size_t ca = c->xpose_a_cap, cb = c->xpose_b_cap;
      const int64_t k4 = (K + 3) / 4 * 4;
      if (!tc(c) && c->tf32x3) {
        c->xpose_a = dalloc<float>((int64_t)M * k4);
        c->xpose_b = dalloc<float>((int64_t)N * k4);
        c->xpose_a_cap = (size_t)M * k4;
        c->xpose_b_cap = (size_t)N * k4;
      }
      gemm(c, g);
      if (!tc(c) && c->tf32x3) {
        DL_CUDA(cudaStreamSynchronize(c->st));
        cudaFree(c->xpose_a);
        cudaFree(c->xpose_b);
        c->xpose_a = sa;
        c->xpose_b = sb;
        c->xpose_a_cap = ca;
        c->xpose_b_cap = cb;
      }
      reduce_splits(out, s, (int64_t)M * N, (int64_t)M * N, red, 0.f, 0, nullptr, c->st);
      DL_CUDA(cudaMemcpyAsync(Cout, red, (size_t)M * N * 4, cudaMemcpyDeviceToHost, c->st));
      DL_CUDA(cudaStreamSynchronize(c->st));
      cudaFree(out);
      cudaFree(red);
    }
    DL_CUDA(cudaStreamSynchronize(c->st));
    cudaFree(a32); cudaFree(b32);
    if (a16) cudaFree(a16);
    if (b16) cudaFree(b16);
  });
}

uint64_t dl_launch_count(const dl_ctx* c) { return c ? c->launches.load() : 0; }

void* dl_cuda_stream(const dl_ctx* c) { return c ? static_cast<void*>(c->st) : nullptr; }

int dl_set_profiling(dl_ctx* c, int on) {
  if (!c) return fail(c, DL_EINVAL, "null ctx");
  c->profiling = on != 0;
  c->prof.clear();
  return DL_OK;
}

double dl_kernel_ms(const dl_ctx* c, const char* name) {
  if (!c || !name) return -1.0;
  auto it = c->prof.find(name);
  if (it == c->prof.end() || it->second.second == 0) return -1.0;
  return it->second.first / (double)it->second.second;
}

}  // extern "C"
