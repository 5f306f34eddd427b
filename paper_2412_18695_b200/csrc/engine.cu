// engine.cu — host runtime behind the C ABI (include/rt.h).
//
// One engine per GPU/process.  A round (rt_step) is, on one CUDA stream:
//   [H2D staged submissions + apply kernel] -> sched_pre (1 CTA) -> plan handshake
//   (the only host sync: 1 small mapped-memory read) -> forward pass over the
//   round's rows (prefill chunks + decode rows) -> lm_head+argmax -> sched_post.
// With world > 1 the per-rank top-K candidates are allgathered with NCCL on a
// side stream and merged on device (BASELINE.json: "one NCCL allgather over
// NVLink per scheduling round").
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdio.h>
#include <string.h>
#include <algorithm>
#include <string>
#include <unordered_map>
#include <vector>
#include <atomic>

#include "rt.h"
#include "internal.h"
#include "model.h"

using namespace rt;
static_assert(sizeof(SegRec) == sizeof(rt_segment), "segment record layout");

// ----------------------------------------------------------------- NCCL (dlopen)
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
typedef int (*pfn_comm_init_rank)(nccl_comm_t*, int, nccl_uid_t, int);
typedef int (*pfn_all_gather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t);
typedef int (*pfn_comm_destroy)(nccl_comm_t);
typedef const char* (*pfn_get_error_string)(int);
typedef int (*pfn_get_unique_id)(nccl_uid_t*);
struct NcclApi {
  void* h = nullptr;
  pfn_comm_init_rank init = nullptr;
  pfn_all_gather allgather = nullptr;
  pfn_comm_destroy destroy = nullptr;
  pfn_get_error_string errstr = nullptr;
  pfn_get_unique_id get_uid = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    init = (pfn_comm_init_rank)dlsym(h, "ncclCommInitRank");
    allgather = (pfn_all_gather)dlsym(h, "ncclAllGather");
    destroy = (pfn_comm_destroy)dlsym(h, "ncclCommDestroy");
    errstr = (pfn_get_error_string)dlsym(h, "ncclGetErrorString");
    get_uid = (pfn_get_unique_id)dlsym(h, "ncclGetUniqueId");
    return init && allgather && destroy;
  }
};
static NcclApi g_nccl;
static const int kNcclFloat64 = 8;

struct LayerW {
  bf16 *qkv, *o, *gu, *d;

};

struct rt_engine {
  rt_config cfg{};
  std::vector<int16_t> tok_skill;
  std::vector<int32_t> tok_exec;
  std::vector<int16_t> tok_class;                 // stop grammar (NEXT-4)
  std::vector<int32_t> skill_base, skill_unit;
  int qkv_dim = 0, pt_stride = 0, rows_cap = 0, fwd_rows = 0, part_rows = 0;
  int64_t pool_layer_bytes = 0;
  cudaStream_t stream = nullptr, side = nullptr;
  cudaEvent_t ev_plan = nullptr, ev_post = nullptr, ev_cand = nullptr, ev_merge = nullptr;
  bool post_pending = false, merge_pending = false, exchange = false;
  // weights
  void* d_wbuf = nullptr;
  bf16 *emb = nullptr, *lm = nullptr;
  std::vector<LayerW> layers;

  // KV pool
  unsigned char* d_pool = nullptr;
  // scheduler state
  TaskTable tt{};
  std::vector<void*> allocs;
  DevState* d_st = nullptr;
  void *h_hpool = nullptr, *d_hpool = nullptr;  // host KV pool (R-EVICT), mapped pinned
  int64_t hpool_page_bytes = 0;
  HostMailbox* h_mb = nullptr;
  HostMailbox* d_mb = nullptr;
  SegRec* h_ring = nullptr;
  SegRec* d_ring = nullptr;
  int64_t ring_cap = 32768;
  SchedParams sp{};
  // activations
  float *d_x = nullptr, *d_part = nullptr, *d_attn_ws = nullptr, *d_logits = nullptr, *d_am_val = nullptr;
  int32_t* d_am_idx = nullptr;
  bf16 *d_h = nullptr, *d_q = nullptr, *d_o = nullptr, *d_act = nullptr, *d_hfin = nullptr;
  float *d_cap_q = nullptr, *d_cap_o = nullptr, *d_rope_cos = nullptr, *d_rope_sin = nullptr;
  float* d_qkv_part = nullptr;   // decode QKV split-K partials folded into the attention
  int qkv_part_rows = 0;         // decode rows the fold serves (its partials are sized for)
  // RT_FLAG_CAPTURE_LAYERS: per-layer intermediates of the last round's first forward chunk
  float *d_lc_x = nullptr, *d_lc_xmid = nullptr;   // [L + 1][fwd_rows][d], [L][fwd_rows][d]
  bf16 *d_lc_q = nullptr, *d_lc_o = nullptr, *d_lc_act = nullptr;  // [L][fwd_rows][...]
  int lc_rows = 0;                                   // rows captured in the last round
  int64_t attn_ws_cap = 0, gemm_ws_cap = 0;
  float *d_gemm_ws = nullptr, *d_ss = nullptr;
  int* d_attn_tickets = nullptr;
  int* d_gemm_cnt = nullptr;
  GemmTmaSet x_h, x_o, x_act, x_hfin;
  float* d_dec_ws = nullptr;     // decode-pair split-K exchange (k_gemm_dec)
  int64_t dec_ws_floats = 0;
  unsigned* d_dec_flags = nullptr;
  unsigned dec_epoch = 0;
  float* d_sk_ws = nullptr;      // stream-K partial tiles (prefill projections, N > 128 rows)
  unsigned* d_sk_cnt = nullptr;  // stream-K tile tickets
  int sk_cnt_cap = 0;
  // submissions
  SubmitRec* h_recs = nullptr;
  int32_t* h_toks = nullptr;
  SubmitRec* d_recs = nullptr;
  int32_t* d_toks = nullptr;
  int n_staged = 0, recs_cap = 0;
  int64_t toks_staged = 0, toks_cap = 0;
  std::vector<int> free_slots;
  // registered shared prompt prefixes (rt_register_prefix): tokens (a multiple of 16) and
  // their read-only pages = page-table row max_tasks + id
  std::vector<std::vector<int32_t>> prefixes;
  int32_t pfx_pages = 0;  // pages held by registered prefixes (never freed)
  std::unordered_map<int64_t, int> rid_slot;
  int64_t n_submitted = 0;
  int64_t seg_read = 0;
  HostMailbox plan{};
  // RT_FLAG_TRACE: per-CTA kernel records (common.cuh TraceScope)
  uint64_t* d_trace = nullptr;
  unsigned* d_trace_n = nullptr;
  unsigned trace_cap = 0;
  // timing
  std::vector<cudaEvent_t> ev_attn;  // 2 per layer
  cudaEvent_t ev_f0 = nullptr, ev_f1 = nullptr, ev_s0 = nullptr, ev_s1 = nullptr, ev_q1 = nullptr;
  cudaEvent_t ev_m0 = nullptr, ev_m1 = nullptr;
  bool timing_pending = false;
  int timing_layers = 0;
  double attn_bytes_pending = 0.0;
  rt_stats stats{};
  // nccl
  nccl_comm_t comm = nullptr;
  double *d_cand_all = nullptr, *d_merged = nullptr;
  // errors
  bool sticky = false;
  std::string err;
};

static std::string g_last_err;

static rt_status fail(rt_engine* e, rt_status code, const std::string& msg) {
  if (e) {
    e->err = msg;
    if (code == RT_E_CUDA || code == RT_E_NCCL) e->sticky = true;
  }
  g_last_err = msg;
  return code;
}

#define CK(e, x)                                                                       \
  do {                                                                                 \
    cudaError_t _r = (x);                                                              \
    if (_r != cudaSuccess)                                                             \
      return fail(e, RT_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(_r));       \
  } while (0)

template <typename T>
static cudaError_t dalloc(rt_engine* e, T** p, size_t n) {
  void* q = nullptr;
  cudaError_t r = cudaMalloc(&q, std::max<size_t>(n * sizeof(T), 16));
  if (r == cudaSuccess) {
    e->allocs.push_back(q);
    cudaMemset(q, 0, std::max<size_t>(n * sizeof(T), 16));
    *p = (T*)q;
  }
  return r;
}

extern "C" const char* rt_version(void) {
  return "paper_2412_18695_b200 rt 0.1 (sm_100a: tcgen05 GEMM, bulk-copy paged attention, device scheduler)";
}

extern "C" const char* rt_last_error(rt_engine* e) { return e ? e->err.c_str() : g_last_err.c_str(); }

// ------------------------------------------------------------------ create
static rt_status validate(const rt_config* c) {
  if (!c) return RT_E_INVAL;
  if (c->page_tokens != 16) return RT_E_INVAL;
  if (c->max_batch < 1 || c->max_batch > 1024) return RT_E_INVAL;
  if (c->max_tasks < 1 || c->max_tasks > kMaxTasks) return RT_E_INVAL;
  if (c->max_ctx < 2) return RT_E_INVAL;
  if (c->max_seg_tokens < 1 || c->max_seg_tokens > kMaxSegTok) return RT_E_INVAL;
  if (c->speed_window < 1 || c->speed_window > 8) return RT_E_INVAL;
  if (c->g_us <= 0 || c->eps_l_us <= 0 || c->net_us < 0) return RT_E_INVAL;
  if (c->policy < 0 || c->policy > 2 || c->clock_mode < 0 || c->clock_mode > 1) return RT_E_INVAL;
  if (c->seg_mode < RT_SEG_SUSPEND || c->seg_mode > RT_SEG_NONE || c->wcet_off < 0 || c->wcet_off > 1)
    return RT_E_INVAL;
  if (c->host_pages < 0 || c->swap_us_per_page < 0) return RT_E_INVAL;
  if (c->stop_grammar < RT_GRAMMAR_TOKEN || c->stop_grammar > RT_GRAMMAR_PARAGRAPH || c->word_us < 0) return RT_E_INVAL;
  if (c->stop_grammar != RT_GRAMMAR_TOKEN &&
      (!c->tok_class || (c->stop_grammar == RT_GRAMMAR_SKILL && (!c->skill_base_us || !c->skill_unit_us))))
    return RT_E_INVAL;
  if (c->vocab < 2 || !c->tok_skill || !c->tok_exec_min_us) return RT_E_INVAL;
  if (c->gemm_path < RT_GEMM_PATH_AUTO || c->gemm_path > RT_GEMM_PATH_DECPAIR) return RT_E_INVAL;
  if (c->eos_id < 0 || c->eos_id >= c->vocab) return RT_E_INVAL;
  // the device merge of the per-round candidates (k_merge_cand) holds world x kTopK keys in
  // shared memory: one node of <= 8 GPUs (BASELINE.json: one 8xB200 box)
  if (c->world < 1 || c->world > 8 || c->rank < 0 || c->rank >= c->world) return RT_E_INVAL;
  if (!(c->flags & RT_FLAG_NO_MODEL)) {
    if (c->n_layers < 1 || c->d_model % 64 || c->d_ff % 64 || c->n_q_heads < 1 || c->n_kv_heads < 1) return RT_E_INVAL;
    if (c->n_q_heads % c->n_kv_heads || c->n_q_heads / c->n_kv_heads > 8) return RT_E_INVAL;
    if (c->head_dim != 32 && c->head_dim != 64 && c->head_dim != 128) return RT_E_INVAL;
    if ((c->n_q_heads * c->head_dim) % 64) return RT_E_INVAL;
  }
  return RT_OK;
}

static rt_status create_impl(rt_engine* e, const rt_config* cfg);

extern "C" rt_status rt_create(const rt_config* cfg, rt_engine** out) {
  if (!out) return RT_E_INVAL;
  *out = nullptr;
  rt_status v = validate(cfg);
  if (v != RT_OK) return fail(nullptr, v, "invalid rt_config");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= cfg->device)
    return fail(nullptr, RT_E_CUDA, "no CUDA device (this library has no CPU fallback)");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10)
    return fail(nullptr, RT_E_CUDA, "an sm_100 (B200) device is required");
  rt_engine* e = new rt_engine();
  rt_status s = create_impl(e, cfg);
  if (s != RT_OK) {
    g_last_err = e->err;
    rt_destroy(e);
    return s;
  }
  *out = e;
  return RT_OK;
}

static rt_status create_impl(rt_engine* e, const rt_config* cfg) {
  e->cfg = *cfg;
  const rt_config& c = e->cfg;
  e->tok_skill.assign(cfg->tok_skill, cfg->tok_skill + cfg->vocab);
  e->tok_exec.assign(cfg->tok_exec_min_us, cfg->tok_exec_min_us + cfg->vocab);
  e->cfg.tok_skill = nullptr;
  if (cfg->tok_class) e->tok_class.assign(cfg->tok_class, cfg->tok_class + cfg->vocab);
  else e->tok_class.assign(cfg->vocab, (int16_t)RT_TC_OTHER);
  e->skill_base.assign(RT_MAX_SKILL_NAMES, 0);
  e->skill_unit.assign(RT_MAX_SKILL_NAMES, 0);
  if (cfg->skill_base_us) e->skill_base.assign(cfg->skill_base_us, cfg->skill_base_us + RT_MAX_SKILL_NAMES);
  if (cfg->skill_unit_us) e->skill_unit.assign(cfg->skill_unit_us, cfg->skill_unit_us + RT_MAX_SKILL_NAMES);
  e->cfg.tok_class = nullptr;
  e->cfg.skill_base_us = nullptr;
  e->cfg.skill_unit_us = nullptr;
  e->cfg.tok_exec_min_us = nullptr;
  e->cfg.nccl_id = nullptr;
  if (e->cfg.max_admit_per_round <= 0) e->cfg.max_admit_per_round = 1 << 30;
  if (e->cfg.max_rows_per_forward < c.max_batch) e->cfg.max_rows_per_forward = std::max(c.max_batch, 2048);
  const bool model = !(c.flags & RT_FLAG_NO_MODEL);
  auto done = [&](rt_status s) { return s; };
  if (cudaSetDevice(c.device) != cudaSuccess) return done(fail(e, RT_E_CUDA, "cudaSetDevice"));
  if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking) != cudaSuccess)
    return done(fail(e, RT_E_CUDA, "stream create"));
  cudaEventCreateWithFlags(&e->ev_plan, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_post, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_cand, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_merge, cudaEventDisableTiming);
  cudaEventCreate(&e->ev_f0);
  cudaEventCreate(&e->ev_f1);
  cudaEventCreate(&e->ev_s0);
  cudaEventCreate(&e->ev_s1);
  cudaEventCreate(&e->ev_q1);
  cudaEventCreate(&e->ev_m0);
  cudaEventCreate(&e->ev_m1);

  e->pt_stride = (c.max_ctx + 15) / 16;
  e->rows_cap = c.max_batch * c.max_ctx;
  e->fwd_rows = e->cfg.max_rows_per_forward;
  const int d = c.d_model, hd = c.head_dim, nq = c.n_q_heads, nkv = c.n_kv_heads, L = c.n_layers;
  e->qkv_dim = (nq + 2 * nkv) * hd;

  // ---- page pool
  int n_pages = c.n_pages;
  const int64_t page_bytes_all_layers = model ? (int64_t)L * nkv * 64 * hd : 0;
  if (n_pages <= 0) {
    if (!model || c.kv_pool_bytes <= 0) return done(fail(e, RT_E_INVAL, "n_pages or kv_pool_bytes required"));
    n_pages = (int)std::min<int64_t>(c.kv_pool_bytes / page_bytes_all_layers, INT32_MAX / 2);
  }
  if (n_pages < 1) return done(fail(e, RT_E_INVAL, "empty page pool"));
  e->cfg.n_pages = n_pages;

  // ---- task table
  TaskTable& T = e->tt;
  const int MT = c.max_tasks;
#define A(f, n) CK(e, dalloc(e, &T.f, (size_t)(n)))
  A(rid, MT); A(arrival, MT); A(ert, MT); A(D, MT); A(ref, MT); A(end_est, MT); A(seg_exec, MT);
  A(alpha, MT); A(beta, MT); A(pri, MT);
  A(state, MT); A(agent, MT); A(k, MT); A(n_prompt, MT); A(max_new, MT); A(window, MT); A(scripted, MT);
  A(n_gen, MT); A(seg_tok, MT); A(n_skills, MT); A(pending, MT); A(ctx, MT); A(n_pages, MT); A(R, MT);
  A(holder, MT); A(argmax_last, MT); A(pfx, MT); A(n_pfx, MT); A(evicted, MT); A(n_hpages, MT);
  A(dfa_s, MT); A(dfa_n, MT); A(dfa_v, MT);
  A(hpage_table, (size_t)MT * e->pt_stride);
  A(page_table, (size_t)(MT + kMaxPrefixes) * e->pt_stride);
  A(prompt, (size_t)MT * c.max_ctx);
  A(script, (size_t)MT * c.max_ctx);
  A(out, (size_t)MT * c.max_ctx);
#undef A
  {
    std::vector<int32_t> fs(MT, T_FREE);
    CK(e, cudaMemcpy(T.state, fs.data(), MT * 4, cudaMemcpyHostToDevice));
  }
  SchedParams& P = e->sp;
  CK(e, dalloc(e, &e->d_st, 1));
  {
    DevState st{};
    st.t = c.t0_us;
    st.free_top = n_pages;
    st.hfree_top = c.host_pages;
    CK(e, cudaMemcpy(e->d_st, &st, sizeof(st), cudaMemcpyHostToDevice));
  }
  // KV eviction to host (R-EVICT): host free stack, per-round copy list, pinned mapped
  // host pool of host_pages pages x all layers (zero-copy target of k_kv_swap)
  P.host_pages = c.host_pages;
  P.swap_us_per_page = c.swap_us_per_page;
  P.swap_cap = 2 * n_pages;
  CK(e, dalloc(e, &P.hfree_stack, std::max(1, c.host_pages)));
  if (c.host_pages > 0) launch_init_free_stack(P.hfree_stack, c.host_pages, e->stream);
  CK(e, dalloc(e, &P.swap, (size_t)P.swap_cap));
  if (model && c.host_pages > 0) {
    e->hpool_page_bytes = page_bytes_all_layers;
    if (cudaHostAlloc(&e->h_hpool, (size_t)c.host_pages * page_bytes_all_layers, cudaHostAllocMapped) !=
        cudaSuccess)
      return done(fail(e, RT_E_NOMEM, "host KV pool (pinned) allocation failed"));
    CK(e, cudaHostGetDevicePointer(&e->d_hpool, e->h_hpool, 0));
  }
  CK(e, cudaHostAlloc((void**)&e->h_mb, sizeof(HostMailbox), cudaHostAllocMapped));
  memset(e->h_mb, 0, sizeof(HostMailbox));
  CK(e, cudaHostGetDevicePointer((void**)&e->d_mb, e->h_mb, 0));
  CK(e, cudaHostAlloc((void**)&e->h_ring, sizeof(SegRec) * e->ring_cap, cudaHostAllocMapped));
  CK(e, cudaHostGetDevicePointer((void**)&e->d_ring, e->h_ring, 0));
  CK(e, dalloc(e, &P.free_stack, n_pages));
  launch_init_free_stack(P.free_stack, n_pages, e->stream);
  CK(e, dalloc(e, &P.slot_task, c.max_batch));
  CK(e, dalloc(e, &P.round_slots, c.max_batch));
  CK(e, dalloc(e, &P.slot_is_prefill, c.max_batch));
  CK(e, dalloc(e, &P.slot_row, c.max_batch));
  CK(e, dalloc(e, &P.admitted, c.max_batch));
  CK(e, dalloc(e, &P.row_task, e->rows_cap));
  CK(e, dalloc(e, &P.row_pos, e->rows_cap));
  CK(e, dalloc(e, &P.dec_rows, c.max_batch));
  P.pf_tiles_cap = e->rows_cap / 16 + c.max_batch;
  CK(e, dalloc(e, &P.pf_tiles, (size_t)P.pf_tiles_cap));
  CK(e, dalloc(e, &P.row_tok, e->rows_cap));
  CK(e, dalloc(e, &P.argmax_tok, c.max_batch));
  CK(e, dalloc(e, &P.slot_tok, c.max_batch));
  CK(e, dalloc(e, &P.popped, 2 * ((size_t)n_pages + c.max_batch)));
  CK(e, dalloc(e, &P.cand, kTopK * 4));
  int16_t* d_skill;
  int32_t* d_exec;
  CK(e, dalloc(e, &d_skill, c.vocab));
  CK(e, dalloc(e, &d_exec, c.vocab));
  CK(e, cudaMemcpy(d_skill, e->tok_skill.data(), c.vocab * 2, cudaMemcpyHostToDevice));
  CK(e, cudaMemcpy(d_exec, e->tok_exec.data(), c.vocab * 4, cudaMemcpyHostToDevice));
  P.tt = T;
  P.pfx_pages = T.page_table + (size_t)MT * e->pt_stride;
  P.st = e->d_st;
  P.mb = e->d_mb;
  P.seg_ring = e->d_ring;
  P.seg_ring_cap = e->ring_cap;
  P.tok_skill = d_skill;
  P.tok_exec = d_exec;
  {
    int16_t* d_class;
    int32_t *d_base, *d_unit;
    CK(e, dalloc(e, &d_class, c.vocab));
    CK(e, dalloc(e, &d_base, RT_MAX_SKILL_NAMES));
    CK(e, dalloc(e, &d_unit, RT_MAX_SKILL_NAMES));
    CK(e, cudaMemcpy(d_class, e->tok_class.data(), c.vocab * 2, cudaMemcpyHostToDevice));
    CK(e, cudaMemcpy(d_base, e->skill_base.data(), RT_MAX_SKILL_NAMES * 4, cudaMemcpyHostToDevice));
    CK(e, cudaMemcpy(d_unit, e->skill_unit.data(), RT_MAX_SKILL_NAMES * 4, cudaMemcpyHostToDevice));
    P.tok_class = d_class;
    P.skill_base_us = d_base;
    P.skill_unit_us = d_unit;
    P.stop_grammar = c.stop_grammar;
    P.word_us = c.word_us;
  }
  P.max_tasks = MT;
  P.max_batch = c.max_batch;
  P.max_ctx = c.max_ctx;
  P.pt_stride = e->pt_stride;
  P.n_pages = n_pages;
  P.page_tokens = 16;
  P.rows_cap = e->rows_cap;
  P.max_seg_tokens = c.max_seg_tokens;
  P.g_us = c.g_us;
  P.net_us = c.net_us;
  P.eps_l_us = c.eps_l_us;
  P.speed_window = c.speed_window;
  P.max_admit = e->cfg.max_admit_per_round;
  P.policy = c.policy;
  P.seg_mode = c.seg_mode;
  P.wcet_off = c.wcet_off;
  P.clock_mode = c.clock_mode;
  P.base_us = c.base_us;
  P.gamma_ppm = c.gamma_ppm;
  P.kv_us_per_1k = c.kv_us_per_1k;
  P.prefill_us_per_tok = c.prefill_us_per_tok;
  P.eos_id = c.eos_id;
  P.rank = c.rank;
  P.world = c.world;
  P.no_model = model ? 0 : 1;

  // ---- submission staging (pinned)
  e->recs_cap = std::min(MT, 1024);
  e->toks_cap = (int64_t)std::max(4 * c.max_ctx, 1 << 20);
  CK(e, cudaHostAlloc((void**)&e->h_recs, sizeof(SubmitRec) * e->recs_cap, cudaHostAllocDefault));
  CK(e, cudaHostAlloc((void**)&e->h_toks, 4 * e->toks_cap, cudaHostAllocDefault));
  CK(e, dalloc(e, &e->d_recs, e->recs_cap));
  CK(e, dalloc(e, &e->d_toks, e->toks_cap));
  for (int i = MT - 1; i >= 0; --i) e->free_slots.push_back(i);

  // ---- model
  if (model) {
    const int ff = c.d_ff, V = c.vocab;
    // projection weights live in the UMMA-tiled layout; the embedding is
    // row-major (gathered by token id)
    const size_t n_emb = (size_t)V * d, n_lm = tiled_elems(V, d), n_qkv = tiled_elems(e->qkv_dim, d),
                 n_o = tiled_elems(d, nq * hd), n_gu = tiled_elems(2 * ff, d), n_d = tiled_elems(d, ff);
    const size_t total = n_emb + n_lm + L * (n_qkv + n_o + n_gu + n_d);
    if (cudaMalloc(&e->d_wbuf, total * 2) != cudaSuccess) return done(fail(e, RT_E_NOMEM, "weights do not fit in HBM"));
    bf16* w = (bf16*)e->d_wbuf;
    const float sig = c.init_std > 0 ? c.init_std : 0.02f;
    e->emb = w;
    w += n_emb;
    e->lm = w;
    w += n_lm;
    launch_init_weights(e->emb, n_emb, c.weight_seed, 0, sig, e->stream);
    launch_init_weights_tiled(e->lm, V, d, 0, 0, c.weight_seed, 1, sig, e->stream);
    e->layers.resize(L);
    for (int l = 0; l < L; ++l) {
      LayerW& lw = e->layers[l];
      lw.qkv = w; w += n_qkv;
      lw.o = w; w += n_o;
      lw.gu = w; w += n_gu;
      lw.d = w; w += n_d;
      launch_init_weights_tiled(lw.qkv, e->qkv_dim, d, 0, hd, c.weight_seed, 16 + 8 * l + 0, sig, e->stream);
      launch_init_weights_tiled(lw.o, d, nq * hd, 0, 0, c.weight_seed, 16 + 8 * l + 1, sig, e->stream);
      launch_init_weights_tiled(lw.gu, 2 * ff, d, ff, 0, c.weight_seed, 16 + 8 * l + 2, sig, e->stream);
      launch_init_weights_tiled(lw.d, d, ff, 0, 0, c.weight_seed, 16 + 8 * l + 3, sig, e->stream);
    }
    // KV pool
    e->pool_layer_bytes = (int64_t)n_pages * nkv * 64 * hd;
    if (cudaMalloc(&e->d_pool, (size_t)e->pool_layer_bytes * L) != cudaSuccess)
      return done(fail(e, RT_E_NOMEM, "KV pool does not fit in HBM"));
    CK(e, cudaMemsetAsync(e->d_pool, 0, (size_t)e->pool_layer_bytes * L, e->stream));
    // activations (one forward chunk of fwd_rows rows)
    const int R = e->fwd_rows;
    e->part_rows = std::max(R, 16 * c.max_batch);
    const int max_out = std::max(std::max(e->qkv_dim, d), 2 * ff);
    CK(e, dalloc(e, &e->d_x, (size_t)R * d));
    CK(e, dalloc(e, &e->d_h, (size_t)R * d));
    CK(e, dalloc(e, &e->d_q, (size_t)R * nq * hd));
    CK(e, dalloc(e, &e->d_o, (size_t)R * nq * hd));
    CK(e, dalloc(e, &e->d_act, (size_t)R * ff));
    (void)max_out;
    CK(e, dalloc(e, &e->d_ss, (size_t)R * ((d + 127) / 128)));
    CK(e, dalloc(e, &e->d_hfin, (size_t)c.max_batch * d));
    const int mt = (V + 127) / 128;
    CK(e, dalloc(e, &e->d_am_val, (size_t)mt * c.max_batch));
    CK(e, dalloc(e, &e->d_am_idx, (size_t)mt * c.max_batch));
    if (c.flags & RT_FLAG_KEEP_LOGITS) CK(e, dalloc(e, &e->d_logits, (size_t)c.max_batch * V));
    e->attn_ws_cap = (int64_t)(148 * 8 + (int64_t)R * nkv) * 8 * (hd + 2) * 2;
    CK(e, dalloc(e, &e->d_attn_ws, (size_t)e->attn_ws_cap));
    CK(e, dalloc(e, &e->d_attn_tickets, (size_t)R * nkv));
    if (c.flags & RT_FLAG_CAPTURE) {
      CK(e, dalloc(e, &e->d_cap_q, (size_t)e->rows_cap * nq * hd));
      CK(e, dalloc(e, &e->d_cap_o, (size_t)e->rows_cap * nq * hd));
    }
    if (c.flags & RT_FLAG_CAPTURE_LAYERS) {
      CK(e, dalloc(e, &e->d_lc_x, (size_t)(L + 1) * R * d));
      CK(e, dalloc(e, &e->d_lc_xmid, (size_t)L * R * d));
      CK(e, dalloc(e, &e->d_lc_q, (size_t)L * R * nq * hd));
      CK(e, dalloc(e, &e->d_lc_o, (size_t)L * R * nq * hd));
      CK(e, dalloc(e, &e->d_lc_act, (size_t)L * R * ff));
    }
    // RoPE tables (rotate-half, theta 500000), fp64 on host -> fp32
    std::vector<float> cs((size_t)c.max_ctx * hd / 2), sn((size_t)c.max_ctx * hd / 2);
    for (int p = 0; p < c.max_ctx; ++p)
      for (int i = 0; i < hd / 2; ++i) {
        const double inv = pow(500000.0, -2.0 * i / hd);
        const double ang = (double)p * inv;
        cs[(size_t)p * hd / 2 + i] = (float)cos(ang);
        sn[(size_t)p * hd / 2 + i] = (float)sin(ang);
      }
    CK(e, dalloc(e, &e->d_rope_cos, cs.size()));
    CK(e, dalloc(e, &e->d_rope_sin, sn.size()));
    CK(e, cudaMemcpy(e->d_rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
    CK(e, cudaMemcpy(e->d_rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
    bool ok = make_gemm_act_maps(&e->x_h, e->d_h, d, R) && make_gemm_act_maps(&e->x_o, e->d_o, nq * hd, R) &&
              make_gemm_act_maps(&e->x_act, e->d_act, ff, R) &&
              make_gemm_act_maps(&e->x_hfin, e->d_hfin, d, c.max_batch);
    if (!ok) return done(fail(e, RT_E_CUDA, "cuTensorMapEncodeTiled failed (activations)"));
    e->ev_attn.resize(2 * L);
    for (auto& ev : e->ev_attn) cudaEventCreate(&ev);
    // decode QKV folded into the attention (EPI_PART): raw split-K partials of up to
    // min(max_batch, 256, fwd_rows) decode rows
    {
      e->qkv_part_rows = std::min(std::min(c.max_batch, 256), R);
      int64_t need = 0;  // the QKV, O and down projections' partials share one buffer
      const int shapes[3][2] = {{e->qkv_dim, d}, {d, nq * hd}, {d, ff}};
      for (int n = 1; n <= e->qkv_part_rows; ++n)
        for (auto& sh : shapes) need = std::max(need, (int64_t)gemm_part_splits(sh[0], sh[1], n) * sh[0]);
      if (need > 0 && hd % 16 == 0 && nq / nkv <= 8)
        CK(e, dalloc(e, &e->d_qkv_part, (size_t)need * e->qkv_part_rows));
    }
    // decode-pair split-K exchange workspace (k_gemm_dec), sized for the model's projections
    {
      const int shapes[4][2] = {{e->qkv_dim, d}, {d, nq * hd}, {2 * ff, d}, {d, ff}};
      for (auto& sh : shapes)
        e->dec_ws_floats = std::max(e->dec_ws_floats, gemm_dec_ws_floats(sh[0], 256, sh[1]));
      if (e->dec_ws_floats > 0) {
        CK(e, dalloc(e, &e->d_dec_ws, (size_t)e->dec_ws_floats));
        CK(e, dalloc(e, &e->d_dec_flags, (size_t)kDecFlags));
      }
    }
    // hybrid DP + stream-K workspace of the prefill projections (gemm_tc.cu k_gemm_sk)
    {
      const int max_mt = (std::max(std::max(e->qkv_dim, d), 2 * ff) + 127) / 128;
      e->sk_cnt_cap = max_mt * ((R + 159) / 160);
      CK(e, dalloc(e, &e->d_sk_ws, (size_t)gemm_sk_ws_floats()));
      CK(e, dalloc(e, &e->d_sk_cnt, (size_t)e->sk_cnt_cap));
    }
  }
  if (c.flags & RT_FLAG_TRACE) {  // 48-byte records, bound process-wide (last engine wins)
    e->trace_cap = 1u << 20;
    CK(e, dalloc(e, &e->d_trace, (size_t)e->trace_cap * 6));
    CK(e, dalloc(e, &e->d_trace_n, 1));
    trace_bind_model(e->d_trace, e->d_trace_n, e->trace_cap);
    trace_bind_attn(e->d_trace, e->d_trace_n, e->trace_cap);
    trace_bind_gemm(e->d_trace, e->d_trace_n, e->trace_cap);
    trace_bind_sched(e->d_trace, e->d_trace_n, e->trace_cap);
    CK(e, cudaGetLastError());
  }
  // ---- replicas: NCCL communicator (one allgather of top-K candidates per round)
  e->exchange = c.world > 1 || (c.flags & RT_FLAG_FORCE_EXCHANGE);
  if (e->exchange) {
    if (c.world > 1 && !cfg->nccl_id) return done(fail(e, RT_E_INVAL, "nccl_id required when world > 1"));
    if (!g_nccl.load()) return done(fail(e, RT_E_NCCL, "libnccl.so.2 not loadable"));
    nccl_uid_t uid;
    if (cfg->nccl_id) {
      memcpy(uid.internal, cfg->nccl_id, 128);
    } else if (!g_nccl.get_uid || g_nccl.get_uid(&uid) != 0) {  // single-rank communicator
      return done(fail(e, RT_E_NCCL, "ncclGetUniqueId failed"));
    }
    int r = g_nccl.init(&e->comm, c.world, uid, c.rank);
    if (r != 0) return done(fail(e, RT_E_NCCL, std::string("ncclCommInitRank: ") + (g_nccl.errstr ? g_nccl.errstr(r) : "?")));
    CK(e, dalloc(e, &e->d_cand_all, (size_t)c.world * kTopK * 4));
    CK(e, dalloc(e, &e->d_merged, (size_t)kTopK * 4));
  }
  CK(e, cudaStreamSynchronize(e->stream));
  CK(e, cudaGetLastError());
  return done(RT_OK);
}

extern "C" rt_status rt_destroy(rt_engine* e) {
  if (!e) return RT_OK;
  if (e->stream) cudaStreamSynchronize(e->stream);
  if (e->side) cudaStreamSynchronize(e->side);
  if (e->comm && g_nccl.destroy) g_nccl.destroy(e->comm);
  if (e->d_trace) {  // unbind before the buffer goes away
    trace_bind_model(nullptr, nullptr, 0);
    trace_bind_attn(nullptr, nullptr, 0);
    trace_bind_gemm(nullptr, nullptr, 0);
    trace_bind_sched(nullptr, nullptr, 0);
  }
  for (void* p : e->allocs) cudaFree(p);
  if (e->d_wbuf) cudaFree(e->d_wbuf);
  if (e->d_pool) cudaFree(e->d_pool);
  if (e->h_mb) cudaFreeHost(e->h_mb);
  if (e->h_ring) cudaFreeHost(e->h_ring);
  if (e->h_hpool) cudaFreeHost(e->h_hpool);
  if (e->h_recs) cudaFreeHost(e->h_recs);
  if (e->h_toks) cudaFreeHost(e->h_toks);
  for (auto ev : e->ev_attn) cudaEventDestroy(ev);
  cudaEvent_t evs[] = {e->ev_plan, e->ev_post, e->ev_cand, e->ev_merge, e->ev_f0, e->ev_f1, e->ev_s0, e->ev_s1, e->ev_q1, e->ev_m0, e->ev_m1};
  for (auto ev : evs)
    if (ev) cudaEventDestroy(ev);
  if (e->stream) cudaStreamDestroy(e->stream);
  if (e->side) cudaStreamDestroy(e->side);
  delete e;
  return RT_OK;
}

// ------------------------------------------------------------------ submit
static rt_status flush_staging(rt_engine* e) {
  if (e->n_staged == 0) return RT_OK;
  CK(e, cudaMemcpyAsync(e->d_recs, e->h_recs, sizeof(SubmitRec) * e->n_staged, cudaMemcpyHostToDevice, e->stream));
  if (e->toks_staged)
    CK(e, cudaMemcpyAsync(e->d_toks, e->h_toks, 4 * e->toks_staged, cudaMemcpyHostToDevice, e->stream));
  launch_apply_submits(e->sp, e->d_recs, e->d_toks, e->n_staged, e->stream);
  e->n_staged = 0;
  e->toks_staged = 0;
  return RT_OK;
}

extern "C" rt_status rt_submit_request(rt_engine* e, int32_t agent_id, const int32_t* prompt, int32_t n_prompt,
                                       int64_t arrival_us, int64_t deadline_us, rt_utility fn,
                                       int32_t exec_window_us, int32_t max_new_tokens, const int32_t* script,
                                       int32_t n_script, int64_t* request_id_out) {
  if (!e) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  const rt_config& c = e->cfg;
  if (!(fn.alpha <= 0.0) || deadline_us < 0 || !isfinite(fn.beta) || exec_window_us < 0 || agent_id < 0)
    return fail(e, RT_E_INVAL, "bad utility function / agent");
  if (!prompt || n_prompt < 1) return fail(e, RT_E_INVAL, "empty prompt");
  for (int i = 0; i < n_prompt; ++i)
    if (prompt[i] < 0 || prompt[i] >= c.vocab) return fail(e, RT_E_INVAL, "prompt token out of range");
  const bool scripted = script != nullptr;
  if (scripted) {
    if (n_script < 1) return fail(e, RT_E_INVAL, "empty script");
    for (int i = 0; i < n_script; ++i)
      if (script[i] < 0 || script[i] >= c.vocab) return fail(e, RT_E_INVAL, "script token out of range");
    max_new_tokens = n_script;
  } else if (c.flags & RT_FLAG_NO_MODEL) {
    return fail(e, RT_E_INVAL, "engine without model needs scripted requests");
  }
  if (max_new_tokens < 1 || (int64_t)n_prompt + max_new_tokens > c.max_ctx)
    return fail(e, RT_E_INVAL, "n_prompt + max_new_tokens > max_ctx");
  const int R = (n_prompt + max_new_tokens + 15) / 16;
  // shared prefix: the longest registered prefix that is a proper head of the prompt
  int pfx = -1, n_pfx = 0;
  for (int i = 0; i < (int)e->prefixes.size(); ++i) {
    const std::vector<int32_t>& pt = e->prefixes[i];
    const int lp = (int)pt.size();
    if (lp < n_prompt && lp / 16 > n_pfx && memcmp(pt.data(), prompt, 4 * (size_t)lp) == 0) {
      pfx = i;
      n_pfx = lp / 16;
    }
  }
  // the request's own pages must fit beside the prefixes' permanent pages, or it could never
  // be admitted (and, R-MEM, would refuse every later k = 0 request of each round)
  if (R - n_pfx > c.n_pages - e->pfx_pages) return fail(e, RT_E_NOMEM, "request larger than the page pool");
  if (e->free_slots.empty()) return fail(e, RT_E_NOMEM, "task table full");
  const int64_t need = (int64_t)n_prompt + (scripted ? n_script : 0);
  if (e->n_staged >= e->recs_cap || e->toks_staged + need > e->toks_cap) {
    rt_status s = flush_staging(e);
    if (s != RT_OK) return s;
    CK(e, cudaStreamSynchronize(e->stream));
  }
  const int slot = e->free_slots.back();
  e->free_slots.pop_back();
  SubmitRec& r = e->h_recs[e->n_staged++];
  r.rid = e->n_submitted * c.world + c.rank;
  e->n_submitted++;
  r.arrival = arrival_us;
  r.ert = deadline_us;
  r.alpha = fn.alpha;
  r.beta = fn.beta;
  r.slot = slot;
  r.agent = agent_id;
  r.n_prompt = n_prompt;
  r.max_new = max_new_tokens;
  r.window = exec_window_us;
  r.scripted = scripted ? 1 : 0;
  r.pfx = pfx;
  r.n_pfx = n_pfx;
  r.tok_off = e->toks_staged;
  memcpy(e->h_toks + e->toks_staged, prompt, 4 * (size_t)n_prompt);
  e->toks_staged += n_prompt;
  if (scripted) {
    memcpy(e->h_toks + e->toks_staged, script, 4 * (size_t)n_script);
    e->toks_staged += n_script;
  }
  e->rid_slot[r.rid] = slot;
  if (request_id_out) *request_id_out = r.rid;
  return RT_OK;
}

static rt_status forward(rt_engine* e, const HostMailbox& plan, bool embed0_done = false);

// ------------------------------------------------------------ shared prefixes
// NEXT-1 (fixed prompt components pre-stored on the server): the prefix's pages are
// popped from the free stack like an admission's and never freed; its KV is computed once by
// a forward over its rows (B = 0: no logits).  Later submissions whose prompt starts with it
// point their first page-table entries at these pages and prefill only the rest (DESIGN R-PFX).
extern "C" rt_status rt_register_prefix(rt_engine* e, const int32_t* tokens, int32_t n_tokens,
                                        int32_t* prefix_id_out) {
  if (!e) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  const rt_config& c = e->cfg;
  if (!tokens || n_tokens < 16 || n_tokens % 16 != 0 || n_tokens >= c.max_ctx)
    return fail(e, RT_E_INVAL, "prefix length must be a positive multiple of 16 below max_ctx");
  for (int i = 0; i < n_tokens; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) return fail(e, RT_E_INVAL, "prefix token out of range");
  if ((int)e->prefixes.size() >= kMaxPrefixes) return fail(e, RT_E_NOMEM, "too many prefixes");
  rt_status st = flush_staging(e);
  if (st != RT_OK) return st;
  st = rt_sync(e);
  if (st != RT_OK) return st;
  const int MT = c.max_tasks, n = n_tokens / 16, pid = (int)e->prefixes.size();
  // pages available = free stack - outstanding reservations of admitted requests (AMB-26)
  DevState ds;
  CK(e, cudaMemcpy(&ds, e->d_st, sizeof(ds), cudaMemcpyDeviceToHost));
  std::vector<int32_t> holder(MT), R(MT), np(MT);
  CK(e, cudaMemcpy(holder.data(), e->tt.holder, 4 * MT, cudaMemcpyDeviceToHost));
  CK(e, cudaMemcpy(R.data(), e->tt.R, 4 * MT, cudaMemcpyDeviceToHost));
  CK(e, cudaMemcpy(np.data(), e->tt.n_pages, 4 * MT, cudaMemcpyDeviceToHost));
  int64_t outstanding = 0;
  for (int i = 0; i < MT; ++i)
    if (holder[i]) outstanding += R[i] - np[i];
  if (ds.free_top - outstanding < n) return fail(e, RT_E_NOMEM, "not enough free pages for the prefix");
  // pop n pages in stack order (the same order an admission pops them)
  std::vector<int32_t> top(n), pages(n);
  CK(e, cudaMemcpy(top.data(), e->sp.free_stack + ds.free_top - n, 4 * (size_t)n, cudaMemcpyDeviceToHost));
  for (int m = 0; m < n; ++m) pages[m] = top[n - 1 - m];
  const int slot = MT + pid;  // the prefix's page-table row
  // every write below is ordered on the engine stream (non-blocking: the legacy default
  // stream does not synchronise with it), and the host buffers live until the final sync
  CK(e, cudaMemcpyAsync(e->tt.page_table + (size_t)slot * e->pt_stride, pages.data(), 4 * (size_t)n,
                        cudaMemcpyHostToDevice, e->stream));
  const int32_t new_top = ds.free_top - n;
  CK(e, cudaMemcpyAsync(&e->d_st->free_top, &new_top, 4, cudaMemcpyHostToDevice, e->stream));
  if (!(c.flags & RT_FLAG_NO_MODEL)) {
    // rows (slot, position, token) and 16-position tiles of the prefix, then the forward
    if (n_tokens > e->rows_cap) return fail(e, RT_E_INVAL, "prefix longer than the forward row capacity");
    std::vector<int32_t> rt(n_tokens, slot), rp(n_tokens);
    for (int j = 0; j < n_tokens; ++j) rp[j] = j;
    std::vector<int4> tiles(n);
    for (int t = 0; t < n; ++t) tiles[t] = make_int4(16 * t, 16, 16 * t, slot);
    CK(e, cudaMemcpyAsync(e->sp.row_task, rt.data(), 4 * (size_t)n_tokens, cudaMemcpyHostToDevice, e->stream));
    CK(e, cudaMemcpyAsync(e->sp.row_pos, rp.data(), 4 * (size_t)n_tokens, cudaMemcpyHostToDevice, e->stream));
    CK(e, cudaMemcpyAsync(e->sp.row_tok, tokens, 4 * (size_t)n_tokens, cudaMemcpyHostToDevice, e->stream));
    CK(e, cudaMemcpyAsync(e->sp.pf_tiles, tiles.data(), sizeof(int4) * (size_t)n, cudaMemcpyHostToDevice,
                          e->stream));
    HostMailbox plan{};
    plan.B = 0;
    plan.n_rows = n_tokens;
    plan.n_prefill_rows = n_tokens;
    plan.n_pf_tiles = n;
    plan.n_dec_rows = 0;
    plan.max_seqlen = n_tokens;
    st = forward(e, plan);
    if (st != RT_OK) return st;
  }
  CK(e, cudaStreamSynchronize(e->stream));
  e->prefixes.emplace_back(tokens, tokens + n_tokens);
  e->pfx_pages += n;
  if (prefix_id_out) *prefix_id_out = pid;
  return RT_OK;
}

// ------------------------------------------------------------------ timing
static void harvest_timing(rt_engine* e) {
  if (!e->timing_pending) return;
  float ms = 0.f;
  for (int l = 0; l < e->timing_layers; ++l) {
    if (cudaEventElapsedTime(&ms, e->ev_attn[2 * l], e->ev_attn[2 * l + 1]) == cudaSuccess) {
      e->stats.attn_ms += ms;
      e->stats.attn_launches++;
    }
  }
  if (cudaEventElapsedTime(&ms, e->ev_s0, e->ev_q1) == cudaSuccess) e->stats.step_ms += ms;
  if (cudaEventElapsedTime(&ms, e->ev_s0, e->ev_s1) == cudaSuccess) e->stats.sched_ms += ms;
  if (cudaEventElapsedTime(&ms, e->ev_f1, e->ev_q1) == cudaSuccess) e->stats.sched_ms += ms;
  if (cudaEventElapsedTime(&ms, e->ev_f0, e->ev_f1) == cudaSuccess) e->stats.gemm_ms += ms;
  e->stats.attn_bytes += e->attn_bytes_pending;
  e->timing_pending = false;
  // an event pair that was not recorded this round (e.g. no forward) is not an error of the
  // step: drop the non-sticky error it left so the next CK(cudaGetLastError()) does not see it
  cudaError_t le = cudaPeekAtLastError();
  if (le == cudaErrorInvalidResourceHandle || le == cudaErrorNotReady || le == cudaErrorInvalidValue)
    cudaGetLastError();
}

// ------------------------------------------------------------------ forward
static void record_timing_event(cudaEvent_t ev, cudaStream_t s) { cudaEventRecord(ev, s); }

#ifndef RT_QKV_FOLD
#define RT_QKV_FOLD 1
#endif
#ifndef RT_RESID_PART
#define RT_RESID_PART 1
#endif
static rt_status forward(rt_engine* e, const HostMailbox& plan, bool embed0_done) {
  const rt_config& c = e->cfg;
  const int d = c.d_model, hd = c.head_dim, nq = c.n_q_heads, nkv = c.n_kv_heads, ff = c.d_ff, V = c.vocab;
  const int B = plan.B, n_rows = plan.n_rows;
  const bool timing = (c.flags & RT_FLAG_TIMING) != 0;
  cudaStream_t s = e->stream;
  SchedParams& P = e->sp;
  const float sl2 = (float)(1.4426950408889634 / sqrt((double)hd));
  const int d_tiles = (d + 127) / 128;
  int launches = 0;
  const bool lcap = e->d_lc_x != nullptr;
  if (lcap) e->lc_rows = std::min(n_rows, e->fwd_rows);
  // RT_FLAG_CAPTURE_LAYERS: device copy of a forward buffer of this chunk (first chunk only)
  auto lc_copy = [&](void* dst_base, const void* src, int l, size_t row_bytes, int row0_) {
    if (!lcap || row0_ != 0) return;
    cudaMemcpyAsync((char*)dst_base + ((size_t)l * e->fwd_rows) * row_bytes, src, (size_t)e->lc_rows * row_bytes,
                    cudaMemcpyDeviceToDevice, s);
  };
  for (int row0 = 0; row0 < n_rows; row0 += e->fwd_rows) {
    const int n = std::min(e->fwd_rows, n_rows - row0);
    if (!(row0 == 0 && embed0_done)) {  // chunk 0 of a scheduler round: k_embed_plan (rt_step)
      launch_embed(P.row_tok, row0, n, e->emb, d, e->d_x, e->d_h, e->d_ss, s);  // d_h = bf16(x), un-normed
      ++launches;
    }
    AttnArgs aa{};
    aa.q = e->d_q;
    aa.page_table = e->tt.page_table;
    aa.pt_stride = e->pt_stride;
    aa.row_task = P.row_task;
    aa.row_pos = P.row_pos;
    aa.row_seqlen = nullptr;
    aa.row0 = row0;
    aa.n_rows = n;
    aa.nq = nq;
    aa.nkv = nkv;
    aa.hd = hd;
    aa.G = nq / nkv;
    attn_plan(n, nkv, plan.max_seqlen, &aa.chunk_pages, &aa.max_chunks);
    if (attn_ws_floats(n, nq, hd, aa.max_chunks) > e->attn_ws_cap) aa.max_chunks = 1;
    if (aa.max_chunks == 1) aa.chunk_pages = e->pt_stride;
    aa.out = e->d_o;
    aa.ws = e->d_attn_ws;
    aa.tickets = e->d_attn_tickets;
    aa.scale_log2 = sl2;
    // decode rows in the scheduler's longest-context-first order (prompt rows: k_attn_prefill)
    {
      aa.row_list = P.dec_rows;
      aa.chunk_rows = n;
      aa.n_rows = plan.n_dec_rows;
      attn_plan(plan.n_dec_rows, nkv, plan.max_seqlen, &aa.chunk_pages, &aa.max_chunks);
      if (attn_ws_floats(n, nq, hd, aa.max_chunks) > e->attn_ws_cap) aa.max_chunks = 1;
      if (aa.max_chunks == 1) aa.chunk_pages = e->pt_stride;
    }
    PrefillArgs pa{};
    pa.q = e->d_q;
    pa.page_table = e->tt.page_table;
    pa.pt_stride = e->pt_stride;
    pa.tiles = P.pf_tiles;
    pa.n_tiles = plan.n_pf_tiles;
    pa.row0 = row0;
    pa.n_rows = n;
    pa.nq = nq;
    pa.nkv = nkv;
    pa.hd = hd;
    pa.G = nq / nkv;
    pa.out = e->d_o;
    pa.scale_log2 = sl2;
    const bool any_decode = plan.n_rows > plan.n_prefill_rows;
    // decode-only rounds: the QKV projection writes its raw split-K partials and the decode
    // attention runs the QKV epilogue (sum, RMSNorm scale, RoPE, KV append) for its own (row,
    // kv head) — no split-K exchange or fused epilogue on the projection's critical path
    int fold_S = (RT_QKV_FOLD && e->d_qkv_part && c.gemm_path == GEMM_PATH_AUTO &&
                  n_rows <= e->fwd_rows && n <= e->qkv_part_rows && plan.n_pf_tiles <= e->sp.pf_tiles_cap)
                     ? gemm_part_splits(e->qkv_dim, d, n)
                     : 0;
    if (fold_S > 8 || d / 128 > 64) fold_S = 0;  // the attention's fold holds <= 8 partials, <= 64 tiles
    // ... and the O / down projections write theirs too, finished by k_resid_reduce (residual
    // add, bf16 copy, RMSNorm sums) instead of a split-K exchange inside the GEMM
    auto part_s = [&](int M, int K) {
      // (at <= 128 rows the single-SM kernel's in-cluster DSMEM exchange is cheaper than the
      // extra reduce launch: measured equal or slower at C2)
      const int S = (RT_RESID_PART && fold_S > 0 && n > 128) ? gemm_part_splits(M, K, n) : 0;
      return (S > 0 && S <= 8 && M % 128 == 0) ? S : 0;
    };
    const int o_S = part_s(d, nq * hd), dn_S = part_s(d, ff);
    if (fold_S > 0) {
      aa.part = e->d_qkv_part;
      aa.part_splits = fold_S;
      aa.part_ld_n = n;
      aa.part_m = e->qkv_dim;
      aa.rs_ss = e->d_ss;
      aa.rs_tiles = d_tiles;
      aa.d_model = d;
      aa.cos = e->d_rope_cos;
      aa.sin = e->d_rope_sin;
      aa.q_out = e->d_q;
    }
    auto gemm = [&](const bf16* w, const GemmTmaSet& x, int M, int K, GemmArgs g) {
      g.M = M;
      g.N = n;
      g.K = K;
      g.sk_ws = e->d_sk_ws;
      g.sk_cnt = e->d_sk_cnt;
      g.sk_cnt_cap = e->sk_cnt_cap;
      g.force_path = c.gemm_path;
      g.dec_ws = e->d_dec_ws;
      g.dec_ws_floats = e->dec_ws_floats;
      g.dec_flags = e->d_dec_flags;
      g.dec_flags_cap = kDecFlags;
      g.dec_epoch = ++e->dec_epoch;
      launch_gemm_epi(w, x, g, 0, s);
      ++launches;
    };
    // epilogue arguments of the four decode-layer projections (a6)
    auto args_qkv = [&](int l) {  // QKV projection + RoPE + KV append (a6 -> a4 pages)
      GemmArgs g{};
      g.mode = EPI_QKV;
      QkvFuse& q = g.qkv;
      q.row_task = P.row_task;
      q.row_pos = P.row_pos;
      q.page_table = e->tt.page_table;
      q.row0 = row0;
      q.pt_stride = e->pt_stride;
      q.nq = nq;
      q.nkv = nkv;
      q.hd = hd;
      q.cos = e->d_rope_cos;
      q.sin = e->d_rope_sin;
      q.q_out = e->d_q;
      q.pool = e->d_pool + (size_t)l * e->pool_layer_bytes;
      q.q_cap = (e->d_cap_q && l == c.capture_layer) ? e->d_cap_q : nullptr;
      g.rs_ss = e->d_ss;  // attention RMSNorm applied as the epilogue's row scale
      g.rs_tiles = d_tiles;
      g.M = e->qkv_dim;
      g.N = n;
      g.K = d;
      return g;
    };
    auto args_resid = [&](int M, int K) {  // O / down projection + residual
      GemmArgs g{};
      g.mode = EPI_RESID;
      g.x = e->d_x;
      g.ss = e->d_ss;
      g.xb = e->d_h;
      g.M = M;
      g.N = n;
      g.K = K;
      return g;
    };
    auto args_gu = [&]() {  // gate/up projection (FFN RMSNorm as row scale) + SwiGLU
      GemmArgs g{};
      g.mode = EPI_SWIGLU;
      g.act = e->d_act;
      g.ff = ff;
      g.rs_ss = e->d_ss;
      g.rs_tiles = d_tiles;
      g.M = 2 * ff;
      g.N = n;
      g.K = d;
      return g;
    };
    for (int l = 0; l < c.n_layers; ++l) {
      LayerW& w = e->layers[l];
      void* pool_l = e->d_pool + (size_t)l * e->pool_layer_bytes;
      lc_copy(e->d_lc_x, e->d_x, l, (size_t)d * 4, row0);
      {
        GemmArgs g = args_qkv(l);
        if (fold_S > 0) {
          g.mode = EPI_PART;
          g.part = e->d_qkv_part;
          g.part_ld_n = n;
          g.rs_ss = nullptr;  // the row scale is applied by the attention
        }
        gemm(w.qkv, e->x_h, e->qkv_dim, d, g);
      }
      aa.pool = pool_l;
      aa.q_cap = (fold_S > 0 && e->d_cap_q && l == c.capture_layer) ? e->d_cap_q : nullptr;
      aa.out_f32 = (e->d_cap_o && l == c.capture_layer) ? e->d_cap_o : nullptr;
      if (timing && row0 == 0) record_timing_event(e->ev_attn[2 * l], s);
      if (any_decode) {
        launch_attention(aa, s);
        ++launches;
      }
      if (timing && row0 == 0) record_timing_event(e->ev_attn[2 * l + 1], s);
      if (fold_S > 0 && pa.n_tiles > 0) {  // the folded QKV epilogue of the prompt rows
        launch_qkv_finish(aa, P.pf_tiles, pa.n_tiles, s);
        ++launches;
      }
      if (pa.n_tiles > 0) {  // prompt rows of k = 0 admissions
        pa.pool = pool_l;
        pa.out_f32 = aa.out_f32;
        launch_attention_prefill(pa, s);
        ++launches;
      }
      lc_copy(e->d_lc_q, e->d_q, l, (size_t)nq * hd * 2, row0);  // (after the attention: q of a fold)
      lc_copy(e->d_lc_o, e->d_o, l, (size_t)nq * hd * 2, row0);
      {  // O projection + residual
        GemmArgs g = args_resid(d, nq * hd);
        if (o_S > 0) {
          g.mode = EPI_PART;
          g.part = e->d_qkv_part;
          g.part_ld_n = n;
        }
        gemm(w.o, e->x_o, d, nq * hd, g);
        if (o_S > 0) {
          launch_resid_reduce(e->d_qkv_part, o_S, n, n, d, e->d_x, e->d_h, e->d_ss, s);
          ++launches;
        }
      }
      lc_copy(e->d_lc_xmid, e->d_x, l, (size_t)d * 4, row0);
      {  // gate/up projection (FFN RMSNorm as row scale) + SwiGLU
        GemmArgs g = args_gu();
        gemm(w.gu, e->x_h, 2 * ff, d, g);
      }
      lc_copy(e->d_lc_act, e->d_act, l, (size_t)ff * 2, row0);
      {  // down projection + residual
        GemmArgs g = args_resid(d, ff);
        if (dn_S > 0) {
          g.mode = EPI_PART;
          g.part = e->d_qkv_part;
          g.part_ld_n = n;
        }
        gemm(w.d, e->x_act, d, ff, g);
        if (dn_S > 0) {
          launch_resid_reduce(e->d_qkv_part, dn_S, n, n, d, e->d_x, e->d_h, e->d_ss, s);
          ++launches;
        }
      }
    }
    lc_copy(e->d_lc_x, e->d_x, c.n_layers, (size_t)d * 4, row0);
    // logits rows: final RMSNorm applied while gathering them
    if (B > 0) {
      launch_gather_norm(P.slot_row, B, row0, n, e->d_x, e->d_ss, d, e->d_hfin, s);
      ++launches;
    }
  }
  if (B > 0) {  // lm_head + greedy argmax (a8); B = 0: prefix registration (KV only)
    GemmArgs g{};
    g.mode = EPI_ARGMAX;
    g.M = V;
    g.N = B;
    g.K = d;
    g.out = e->d_logits;
    g.part_val = e->d_am_val;
    g.part_idx = e->d_am_idx;
    launch_gemm_epi(e->lm, e->x_hfin, g, 0, s);
    launch_argmax_reduce(e->d_am_val, e->d_am_idx, (V + 127) / 128, B, P.argmax_tok, s);
    launches += 2;
  }
  CK(e, cudaGetLastError());
  e->stats.kernel_launches += launches;
  if (timing) e->timing_layers = c.n_layers;
  return RT_OK;
}

// -------------------------------------------------------------------- step
extern "C" rt_status rt_step(rt_engine* e, int64_t now_us, rt_round_info* info) {
  if (!e) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  const rt_config& c = e->cfg;
  cudaStream_t s = e->stream;
  const bool timing = (c.flags & RT_FLAG_TIMING) != 0;
  if (e->merge_pending) CK(e, cudaStreamWaitEvent(s, e->ev_merge, 0));
  if (e->timing_pending) {
    CK(e, cudaEventSynchronize(e->ev_post));
    harvest_timing(e);
  }
  rt_status st = flush_staging(e);
  if (st != RT_OK) return st;
  if (timing) cudaEventRecord(e->ev_s0, s);
  const volatile HostMailbox* mb = e->h_mb;
  const int64_t seq0 = mb->plan_seq;
  launch_sched_pre(e->sp, now_us, s);
  if (timing) cudaEventRecord(e->ev_s1, s);
  // the first chunk's embedding goes in right behind the scheduler, before the handshake: it
  // reads the row count from the device state, so it runs while the host spins on the plan
  // and launches the layers (hides the plan handshake behind the embedding)
  const bool embed0 = !(c.flags & RT_FLAG_NO_MODEL);
  if (embed0) {
    launch_embed_plan(e->sp.row_tok, &e->d_st->n_rows, e->fwd_rows, e->emb, c.d_model, e->d_x, e->d_h, e->d_ss, s);
    e->stats.kernel_launches++;
  }
  CK(e, cudaGetLastError());
  // plan handshake: spin on the sequence number k_sched_pre writes last into the mapped
  // mailbox (an event record + synchronize cost ~5 us more per round); the stream is polled
  // now and then so a device fault cannot hang the host
  for (uint32_t it = 1; mb->plan_seq == seq0; ++it) {
    if ((it & 1023) == 0) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q != cudaSuccess && q != cudaErrorNotReady) return fail(e, RT_E_CUDA, cudaGetErrorString(q));
      if (q == cudaSuccess && mb->plan_seq == seq0) return fail(e, RT_E_STATE, "plan handshake: no plan published");
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  HostMailbox plan;
  memcpy(&plan, (const void*)mb, sizeof(plan));
  e->plan = plan;
  if (info) {
    memset(info, 0, sizeof(*info));
    info->t_us = plan.t_us;
    info->round_us = plan.round_us;
    info->n_waiting = plan.n_waiting;
    info->n_running = plan.idle ? 0 : plan.B;
    info->n_admitted = plan.n_admitted;
    info->n_refused_mem = plan.n_refused_mem;
    info->n_refused_wcet = plan.n_refused_wcet;
    info->n_rows = plan.n_rows;
    info->n_prefill_rows = plan.n_prefill_rows;
    info->n_evicted = plan.n_evicted;
    info->n_restored = plan.n_restored;
  }
  // a12: allgather of this round's local top-K candidates on the side stream.  EVERY round
  // (idle and B == 0 rounds too, whose candidates are empty): the allgather is a collective,
  // so every rank must issue exactly one per rt_step call
  if (e->exchange) {
    CK(e, cudaEventRecord(e->ev_cand, s));
    CK(e, cudaStreamWaitEvent(e->side, e->ev_cand, 0));
    int r = g_nccl.allgather(e->sp.cand, e->d_cand_all, kTopK * 4, kNcclFloat64, e->comm, e->side);
    if (r != 0) return fail(e, RT_E_NCCL, "ncclAllGather failed");
    launch_merge_cand(e->d_cand_all, c.world, e->d_merged, e->side);
    CK(e, cudaEventRecord(e->ev_merge, e->side));
    e->merge_pending = true;
  }
  if (plan.idle || plan.B == 0) return RT_OK;
  // KV eviction / restore copies of this round (before the forward reuses the pages):
  // evictions first (a restore may re-pop a page an eviction just released)
  if (plan.n_swap > 0 && e->h_hpool) {
    const int L = c.n_layers;
    const int64_t blk = e->hpool_page_bytes / L;
    launch_kv_swap(e->sp.swap, plan.n_swap_ev, e->d_pool, e->pool_layer_bytes, e->d_hpool, blk, L, s);
    launch_kv_swap(e->sp.swap + plan.n_swap_ev, plan.n_swap - plan.n_swap_ev, e->d_pool, e->pool_layer_bytes,
                   e->d_hpool, blk, L, s);
    CK(e, cudaGetLastError());
  }
  if (timing) cudaEventRecord(e->ev_f0, s);
  if (!(c.flags & RT_FLAG_NO_MODEL)) {
    st = forward(e, plan, embed0);
    if (st != RT_OK) return st;
  }
  if (timing) {
    cudaEventRecord(e->ev_f1, s);
    e->timing_pending = true;
    if (c.flags & RT_FLAG_NO_MODEL) e->timing_layers = 0;
  }
  launch_sched_post(e->sp, s);
  if (timing) {
    cudaEventRecord(e->ev_q1, s);
    const rt_config& cc = e->cfg;
    e->attn_bytes_pending = (double)cc.n_layers *
        ((double)plan.attn_tokens * cc.n_kv_heads * cc.head_dim * 4.0 +
         (double)std::min(plan.n_rows, e->fwd_rows) * cc.n_q_heads * cc.head_dim * 4.0);
  }
  CK(e, cudaEventRecord(e->ev_post, s));
  CK(e, cudaGetLastError());
  e->post_pending = true;
  e->stats.rounds++;
  e->stats.tokens += plan.B;
  e->stats.prefill_tokens += plan.n_prefill_rows;
  return RT_OK;
}

static rt_status wait_post(rt_engine* e) {
  if (e->post_pending) {
    CK(e, cudaEventSynchronize(e->ev_post));
    e->post_pending = false;
  }
  return RT_OK;
}

extern "C" rt_status rt_sync(rt_engine* e) {
  if (!e) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  CK(e, cudaStreamSynchronize(e->stream));
  CK(e, cudaStreamSynchronize(e->side));
  e->post_pending = false;
  harvest_timing(e);
  return RT_OK;
}

// Drains the mapped segment ring up to the count k_sched_post published last.  `wait`:
// first block until the last launched round is complete (rt_poll_segment); without it
// (rt_poll_segment_ready) only the rounds the device has already retired are visible —
// k_sched_post writes every record, then (after a barrier and a system-scope fence) the
// count, so a count read here covers only complete records.
static rt_status poll_ring(rt_engine* e, rt_segment* out, int32_t cap, int32_t* n_out, bool wait) {
  if (!e || !n_out || (cap > 0 && !out)) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  *n_out = 0;
  if (wait) {
    rt_status st = wait_post(e);
    if (st != RT_OK) return st;
  }
  const volatile HostMailbox* mb = e->h_mb;
  const int64_t published = mb->seg_written;
  std::atomic_thread_fence(std::memory_order_acquire);
  if (published - e->seg_read > e->ring_cap) return fail(e, RT_E_STATE, "segment ring overflow (poll more often)");
  int32_t n = 0;
  while (n < cap && e->seg_read < published) {
    const SegRec& r = e->h_ring[e->seg_read % e->ring_cap];
    memcpy(&out[n], &r, sizeof(rt_segment));
    ++n;
    ++e->seg_read;
  }
  // the host saw the final segment: the task slot may be reused (the device
  // ignores T_FINISHED slots; apply_submits overwrites every field)
  for (int i = 0; i < n; ++i) {
    if (out[i].reason != RT_STOP_EOS && out[i].reason != RT_STOP_MAXNEW) continue;
    auto it = e->rid_slot.find(out[i].request_id);
    if (it != e->rid_slot.end()) {
      e->free_slots.push_back(it->second);
      e->rid_slot.erase(it);
    }
  }
  e->stats.segments += n;
  *n_out = n;
  return RT_OK;
}

extern "C" rt_status rt_poll_segment(rt_engine* e, rt_segment* out, int32_t cap, int32_t* n_out) {
  return poll_ring(e, out, cap, n_out, true);
}

extern "C" rt_status rt_poll_segment_ready(rt_engine* e, rt_segment* out, int32_t cap, int32_t* n_out) {
  return poll_ring(e, out, cap, n_out, false);
}

extern "C" rt_status rt_last_round(rt_engine* e, rt_round_info* info) {
  if (!e || !info) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  rt_status st = wait_post(e);
  if (st != RT_OK) return st;
  const volatile HostMailbox* mb = e->h_mb;
  memset(info, 0, sizeof(*info));
  info->t_us = mb->t_us;
  info->round_us = mb->round_us;
  info->n_waiting = mb->n_waiting;
  info->n_running = mb->idle ? 0 : mb->B;
  info->n_admitted = mb->n_admitted;
  info->n_stopped = mb->idle ? 0 : mb->n_stopped;
  info->n_refused_mem = mb->n_refused_mem;
  info->n_refused_wcet = mb->n_refused_wcet;
  info->n_rows = mb->n_rows;
  info->n_prefill_rows = mb->n_prefill_rows;
  return RT_OK;
}

extern "C" rt_status rt_set_timing(rt_engine* e, int32_t on) {
  if (!e || on < 0 || on > 1) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  if (on) e->cfg.flags |= RT_FLAG_TIMING;
  else e->cfg.flags &= ~RT_FLAG_TIMING;
  return RT_OK;
}

extern "C" rt_status rt_mark(rt_engine* e, int32_t which) {
  if (!e || which < 0 || which > 1) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  CK(e, cudaEventRecord(which == 0 ? e->ev_m0 : e->ev_m1, e->stream));
  return RT_OK;
}

extern "C" rt_status rt_elapsed_ms(rt_engine* e, double* ms_out) {
  if (!e || !ms_out) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  CK(e, cudaEventSynchronize(e->ev_m1));
  float ms = 0.f;
  CK(e, cudaEventElapsedTime(&ms, e->ev_m0, e->ev_m1));
  *ms_out = ms;
  return RT_OK;
}

extern "C" rt_status rt_nccl_unique_id(uint8_t* out128) {
  if (!out128) return RT_E_INVAL;
  if (!g_nccl.load() || !g_nccl.get_uid) return fail(nullptr, RT_E_NCCL, "libnccl.so.2 not loadable");
  nccl_uid_t uid;
  const int r = g_nccl.get_uid(&uid);
  if (r != 0) return fail(nullptr, RT_E_NCCL, "ncclGetUniqueId failed");
  memcpy(out128, uid.internal, 128);
  return RT_OK;
}

extern "C" rt_status rt_get_stats(rt_engine* e, rt_stats* out) {
  if (!e || !out) return RT_E_INVAL;
  rt_status st = rt_sync(e);
  if (st != RT_OK) return st;
  *out = e->stats;
  return RT_OK;
}

extern "C" rt_status rt_reset_stats(rt_engine* e) {
  if (!e) return RT_E_INVAL;
  rt_status st = rt_sync(e);
  if (st != RT_OK) return st;
  memset(&e->stats, 0, sizeof(e->stats));
  if (e->d_trace_n) CK(e, cudaMemset(e->d_trace_n, 0, sizeof(unsigned)));
  return RT_OK;
}

// -------------------------------------------------------------------- dumps
static rt_status copy_out(rt_engine* e, void* dst, int64_t bytes, const void* src, int64_t need,
                          int64_t* bytes_out, bool device_src = true) {
  if (bytes_out) *bytes_out = need;
  if (!dst) return RT_OK;
  if (bytes < need) return fail(e, RT_E_INVAL, "dump buffer too small");
  if (need == 0) return RT_OK;
  if (device_src) CK(e, cudaMemcpy(dst, src, need, cudaMemcpyDeviceToHost));
  else memcpy(dst, src, need);
  return RT_OK;
}

extern "C" rt_status rt_debug_dump(rt_engine* e, int32_t what, void* dst, int64_t bytes, int64_t* bytes_out) {
  if (!e) return RT_E_INVAL;
  if (e->sticky) return RT_E_CUDA;
  rt_status st = rt_sync(e);
  if (st != RT_OK) return st;
  const rt_config& c = e->cfg;
  const int MT = c.max_tasks;
  DevState ds;
  CK(e, cudaMemcpy(&ds, e->d_st, sizeof(ds), cudaMemcpyDeviceToHost));
  const int B = ds.B, n_rows = ds.n_rows;
  const int layer = (what >> 16) & 0x7FFF;
  what &= 0xFFFF;
  if (what >= RT_DUMP_LAYER_X && what <= RT_DUMP_LAYER_ACT) {
    if (!e->d_lc_x) return fail(e, RT_E_STATE, "RT_FLAG_CAPTURE_LAYERS not set");
    if (layer > c.n_layers || (layer == c.n_layers && what != RT_DUMP_LAYER_X))
      return fail(e, RT_E_INVAL, "layer out of range");
    const int R = e->fwd_rows, nr = e->lc_rows;
    const size_t qb = (size_t)c.n_q_heads * c.head_dim * 2;
    switch (what) {
      case RT_DUMP_LAYER_X:
        return copy_out(e, dst, bytes, e->d_lc_x + (size_t)layer * R * c.d_model, (int64_t)nr * c.d_model * 4, bytes_out);
      case RT_DUMP_LAYER_XMID:
        return copy_out(e, dst, bytes, e->d_lc_xmid + (size_t)layer * R * c.d_model, (int64_t)nr * c.d_model * 4,
                        bytes_out);
      case RT_DUMP_LAYER_Q:
        return copy_out(e, dst, bytes, (const char*)e->d_lc_q + (size_t)layer * R * qb, (int64_t)nr * qb, bytes_out);
      case RT_DUMP_LAYER_O:
        return copy_out(e, dst, bytes, (const char*)e->d_lc_o + (size_t)layer * R * qb, (int64_t)nr * qb, bytes_out);
      default:
        return copy_out(e, dst, bytes, e->d_lc_act + (size_t)layer * R * c.d_ff, (int64_t)nr * c.d_ff * 2, bytes_out);
    }
  }
  switch (what) {
    case RT_DUMP_TASKS: {
      std::vector<int64_t> v((size_t)MT * 10);
      std::vector<int64_t> rid(MT);
      std::vector<int32_t> a(MT);
      CK(e, cudaMemcpy(rid.data(), e->tt.rid, 8 * MT, cudaMemcpyDeviceToHost));
      for (int i = 0; i < MT; ++i) v[(size_t)i * 10] = rid[i];
      int32_t* fields[] = {e->tt.state, e->tt.k,       e->tt.ctx, e->tt.n_pages, e->tt.n_gen,
                           e->tt.seg_tok, e->tt.R, e->tt.evicted, e->tt.n_hpages};
      for (int f = 0; f < 9; ++f) {
        CK(e, cudaMemcpy(a.data(), fields[f], 4 * MT, cudaMemcpyDeviceToHost));
        for (int i = 0; i < MT; ++i) v[(size_t)i * 10 + 1 + f] = a[i];
      }
      return copy_out(e, dst, bytes, v.data(), (int64_t)v.size() * 8, bytes_out, false);
    }
    case RT_DUMP_PAGE_TABLES:
      return copy_out(e, dst, bytes, e->tt.page_table, (int64_t)MT * e->pt_stride * 4, bytes_out);
    case RT_DUMP_ROUND: {
      std::vector<int32_t> v;
      v.push_back(B);
      v.push_back(n_rows);
      v.push_back(ds.n_admitted);
      v.push_back(ds.free_top);
      std::vector<int32_t> slots(std::max(B, 1)), toks(std::max(B, 1)), am(std::max(B, 1)),
          adm(std::max(ds.n_admitted, 1));
      std::vector<int64_t> rid(MT);
      CK(e, cudaMemcpy(rid.data(), e->tt.rid, 8 * MT, cudaMemcpyDeviceToHost));
      if (B > 0) {
        CK(e, cudaMemcpy(slots.data(), e->sp.round_slots, 4 * B, cudaMemcpyDeviceToHost));
        CK(e, cudaMemcpy(toks.data(), e->sp.slot_tok, 4 * B, cudaMemcpyDeviceToHost));
        CK(e, cudaMemcpy(am.data(), e->sp.argmax_tok, 4 * B, cudaMemcpyDeviceToHost));
      }
      if (ds.n_admitted > 0) CK(e, cudaMemcpy(adm.data(), e->sp.admitted, 4 * ds.n_admitted, cudaMemcpyDeviceToHost));
      for (int i = 0; i < B; ++i) v.push_back((int32_t)rid[slots[i]]);
      for (int i = 0; i < B; ++i) v.push_back(toks[i]);
      for (int i = 0; i < B; ++i) v.push_back((c.flags & RT_FLAG_NO_MODEL) ? -1 : am[i]);
      for (int i = 0; i < ds.n_admitted; ++i) v.push_back((int32_t)rid[adm[i]]);
      return copy_out(e, dst, bytes, v.data(), (int64_t)v.size() * 4, bytes_out, false);
    }
    case RT_DUMP_LOGITS:
      if (!e->d_logits) return fail(e, RT_E_STATE, "RT_FLAG_KEEP_LOGITS not set");
      return copy_out(e, dst, bytes, e->d_logits, (int64_t)B * c.vocab * 4, bytes_out);
    case RT_DUMP_HIDDEN:
      if (!e->d_hfin) return fail(e, RT_E_STATE, "no model");
      return copy_out(e, dst, bytes, e->d_hfin, (int64_t)B * c.d_model * 2, bytes_out);
    case RT_DUMP_CAPTURE_Q:
      if (!e->d_cap_q) return fail(e, RT_E_STATE, "RT_FLAG_CAPTURE not set");
      return copy_out(e, dst, bytes, e->d_cap_q, (int64_t)n_rows * c.n_q_heads * c.head_dim * 4, bytes_out);
    case RT_DUMP_CAPTURE_O:
      if (!e->d_cap_o) return fail(e, RT_E_STATE, "RT_FLAG_CAPTURE not set");
      return copy_out(e, dst, bytes, e->d_cap_o, (int64_t)n_rows * c.n_q_heads * c.head_dim * 4, bytes_out);
    case RT_DUMP_ROWS: {
      std::vector<int32_t> a(std::max(n_rows, 1)), b(std::max(n_rows, 1)), t(std::max(n_rows, 1)), v;
      if (n_rows > 0) {
        CK(e, cudaMemcpy(a.data(), e->sp.row_task, 4 * n_rows, cudaMemcpyDeviceToHost));
        CK(e, cudaMemcpy(b.data(), e->sp.row_pos, 4 * n_rows, cudaMemcpyDeviceToHost));
        CK(e, cudaMemcpy(t.data(), e->sp.row_tok, 4 * n_rows, cudaMemcpyDeviceToHost));
      }
      for (int i = 0; i < n_rows; ++i) {
        v.push_back(a[i]);
        v.push_back(b[i]);
        v.push_back(t[i]);
      }
      return copy_out(e, dst, bytes, v.data(), (int64_t)v.size() * 4, bytes_out, false);
    }
    case RT_DUMP_KV_LAYER:
    case RT_DUMP_LAYER_KV: {
      if (!e->d_pool) return fail(e, RT_E_STATE, "no model");
      const int kl = what == RT_DUMP_LAYER_KV ? layer : c.capture_layer;
      if (kl >= c.n_layers) return fail(e, RT_E_INVAL, "layer out of range");
      const int64_t need = (int64_t)c.n_pages * 2 * c.n_kv_heads * 16 * c.head_dim * 2;
      if (bytes_out) *bytes_out = need;
      if (!dst) return RT_OK;
      if (bytes < need) return fail(e, RT_E_INVAL, "dump buffer too small");
      bf16* tmp = nullptr;
      CK(e, cudaMalloc(&tmp, need));
      launch_kv_read(e->d_pool + (size_t)kl * e->pool_layer_bytes, tmp, c.n_pages, c.n_kv_heads,
                     c.head_dim, e->stream);
      CK(e, cudaStreamSynchronize(e->stream));
      cudaError_t r = cudaMemcpy(dst, tmp, need, cudaMemcpyDeviceToHost);
      cudaFree(tmp);
      CK(e, r);
      return RT_OK;
    }
    case RT_DUMP_FREE_STACK:
      return copy_out(e, dst, bytes, e->sp.free_stack, (int64_t)ds.free_top * 4, bytes_out);
    case RT_DUMP_HOST_PAGE_TABLES:
      return copy_out(e, dst, bytes, e->tt.hpage_table, (int64_t)MT * e->pt_stride * 4, bytes_out);
    case RT_DUMP_HOST_FREE_STACK:
      return copy_out(e, dst, bytes, e->sp.hfree_stack, (int64_t)ds.hfree_top * 4, bytes_out);
    case RT_DUMP_TASK_SLOTS:
      return copy_out(e, dst, bytes, e->sp.round_slots, (int64_t)B * 4, bytes_out);
    case RT_DUMP_MERGED: {
      if (!e->d_merged) return fail(e, RT_E_STATE, "world == 1");
      std::vector<double> m(kTopK * 4);
      CK(e, cudaMemcpy(m.data(), e->d_merged, 8 * m.size(), cudaMemcpyDeviceToHost));
      std::vector<int64_t> v(kTopK * 4);
      for (int i = 0; i < kTopK * 4; ++i) memcpy(&v[i], &m[i], 8);
      return copy_out(e, dst, bytes, v.data(), (int64_t)v.size() * 8, bytes_out, false);
    }
    case RT_DUMP_TRACE: {
      if (!e->d_trace) return fail(e, RT_E_STATE, "RT_FLAG_TRACE not set");
      unsigned n = 0;
      CK(e, cudaMemcpy(&n, e->d_trace_n, sizeof n, cudaMemcpyDeviceToHost));
      n = std::min(n, e->trace_cap);
      return copy_out(e, dst, bytes, e->d_trace, (int64_t)n * 48, bytes_out);
    }
    default:
      return fail(e, RT_E_INVAL, "unknown dump kind");
  }
}
