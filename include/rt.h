/* rt.h — C ABI of the B200 segmented-decode serving engine (arxiv 2412.18695).
 *
 * The calls follow the paper's problem statement: "A robotic agent submits a
 * request, along with its time-sensitive requirement in terms of the Expected
 * Response Time or deadline (ERT in TUF), the tolerance level for missing
 * deadlines (alpha in TUF), and the time-sensitive degree (beta in TUF)"
 * (§3); the system "evaluates resource availability whenever the
 * LLM inference engine completes a decoding iteration" and
 * "dispatches the generated segment to the corresponding agent for immediate
 * action".  BASELINE.json fixes the verbs
 * submit_request(agent, prompt, deadline, utility_fn), step(), poll_segment().
 *
 * Conventions
 *   - Every call returns rt_status (0 = RT_OK, < 0 = error).  No C++ exception
 *     or longjmp crosses the ABI.  RT_E_CUDA / RT_E_NCCL are sticky: the engine
 *     is unusable afterwards (only rt_destroy / rt_last_error are valid).
 *   - Times are int64 microseconds (reading AMB-23).
 *   - All pointers are HOST pointers unless stated otherwise; the engine copies
 *     what it needs before returning (caller keeps ownership).
 *   - One thread per engine; one engine per GPU/process.  rt_step is
 *     asynchronous except for one small pinned-memory handshake (the round plan).
 *   - No CPU fallback: rt_create fails with RT_E_CUDA when no sm_100 device is
 *     present.
 */
#ifndef RT_H_
#define RT_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t rt_status;
enum {
  RT_OK = 0,
  RT_E_INVAL = -1,   /* bad argument (see each call) */
  RT_E_NOMEM = -2,   /* task table full, request larger than the page pool, HBM exhausted */
  RT_E_CUDA = -3,    /* CUDA error (sticky) */
  RT_E_NCCL = -4,    /* NCCL error (sticky) */
  RT_E_STATE = -5    /* call not valid in the engine's current state */
};

enum { RT_CLOCK_VIRTUAL = 0, RT_CLOCK_WALL = 1 };
enum { RT_POLICY_PUD = 0, RT_POLICY_FCFS = 1, RT_POLICY_EDF = 2 };
/* Stop reasons, in priority order EOS > MAXNEW > SKILL_WINDOW > CAP (DESIGN.md a9). */
enum { RT_STOP_NONE = 0, RT_STOP_EOS = 1, RT_STOP_MAXNEW = 2, RT_STOP_SKILL = 3, RT_STOP_CAP = 4 };
/* Segmentation modes (rt_config.seg_mode, the paper's comparison systems,
 * PAPER.md:576-584, 657-661):
 *   RT_SEG_SUSPEND  the method: a segment ends at the stop checker's boundary, the request
 *                   is suspended (KV retained) and re-enters the priority queue
 *   RT_SEG_STREAM   "vLLM-stream": a segment record is delivered at every skill boundary
 *                   (window rule) but the request keeps decoding in its slot (no suspension,
 *                   no CAP boundary)
 *   RT_SEG_NONE     "vLLM": no segmentation, one record at EOS / max_new_tokens
 * In STREAM / NONE modes a delivered segment is at most RT_SEG_MAX_TOKENS tokens (a longer
 * run is cut there with reason RT_STOP_CAP). */
enum { RT_SEG_SUSPEND = 0, RT_SEG_STREAM = 1, RT_SEG_NONE = 2 };
enum { RT_GRAMMAR_TOKEN = 0, RT_GRAMMAR_SKILL = 1, RT_GRAMMAR_SENTENCE = 2, RT_GRAMMAR_PARAGRAPH = 3 };
/* token classes of rt_config.tok_class: 1 .. 63 skill names, digits RT_TC_DIGIT0 + d */
enum { RT_TC_OTHER = 0, RT_TC_DIGIT0 = 64, RT_TC_LPAREN = 80, RT_TC_RPAREN = 81, RT_TC_SEMI = 82,
       RT_TC_WORD = 90, RT_TC_SENT_END = 91, RT_TC_PARA_END = 92 };
#define RT_MAX_SKILL_NAMES 63
#define RT_SEG_MAX_TOKENS 128
/* rt_config.flags */
enum {
  RT_FLAG_NO_MODEL = 1,     /* scheduling-only engine: scripted tokens, no forward pass */
  RT_FLAG_KEEP_LOGITS = 2,  /* materialise fp32 logits of the last round (parity tests) */
  RT_FLAG_CAPTURE = 4,      /* keep q / attention output (fp32) of layer capture_layer */
  RT_FLAG_TIMING = 8,       /* CUDA-event timing of attention / GEMM launches (rt_stats) */
  RT_FLAG_FORCE_EXCHANGE = 16, /* run the per-round NCCL allgather + merge even when world == 1 */
  RT_FLAG_TRACE = 64,          /* per-CTA %globaltimer records of every kernel (RT_DUMP_TRACE) */
  RT_FLAG_CAPTURE_LAYERS = 128 /* keep every layer's intermediates of the last round (RT_DUMP_LAYER_*;
                                  the round's first max_rows_per_forward rows; parity tests only:
                                  a device copy after each projection / attention launch) */
};
/* Projection kernel path (rt_config.gemm_path, rt_op_gemm_tiled): AUTO = the measured dispatch
 * (DESIGN.md §6); the others force one kernel wherever it applies, for parity tests:
 *   RT_GEMM_PATH_SPLITK   k_gemm_tc: one 128-row tile per CTA, cluster split-K
 *   RT_GEMM_PATH_STREAMK  k_gemm_sk: hybrid data-parallel + stream-K (N > 128 rows)
 *   RT_GEMM_PATH_PAIR     k_gemm_2sm: CTA pairs, tcgen05.mma.cta_group::2 (N > 128 rows)
 *   RT_GEMM_PATH_DECPAIR  k_gemm_dec: CTA pairs + cluster split-K over pairs (N <= 256 rows,
 *                         weight rows a multiple of 256, few pair-tiles; the default for
 *                         129..256-row rounds) */
enum { RT_GEMM_PATH_AUTO = 0, RT_GEMM_PATH_SPLITK = 1, RT_GEMM_PATH_STREAMK = 2, RT_GEMM_PATH_PAIR = 3,
       RT_GEMM_PATH_DECPAIR = 4 };

typedef struct rt_engine rt_engine;

/* Eq. 1 family only: TUF(t) = min(beta, alpha (t - ERT) + beta), alpha <= 0
 * (SPEC.md:32-35). */
typedef struct { double alpha, beta; } rt_utility;

typedef struct {
  /* replicas (BASELINE.json: agents partitioned over GPUs, one allgather per round):
   * 1 <= world <= 8 (one node).  With world > 1 every rt_step call is a collective (one
   * ncclAllGather of the round's candidates, idle rounds included): every rank must call
   * rt_step the same number of times. */
  int32_t rank, world;
  const uint8_t* nccl_id;           /* 128-byte ncclUniqueId (host); NULL when world == 1 */
  int32_t device;                   /* CUDA device ordinal */
  /* model shape (Llama-3 family; random init, DESIGN.md AMB-15) */
  int32_t n_layers, d_model, n_q_heads, n_kv_heads, head_dim, d_ff, vocab;
  uint64_t weight_seed;
  float init_std;                   /* 0.02 */
  /* paged KV pool + tables */
  int32_t page_tokens;              /* must be 16 */
  int32_t max_batch;                /* running slots per round */
  int32_t max_tasks;                /* task-table capacity (<= 2048) */
  int32_t max_ctx;                  /* prompt + max_new_tokens bound */
  int32_t n_pages;                  /* KV pages in the pool (0: derive from kv_pool_bytes) */
  int64_t kv_pool_bytes;
  int32_t max_rows_per_forward;     /* prefill chunk size (rows), >= max_batch */
  /* method parameters */
  int32_t max_seg_tokens;           /* 10, <= 16 */
  int32_t g_us;                     /* G(s_k) = 90000 */
  int32_t net_us;                   /* 8000 */
  int32_t eps_l_us;                 /* 1000 */
  int32_t speed_window;             /* 5, <= 8 */
  int32_t max_admit_per_round;      /* AMB-8; <= 0 means unbounded */
  int32_t policy;                   /* RT_POLICY_* */
  int32_t clock_mode;               /* RT_CLOCK_* */
  /* VIRTUAL clock cost model (DESIGN.md AMB-24), integers in microseconds */
  int32_t base_us, gamma_ppm, kv_us_per_1k, prefill_us_per_tok;
  int64_t t0_us;
  /* stop-checker tables [vocab], copied at create (token -> skill id / E_min µs) */
  const int16_t* tok_skill;
  const int32_t* tok_exec_min_us;
  int32_t eos_id;
  int32_t flags;                    /* RT_FLAG_* */
  int32_t capture_layer;
  int32_t seg_mode;                 /* RT_SEG_* (0 = the method) */
  int32_t wcet_off;                 /* 1: no WCET admission gate (the baselines) */
  /* KV eviction to host memory + restore (PAPER.md:226-229 context caching; DESIGN.md
   * R-EVICT): host_pages pinned host pages of one 16-token page across all layers
   * (n_layers x n_kv_heads x 2 x 16 x head_dim bf16 = 2 MiB at 8B dims); 0 = off.
   * swap_us_per_page: VIRTUAL clock cost of one evicted or restored page. */
  int32_t host_pages;
  int32_t swap_us_per_page;
  /* Stop grammar ("detokenizes token IDs as they are
   * generated in order to check an executable skill has been generated"
   * "regular expression matching", PAPER.md:606-609 chatbot sentence / paragraph segments):
   *   RT_GRAMMAR_TOKEN      one token = one (skill, parameter): tok_skill / tok_exec_min_us
   *   RT_GRAMMAR_SKILL      multi-token statements  name ( digits ) ;  recognised by a DFA over
   *                         tok_class; E_min = skill_base_us[name] + skill_unit_us[name] * arg
   *   RT_GRAMMAR_SENTENCE   chatbot: every word token adds word_us of reading time, a sentence
   *                         end (or paragraph end) is the boundary
   *   RT_GRAMMAR_PARAGRAPH  chatbot: a paragraph end is the boundary
   * tok_class [vocab] (copied; NULL only with RT_GRAMMAR_TOKEN): RT_TC_* below; names are
   * classes 1 .. 63 (skill index + 1).  skill_base_us / skill_unit_us [63] (copied). */
  int32_t stop_grammar;
  const int16_t* tok_class;
  const int32_t* skill_base_us;
  const int32_t* skill_unit_us;
  int32_t word_us;
  int32_t gemm_path;                /* RT_GEMM_PATH_* (0: measured dispatch) */
} rt_config;

typedef struct {
  int64_t request_id;
  int32_t agent_id, k, tok_begin, tok_end, n_skills, reason;
  int64_t est_exec_us;              /* sum of E_min over the segment's skills */
  int64_t dispatch_us;              /* clock at the end of the producing round */
  int32_t tokens[RT_SEG_MAX_TOKENS]; /* the first tok_end - tok_begin are valid */
} rt_segment;

typedef struct {
  int64_t t_us, round_us;
  int32_t n_waiting, n_running, n_admitted, n_stopped, n_refused_mem, n_refused_wcet;
  int32_t n_rows, n_prefill_rows;
  int32_t n_evicted, n_restored;    /* requests whose KV went to / came back from host */
} rt_round_info;

typedef struct {
  int64_t rounds, tokens, segments, prefill_tokens;
  double attn_ms, gemm_ms, sched_ms, step_ms;   /* CUDA-event sums (RT_FLAG_TIMING) */
  int64_t attn_launches, gemm_launches, kernel_launches;
  double attn_bytes;                            /* algorithmic KV+q+o bytes of timed attention */
} rt_stats;

/* Create an engine on cfg->device.  Allocates weights (counter-based init on
 * device), the KV page pool, task table and pinned rings.  Errors:
 * RT_E_INVAL (shape / limits invalid), RT_E_NOMEM, RT_E_CUDA (no sm_100 GPU),
 * RT_E_NCCL (world > 1 and communicator init failed). */
rt_status rt_create(const rt_config* cfg, rt_engine** out);
rt_status rt_destroy(rt_engine* e);

/* Submit one request.  prompt[n_prompt] token ids; deadline_us = ERT relative to
 * arrival; fn = (alpha, beta) of Eq. 1; exec_window_us = execution time a
 * segment must cover before it ends at a skill (0 = end at any skill, the
 * paper's rule); script[n_script] (optional) = scripted output tokens (then
 * max_new_tokens := n_script).  request_id_out receives a global id
 * (local_seq * world + rank).  Errors: RT_E_INVAL for alpha > 0, ERT < 0,
 * non-finite beta, token ids outside [0, vocab), n_prompt < 1,
 * n_prompt + max_new_tokens > max_ctx; RT_E_NOMEM for a full task table or a
 * reservation larger than the pool.  Admission refusal is NOT an error. */
rt_status rt_submit_request(rt_engine* e, int32_t agent_id, const int32_t* prompt, int32_t n_prompt,
                            int64_t arrival_us, int64_t deadline_us, rt_utility fn,
                            int32_t exec_window_us, int32_t max_new_tokens,
                            const int32_t* script, int32_t n_script, int64_t* request_id_out);

/* Register a shared prompt prefix ("fixed prompt components
 * ... pre-stored on the server"; DESIGN.md R-PFX).  tokens[n_tokens], n_tokens a positive
 * multiple of page_tokens (16) below max_ctx.  Pops n_tokens/16 pages from the free stack
 * (the order an admission pops them), computes their KV once (a forward over the prefix
 * rows, no logits) and keeps them for the engine's lifetime, read-only.  Every later
 * rt_submit_request whose prompt starts with a registered prefix and is longer than it (the
 * longest such prefix) shares those pages: its reservation, page pops and prefill cover only
 * the rest of the prompt, and finishing frees only its own pages.  Synchronises.  Errors:
 * RT_E_INVAL (length / token ids), RT_E_NOMEM (more than 8 prefixes, or fewer than
 * n_tokens/16 pages free after the outstanding reservations). */
rt_status rt_register_prefix(rt_engine* e, const int32_t* tokens, int32_t n_tokens, int32_t* prefix_id_out);

/* One scheduling round + one decoding iteration (DESIGN.md R-ROUND).  now_us is
 * the round start in WALL mode and ignored in VIRTUAL mode.  info (nullable)
 * receives the round summary available at return (t_us, n_waiting, n_running,
 * n_admitted, refusals, n_rows); n_stopped / round_us of this round are
 * reported by rt_last_round after the next synchronising call. */
rt_status rt_step(rt_engine* e, int64_t now_us, rt_round_info* info);

/* Drain up to cap segment records produced so far (synchronises with the
 * device).  n_out receives the number written.  Records come in round order,
 * slot order within a round. */
rt_status rt_poll_segment(rt_engine* e, rt_segment* out, int32_t cap, int32_t* n_out);

/* Non-blocking rt_poll_segment: drains only the records of rounds the device has
 * already retired (k_sched_post published them to the mapped ring), without waiting
 * for the round in flight.  A serving loop that calls it right after rt_step overlaps
 * its own host work (polling, submitting the next requests) with the round running on
 * the GPU; a round's records appear here at the latest once the next rt_step has
 * returned (that call's plan handshake follows the round's k_sched_post on the stream).
 * Same arguments, ownership and errors as rt_poll_segment (§8(b)). */
rt_status rt_poll_segment_ready(rt_engine* e, rt_segment* out, int32_t cap, int32_t* n_out);

/* Completed summary of the last executed round (synchronises). */
rt_status rt_last_round(rt_engine* e, rt_round_info* info);

/* Block until all device work of this engine is complete. */
rt_status rt_sync(rt_engine* e);

rt_status rt_get_stats(rt_engine* e, rt_stats* out);
rt_status rt_reset_stats(rt_engine* e);

/* Parity-test dumps (synchronise).  bytes_out receives the size needed; a
 * NULL dst only queries the size.
 *   RT_DUMP_TASKS       int64 per task slot: [rid, state, k, ctx, n_pages, n_gen, seg_tok, R]
 *   RT_DUMP_PAGE_TABLES int32 [max_tasks][pages_per_task]
 *   RT_DUMP_ROUND       int32: [B, n_rows, n_admitted, free_top, slot_rid_lo[B], tokens[B],
 *                        argmax[B], admitted_rid_lo[n_admitted]]
 *   RT_DUMP_LOGITS      fp32 [B][vocab]       (RT_FLAG_KEEP_LOGITS)
 *   RT_DUMP_HIDDEN      bf16 [B][d_model]     final-normed hidden of the logits rows
 *   RT_DUMP_CAPTURE_Q   fp32 [n_rows][n_q_heads][head_dim]   (RT_FLAG_CAPTURE)
 *   RT_DUMP_CAPTURE_O   fp32 [n_rows][n_q_heads][head_dim]
 *   RT_DUMP_ROWS        int32 [n_rows][3] (task slot, position, token) of the last round
 *   RT_DUMP_KV_LAYER    bf16 logical [n_pages][2][n_kv_heads][16][head_dim] of capture_layer
 *   RT_DUMP_FREE_STACK  int32 [free_top]
 *   RT_DUMP_HOST_PAGE_TABLES int32 [max_tasks][pages_per_task] host pages of evicted requests
 *                       (RT_DUMP_TASKS column 8 = evicted, 9 = host pages held)
 *   RT_DUMP_HOST_FREE_STACK  int32 [host free top]
 *   RT_DUMP_TASK_SLOTS  int32 [B] task slot of each batch slot of the last round
 *   RT_DUMP_MERGED      int64 [K][4] merged global top-K (world > 1)
 *   RT_DUMP_TRACE       rt_trace_rec [n] since the last rt_reset_stats (RT_FLAG_TRACE; at most
 *                       2^20 records, one per CTA; the buffer is process-wide: with several
 *                       traced engines in one process the last created one owns it)
 * Per-layer dumps (RT_FLAG_CAPTURE_LAYERS), layer l in bits 16..30 of `what`
 * (what = RT_DUMP_LAYER_* | l << 16), rows of the last round's first forward chunk:
 *   RT_DUMP_LAYER_X     fp32 [n_rows][d_model]  residual stream entering layer l (l = n_layers:
 *                       leaving the last layer)
 *   RT_DUMP_LAYER_Q     bf16 [n_rows][n_q_heads][head_dim]  q after RoPE
 *   RT_DUMP_LAYER_O     bf16 [n_rows][n_q_heads][head_dim]  attention output
 *   RT_DUMP_LAYER_XMID  fp32 [n_rows][d_model]  residual after the O projection
 *   RT_DUMP_LAYER_ACT   bf16 [n_rows][d_ff]     SwiGLU activation (down projection input)
 *   RT_DUMP_LAYER_KV    bf16 logical [n_pages][2][n_kv_heads][16][head_dim] of layer l (any engine
 *                       with a model; no flag needed) */
enum {
  RT_DUMP_TASKS = 1, RT_DUMP_PAGE_TABLES = 2, RT_DUMP_ROUND = 3, RT_DUMP_LOGITS = 4,
  RT_DUMP_HIDDEN = 5, RT_DUMP_CAPTURE_Q = 6, RT_DUMP_CAPTURE_O = 7, RT_DUMP_ROWS = 8,
  RT_DUMP_KV_LAYER = 9, RT_DUMP_FREE_STACK = 10, RT_DUMP_TASK_SLOTS = 11, RT_DUMP_MERGED = 12,
  RT_DUMP_TRACE = 13, RT_DUMP_HOST_PAGE_TABLES = 14, RT_DUMP_HOST_FREE_STACK = 15,
  RT_DUMP_LAYER_X = 16, RT_DUMP_LAYER_Q = 17, RT_DUMP_LAYER_O = 18, RT_DUMP_LAYER_XMID = 19,
  RT_DUMP_LAYER_ACT = 20, RT_DUMP_LAYER_KV = 21
};
/* One kernel CTA: grid = %gridid (unique per launch); kind = 1 GEMM (| epilogue mode << 8 |
 * cluster split << 16), 2 attention, 3 norm, 4 embed, 5/6 scheduler pre/post, 7 gather,
 * 8 argmax reduce, 9 candidate merge, 10 prefill attention; t_* = %globaltimer ns at CTA entry, after its
 * dependency wait (griddepcontrol.wait; = entry for kernels without one), t_aux = GEMM:
 * accumulator complete (last tcgen05.mma retired, seen by the epilogue; 0 elsewhere) and
 * t_exit at CTA exit. */
typedef struct {
  uint64_t grid;
  uint32_t kind, smid;
  uint64_t t_entry, t_ready, t_aux, t_exit;
} rt_trace_rec;
rt_status rt_debug_dump(rt_engine* e, int32_t what, void* dst, int64_t bytes, int64_t* bytes_out);

/* Device-time markers on the engine's stream (CUDA events): which = 0 records the
 * start mark, 1 the stop mark; rt_elapsed_ms synchronises and returns stop - start. */
rt_status rt_mark(rt_engine* e, int32_t which);
rt_status rt_elapsed_ms(rt_engine* e, double* ms_out);
/* Switch the per-launch CUDA-event timing of RT_FLAG_TIMING on (1) or off (0) from the next
 * rt_step.  The events recorded around every attention launch sit between dependent kernels
 * and cost the programmatic-dependent-launch overlap there (measured ~0.45 ms per 8B round),
 * so throughput is timed with it off and the per-kernel roofline in a separate pass. */
rt_status rt_set_timing(rt_engine* e, int32_t on);

/* Create a 128-byte ncclUniqueId (rank 0 calls it and broadcasts the bytes;
 * libnccl.so.2 is loaded with dlopen).  RT_E_NCCL if NCCL is unavailable. */
rt_status rt_nccl_unique_id(uint8_t* out128);

/* Human-readable description of the last error (engine may be NULL). */
const char* rt_last_error(rt_engine* e);

/* Library build / device information string ("sm_100a ..."). */
const char* rt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RT_H_ */
