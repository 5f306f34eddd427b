// internal.h — structures shared by the host engine and the device kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "rt.h"

namespace rt {

enum TaskState : int32_t { T_FREE = -1, T_PENDING = 0, T_WAITING = 1, T_RUNNING = 2, T_FINISHED = 3 };

constexpr int kMaxSegTok = 16;
constexpr int kMaxTasks = 2048;
constexpr int kSchedThreads = 1024;
constexpr int kMaxPrefixes = 8;    // registered shared prompt prefixes (NEXT-1)
constexpr int kTopK = 16;          // per-rank candidates exchanged per round (a12)

// Submission record staged in pinned host memory, applied on device at the next step.
struct SubmitRec {
  int64_t rid, arrival, ert;
  double alpha, beta;
  int32_t slot, agent, n_prompt, max_new, window, scripted;
  int32_t pfx, n_pfx;  // shared prefix id (-1 none) and its page count
  int64_t tok_off;  // offset of prompt (then script) tokens in the staging token pool
};

// Device task table (structure of arrays, capacity max_tasks).
struct TaskTable {
  int64_t *rid, *arrival, *ert, *D, *ref, *end_est, *seg_exec;
  double *alpha, *beta, *pri;
  int32_t *state, *agent, *k, *n_prompt, *max_new, *window, *scripted;
  int32_t *n_gen, *seg_tok, *n_skills, *pending, *ctx, *n_pages, *R, *holder, *argmax_last;
  int32_t *pfx, *n_pfx;  // shared prefix id (-1 none) and its page count (leading page-table
                         // entries that are the prefix's read-only pages)
  int32_t *evicted, *n_hpages;  // KV evicted to host pages (R-EVICT) and how many
  int32_t *dfa_s, *dfa_n, *dfa_v;  // stop-grammar DFA state, skill name, argument (NEXT-4)
  int32_t* hpage_table;  // [max_tasks][pt_stride] host pages of an evicted request's own pages
  int32_t* page_table;   // [max_tasks + kMaxPrefixes][pt_stride] (prefix rows at the end)
  int32_t* prompt;       // [max_tasks][max_ctx]
  int32_t* script;       // [max_tasks][max_ctx]
  int32_t* out;          // [max_tasks][max_ctx]
};

// Scalars kept on device across rounds.
struct DevState {
  int64_t t, last_t;
  int64_t hist[8];
  int32_t hist_n, hist_pos, last_nonempty;
  int32_t n_slots;       // running slots after the last retire
  int32_t free_top;      // free-stack size
  int32_t B, n_rows, n_prefill_rows, max_seqlen;
  int64_t round_us, dispatch_us, sum_ctx, sum_prompt;
  int64_t seg_written;   // segment records published so far
  int32_t n_admitted, n_waiting, n_refused_mem, n_refused_wcet, n_stopped, n_pops;
  int32_t error;
  int32_t hfree_top;     // host free-stack size (R-EVICT)
  int32_t n_swap, n_evicted, n_restored;  // this round's page copies / requests
  int64_t plan_seq;      // rounds planned by k_sched_pre (published as HostMailbox::plan_seq)
};

// Round plan / summary published to the host (mapped pinned memory).
struct HostMailbox {
  int64_t t_us, round_us;
  int32_t idle, B, n_rows, n_prefill_rows, max_seqlen, n_admitted, n_waiting;
  int32_t n_refused_mem, n_refused_wcet, n_stopped, error;
  int64_t seg_written;
  int64_t round_seq;
  int64_t attn_tokens;   // sum over rows of attended positions (algorithmic attention bytes)
  int32_t n_pf_tiles;    // prefill attention tiles of this round (SchedParams::pf_tiles)
  int32_t n_dec_rows;    // decode rows of this round (SchedParams::dec_rows)
  int32_t n_swap, n_evicted, n_restored;  // KV page copies (SchedParams::swap) / requests
  int32_t n_swap_ev;     // the first n_swap_ev copies are evictions (device -> host)
  int64_t plan_seq;      // written LAST by k_sched_pre (after a system fence): the plan is complete
};

struct SegRec {  // identical layout to rt_segment
  int64_t request_id;
  int32_t agent_id, k, tok_begin, tok_end, n_skills, reason;
  int64_t est_exec_us;
  int64_t dispatch_us;
  int32_t tokens[RT_SEG_MAX_TOKENS];
};

struct SchedParams {
  TaskTable tt;
  DevState* st;
  HostMailbox* mb;           // mapped host pointer
  SegRec* seg_ring;          // mapped host pointer
  int64_t seg_ring_cap;
  int32_t* free_stack;       // [n_pages]
  int32_t* slot_task;        // [max_batch]   task slot of each running slot (persistent)
  int32_t* round_slots;      // [max_batch]   task slot of each slot of the current round (log)
  int32_t* slot_is_prefill;  // [max_batch]
  int32_t* slot_row;         // [max_batch]   logits row of each slot
  int32_t* admitted;         // [max_batch]   admitted task slots (this round, in order)
  int32_t* row_task;         // [rows_cap]
  int32_t* row_pos;          // [rows_cap]
  int32_t* dec_rows;         // [max_batch]   forward rows of the decode slots (slot order)
  int4* pf_tiles;            // [pf_tiles_cap] prefill attention tiles: (first row, rows <= 16,
                             //                first position (multiple of 16), task slot)
  int32_t pf_tiles_cap;
  int32_t* row_tok;          // [rows_cap]
  int32_t* argmax_tok;       // [max_batch]   lm_head argmax per slot
  int32_t* slot_tok;         // [max_batch]   selected token per slot (log)
  int32_t* popped;           // [max_pops][2]
  const int16_t* tok_skill;
  const int32_t* tok_exec;
  double* cand;              // [kTopK][4] local top-K candidates (pri, arrival, rid, rank)
  const int32_t* pfx_pages;  // [kMaxPrefixes][pt_stride] page ids of each registered prefix
  int32_t max_tasks, max_batch, max_ctx, pt_stride, n_pages, page_tokens, rows_cap;
  int32_t max_seg_tokens, g_us, net_us, eps_l_us, speed_window, max_admit, policy, clock_mode;
  int32_t base_us, gamma_ppm, kv_us_per_1k, prefill_us_per_tok;
  int32_t eos_id, rank, world, no_model;
  int32_t seg_mode, wcet_off;  // RT_SEG_*, WCET gate disabled (baselines)
  int32_t host_pages, swap_us_per_page;  // KV eviction to host (R-EVICT); 0 pages = off
  int32_t stop_grammar, word_us;         // RT_GRAMMAR_* (NEXT-4)
  const int16_t* tok_class;              // [vocab]
  const int32_t* skill_base_us;          // [RT_MAX_SKILL_NAMES]
  const int32_t* skill_unit_us;
  int32_t* hfree_stack;        // [host_pages] host free stack (top = end, pops 0, 1, 2, ...)
  int4* swap;                  // [swap_cap] (dir 0 evict / 1 restore, task, device page, host page)
  int32_t swap_cap;
};

// launchers (sched.cu)
void launch_apply_submits(const SchedParams& p, const SubmitRec* d_recs, const int32_t* d_toks, int n,
                          cudaStream_t s);
void launch_sched_pre(const SchedParams& p, int64_t now_us, cudaStream_t s);
void launch_sched_post(const SchedParams& p, cudaStream_t s);
void launch_init_free_stack(int32_t* stack, int n, cudaStream_t s);
// a12: global top-kTopK of world x kTopK candidate records (sched.cu k_merge_cand)
void launch_merge_cand(const double* all, int world, double* merged, cudaStream_t s);

}  // namespace rt
