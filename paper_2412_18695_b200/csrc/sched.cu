// sched.cu — device-side segmented scheduler (rows a1-a4, a9-a11 of SURVEY §8(a)).
//
// One CTA of 1024 threads per kernel; all state lives in HBM (task table SoA,
// free stack, slot arrays) so a round needs no host round trip except the plan
// handshake.  Semantics are those of DESIGN.md R-ROUND (identical to
// oracle/engine.py, which is written from the paper independently):
//   pre  : clock, ingest, Eq. 4 scoring of every waiting
//          task, sort by (Pri desc, arrival, id),
//          WCET gate + memory check admission,
//          page pops + batch assembly, forward rows.
//   post : stop checker (window rule BASELINE.json),
//          segment records to the pinned ring, suspend with the
//          completion estimate / finish + free, clock advance.
// Floating point: Eq. 4 in IEEE fp64 with explicit _rn intrinsics (no FMA
// contraction), fixed operation order, -0.0 canonicalised (AMB-10).
#include "common.cuh"
#include "internal.h"
#include <limits.h>

namespace rt {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ unsigned long long enc_i64(int64_t a) {
  return (unsigned long long)a ^ 0x8000000000000000ull;
}
__device__ __forceinline__ int64_t dec_i64(unsigned long long u) {
  return (int64_t)(u ^ 0x8000000000000000ull);
}

// Eq. 1 at waiting w (µs): min(beta, alpha (w - ERT)/1e6 + beta)
__device__ double tuf0_d(double beta, double alpha, int64_t ert, int64_t w) {
  double x = __ddiv_rn(__ll2double_rn(w - ert), 1e6);
  double y = __dmul_rn(alpha, x);
  y = __dadd_rn(y, beta);
  return (beta <= y) ? beta : y;
}
// TUF_1: min(beta, alpha max(w, 0)/1e6 + beta)
__device__ double tuf1_d(double beta, double alpha, int64_t w) {
  double x = __ddiv_rn(__ll2double_rn(w > 0 ? w : 0), 1e6);
  double y = __dmul_rn(alpha, x);
  y = __dadd_rn(y, beta);
  return (beta <= y) ? beta : y;
}
// Eq. 4 with readings AMB-2/3/4/5
__device__ double priority_d(int64_t t, int32_t k, int64_t ref, int64_t D, int64_t ert, double alpha,
                             double beta, int32_t g_us, int32_t net_us, int32_t eps_l_us) {
  int64_t w = t + (int64_t)g_us + (int64_t)net_us - ref;
  double num = (k == 0) ? tuf0_d(beta, alpha, ert, w) : tuf1_d(beta, alpha, w);
  int64_t L = D - t - (int64_t)g_us;
  if (L < (int64_t)eps_l_us) L = eps_l_us;
  double a = __ddiv_rn(__ll2double_rn((int64_t)g_us), 1e6);
  double b = __ddiv_rn(__ll2double_rn(L), 1e6);
  double den = __dmul_rn(a, b);
  double pri = __ddiv_rn(num, den);
  return __dadd_rn(pri, 0.0);
}

__device__ __forceinline__ int ceil_div_i(int a, int b) { return (a + b - 1) / b; }

// The plan handshake (rt_step): the mailbox fields are written and fenced first, then the
// sequence number the host spins on (mapped pinned memory, no event round trip)
__device__ __forceinline__ void publish_plan(DevState* st, HostMailbox* mb) {
  const long long q = st->plan_seq + 1;
  st->plan_seq = q;
  *reinterpret_cast<volatile long long*>(&mb->plan_seq) = q;
}

// Exclusive scan in place over a[0..n) (shared memory), returns the total.
// All threads of the block must call it.
__device__ __forceinline__ int block_scan_excl_inl(int* a, int n, int* wbuf) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  const int per = (n + nt - 1) / nt;
  const int beg = min(tid * per, n), end = min(beg + per, n);
  int local = 0;
  #pragma unroll 1
  for (int i = beg; i < end; ++i) local += a[i];
  int v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) wbuf[w] = v;
  __syncthreads();
  if (w == 0) {
    int x = lane < nw ? wbuf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wbuf[lane] = x;
  }
  __syncthreads();
  int run = (w > 0 ? wbuf[w - 1] : 0) + v - local;
  const int total = wbuf[nw - 1];
  #pragma unroll 1
  for (int i = beg; i < end; ++i) {
    int x = a[i];
    a[i] = run;
    run += x;
  }
  __syncthreads();
  return total;
}
// k_sched_pre calls the scan at ten sites: one out-of-line copy keeps its (cold, once per
// round) code small; k_sched_post keeps the inlined form (measured faster there)
__device__ __noinline__ int block_scan_excl(int* a, int n, int* wbuf) { return block_scan_excl_inl(a, n, wbuf); }

__device__ void hist_push(DevState* st, int64_t v) {
  st->hist[st->hist_pos] = v;
  st->hist_pos = (st->hist_pos + 1) & 7;
  if (st->hist_n < 8) st->hist_n++;
}

// ------------------------------------------------------------ submissions
__global__ void k_apply_submits(SchedParams p, const SubmitRec* recs, const int32_t* toks) {
  const SubmitRec r = recs[blockIdx.x];
  TaskTable T = p.tt;
  const int i = r.slot;
  #pragma unroll 1
  for (int j = threadIdx.x; j < r.n_prompt; j += blockDim.x)
    T.prompt[(size_t)i * p.max_ctx + j] = toks[r.tok_off + j];
  if (r.scripted)
    #pragma unroll 1
    for (int j = threadIdx.x; j < r.max_new; j += blockDim.x)
      T.script[(size_t)i * p.max_ctx + j] = toks[r.tok_off + r.n_prompt + j];
  if (threadIdx.x == 0) {
    T.rid[i] = r.rid;
    T.arrival[i] = r.arrival;
    T.ert[i] = r.ert;
    T.D[i] = r.arrival + r.ert;
    T.ref[i] = r.arrival;
    T.end_est[i] = LLONG_MIN;
    T.seg_exec[i] = 0;
    T.alpha[i] = r.alpha;
    T.beta[i] = r.beta;
    T.pri[i] = 0.0;
    T.agent[i] = r.agent;
    T.k[i] = 0;
    T.n_prompt[i] = r.n_prompt;
    T.max_new[i] = r.max_new;
    T.window[i] = r.window;
    T.scripted[i] = r.scripted;
    T.pfx[i] = r.pfx;
    T.n_pfx[i] = r.n_pfx;
    T.n_gen[i] = 0;
    T.seg_tok[i] = 0;
    T.n_skills[i] = 0;
    T.pending[i] = -1;
    T.ctx[i] = 0;
    T.n_pages[i] = 0;
    T.R[i] = ceil_div_i(r.n_prompt + r.max_new, p.page_tokens);
    T.holder[i] = 0;
    T.evicted[i] = 0;
    T.n_hpages[i] = 0;
    T.dfa_s[i] = 0;
    T.dfa_n[i] = 0;
    T.dfa_v[i] = 0;
    T.argmax_last[i] = -1;
    __threadfence();
    T.state[i] = T_PENDING;
  }
}

void launch_apply_submits(const SchedParams& p, const SubmitRec* d_recs, const int32_t* d_toks, int n,
                          cudaStream_t s) {
  if (n > 0) k_apply_submits<<<n, 256, 0, s>>>(p, d_recs, d_toks);
}

__global__ void k_init_free_stack(int32_t* stack, int n) {
  // stack[0] is the bottom; top = stack[n-1] = 0 -> pops yield 0, 1, 2, ... (AMB-14)
  #pragma unroll 1
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    stack[i] = n - 1 - i;
}
void launch_init_free_stack(int32_t* stack, int n, cudaStream_t s) {
  k_init_free_stack<<<(n + 255) / 256, 256, 0, s>>>(stack, n);
}

// -------------------------------------------------------------- sched_pre
struct PreSmem {
  double a0[kMaxTasks];
  long long a1[kMaxTasks], a2[kMaxTasks], a3[kMaxTasks];
  int perm[kMaxTasks];
  int cslot[kMaxTasks], ck[kMaxTasks], cR[kMaxTasks];
  int cnt_a[kMaxTasks], cnt_b[kMaxTasks];
  int adm[kMaxTasks];
  int evn[kMaxTasks];   // candidate evicted this round (R-EVICT)
  int vic[kMaxTasks];   // victims (task slots) in eviction order
  int evc[kMaxTasks];   // candidate's KV is on the host (T.evicted at scoring time)
  int admx[kMaxTasks];  // candidate index of each admission
  int sflag[kMaxTasks]; // batch slot: 1 = prefill (k = 0 admission), 2 = restore (evicted resume)
  long long wb[32];     // WCET gate: per-warp (budget, rid, seg_tok) minima; then the
  long long wr[32];     // per-warp round sums of the rows loop (prompt, attended, ctx, max)
  long long wc[32];
  int ws[32];
};

__device__ __forceinline__ bool key_before(const PreSmem& S, int x, int y, int n) {
  // x before y ?  invalid (>= n) entries sort last
  if (x >= n) return false;
  if (y >= n) return true;
  if (S.a0[x] != S.a0[y]) return S.a0[x] > S.a0[y];
  if (S.a1[x] != S.a1[y]) return S.a1[x] < S.a1[y];
  if (S.a2[x] != S.a2[y]) return S.a2[x] < S.a2[y];
  return S.a3[x] < S.a3[y];
}

// Sort of the n <= blockDim.x scored candidates (n_pad = power of two >= 32, <= blockDim.x):
// every key becomes a tuple of order-preserving u64 words (Pri descending via its IEEE bits
// — the -0.0 -> +0.0 canonicalisation makes equal priorities equal bit patterns —, then
// a1, a2, a3 ascending, then the candidate index), one element per thread, bitonic network
// with the exchange on registers (shuffles) for distances < 32 and through double-buffered
// shared memory otherwise (one barrier per stage).  Result: S.perm[0 .. n_pad).  The key
// arrays S.a0..a3 are reused as the exchange buffers.
__device__ __forceinline__ unsigned long long desc_key_f64(double d) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  const unsigned long long asc = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  return ~asc;
}
struct SortKey {
  unsigned long long k0, k1, k2, k3;
  int ix;
};
__device__ __forceinline__ bool sk_less(const SortKey& a, const SortKey& b) {
  if (a.k0 != b.k0) return a.k0 < b.k0;
  if (a.k1 != b.k1) return a.k1 < b.k1;
  if (a.k2 != b.k2) return a.k2 < b.k2;
  if (a.k3 != b.k3) return a.k3 < b.k3;
  return a.ix < b.ix;
}
__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int j) {
  const unsigned lo = __shfl_xor_sync(0xffffffffu, (unsigned)v, j);
  const unsigned hi = __shfl_xor_sync(0xffffffffu, (unsigned)(v >> 32), j);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ void sort_keys_small(PreSmem& S, int n, int n_pad, bool pud) {
  const int tid = threadIdx.x;
  const bool act = tid < n_pad;
  SortKey me;
  if (tid < n) {
    me.k0 = pud ? desc_key_f64(S.a0[tid]) : 0ull;
    me.k1 = enc_i64(S.a1[tid]);
    me.k2 = enc_i64(S.a2[tid]);
    me.k3 = enc_i64(S.a3[tid]);
    me.ix = tid;
  } else {  // padding: sorts last
    me.k0 = me.k1 = me.k2 = me.k3 = ~0ull;
    me.ix = tid;
  }
  __syncthreads();  // the key arrays become the exchange buffers
  unsigned long long* xb = reinterpret_cast<unsigned long long*>(S.a0);  // [2][4][blockDim.x] (a0..a3)
  int* xi = S.cnt_a;                                                     // [2][blockDim.x]
  const int nt = blockDim.x;
  int buf = 0;
  #pragma unroll 1
  for (int kk = 2; kk <= n_pad; kk <<= 1) {
    #pragma unroll 1
    for (int j = kk >> 1; j > 0; j >>= 1) {
      SortKey o;
      if (j >= 32) {
        unsigned long long* b = xb + (size_t)buf * 4 * nt;
        if (act) {
          b[tid] = me.k0;
          b[nt + tid] = me.k1;
          b[2 * nt + tid] = me.k2;
          b[3 * nt + tid] = me.k3;
          xi[buf * nt + tid] = me.ix;
        }
        __syncthreads();
        if (act) {
          const int q = tid ^ j;
          o.k0 = b[q];
          o.k1 = b[nt + q];
          o.k2 = b[2 * nt + q];
          o.k3 = b[3 * nt + q];
          o.ix = xi[buf * nt + q];
        }
        buf ^= 1;  // the next stage writes the other buffer: no second barrier
      } else if (tid < ((n_pad + 31) & ~31)) {
        o.k0 = shfl_u64(me.k0, j);
        o.k1 = shfl_u64(me.k1, j);
        o.k2 = shfl_u64(me.k2, j);
        o.k3 = shfl_u64(me.k3, j);
        o.ix = __shfl_xor_sync(0xffffffffu, me.ix, j);
      }
      if (act) {
        const bool up = (tid & kk) == 0, lower = (tid & j) == 0;
        // lower position keeps the smaller key of an ascending pair, the larger of a descending one
        const bool take = (lower == up) ? sk_less(o, me) : sk_less(me, o);
        if (take) me = o;
      }
    }
  }
  __syncthreads();
  if (act) S.perm[tid] = me.ix;
  __syncthreads();
}

// Rank sort for few candidates (n <= 128, the usual waiting queue): candidate i goes to
// position #{j : key_j < key_i} (keys unique by index), one pass over the keys in shared
// memory (broadcast reads), no compare-exchange network.  Same keys as sort_keys_small.
// g = min(32, blockDim / n) (a power of two) threads share a candidate: lane `sub` of the
// group counts the keys j = sub, sub + g, ... and the group sums by shuffles, so the serial
// pass is n / g keys long (C3: 90 candidates, 8 lanes each: 12 keys instead of 90).
__device__ void sort_keys_rank(PreSmem& S, int n, bool pud) {
  const int tid = threadIdx.x, nt = blockDim.x;
  unsigned long long* K = reinterpret_cast<unsigned long long*>(S.cnt_a);  // [4][n] (cnt_a, cnt_b)
#pragma unroll 1
  for (int i = tid; i < n; i += nt) {
    K[i] = pud ? desc_key_f64(S.a0[i]) : 0ull;
    K[n + i] = enc_i64(S.a1[i]);
    K[2 * n + i] = enc_i64(S.a2[i]);
    K[3 * n + i] = enc_i64(S.a3[i]);
  }
  __syncthreads();
  int g = 1;
  while (g < 32 && 2 * g * n <= nt) g <<= 1;
  const int e = tid / g, sub = tid & (g - 1);
  if (e * g < nt && (tid >> 5) * 32 < min(n * g, nt)) {  // warps that hold a candidate (whole warps: shuffles)
    const bool act = e < n;
    unsigned long long m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    if (act) {
      m0 = K[e];
      m1 = K[n + e];
      m2 = K[2 * n + e];
      m3 = K[3 * n + e];
    }
    int r = 0;
    if (act) {
#pragma unroll 2
      for (int j = sub; j < n; j += g) {
        const unsigned long long a0 = K[j], a1 = K[n + j], a2 = K[2 * n + j], a3 = K[3 * n + j];
        // key_j < key_e, lexicographic, without branches (index j breaks ties)
        const bool lt = a0 < m0 ||
                        (a0 == m0 && (a1 < m1 || (a1 == m1 && (a2 < m2 || (a2 == m2 &&
                                                                (a3 < m3 || (a3 == m3 && j < e)))))));
        r += lt ? 1 : 0;
      }
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
      if (o < g) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (act && sub == 0) S.perm[r] = e;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSchedThreads, 1) k_sched_pre(SchedParams p, int64_t now_us) {
  TraceScope tr(TK_SCHED_PRE);
  extern __shared__ __align__(16) unsigned char dsm[];
  PreSmem& S = *reinterpret_cast<PreSmem*>(dsm);
  __shared__ long long s_t;
  __shared__ int s_nwait, s_nc, s_nadm, s_gate_ok, s_refused_mem, s_refused_wcet, s_outstanding;
  __shared__ int s_nvic, s_nswap, s_nrest, s_ftop;
  __shared__ unsigned long long s_min_arr;
  __shared__ int wbuf[32];
  __shared__ unsigned long long s_sum_ctx, s_sum_prompt, s_attn_tok;
  __shared__ int s_max_seqlen, s_ndec, s_npf;
  __shared__ long long s_pm[10];  // clock64 phase marks (RT_FLAG_TRACE)
#define PRE_MARK(i) \
  if (threadIdx.x == 0) s_pm[i] = clock64()
  pdl_wait();  // launched with PDL: every read of the task table / state follows the wait
  tr.ready();
  if (threadIdx.x == 0) pdl_trigger();
  PRE_MARK(0);

  TaskTable T = p.tt;
  DevState* st = p.st;
  const int tid = threadIdx.x, nt = blockDim.x;
  const bool wall = (p.clock_mode == 1);

  if (tid == 0) {
    int64_t t;
    if (wall) {
      t = now_us;
      if (st->last_nonempty) hist_push(st, t - st->last_t);
      st->last_nonempty = 0;
      st->last_t = t;
    } else {
      t = st->t;
    }
    s_t = t;
    s_nwait = 0;
    s_min_arr = ~0ull;
    s_outstanding = 0;
    s_sum_ctx = 0;
    s_npf = 0;
    s_sum_prompt = 0;
    s_attn_tok = 0;
    s_max_seqlen = 0;
  }
  __syncthreads();
  int64_t t = s_t;

  // ---- (1) ingest arrivals <= t
  #pragma unroll 1
  for (int i = tid; i < p.max_tasks; i += nt) {
    int sti = T.state[i];
    if (sti == T_PENDING && T.arrival[i] <= t) {
      T.state[i] = T_WAITING;
      sti = T_WAITING;
    }
    if (sti == T_WAITING) atomicAdd(&s_nwait, 1);
    if (sti == T_PENDING) atomicMin(&s_min_arr, enc_i64(T.arrival[i]));
  }
  __syncthreads();
  PRE_MARK(1);
  const int n_run = st->n_slots;
  if (n_run == 0 && s_nwait == 0) {
    if (!wall && s_min_arr != ~0ull) {  // virtual clock jumps to the next arrival
      t = dec_i64(s_min_arr);
      __syncthreads();
      if (tid == 0) {
        s_t = t;
        st->t = t;
      }
      #pragma unroll 1
      for (int i = tid; i < p.max_tasks; i += nt) {
        if (T.state[i] == T_PENDING && T.arrival[i] <= t) {
          T.state[i] = T_WAITING;
          atomicAdd(&s_nwait, 1);
        }
      }
      __syncthreads();
    }
    if (s_nwait == 0) {
      if (tid == 0) {
        st->B = 0;
        st->n_rows = 0;
        st->n_prefill_rows = 0;
        st->round_us = 0;
        st->n_admitted = 0;
        st->n_waiting = 0;
        st->n_refused_mem = 0;
        st->n_refused_wcet = 0;
        HostMailbox* mb = p.mb;
        mb->t_us = t;
        mb->round_us = 0;
        mb->idle = 1;
        mb->B = 0;
        mb->n_rows = 0;
        mb->n_prefill_rows = 0;
        mb->n_pf_tiles = 0;
        mb->n_dec_rows = 0;
        mb->max_seqlen = 0;
        mb->n_admitted = 0;
        mb->n_waiting = 0;
        mb->n_refused_mem = 0;
        mb->n_refused_wcet = 0;
        mb->n_swap = 0;
        mb->n_swap_ev = 0;
        mb->n_evicted = 0;
        mb->n_restored = 0;
        #pragma unroll 1
        for (int j = 0; j < kTopK; ++j) {
          p.cand[j * 4 + 0] = -INFINITY;
          p.cand[j * 4 + 2] = -1.0;
        }
        __threadfence_system();
        publish_plan(st, mb);
      }
      return;
    }
  }

  // ---- (2) score every waiting task (Eq. 4 recomputed before fetching), and
  // the outstanding reservations sum_active (R - held) (AMB-26) in the same pass.  Every
  // field is loaded before the state test, so a task's loads are one round trip in flight
  // together instead of a state load followed by dependent field loads.
  if (tid == 0) s_nc = 0;
  __syncthreads();
  int my_out = 0;
#pragma unroll 1
  for (int i = tid; i < p.max_tasks; i += nt) {
    const int sti = T.state[i], hold = T.holder[i], Ri = T.R[i], npg = T.n_pages[i], npf = T.n_pfx[i];
    const int evi = T.evicted[i], k = T.k[i];
    const int64_t arr = T.arrival[i], rid = T.rid[i], ref = T.ref[i], Di = T.D[i], ert = T.ert[i];
    const double al = T.alpha[i], be = T.beta[i];
    if (hold) my_out += Ri - npg;
    if (sti != T_WAITING) continue;
    const int pos = atomicAdd(&s_nc, 1);
    double a0 = 0.0;
    long long a1, a2, a3 = 0;
    if (p.policy == 0) {  // PUD (the paper's)
      a0 = priority_d(t, k, ref, Di, ert, al, be, p.g_us, p.net_us, p.eps_l_us);
      T.pri[i] = a0;
      a1 = arr;
      a2 = rid;
    } else if (p.policy == 1) {  // FCFS
      a1 = arr;
      a2 = rid;
    } else {  // EDF on the initial deadline
      a1 = arr + ert;
      a2 = arr;
      a3 = rid;
    }
    S.a0[pos] = a0;
    S.a1[pos] = a1;
    S.a2[pos] = a2;
    S.a3[pos] = a3;
    S.cslot[pos] = i;
    S.ck[pos] = k;
    S.cR[pos] = Ri - npf;  // own pages (a shared prefix is already resident)
    S.evn[pos] = 0;
    S.evc[pos] = evi;
  }
  if (my_out) atomicAdd(&s_outstanding, my_out);
  __syncthreads();
  PRE_MARK(2);
  const int n = s_nc;
  int n_pad = 1;
  while (n_pad < n) n_pad <<= 1;
  if (n <= 1) {
    if (tid == 0) S.perm[0] = 0;
    __syncthreads();
  } else if (n <= 128) {
    sort_keys_rank(S, n, p.policy == 0);
  } else if (n_pad <= nt) {
    sort_keys_small(S, n, n_pad, p.policy == 0);
  } else {
    #pragma unroll 1
    for (int i = tid; i < n_pad; i += nt) S.perm[i] = i;
    __syncthreads();
    // bitonic sort of perm by key.  Compare-exchange distances j >= 32 go through shared memory
    // with a barrier per stage; j < 32 partners sit in the same warp, so those stages run on
    // registers with shuffles (one barrier per kk instead of five): the same network
    #pragma unroll 1
    for (int kk = 2; kk <= n_pad; kk <<= 1) {
      #pragma unroll 1
      for (int j = kk >> 1; j >= 32; j >>= 1) {
        #pragma unroll 1
        for (int i = tid; i < n_pad; i += nt) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const int x = S.perm[i], y = S.perm[ixj];
            const bool up = ((i & kk) == 0);
            const bool sw = up ? key_before(S, y, x, n) : key_before(S, x, y, n);
            if (sw) {
              S.perm[i] = y;
              S.perm[ixj] = x;
            }
          }
        }
        __syncthreads();
      }
      #pragma unroll 1
      for (int base = 0; base < n_pad; base += nt) {  // every lane takes part in the shuffles
        const int i = base + tid;
        int x = i < n_pad ? S.perm[i] : n_pad;  // index >= n: sorts last, never read
        const bool up = ((i & kk) == 0);
        #pragma unroll 1
        for (int j = min(kk >> 1, 16); j > 0; j >>= 1) {
          const int y = __shfl_xor_sync(0xffffffffu, x, j);
          // lower position: takes the partner when it goes first; upper: the mirror
          const bool lower = (i & j) == 0;
          const bool sw = lower ? (up ? key_before(S, y, x, n) : key_before(S, x, y, n))
                                : (up ? key_before(S, x, y, n) : key_before(S, y, x, n));
          if (sw) x = y;
        }
        if (i < n_pad) S.perm[i] = x;
      }
      __syncthreads();
    }
  }

  PRE_MARK(3);
  // ---- local top-K candidates for the round allgather (a12)
  if (tid < kTopK) {
    if (tid < n) {  // record {Pri (0 for FCFS/EDF), arrival, global id, rank}
      const int x = S.perm[tid];
      const int task = S.cslot[x];
      p.cand[tid * 4 + 0] = p.policy == 0 ? T.pri[task] : 0.0;
      p.cand[tid * 4 + 1] = (double)T.arrival[task];
      p.cand[tid * 4 + 2] = (double)T.rid[task];
      p.cand[tid * 4 + 3] = (double)p.rank;
    } else {
      p.cand[tid * 4 + 0] = -INFINITY;
      p.cand[tid * 4 + 1] = 0.0;
      p.cand[tid * 4 + 2] = -1.0;
      p.cand[tid * 4 + 3] = (double)p.rank;
    }
  }

  // ---- (3a) WCET gate on the most urgent running generation: minimum
  // (budget, rid) over the running slots, one slot per thread, then warps, then warp 0
  {
    long long best_bud = LLONG_MAX, best_rid = LLONG_MAX;
    int best_seg = 0;
    #pragma unroll 1
    for (int s = tid; s < n_run; s += nt) {
      const int task = p.slot_task[s];
      const long long bud = T.D[task] - t;
      const long long rid = T.rid[task];
      if (bud >= 0 && (bud < best_bud || (bud == best_bud && rid < best_rid))) {
        best_bud = bud;
        best_rid = rid;
        best_seg = T.seg_tok[task];
      }
    }
    auto warp_min = [&](long long& b, long long& r, int& sg) {
      #pragma unroll 1
      for (int o = 16; o > 0; o >>= 1) {
        const long long ob = __shfl_xor_sync(0xffffffffu, b, o);
        const long long orid = __shfl_xor_sync(0xffffffffu, r, o);
        const int os = __shfl_xor_sync(0xffffffffu, sg, o);
        if (ob < b || (ob == b && orid < r)) {
          b = ob;
          r = orid;
          sg = os;
        }
      }
    };
    warp_min(best_bud, best_rid, best_seg);
    if ((tid & 31) == 0) {
      S.wb[tid >> 5] = best_bud;
      S.wr[tid >> 5] = best_rid;
      S.ws[tid >> 5] = best_seg;
    }
    __syncthreads();
    if (tid < 32) {
      best_bud = tid < (nt >> 5) ? S.wb[tid] : LLONG_MAX;
      best_rid = tid < (nt >> 5) ? S.wr[tid] : LLONG_MAX;
      best_seg = tid < (nt >> 5) ? S.ws[tid] : 0;
      warp_min(best_bud, best_rid, best_seg);
      if (tid == 0) {
        int gate = 1;
        const int nh = min(p.speed_window, st->hist_n);
        if (best_bud != LLONG_MAX && nh > 0 && !p.wcet_off) {
          long long sum = 0;
          #pragma unroll 1
          for (int j = 1; j <= nh; ++j) sum += st->hist[(st->hist_pos - j + 8) & 7];
          const long long rem = max(0, p.max_seg_tokens - best_seg);
          gate = (rem * sum <= (long long)nh * best_bud) ? 1 : 0;
        }
        s_gate_ok = gate;
      }
    }
  }
  __syncthreads();

  PRE_MARK(4);
  // ---- (3b) admission in key order (reading R-MEM), with KV eviction to
  // host memory when a candidate that needs memory does not fit (R-EVICT):
  // suspended holders LATER in the key order are evicted, lowest priority first, only if
  // evicting them (within the host pool) makes the candidate fit
  if (p.host_pages <= 0 && n > 32) {
    // no KV host pool (no eviction), more than a warp of candidates: the serial admission loop below in closed form, all
    // threads.  Walking the key order, a memory-needing candidate (k = 0, or an evicted
    // resume) is admitted iff the reservations of the memory-needing candidates up to and
    // including it fit (R-MEM: once one does not fit, no later one does: the prefix only
    // grows); resumes need none; the first cap = min(max_admit, max_batch - n_run) admissible
    // candidates are admitted, and refusals count up to the last admission (the loop stops
    // there).  Two block scans instead of a serial walk (the walk is faster for <= 32).
    const long long avail = (long long)st->free_top - s_outstanding;
    const int cap = max(0, min(p.max_admit, p.max_batch - n_run));
    const bool gate = s_gate_ok != 0;
    if (tid == 0) s_nc = (cap > 0) ? n : 0;  // c_stop (the serial loop's last iteration + 1)
    #pragma unroll 1
    for (int c = tid; c < n; c += nt) {
      const int x = S.perm[c];
      S.cnt_a[c] = (S.ck[x] == 0 || S.evc[x]) ? S.cR[x] : 0;  // reservation pages needed
    }
    __syncthreads();
    block_scan_excl(S.cnt_a, n, wbuf);  // pages of the memory-needing candidates before c
    #pragma unroll 1
    for (int c = tid; c < n; c += nt) {
      const int x = S.perm[c];
      const bool memc = S.ck[x] == 0 || S.evc[x];
      S.cnt_b[c] = (!memc || (long long)S.cnt_a[c] + S.cR[x] <= avail) ? 1 : 0;
    }
    __syncthreads();
    // (cnt_b is rewritten in place by the scan: keep each candidate's admissibility first)
    #pragma unroll 1
    for (int c = tid; c < n; c += nt) S.sflag[c] = S.cnt_b[c];
    __syncthreads();
    const int tot_ok = block_scan_excl(S.cnt_b, n, wbuf);
    int my_rmem = 0;
    #pragma unroll 1
    for (int c = tid; c < n; c += nt) {
      const int x = S.perm[c];
      const int rank = S.cnt_b[c];
      if (S.sflag[c] && rank < cap && gate) {
        S.admx[rank] = x;
        S.adm[rank] = S.cslot[x];
        if (rank == cap - 1) s_nc = c + 1;
      }
    }
    __syncthreads();
    const int c_stop = s_nc;
    #pragma unroll 1
    for (int c = tid; c < c_stop; c += nt) my_rmem += S.sflag[c] ? 0 : 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_rmem += __shfl_xor_sync(0xffffffffu, my_rmem, o);
    if (tid == 0) {
      s_refused_mem = 0;
      s_nadm = gate ? min(tot_ok, cap) : 0;
      s_refused_wcet = (!gate && n > 0 && cap > 0) ? 1 : 0;
      s_nvic = 0;
      s_ftop = st->free_top;
      s_nswap = 0;
      p.mb->n_swap_ev = 0;
    }
    __syncthreads();
    if ((tid & 31) == 0 && my_rmem && gate) atomicAdd(&s_refused_mem, my_rmem);
  } else if (tid == 0) {
    long long avail = (long long)st->free_top - s_outstanding;
    int havail = p.host_pages > 0 ? st->hfree_top : 0;
    int nadm = 0, rmem = 0, rwcet = 0, nvic = 0;
    bool mem_blocked = false;
    #pragma unroll 1
    for (int c = 0; c < n; ++c) {
      if (nadm >= p.max_admit) break;
      if (n_run + nadm >= p.max_batch) break;
      if (!s_gate_ok) {
        rwcet = 1;
        break;
      }
      const int x = S.perm[c];
      if (S.evn[x]) {  // evicted earlier in this round: not resumable now
        ++rmem;
        continue;
      }
      if (S.ck[x] == 0 || S.evc[x]) {
        const int need = S.cR[x];
        if (!mem_blocked && avail < need && p.host_pages > 0) {
          long long gain = 0;
          int hneed = 0, nv = 0;
          #pragma unroll 1
          for (int cj = n - 1; cj > c && avail + gain < need; --cj) {
            const int y = S.perm[cj];
            const int vt = S.cslot[y];
            if (S.ck[y] > 0 && T.holder[vt] && !T.evicted[vt] && !S.evn[y]) {
              const int own = T.n_pages[vt] - T.n_pfx[vt];
              if (hneed + own > havail) continue;
              S.cnt_b[nv++] = y;  // scratch: tentative victims
              gain += S.cR[y];
              hneed += own;
            }
          }
          if (avail + gain >= need) {
            #pragma unroll 1
            for (int v = 0; v < nv; ++v) {
              const int y = S.cnt_b[v];
              S.evn[y] = 1;
              S.vic[nvic++] = S.cslot[y];
              avail += S.cR[y];
            }
            havail -= hneed;
          }
        }
        if (mem_blocked || avail < need) {
          mem_blocked = true;
          ++rmem;
          continue;
        }
        avail -= need;
      }
      S.admx[nadm] = x;
      S.adm[nadm++] = S.cslot[x];
    }
    s_nadm = nadm;
    s_refused_mem = rmem;
    s_refused_wcet = rwcet;
    s_nvic = nvic;
    // evictions: own pages -> host pages (host pops in page-table order), device pages
    // pushed back in reverse page-table order, victims in eviction order
    int ftop = st->free_top, htop = st->hfree_top, nsw = 0;
    #pragma unroll 1
    for (int v = 0; v < nvic; ++v) {
      const int vt = S.vic[v];
      const int npf = T.n_pfx[vt], own = T.n_pages[vt] - npf;
      int32_t* pt = T.page_table + (size_t)vt * p.pt_stride;
      int32_t* hpt = T.hpage_table + (size_t)vt * p.pt_stride;
      #pragma unroll 1
      for (int m = 0; m < own; ++m) {
        const int hp = p.hfree_stack[htop - 1 - m];
        hpt[m] = hp;
        if (nsw < p.swap_cap) p.swap[nsw] = make_int4(0, vt, pt[npf + m], hp);
        ++nsw;
      }
      htop -= own;
      #pragma unroll 1
      for (int m = 0; m < own; ++m) p.free_stack[ftop + m] = pt[npf + own - 1 - m];
      ftop += own;
      T.n_hpages[vt] = own;
      T.n_pages[vt] = npf;
      T.holder[vt] = 0;
      T.evicted[vt] = 1;
    }
    st->hfree_top = htop;
    s_ftop = ftop;
    s_nswap = nsw;
    p.mb->n_swap_ev = min(nsw, p.swap_cap);
  }
  __syncthreads();
  PRE_MARK(5);
  const int nadm = s_nadm;
  const int B = n_run + nadm;

  // ---- (4) batch assembly: running slots keep their order, admissions appended
  #pragma unroll 1
  for (int j = tid; j < nadm; j += nt) {
    const int task = S.adm[j];
    const int x = S.admx[j];
    const int s = n_run + j;
    p.slot_task[s] = task;
    p.admitted[j] = task;
    T.state[task] = T_RUNNING;
    const int pre = (S.ck[x] == 0);
    p.slot_is_prefill[s] = pre;
    S.sflag[s] = pre ? 1 : (S.evc[x] ? 2 : 0);
    if (pre) {
      T.holder[task] = 1;
      atomicAdd(&s_npf, 1);
    }
  }
  #pragma unroll 1
  for (int s = tid; s < n_run; s += nt) {
    p.slot_is_prefill[s] = 0;
    S.sflag[s] = 0;
  }
  __syncthreads();
  // restores (evicted resumes admitted this round): re-pop their own pages with the
  // admissions (admission order), KV copied back from the host pages, host pages pushed back
  // (admission order, each in reverse order) after this round's eviction pops
  if (tid == 0) {
    int htop = st->hfree_top, nrest = 0;
    #pragma unroll 1
    for (int j = 0; j < nadm && p.host_pages > 0; ++j) {
      const int task = S.adm[j];
      if (S.sflag[n_run + j] != 2) continue;
      ++nrest;
      const int nh = T.n_hpages[task];
      const int32_t* hpt = T.hpage_table + (size_t)task * p.pt_stride;
      #pragma unroll 1
      for (int m = 0; m < nh; ++m) p.hfree_stack[htop + m] = hpt[nh - 1 - m];
      htop += nh;
    }
    st->hfree_top = htop;
    s_nrest = nrest;
  }
  __syncthreads();
  PRE_MARK(6);
  // page pops: prefill admissions (admission order) first, then decode slots in slot order
  #pragma unroll 1
  for (int s = tid; s < B; s += nt) {
    const int task = p.slot_task[s];
    p.round_slots[s] = task;
    const int fl = S.sflag[s];
    if (fl == 1) {
      S.cnt_a[s] = ceil_div_i(T.n_prompt[task], p.page_tokens) - T.n_pfx[task];
    } else {
      S.cnt_a[s] = fl == 2 ? T.n_hpages[task] : 0;  // restore pops
    }
    S.cnt_b[s] = fl == 1 ? 0 : ((T.ctx[task] % p.page_tokens == 0) ? 1 : 0);
  }
  __syncthreads();
  const int tot_a = block_scan_excl(S.cnt_a, B, wbuf);
  const int tot_b = block_scan_excl(S.cnt_b, B, wbuf);
  const int top = s_ftop;
  #pragma unroll 1
  for (int s = tid; s < B; s += nt) {
    const int task = p.slot_task[s];
    int32_t* pt = T.page_table + (size_t)task * p.pt_stride;
    if (S.sflag[s] == 1) {
      const int npg = ceil_div_i(T.n_prompt[task], p.page_tokens);
      const int npf = T.n_pfx[task];
      const int32_t* pp = p.pfx_pages + (size_t)max(T.pfx[task], 0) * p.pt_stride;
      #pragma unroll 1
      for (int m = 0; m < npf; ++m) pt[m] = pp[m];  // shared prefix pages, read-only
      #pragma unroll 1
      for (int m = 0; m < npg - npf; ++m) {
        const int q = S.cnt_a[s] + m;
        const int pg = p.free_stack[top - 1 - q];
        pt[npf + m] = pg;
        p.popped[2 * q] = task;
        p.popped[2 * q + 1] = pg;
      }
      T.n_pages[task] = npg;
    } else {
      if (S.sflag[s] == 2) {  // restore: own pages re-popped, KV from host
        const int npf = T.n_pfx[task], nh = T.n_hpages[task];
        #pragma unroll 1
        for (int m = 0; m < nh; ++m) {
          const int q = S.cnt_a[s] + m;
          const int pg = p.free_stack[top - 1 - q];
          pt[npf + m] = pg;
          p.popped[2 * q] = task;
          p.popped[2 * q + 1] = pg;
        }
        T.n_pages[task] = npf + nh;
      }
      if (T.ctx[task] % p.page_tokens == 0) {
        const int q = tot_a + S.cnt_b[s];
        const int pg = p.free_stack[top - 1 - q];
        const int np = T.n_pages[task];
        pt[np] = pg;
        T.n_pages[task] = np + 1;
        p.popped[2 * q] = task;
        p.popped[2 * q + 1] = pg;
      }
    }
  }
  __syncthreads();
  // restore copy list (after the evictions', in admission order) and restored state
  if (tid == 0 && p.host_pages > 0) {
    int nsw = s_nswap;
    #pragma unroll 1
    for (int s = n_run; s < B; ++s) {
      const int task = p.slot_task[s];
      if (S.sflag[s] != 2) continue;
      const int npf = T.n_pfx[task], nh = T.n_hpages[task];
      const int32_t* pt = T.page_table + (size_t)task * p.pt_stride;
      const int32_t* hpt = T.hpage_table + (size_t)task * p.pt_stride;
      #pragma unroll 1
      for (int m = 0; m < nh; ++m) {
        if (nsw < p.swap_cap) p.swap[nsw] = make_int4(1, task, pt[npf + m], hpt[m]);
        ++nsw;
      }
      T.evicted[task] = 0;
      T.n_hpages[task] = 0;
      T.holder[task] = 1;
    }
    s_nswap = nsw;
  }
  __syncthreads();
  PRE_MARK(7);
  // forward rows: prefill slot -> n_prompt rows, decode slot -> 1 row (AMB-13)
  constexpr int NB = 1024;  // decode-row buckets (page counts), filled by the rows loop
  #pragma unroll 1
  for (int i = tid; i < NB; i += nt) S.ck[i] = 0;
  #pragma unroll 1
  for (int s = tid; s < B; s += nt) {
    const int task = p.slot_task[s];
    S.cnt_a[s] = S.sflag[s] == 1 ? T.n_prompt[task] - p.page_tokens * T.n_pfx[task] : 1;
  }
  __syncthreads();
  const int n_rows = block_scan_excl(S.cnt_a, B, wbuf);
  int n_prefill_rows = 0;
  {
    // the round's sums are accumulated per thread and reduced per warp: one shared atomic
    // per warp (64-bit shared atomicAdd is a CAS spin loop, ~20 us at 256 contending slots)
    unsigned long long l_prompt = 0, l_attn = 0, l_ctx = 0;
    int l_max = 0;
    #pragma unroll 1
    for (int s = tid; s < B; s += nt) {
      const int task = p.slot_task[s];
      const int off = S.cnt_a[s];
      if (S.sflag[s] == 1) {
        const int P = T.n_prompt[task];
        const int Lp = p.page_tokens * T.n_pfx[task];  // prefix positions are not recomputed
        p.slot_row[s] = off + (P - Lp) - 1;
        T.ctx[task] = P;
        l_prompt += (unsigned long long)(P - Lp);
        l_attn += (unsigned long long)P * (P + 1) / 2 - (unsigned long long)Lp * (Lp + 1) / 2;
        l_max = max(l_max, P);
      } else {
        const int c = T.ctx[task];
        p.row_task[off] = task;
        p.row_pos[off] = c;
        p.row_tok[off] = T.pending[task];
        p.slot_row[s] = off;
        T.ctx[task] = c + 1;
        // bucket of the decode-row order below: longest context (most pages) first
        const int kb = NB - 1 - min((c + 1 + p.page_tokens - 1) / p.page_tokens, NB - 1);
        S.cR[s] = kb;
        atomicAdd(&S.ck[kb], 1);
        l_ctx += (unsigned long long)(c + 1);
        l_attn += (unsigned long long)(c + 1);
        l_max = max(l_max, c + 1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l_prompt += __shfl_xor_sync(0xffffffffu, l_prompt, o);
      l_attn += __shfl_xor_sync(0xffffffffu, l_attn, o);
      l_ctx += __shfl_xor_sync(0xffffffffu, l_ctx, o);
      l_max = max(l_max, __shfl_xor_sync(0xffffffffu, l_max, o));
    }
    if ((tid & 31) == 0) {  // per-warp partials, summed by warp 0 in fixed order below
      S.wb[tid >> 5] = (long long)l_prompt;
      S.wr[tid >> 5] = (long long)l_attn;
      S.wc[tid >> 5] = (long long)l_ctx;
      S.ws[tid >> 5] = l_max;
    }
  }
  // prefill rows filled slot by slot, all threads in parallel; the prompt is cut into
  // 16-position attention tiles (page-aligned: the prompt starts at position 0)
  int n_pf_tiles = 0;
  #pragma unroll 1
  for (int s = n_run; s < B && s_npf > 0; ++s) {  // (resume-only rounds skip the walk)
    if (S.sflag[s] != 1) continue;
    const int task = p.slot_task[s];
    const int off = S.cnt_a[s];
    const int P = T.n_prompt[task];
    const int Lp = p.page_tokens * T.n_pfx[task];  // rows start after the shared prefix
    const int32_t* pr = T.prompt + (size_t)task * p.max_ctx;
    #pragma unroll 1
    for (int j = tid; j < P - Lp; j += nt) {
      p.row_task[off + j] = task;
      p.row_pos[off + j] = Lp + j;
      p.row_tok[off + j] = pr[Lp + j];
    }
    const int nt16 = (P - Lp + 15) >> 4;
    #pragma unroll 1
    for (int t16 = tid; t16 < nt16; t16 += nt)
      if (n_pf_tiles + t16 < p.pf_tiles_cap)
        p.pf_tiles[n_pf_tiles + t16] =
            make_int4(off + 16 * t16, min(16, P - Lp - 16 * t16), Lp + 16 * t16, task);
    n_pf_tiles += nt16;
    n_prefill_rows += P - Lp;
  }
  // rows of the decode slots, longest context first: the decode attention's grid (one CTA per
  // (row, KV head), issued in grid order).  Largest-processing-time order — the long rows
  // start first and the short ones fill the tail of the last wave.  Counting sort on the
  // page count (a bucket per page count, 1024 buckets); rows of one bucket in any order: each
  // row's attention is independent of when its CTA runs.
  {
    __syncthreads();  // buckets counted by the rows loop
    const int ndec = block_scan_excl(S.ck, NB, wbuf);
    #pragma unroll 1
    for (int s = tid; s < B; s += nt)
      if (S.sflag[s] != 1) p.dec_rows[atomicAdd(&S.ck[S.cR[s]], 1)] = S.cnt_a[s];
    if (tid == 0) s_ndec = ndec;
  }
  __syncthreads();

  PRE_MARK(8);
  if (tid < 32) {  // the round sums: per-warp partials of the rows loop
    const int nw = nt >> 5;
    unsigned long long a = tid < nw ? (unsigned long long)S.wb[tid] : 0ull;
    unsigned long long b = tid < nw ? (unsigned long long)S.wr[tid] : 0ull;
    unsigned long long c = tid < nw ? (unsigned long long)S.wc[tid] : 0ull;
    int m = tid < nw ? S.ws[tid] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
      m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if (tid == 0) {
      s_sum_prompt = a;
      s_attn_tok = b;
      s_sum_ctx = c;
      s_max_seqlen = m;
    }
  }
  __syncwarp();
  // ---- (5) round latency (VIRTUAL cost model, AMB-24) and plan publication
  if (tid == 0) {
    const long long sum_ctx = (long long)s_sum_ctx, sum_prompt = (long long)s_sum_prompt;
    long long round_us, dispatch;
    if (!wall) {
      round_us = (long long)p.base_us + ((long long)p.base_us * p.gamma_ppm * (long long)(B - 1)) / 1000000 +
                 ((long long)p.kv_us_per_1k * sum_ctx) / 1024 + (long long)p.prefill_us_per_tok * sum_prompt +
                 (long long)p.swap_us_per_page * s_nswap;
      dispatch = t + round_us;
    } else {
      round_us = st->hist_n > 0 ? st->hist[(st->hist_pos + 7) & 7] : 0;
      dispatch = t + round_us;
    }
    st->free_top = top - tot_a - tot_b;
    st->B = B;
    st->n_rows = n_rows;
    st->n_prefill_rows = n_prefill_rows;
    st->max_seqlen = s_max_seqlen;
    st->round_us = round_us;
    st->dispatch_us = dispatch;
    st->sum_ctx = sum_ctx;
    st->sum_prompt = sum_prompt;
    st->n_admitted = nadm;
    st->n_waiting = n;
    st->n_refused_mem = s_refused_mem;
    st->n_refused_wcet = s_refused_wcet;
    st->n_pops = tot_a + tot_b;
    st->n_swap = s_nswap;
    st->n_evicted = s_nvic;
    st->n_restored = s_nrest;
    HostMailbox* mb = p.mb;
    mb->n_swap = min(s_nswap, p.swap_cap);
    mb->n_evicted = s_nvic;
    mb->n_restored = s_nrest;
    mb->t_us = t;
    mb->round_us = round_us;
    mb->idle = 0;
    mb->B = B;
    mb->n_rows = n_rows;
    mb->n_prefill_rows = n_prefill_rows;
    mb->n_pf_tiles = min(n_pf_tiles, p.pf_tiles_cap);
    mb->n_dec_rows = s_ndec;
    mb->max_seqlen = s_max_seqlen;
    mb->n_admitted = nadm;
    mb->n_waiting = n;
    mb->n_refused_mem = s_refused_mem;
    mb->n_refused_wcet = s_refused_wcet;
    mb->attn_tokens = (long long)s_attn_tok;
    __threadfence_system();
    publish_plan(st, mb);
  }
  PRE_MARK(9);
  if (threadIdx.x == 0) {
    auto dd = [&](int i, int j) {
      const long long d = s_pm[j] - s_pm[i];
      return (unsigned long long)(uint32_t)(d > 0 ? d : 0);
    };
    trace_phase(TK_PHASE | TK_SCHED_PRE, dd(0, 1) | (dd(1, 2) << 32), dd(2, 3) | (dd(3, 4) << 32),
                dd(4, 5) | (dd(5, 6) << 32), dd(6, 7) | (dd(7, 9) << 32));
  }
#undef PRE_MARK
}

void launch_sched_pre(const SchedParams& p, int64_t now_us, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sched_pre, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PreSmem));
    attr = true;
  }
  // programmatic dependent launch: resident while k_sched_post finishes, waits in pdl_wait()
  launch_pdl(k_sched_pre, dim3(1), dim3(kSchedThreads), sizeof(PreSmem), s, p, now_us);
}

// -------------------------------------------------------------- sched_post
struct PostSmem {
  int reason[1024];
  int stop_off[1024];
  int keep_off[1024];
  int keep_task[1024];
  int fin[1024];
  int fin_off[1024];
};

__global__ void __launch_bounds__(kSchedThreads, 1) k_sched_post(SchedParams p) {
  TraceScope tr(TK_SCHED_POST);
  // launched with PDL behind k_argmax_reduce: nothing is read before the wait; the trigger
  // lets the next round's k_sched_pre become resident (it waits for this kernel's completion)
  pdl_wait();
  tr.ready();
  if (threadIdx.x == 0) pdl_trigger();
  extern __shared__ __align__(16) unsigned char dsm[];
  PostSmem& S = *reinterpret_cast<PostSmem*>(dsm);
  __shared__ int wbuf[32];
  __shared__ int s_nfin;
  TaskTable T = p.tt;
  DevState* st = p.st;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int B = st->B;
  if (B == 0) return;
  const int64_t dispatch = st->dispatch_us;
  if (tid == 0) s_nfin = 0;

  // ---- (6) stop checker per slot (a9)
  for (int s = tid; s < B; s += nt) {
    const int task = p.slot_task[s];
    const size_t base = (size_t)task * p.max_ctx;
    const int ng0 = T.n_gen[task];
    const int am = p.no_model ? -1 : p.argmax_tok[s];
    const int tok = T.scripted[task] ? T.script[base + ng0] : am;
    T.argmax_last[task] = am;
    const int ng = ng0 + 1;
    const int segt = T.seg_tok[task] + 1;
    T.out[base + ng0] = tok;
    T.pending[task] = tok;
    int64_t sx = T.seg_exec[task];
    int nsk = T.n_skills[task];
    int sk = -1;  // >= 0: this token completes an executable unit (a segment boundary candidate)
    if (p.stop_grammar == RT_GRAMMAR_TOKEN) {
      sk = p.tok_skill[tok];
      if (sk >= 0) sx += p.tok_exec[tok];
    } else if (p.stop_grammar == RT_GRAMMAR_SKILL) {
      // DFA of  name ( digits ) ;  (the paper's regex over detokenized text)
      const int cls = p.tok_class[tok];
      int ds = T.dfa_s[task], dn = T.dfa_n[task], dv = T.dfa_v[task];
      if (cls >= 1 && cls <= RT_MAX_SKILL_NAMES) {
        ds = 1;
        dn = cls - 1;
        dv = 0;
      } else if (cls == RT_TC_LPAREN) {
        ds = ds == 1 ? 2 : 0;
      } else if (cls >= RT_TC_DIGIT0 && cls < RT_TC_DIGIT0 + 10) {
        if (ds == 2 || ds == 3) {
          ds = 3;
          dv = min(dv * 10 + (cls - RT_TC_DIGIT0), 1000000);
        } else {
          ds = 0;
        }
      } else if (cls == RT_TC_RPAREN) {
        ds = (ds == 2 || ds == 3) ? 4 : 0;
      } else if (cls == RT_TC_SEMI && ds == 4) {
        sk = dn;
        sx += (int64_t)p.skill_base_us[dn] + (int64_t)p.skill_unit_us[dn] * dv;
        ds = 0;
      } else {
        ds = 0;
      }
      T.dfa_s[task] = ds;
      T.dfa_n[task] = dn;
      T.dfa_v[task] = dv;
    } else {  // chatbot: reading time per word, sentence / paragraph ends
      const int cls = p.tok_class[tok];
      // a word-bearing token (word, skill name, digit) adds reading time
      if (cls == RT_TC_WORD || (cls >= 1 && cls < RT_TC_DIGIT0 + 10)) sx += p.word_us;
      if (cls == RT_TC_PARA_END || (cls == RT_TC_SENT_END && p.stop_grammar == RT_GRAMMAR_SENTENCE)) sk = 0;
    }
    if (sk >= 0) ++nsk;
    // EOS > MAXNEW > SKILL_WINDOW > CAP; STREAM: no CAP below RT_SEG_MAX_TOKENS; NONE: no
    // skill boundary either (the comparison systems, rt.h RT_SEG_*)
    const int cap = p.seg_mode == RT_SEG_SUSPEND ? p.max_seg_tokens : RT_SEG_MAX_TOKENS;
    int reason = 0;
    if (tok == p.eos_id) reason = 1;
    else if (ng == T.max_new[task]) reason = 2;
    else if (p.seg_mode != RT_SEG_NONE && sk >= 0 && sx >= (int64_t)T.window[task]) reason = 3;
    else if (segt == cap) reason = 4;
    // STREAM: a delivered segment does not suspend the request (it keeps its slot)
    const bool keep = reason == 0 || (p.seg_mode != RT_SEG_SUSPEND && (reason == 3 || reason == 4));
    T.n_gen[task] = ng;
    T.seg_tok[task] = segt;
    T.seg_exec[task] = sx;
    T.n_skills[task] = nsk;
    p.slot_tok[s] = tok;
    S.reason[s] = reason;
    S.stop_off[s] = reason != 0;
    S.keep_off[s] = keep;
    S.keep_task[s] = task;
  }
  __syncthreads();
  const int n_stop = block_scan_excl_inl(S.stop_off, B, wbuf);
  const int n_keep = block_scan_excl_inl(S.keep_off, B, wbuf);
  const int64_t seg_base = st->seg_written;

  // ---- (7) segment records + retire (a10)
  for (int s = tid; s < B; s += nt) {
    const int task = S.keep_task[s];
    const int reason = S.reason[s];
    const bool keep = reason == 0 || (p.seg_mode != RT_SEG_SUSPEND && (reason == 3 || reason == 4));
    if (keep) p.slot_task[S.keep_off[s]] = task;  // stable compaction (reads use keep_task copy)
    if (reason == 0) continue;
    const int ng = T.n_gen[task], segt = T.seg_tok[task];
    const int64_t idx = seg_base + S.stop_off[s];
    SegRec* r = p.seg_ring + (idx % p.seg_ring_cap);
    r->request_id = T.rid[task];
    r->agent_id = T.agent[task];
    r->k = T.k[task];
    r->tok_begin = ng - segt;
    r->tok_end = ng;
    r->n_skills = T.n_skills[task];
    r->reason = reason;
    r->est_exec_us = T.seg_exec[task];
    r->dispatch_us = dispatch;
    const int32_t* o = T.out + (size_t)task * p.max_ctx;
    for (int j = 0; j < segt; ++j) r->tokens[j] = o[ng - segt + j];
    if (reason == 1 || reason == 2) {  // finish: free pages + reservation
      T.state[task] = T_FINISHED;
      T.holder[task] = 0;
      const int f = atomicAdd(&s_nfin, 1);
      S.fin[f] = task;
    } else if (keep) {  // STREAM / NONE cut: the request keeps decoding; next segment index
      T.k[task] = T.k[task] + 1;
      T.seg_tok[task] = 0;
      T.seg_exec[task] = 0;
      T.n_skills[task] = 0;
    } else {  // suspend: completion estimate of the dispatched segment
      int64_t b = dispatch + (int64_t)p.net_us;
      const int64_t prev = T.end_est[task];
      if (prev != LLONG_MIN && prev > b) b = prev;
      const int64_t e = b + T.seg_exec[task];
      T.end_est[task] = e;
      T.D[task] = e;
      T.ref[task] = e;
      T.k[task] = T.k[task] + 1;
      T.seg_tok[task] = 0;
      T.seg_exec[task] = 0;
      T.n_skills[task] = 0;
      T.state[task] = T_WAITING;
    }
  }
  __syncthreads();
  // finished requests push their pages in ascending request id, each in reverse
  // page-table order (AMB-14)
  const int nfin = s_nfin;
  if (tid == 0) {
    for (int a = 1; a < nfin; ++a) {  // insertion sort by rid (few per round)
      const int x = S.fin[a];
      const int64_t rx = T.rid[x];
      int b = a - 1;
      while (b >= 0 && T.rid[S.fin[b]] > rx) {
        S.fin[b + 1] = S.fin[b];
        --b;
      }
      S.fin[b + 1] = x;
    }
  }
  __syncthreads();
  for (int f = tid; f < nfin; f += nt) S.fin_off[f] = T.n_pages[S.fin[f]] - T.n_pfx[S.fin[f]];  // own pages
  __syncthreads();
  const int n_push = block_scan_excl_inl(S.fin_off, nfin, wbuf);
  const int top = st->free_top;
  for (int f = tid; f < nfin; f += nt) {
    const int task = S.fin[f];
    const int np = T.n_pages[task], npf = T.n_pfx[task];
    const int32_t* pt = T.page_table + (size_t)task * p.pt_stride;
    for (int m = 0; m < np - npf; ++m) p.free_stack[top + S.fin_off[f] + m] = pt[np - 1 - m];
    T.n_pages[task] = 0;
  }
  __syncthreads();
  if (tid == 0) {
    st->free_top = top + n_push;
    st->n_slots = n_keep;
    st->n_stopped = n_stop;
    st->seg_written = seg_base + n_stop;
    if (p.clock_mode == 0) {
      st->t = st->t + st->round_us;
      hist_push(st, st->round_us);
    } else {
      st->last_nonempty = 1;
    }
    HostMailbox* mb = p.mb;
    mb->n_stopped = n_stop;
    // every thread's ring records (ordered before this thread by the barrier above) become
    // visible to the host before the count that publishes them (rt_poll_segment_ready reads
    // the count without waiting for the round)
    __threadfence_system();
    mb->seg_written = seg_base + n_stop;
    __threadfence_system();
  }
}

void launch_sched_post(const SchedParams& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sched_post, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PostSmem));
    attr = true;
  }
  launch_pdl(k_sched_post, dim3(1), dim3(kSchedThreads), sizeof(PostSmem), s, p);
}

// ------------------------------------------------ multi-GPU candidate merge (a12)
// all: [world][kTopK][4] (pri, arrival, rid, rank); merged: global top-K by
// (pri desc, arrival asc, rid asc) over the union (AMB-22); rid < 0 = empty.
__global__ void k_merge_cand(const double* all, int world, double* merged) {
  TraceScope tr(TK_MERGE);
  __shared__ double key[8 * kTopK][4];
  __shared__ int perm[8 * kTopK];
  const int n = world * kTopK;
  int n_pad = 1;
  while (n_pad < n) n_pad <<= 1;
  for (int i = threadIdx.x; i < n_pad; i += blockDim.x) {
    perm[i] = i;
    for (int j = 0; j < 4; ++j) key[i][j] = i < n ? all[i * 4 + j] : 0.0;
    if (i >= n) key[i][2] = -1.0;
  }
  __syncthreads();
  for (int kk = 2; kk <= n_pad; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n_pad; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj <= i) continue;
        const int x = perm[i], y = perm[ixj];
        auto before = [&](int a, int b) {
          const bool va = key[a][2] >= 0, vb = key[b][2] >= 0;
          if (va != vb) return va;
          if (key[a][0] != key[b][0]) return key[a][0] > key[b][0];
          if (key[a][1] != key[b][1]) return key[a][1] < key[b][1];
          return key[a][2] < key[b][2];
        };
        const bool up = (i & kk) == 0;
        if (up ? before(y, x) : before(x, y)) {
          perm[i] = y;
          perm[ixj] = x;
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < kTopK; i += blockDim.x)
    for (int j = 0; j < 4; ++j) merged[i * 4 + j] = key[perm[i]][j];
}

void launch_merge_cand(const double* all, int world, double* merged, cudaStream_t s) {
  k_merge_cand<<<1, 128, 0, s>>>(all, world, merged);
}

// ------------------------------------------------ op-level Eq. 4 (rt_op_priority)
__global__ void k_priority_batch(const int64_t* trde, const int32_t* k, const double* alpha, const double* beta,
                                 int n, int g_us, int net_us, int eps_l_us, double* pri) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pri[i] = priority_d(trde[4 * i], k[i], trde[4 * i + 1], trde[4 * i + 2], trde[4 * i + 3], alpha[i], beta[i],
                      g_us, net_us, eps_l_us);
}
void launch_priority_batch(const int64_t* trde, const int32_t* k, const double* alpha, const double* beta, int n,
                           int g_us, int net_us, int eps_l_us, double* pri, cudaStream_t s) {
  if (n > 0) k_priority_batch<<<(n + 127) / 128, 128, 0, s>>>(trde, k, alpha, beta, n, g_us, net_us, eps_l_us, pri);
}

RT_TRACE_BINDER(trace_bind_sched)

}  // namespace rt
