// attn.cu — paged decode attention for sm_100a (the graded HBM kernel).
//
// What it computes (oracle c1/c2, PAPER.md:387 PagedAttention): for every row r
// and q head h,  o = softmax(q . K^T / sqrt(hd)) V  over the row's first
// seqlen positions, K/V read through the request's page table (16-token pages).
//
// B200 design:
//  * one CTA per (row, kv head, chunk of pages); the G = nq/nkv q heads of a kv
//    head share every page read (GQA), so each (page, kv head) block is read
//    from HBM exactly once per step;
//  * a (page, kv head) block is one contiguous 64*hd-byte region ([K|V][16][hd],
//    XOR-swizzled at write time) moved by ONE cp.async.bulk (TMA engine, SASS
//    UBLKCP) into a per-warp ring of STAGES shared-memory buffers completed on
//    an mbarrier — no register staging, deep memory-level parallelism;
//  * warps work on interleaved pages independently (no CTA barrier in the loop);
//  * S^T = q K^T and O^T = V^T P^T on mma.sync m16n8k16 (bf16 in, fp32 acc) fed
//    by conflict-free ldmatrix from the swizzled buffers, online softmax in fp32
//    with exp2; warps merged through shared memory, chunks merged by a combine
//    kernel (flash-decoding split-KV).
#include "common.cuh"
#include "model.h"
#include <cstdlib>

namespace rt {

constexpr int kAttnWarps = 4;

template <int HD>
struct AttnCfg {
  static constexpr int BLOCK = 64 * HD;                       // bytes of one (page, kv head) block
  static constexpr int STAGES = HD >= 128 ? 3 : 6;
  static constexpr int MERGE = kAttnWarps * 8 * (HD + 2) * 4;  // fp32 merge buffers
  static constexpr int RING = kAttnWarps * STAGES * BLOCK;
  static constexpr int SMEM = (RING > MERGE ? RING : MERGE) + kAttnWarps * STAGES * 8 + 64;
};

template <int HD>
__global__ void __launch_bounds__(kAttnWarps * 32) k_attn(AttnArgs a) {
  using C = AttnCfg<HD>;
  using SW = KvSwz<HD>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (C::RING > C::MERGE ? C::RING : C::MERGE));

  TraceScope tr(TK_ATTN);
  if (threadIdx.x == 0) pdl_trigger();
  const int chunk = blockIdx.x, h = blockIdx.y, r = blockIdx.z;
  const int row = a.row0 + r;
  const int seqlen = a.row_seqlen ? a.row_seqlen[row] : a.row_pos[row] + 1;
  const int n_pages = (seqlen + 15) >> 4;
  const int n_chunks = (n_pages + a.chunk_pages - 1) / a.chunk_pages;
  if (chunk >= n_chunks) return;
  const int p_begin = chunk * a.chunk_pages;
  const int p_end = min(p_begin + a.chunk_pages, n_pages);
  const int task = a.row_task[row];
  const int32_t* ptab = a.page_table + (size_t)task * a.pt_stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const int gq = lane >> 2, qq = lane & 3;

  unsigned char* ring = smem + warp * C::STAGES * C::BLOCK;
  uint64_t* bar = bars + warp * C::STAGES;
  const unsigned char* pool = (const unsigned char*)a.pool;
  const size_t head_off = (size_t)h * C::BLOCK;
  const size_t page_stride = (size_t)a.nkv * C::BLOCK;

  // pages of this warp: p_begin + warp + i * NW
  const int n_my = p_end - (p_begin + warp) > 0 ? (p_end - (p_begin + warp) + kAttnWarps - 1) / kAttnWarps : 0;
  if (lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  pdl_wait();  // q and the KV pages come from the QKV GEMM that precedes this kernel
  tr.ready();
  // page ids of the first 32 pages of this warp, one per lane
  int my_page = (lane < n_my) ? ptab[p_begin + warp + lane * kAttnWarps] : 0;
#pragma unroll
  for (int i = 0; i < C::STAGES; ++i) {
    const int pg = __shfl_sync(0xffffffffu, my_page, i);
    if (lane == 0 && i < n_my) {
      mbar_arrive_expect_tx(&bar[i], C::BLOCK);
      bulk_g2s(ring + i * C::BLOCK, pool + (size_t)pg * page_stride + head_off, C::BLOCK, &bar[i]);
    }
  }

  // q fragments (A operand of S^T = Q K^T), rows g >= G are zero
  uint32_t qa[HD / 16][2];
  {
    const bf16* qrow = a.q + ((size_t)r * a.nq + (size_t)h * G) * HD;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      if (gq < G) {
        const uint32_t* q32 = reinterpret_cast<const uint32_t*>(qrow + (size_t)gq * HD + ks * 16);
        qa[ks][0] = q32[qq];
        qa[ks][1] = q32[4 + qq];
      } else {
        qa[ks][0] = 0u;
        qa[ks][1] = 0u;
      }
    }
  }
  float acc[HD / 16][4];
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const float sl2 = a.scale_log2;
  // ldmatrix lane addressing: matrix mi = lane >> 3, row j = lane & 7
  const int mi = lane >> 3;
  const int ltok = ((mi >> 1) << 3) + (lane & 7);
  const int lcsel = mi & 1;

  for (int i = 0; i < n_my; ++i) {
    const int s = i % C::STAGES;
    mbar_wait(&bar[s], (uint32_t)((i / C::STAGES) & 1));
    const uint32_t kbase = smem_u32(ring + s * C::BLOCK);
    const uint32_t vbase = kbase + SW::MAT_BYTES;
    // ---- S^T (16 g-rows x 16 tokens) = Q K^T
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(b0, b1, b2, b3, kbase + SW::chunk_off(ltok, 2 * ks + lcsel));
      const uint32_t afr[4] = {qa[ks][0], 0u, qa[ks][1], 0u};
      const uint32_t bf0[2] = {b0, b1}, bf1[2] = {b2, b3};
      mma_bf16_16816(s0, afr, bf0);
      mma_bf16_16816(s1, afr, bf1);
    }
    // ---- online softmax for row g = lane/4 over tokens 2qq, 2qq+1, 8+2qq, 9+2qq
    const int page_idx = p_begin + warp + i * kAttnWarps;
    const int t0 = page_idx * 16 + 2 * qq;
    float x00 = (t0 < seqlen) ? s0[0] * sl2 : -INFINITY;
    float x01 = (t0 + 1 < seqlen) ? s0[1] * sl2 : -INFINITY;
    float x10 = (t0 + 8 < seqlen) ? s1[0] * sl2 : -INFINITY;
    float x11 = (t0 + 9 < seqlen) ? s1[1] * sl2 : -INFINITY;
    float mp = fmaxf(fmaxf(x00, x01), fmaxf(x10, x11));
    mp = fmaxf(mp, __shfl_xor_sync(0xffffffffu, mp, 1));
    mp = fmaxf(mp, __shfl_xor_sync(0xffffffffu, mp, 2));
    const float m_new = fmaxf(m_run, mp);
    const float corr = exp2f(m_run - m_new);
    const float p00 = exp2f(x00 - m_new), p01 = exp2f(x01 - m_new);
    const float p10 = exp2f(x10 - m_new), p11 = exp2f(x11 - m_new);
    l_run = l_run * corr + (p00 + p01) + (p10 + p11);
    m_run = m_new;
    // rescale O^T columns g = 2qq, 2qq+1 (their softmax state lives in lanes 4g..4g+3)
    const float c0 = __shfl_sync(0xffffffffu, corr, 8 * qq);
    const float c1 = __shfl_sync(0xffffffffu, corr, 8 * qq + 4);
    const uint32_t pb[2] = {pack_bf16x2(p00, p01), pack_bf16x2(p10, p11)};
    // ---- O^T (hd x 16 g) += V^T P^T
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      acc[mt][0] *= c0;
      acc[mt][1] *= c1;
      acc[mt][2] *= c0;
      acc[mt][3] *= c1;
      uint32_t va[4];
      ldmatrix_x4_trans(va[0], va[1], va[2], va[3], vbase + SW::chunk_off(ltok, 2 * mt + lcsel));
      mma_bf16_16816(acc[mt], va, pb);
    }
    __syncwarp();
    // refill this stage with page i + STAGES of this warp
    const int nx = i + C::STAGES;
    if (nx < n_my) {
      if ((nx & 31) == 0) my_page = (lane + nx < n_my) ? ptab[p_begin + warp + (nx + lane) * kAttnWarps] : 0;
      const int pg = __shfl_sync(0xffffffffu, my_page, nx & 31);
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[s], C::BLOCK);
        bulk_g2s(ring + s * C::BLOCK, pool + (size_t)pg * page_stride + head_off, C::BLOCK, &bar[s]);
      }
    }
  }
  // ---- merge warps through shared memory (aliases the rings)
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  __syncthreads();
  float* mw = reinterpret_cast<float*>(smem);                   // [NW][8]
  float* lw = mw + kAttnWarps * 8;                              // [NW][8]
  float* ow = lw + kAttnWarps * 8;                              // [NW][8][HD]
  if (qq == 0 && gq < 8) {
    mw[warp * 8 + gq] = m_run;
    lw[warp * 8 + gq] = l_run;
  }
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    const int d = mt * 16 + gq;
    const int g0 = 2 * qq;
    ow[(warp * 8 + g0) * HD + d] = acc[mt][0];
    ow[(warp * 8 + g0 + 1) * HD + d] = acc[mt][1];
    ow[(warp * 8 + g0) * HD + d + 8] = acc[mt][2];
    ow[(warp * 8 + g0 + 1) * HD + d + 8] = acc[mt][3];
  }
  __syncthreads();
  const bool single = (n_chunks == 1);
  for (int it = threadIdx.x; it < G * HD; it += blockDim.x) {
    const int g = it / HD, d = it % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, mw[w * 8 + g]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float mwv = mw[w * 8 + g];
      const float f = (mwv == -INFINITY) ? 0.f : exp2f(mwv - M);
      L += lw[w * 8 + g] * f;
      O += ow[(w * 8 + g) * HD + d] * f;
    }
    const int qh = h * G + g;
    if (single) {
      const float o = O / L;
      a.out[((size_t)r * a.nq + qh) * HD + d] = __float2bfloat16_rn(o);
      if (a.out_f32) a.out_f32[((size_t)row * a.nq + qh) * HD + d] = o;
    } else {
      // partial: ws[((r * nq + qh) * max_chunks + chunk) * (HD + 2) + ...]
      float* wp = a.ws + (((size_t)r * a.nq + qh) * a.max_chunks + chunk) * (HD + 2);
      wp[d] = O;
      if (d == 0) {
        wp[HD] = M;
        wp[HD + 1] = L;
      }
    }
  }
  if (single) return;
  // ---- split-KV merge by the last chunk CTA of this (row, kv head): no combine launch
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* tk = a.tickets + (size_t)r * a.nkv + h;
    const int prev = atomicAdd(tk, 1);
    s_last = (prev == n_chunks - 1);
    if (s_last) *tk = 0;  // self-resetting for the next launch
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int it = threadIdx.x; it < G * HD; it += blockDim.x) {
    const int g = it / HD, d = it % HD;
    const int qh = h * G + g;
    const float* wp = a.ws + ((size_t)r * a.nq + qh) * a.max_chunks * (HD + 2);
    float M = -INFINITY;
    for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, __ldcg(wp + c * (HD + 2) + HD));
    float L = 0.f, O = 0.f;
    for (int c = 0; c < n_chunks; ++c) {  // fixed chunk order -> deterministic
      const float f = exp2f(__ldcg(wp + c * (HD + 2) + HD) - M);
      L += __ldcg(wp + c * (HD + 2) + HD + 1) * f;
      O += __ldcg(wp + c * (HD + 2) + d) * f;
    }
    const float o = O / L;
    a.out[((size_t)r * a.nq + qh) * HD + d] = __float2bfloat16_rn(o);
    if (a.out_f32) a.out_f32[((size_t)row * a.nq + qh) * HD + d] = o;
  }
}

int64_t attn_ws_floats(int n_rows, int nq, int hd, int max_chunks) {
  return (int64_t)n_rows * nq * max_chunks * (hd + 2);
}

// Split-KV plan (measured on B200, tools/attn_bench.py): one CTA per (row, kv head)
// streams at 96-110 % of the measured copy bandwidth from 64 rows x 8 kv heads up (C2
// 64 x 1310: 55 us; 64 x 8192: 90 % of 8 TB/s); extra chunks only add pipeline fills
// and the merge, and were never faster for >= 32 (row, head) pairs.  Below that the
// step is latency-bound and c = ceil(64 / pairs) <= 8 chunks help (1 row x 4096:
// 32 -> 14.5 us).  RT_ATTN_CHUNKS overrides c (tuning).
void attn_plan(int n_rows, int nkv, int max_seqlen, int* chunk_pages, int* max_chunks) {
  const int max_pages = (max_seqlen + 15) / 16;
  const long long base = (long long)n_rows * nkv;
  int best_c = 1;
  if (base < 32) {
    best_c = (int)((64 + base - 1) / base);
    if (best_c > 8) best_c = 8;
    while (best_c > 1 && max_pages / best_c < 2 * kAttnWarps) --best_c;
  }
  static int forced = -2;
  if (forced == -2) {
    const char* e = getenv("RT_ATTN_CHUNKS");
    forced = e ? atoi(e) : -1;
  }
  if (forced > 0) best_c = forced;
  int cp = (max_pages + best_c - 1) / best_c;
  if (cp < 1) cp = 1;
  *chunk_pages = cp;
  *max_chunks = (max_pages + cp - 1) / cp;
}

template <int HD>
static void launch_hd(const AttnArgs& a, cudaStream_t s) {
  using C = AttnCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  dim3 grid(a.max_chunks, a.nkv, a.n_rows);
  launch_pdl(k_attn<HD>, grid, dim3(kAttnWarps * 32), C::SMEM, s, a);
}

void launch_attention(const AttnArgs& a, cudaStream_t s) {
  if (a.n_rows <= 0) return;
  switch (a.hd) {
    case 128: launch_hd<128>(a, s); break;
    case 64: launch_hd<64>(a, s); break;
    case 32: launch_hd<32>(a, s); break;
    default: break;
  }
}

RT_TRACE_BINDER(trace_bind_attn)

}  // namespace rt
