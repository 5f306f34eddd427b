// gemm_tc.cu — dense projections on 5th-gen tensor cores with fused epilogues
// (SURVEY §8(a) a6, a8).
//
//   D[m, n] = sum_k W[m, k] * X[n, k]        (bf16 x bf16 -> fp32 in TMEM)
//
// Decode projections are skinny (N = running batch): the weight matrix goes in the
// UMMA M slot (128 rows per tile) and the batch in N (32..256), so the weights
// stream through HBM once per step (HBM-bound for N <~ 210).
//
// Split-K across a THREAD-BLOCK CLUSTER: the S CTAs of a cluster (grid.x = S, up to
// 16 with the non-portable opt-in) stream disjoint K ranges of the same 128 x BN tile
// into their own TMEM accumulators; each then parks its fp32 partial in its own
// shared memory, and after one cluster barrier CTA r reduces columns
// [r BN / S, (r+1) BN / S) across the S partials through distributed shared memory
// (ld.shared::cluster, fixed rank order -> deterministic) and applies the fused
// epilogue to them.  No global workspace, no atomics, and the reduction runs on all
// S SMs in parallel.  S is chosen per shape so that S x tiles fills the 148 SMs
// (QKV 48 tiles x 6, O / down 32 x 9, gate-up 224 x 5, lm_head 1002 x 2).
// CTA roles (192 threads):
//   warp 0 lane 0 : TMA producer — weights are stored in HBM as UMMA-ready 16 KiB
//                   SW128 tiles, so each k-block of W is ONE
//                   cp.async.bulk of a contiguous range (a CTA streams sequential
//                   HBM); X [BN x 64] tiles come by cp.async.bulk.tensor.2d; the
//                   weight tiles of the first stages are requested BEFORE
//                   griddepcontrol.wait (programmatic dependent launch), so weight
//                   streaming overlaps the previous kernel's tail;
//   warp 1        : TMEM allocator; lane 0 issues tcgen05.mma.cta_group::1.kind::f16
//                   (M=128, N=BN, K=16), tcgen05.commit frees stages / signals the epilogue;
//   warps 2..5    : epilogue — tcgen05.ld.32x32b.x16 (lane quarter = warp % 4), fused
//                   op of oracle c1 applied from registers in 16-column chunks:
//        EPI_STORE  fp32 out[n][m]
//        EPI_ARGMAX lm_head: per-tile (max, lowest index) + optional logits
//        EPI_QKV    RoPE (rotate-half, theta 5e5) on q/k, bf16 q out, bf16 K/V
//                   appended into the swizzled KV page of (row task, position)
//        EPI_RESID  x[n][m] += D (fp32 residual stream) + per-tile sum of squares of
//                   the new x for the following RMSNorm
//        EPI_SWIGLU rows interleaved per tile [64 gate | 64 up]: act = bf16(silu(g) u)
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "model.h"

namespace rt {

constexpr int kGemmThreads = 192;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = 128 * kBK * 2;    // 16 KB
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN <= 64 ? 4 : (BN == 128 ? 3 : 4);
  static constexpr int CTAS_PER_SM = BN <= 128 ? 2 : 1;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int XCH = 16 * 64 * 4;                       // exchange [16][64] fp32
  static constexpr int META = 2 * 256 * 4;                      // per-column pos / page
  static constexpr int RED = 4 * 16 * 8;                        // per-warp column partials
  static constexpr int SMEM = 1024 + STAGES * STAGE + 512 + XCH + META + RED;
  static_assert(BN * 128 * 4 <= STAGES * STAGE, "partial tile must fit in the ring");
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
// UMMA shared-memory descriptor, K-major SWIZZLE_128B (CUTLASS UMMA::SmemDescriptor):
// start>>4 [0,14) | LBO>>4 [16,30) | SBO>>4 [32,46) | version 1 [46,48) | layout 2 [61,64)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;              // version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// instruction descriptor kind::f16: D f32, A/B bf16, K-major, N>>3 at [17,23), M>>4 at [24,29)
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

struct EpiSmem {
  float* xch;    // [16][64]
  int* pos;      // [256]
  int* page;     // [256]
  float* redv;   // [4][16]
  int* redi;     // [4][16]
};

// ------------------------------------------------------------ fused epilogue ops
// v[16] = D[m0 + et][n0 + c0 .. c0 + nv - 1] (nv <= 16 valid columns); executed by
// the 128 epilogue threads of one CTA (every thread must call it: named barriers).
template <int BN>
__device__ void epi_chunk(const GemmArgs& g, const EpiSmem& sm, const float* v, int m_tile, int n0, int c0,
                          int nv, int et) {
  const int NL = min(g.N, n0 + c0 + nv);  // columns >= NL are not owned / out of range
  const int m0 = m_tile * 128;
  const int m = m0 + et;
  const int lane = et & 31, wq = et >> 5;
  switch (g.mode) {
    case EPI_STORE: {
      if (m < g.M)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (n0 + c0 + j < NL) g.out[(size_t)(n0 + c0 + j) * g.M + m] = v[j];
      break;
    }
    case EPI_RESID: {
      float sq[16];
      float xv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c0 + j;
        xv[j] = (n < NL && m < g.M) ? g.x[(size_t)n * g.M + m] : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c0 + j;
        float xn = 0.f;
        if (n < NL && m < g.M) {
          xn = xv[j] + v[j];
          g.x[(size_t)n * g.M + m] = xn;
        }
        sq[j] = xn * xn;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) sq[j] = warp_sum(sq[j]);
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < 16; ++j) sm.redv[wq * 16 + j] = sq[j];
      epi_bar();
      if (et < 16 && n0 + c0 + et < NL) {
        const float s = ((sm.redv[et] + sm.redv[16 + et]) + sm.redv[32 + et]) + sm.redv[48 + et];
        g.ss[(size_t)(n0 + c0 + et) * ((g.M + 127) / 128) + m_tile] = s;
      }
      epi_bar();
      break;
    }
    case EPI_SWIGLU: {
      // rows [0,64) = gate features j0..j0+63, rows [64,128) = up features j0..j0+63
      if (et >= 64)
#pragma unroll
        for (int j = 0; j < 16; ++j) sm.xch[j * 64 + (et - 64)] = v[j];
      epi_bar();
      const int jf = m_tile * 64 + et;
      if (et < 64 && jf < g.ff)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = n0 + c0 + j;
          if (n < NL) {
            const float gv = v[j], uv = sm.xch[j * 64 + et];
            const float sgv = gv / (1.f + __expf(-gv));
            g.act[(size_t)n * g.ff + jf] = __float2bfloat16_rn(sgv * uv);
          }
        }
      epi_bar();
      break;
    }
    case EPI_QKV: {
      const QkvFuse& q = g.qkv;
      const int hd = q.hd, half = hd >> 1;
      const int hl = et / hd, i_full = et % hd;     // head within tile, dim within head
      const bool upper = i_full >= half;
      const int pidx = hl * half + (i_full % half); // pair index in [0, 64)
      if (upper)
#pragma unroll
        for (int j = 0; j < 16; ++j) sm.xch[j * 64 + pidx] = v[j];
      epi_bar();
      const int f = m0 + hl * hd + i_full;          // feature of this (lower) element
      if (!upper && f < g.M) {
        const int head = f / hd, i = i_full;
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
          const int c = c0 + j, n = n0 + c;
          if (n >= NL) break;
          const int pos = sm.pos[c];
          float x1 = v[j], x2 = sm.xch[j * 64 + pidx];
          if (head < q.nq + q.nkv) {
            const float cs = q.cos[(size_t)pos * half + i], sn = q.sin[(size_t)pos * half + i];
            const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
            x1 = y1;
            x2 = y2;
          }
          const bf16 b1 = __float2bfloat16_rn(x1), b2 = __float2bfloat16_rn(x2);
          if (head < q.nq) {
            bf16* qo = q.q_out + ((size_t)n * q.nq + head) * hd;
            qo[i] = b1;
            qo[i + half] = b2;
            if (q.q_cap) {
              float* qc = q.q_cap + ((size_t)(q.row0 + n) * q.nq + head) * hd;
              qc[i] = __bfloat162float(b1);
              qc[i + half] = __bfloat162float(b2);
            }
          } else {
            const int kind = head < q.nq + q.nkv ? 0 : 1;
            const int kvh = kind == 0 ? head - q.nq : head - q.nq - q.nkv;
            const int off = pos & 15;
            unsigned char* blk = (unsigned char*)q.pool +
                                 (((size_t)sm.page[c] * q.nkv + kvh) * 2 + kind) * (size_t)(16 * hd * 2) +
                                 off * hd * 2;
            *(bf16*)(blk + (kv_swz_chunk(hd, off, i >> 3) << 4) + ((i & 7) << 1)) = b1;
            *(bf16*)(blk + (kv_swz_chunk(hd, off, (i + half) >> 3) << 4) + (((i + half) & 7) << 1)) = b2;
          }
        }
      }
      epi_bar();
      break;
    }
    case EPI_ARGMAX: {
      if (g.out && m < g.M)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (n0 + c0 + j < NL) g.out[(size_t)(n0 + c0 + j) * g.M + m] = v[j];
#pragma unroll
      for (int j = 0; j < 16; ++j) {  // greedy: max over the tile's rows, lowest index on ties
        float bv = (m < g.M) ? v[j] : -INFINITY;
        int bi = (m < g.M) ? m : INT_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        if (lane == 0) {
          sm.redv[wq * 16 + j] = bv;
          sm.redi[wq * 16 + j] = bi;
        }
      }
      epi_bar();
      if (et < 16 && n0 + c0 + et < NL) {
        float bv = sm.redv[et];
        int bi = sm.redi[et];
        for (int w = 1; w < 4; ++w) {
          const float ov = sm.redv[w * 16 + et];
          const int oi = sm.redi[w * 16 + et];
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        g.part_val[(size_t)m_tile * g.N + n0 + c0 + et] = bv;
        g.part_idx[(size_t)m_tile * g.N + n0 + c0 + et] = bi;
      }
      epi_bar();
      break;
    }
    default:
      break;
  }
}


template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc(const __grid_constant__ TmaMap tmB, GemmArgs g) {
  using C = GemmCfg<BN>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + C::STAGES * C::A_BYTES;
  unsigned char* ctl = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctl);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* P = reinterpret_cast<float*>(smem);  // [BN][128] partial tile, reuses the ring after the mainloop
  EpiSmem sm;
  sm.xch = reinterpret_cast<float*>(ctl + 512);
  sm.pos = reinterpret_cast<int*>(ctl + 512 + C::XCH);
  sm.page = sm.pos + 256;
  sm.redv = reinterpret_cast<float*>(ctl + 512 + C::XCH + C::META);
  sm.redi = reinterpret_cast<int*>(sm.redv + 64);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.x;                 // cluster = the S split-K CTAs of one tile
  const int rank = S > 1 ? (int)cluster_rank() : 0;
  const int m_tile = blockIdx.y, n_tile = blockIdx.z;
  const int kb0 = (int)(((long long)g.kb_total * rank) / S);
  const int kb1 = (int)(((long long)g.kb_total * (rank + 1)) / S);
  const int nkb = kb1 - kb0;
  const int n0 = n_tile * BN;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // weights do not depend on the previous kernel: request the first stages' W tiles
      // before waiting for it (programmatic dependent launch)
      const int pre = min(C::STAGES, nkb);
      // UMMA-tiled weights: k-block kb of m-tile mt is one contiguous 16 KiB SW128 image
      const bf16* wt = g.w + ((size_t)m_tile * g.kb_total + kb0) * (128 * kBK);
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], C::STAGE);
        bulk_g2s(sA + i * C::A_BYTES, wt + (size_t)i * (128 * kBK), C::A_BYTES, &full[i]);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sB + i * C::B_BYTES, &tmB, (kb0 + i) * kBK, n0, &full[i]);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], C::STAGE);
        bulk_g2s(sA + s * C::A_BYTES, wt + (size_t)i * (128 * kBK), C::A_BYTES, &full[s]);
        tma_load_2d(sB + s * C::B_BYTES, &tmB, (kb0 + i) * kBK, n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc(128, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        mbar_wait(&full[s], (uint32_t)((i / C::STAGES) & 1));
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b0 = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          umma_f16(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                   (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
    __syncwarp();
  } else {
    pdl_wait();
    const int q = warp & 3;
    const int et = q * 32 + lane;  // tile row owned by this thread
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
    mbar_wait(done, 0);
    tc_fence_after();
    if (S == 1) {
      if (g.mode == EPI_QKV) {
        for (int cc = et; cc < BN; cc += 128) {
          const int n = n0 + cc;
          if (n < g.N) {
            const int row = g.qkv.row0 + n;
            const int pos = g.qkv.row_pos[row];
            sm.pos[cc] = pos;
            sm.page[cc] = g.qkv.page_table[(size_t)g.qkv.row_task[row] * g.qkv.pt_stride + (pos >> 4)];
          }
        }
        epi_bar();
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tb + c0, v);
        epi_chunk<BN>(g, sm, v, m_tile, n0, c0, 16, et);
      }
    } else {
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {  // park the partial in this CTA's smem
        float v[16];
        tmem_ld16(tb + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) P[(c0 + j) * 128 + et] = v[j];
      }
    }
  }
  if (S > 1) {
    // ---- cluster reduction: CTA `rank` finishes columns [cb, ce) of the tile
    __syncwarp();        // reconverge the producer / MMA warps (aligned cluster barrier)
    cluster_sync_all();  // every partial of the cluster is in shared memory
    if (warp >= 2) {
      const int et = (warp & 3) * 32 + lane;
      const int cb = (BN * rank) / S, ce = (BN * (rank + 1)) / S;
      if (g.mode == EPI_QKV) {
        for (int cc = cb + et; cc < ce; cc += 128) {
          const int n = n0 + cc;
          if (n < g.N) {
            const int row = g.qkv.row0 + n;
            const int pos = g.qkv.row_pos[row];
            sm.pos[cc] = pos;
            sm.page[cc] = g.qkv.page_table[(size_t)g.qkv.row_task[row] * g.qkv.pt_stride + (pos >> 4)];
          }
        }
        epi_bar();
      }
      const uint32_t pl = smem_u32(P);
#pragma unroll 1
      for (int c0 = cb; c0 < ce; c0 += 16) {
        const int nv = min(16, ce - c0);
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
#pragma unroll 1
        for (int rk = 0; rk < S; ++rk) {  // fixed rank order -> deterministic
          const uint32_t base = dsmem_addr(pl, (uint32_t)rk);
          float w[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) w[j] = (j < nv) ? ld_dsmem(base + (uint32_t)(((c0 + j) * 128 + et) * 4)) : 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += w[j];
        }
        epi_chunk<BN>(g, sm, v, m_tile, n0, c0, nv, et);
      }
    }
    cluster_sync_all();  // keep shared memory alive until every CTA has read it
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

bool make_tma_2d_bf16(TmaMap* out, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                      uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out->bytes), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_gemm_act_maps(GemmTmaSet* out, const void* base, int K, int rows_cap) {
  out->rows_cap = rows_cap;
  return make_tma_2d_bf16(&out->m32, base, K, rows_cap, kBK, 32) &&
         make_tma_2d_bf16(&out->m64, base, K, rows_cap, kBK, 64) &&
         make_tma_2d_bf16(&out->m128, base, K, rows_cap, kBK, 128) &&
         make_tma_2d_bf16(&out->m256, base, K, rows_cap, kBK, 256);
}

int gemm_bn(int N) { return N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256; }

template <int BN>
static void ensure_attrs() {
  using C = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(k_gemm_tc<BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
}

// how many S-CTA clusters of k_gemm_tc<BN> can be co-resident (cached per S)
template <int BN>
static int max_clusters(int S) {
  using C = GemmCfg<BN>;
  static int cache[17] = {0};
  if (S < 1 || S > 16) return 0;
  if (!cache[S]) {
    ensure_attrs<BN>();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(S, 64, 1);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)k_gemm_tc<BN>, &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
    cache[S] = n > 0 ? n : -1;
  }
  return cache[S] > 0 ? cache[S] : 0;
}

static int max_clusters_bn(int bn, int S) {
  if (bn == 32) return max_clusters<32>(S);
  if (bn == 64) return max_clusters<64>(S);
  if (bn == 128) return max_clusters<128>(S);
  return max_clusters<256>(S);
}

// Cluster split count (measured on B200, tools/gemm_bench.py, N = 64): a split-K cluster
// only pays off while every cluster is co-resident in ONE wave; with >= 148 tiles plain
// tiles (S = 1) already cover the SMs.  Measured co-residency of 2-CTA/SM clusters holds
// up to 256 CTAs (O / down: 32 x 8 = 256 -> 11.7 / 26 us) but not 288 (QKV 48 x 6:
// 12 -> 19 us, 32 x 9: 11 -> 19 us), so S = max{S <= 8 : tiles x S <= 256, >= 4 k-blocks
// per CTA} (cudaOccupancyMaxActiveClusters under-reports and is only a cap).
int gemm_choose_splits(int M, int N, int K) {
  const int bn = gemm_bn(N);
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int kb = K / kBK;
  if (tiles >= 148) return 1;
  const int budget = bn <= 128 ? 256 : 128;
  int best = 1;
  for (int s = 2; s <= 8 && kb / s >= 4; ++s)
    if (tiles * s <= budget) best = s;
  (void)max_clusters_bn;
  return best;
}

template <int BN>
static cudaError_t launch_bn(const TmaMap& b, const GemmArgs& g, int S, cudaStream_t s) {
  using C = GemmCfg<BN>;
  ensure_attrs<BN>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(S, (g.M + 127) / 128, (g.N + BN - 1) / BN);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = S;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_tc<BN>, b, g);
}

cudaError_t launch_gemm_epi(const bf16* w_tiled, const GemmTmaSet& x, GemmArgs g, int splits, cudaStream_t s) {
  g.w = w_tiled;
  const int bn = gemm_bn(g.N);
  g.kb_total = g.K / kBK;
  g.m_tiles = (g.M + 127) / 128;
  if (splits <= 0) splits = gemm_choose_splits(g.M, g.N, g.K);
  splits = std::max(1, std::min(splits, std::min(16, g.kb_total)));
  if (bn == 32) return launch_bn<32>(x.m32, g, splits, s);
  if (bn == 64) return launch_bn<64>(x.m64, g, splits, s);
  if (bn == 128) return launch_bn<128>(x.m128, g, splits, s);
  return launch_bn<256>(x.m256, g, splits, s);
}

}  // namespace rt
