// gemm_tc.cu — dense projections on 5th-gen tensor cores with fused epilogues
// (SURVEY §8(a) a6, a8).
//
//   D[m, n] = sum_k W[m, k] * X[n, k]        (bf16 x bf16 -> fp32 in TMEM)
//
// Decode projections are skinny (N = running batch): the weight matrix goes in
// the UMMA M slot (128 rows per CTA tile) and the batch in N (32..256), so the
// weights stream through HBM once per step (HBM-bound for N <~ 210).
// CTA structure (192 threads, one output tile per CTA):
//   warp 0 lane 0 : TMA producer — cp.async.bulk.tensor.2d (SW128 K-major tiles of
//                   W [128 x 64] and X [BN x 64]) into a STAGES-deep smem ring;
//   warp 1        : TMEM allocator; lane 0 issues tcgen05.mma.cta_group::1.kind::f16
//                   (M=128, N=BN, K=16) x 4 per stage; tcgen05.commit frees stages
//                   and finally signals the epilogue;
//   warps 2..5    : epilogue — tcgen05.ld.32x32b.x16 (TMEM lane quarter = warp % 4)
//                   into a [BN][129] fp32 smem tile (reusing the ring), split-K
//                   partials reduced by the LAST CTA of each tile (L2-resident
//                   workspace, fixed split order -> deterministic), then the fused
//                   elementwise op of oracle c1 for this projection:
//        EPI_STORE  fp32 out[n][m]
//        EPI_ARGMAX lm_head: per-tile (max, lowest index) + optional logits
//        EPI_QKV    RoPE (rotate-half, theta 5e5) on q/k, bf16 q out, bf16 K/V
//                   appended into the swizzled KV page of (row task, position)
//        EPI_RESID  x[n][m] += D (fp32 residual stream) + per-tile sum of squares
//                   of the new x for the following RMSNorm
//        EPI_SWIGLU rows interleaved per tile [64 gate | 64 up]: act = bf16(silu(g) u)
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "model.h"

namespace rt {

constexpr int kGemmThreads = 192;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K
constexpr int kSP = 129; // padded row of the smem output tile (conflict-free both ways)

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = 128 * kBK * 2;    // 16 KB
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN <= 64) ? 4 : (BN == 128 ? 3 : 4);
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256;
  static_assert(BN * kSP * 4 <= STAGES * STAGE, "epilogue tile must fit in the ring");
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

// ------------------------------------------------------------ fused epilogue ops
// S: smem tile [BN][kSP] holding D[m0 + r][n0 + c] at S[c * kSP + r]; et = 0..127.
template <int BN>
__device__ void epi_apply(const GemmArgs& g, const float* S, int m_tile, int n_tile, int et) {
  const int m0 = m_tile * 128, n0 = n_tile * BN;
  const int ncol = min(BN, g.N - n0);
  switch (g.mode) {
    case EPI_STORE: {
      const int m = m0 + et;
      if (m < g.M)
        for (int c = 0; c < ncol; ++c) g.out[(size_t)(n0 + c) * g.M + m] = S[c * kSP + et];
      break;
    }
    case EPI_RESID: {
      const int m = m0 + et;
      float* sq = const_cast<float*>(S);  // squares written in place (same thread, same slot)
      float* xb = g.x + (size_t)n0 * g.M + m;
#pragma unroll 1
      for (int c0 = 0; c0 < ncol; c0 += 8) {
        float xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = (m < g.M && c0 + u < ncol) ? xb[(size_t)(c0 + u) * g.M] : 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (c0 + u < ncol) {
            const float v = (m < g.M) ? xv[u] + S[(c0 + u) * kSP + et] : 0.f;
            if (m < g.M) xb[(size_t)(c0 + u) * g.M] = v;
            sq[(c0 + u) * kSP + et] = v * v;
          }
        }
      }
      epi_bar();
      const int mt = (g.M + 127) / 128;
      for (int c = et; c < ncol; c += 128) {  // column sums in fixed row order
        float s = 0.f;
        for (int r = 0; r < 128; ++r) s += S[c * kSP + r];
        g.ss[(size_t)(n0 + c) * mt + m_tile] = s;
      }
      break;
    }
    case EPI_SWIGLU: {
      // tile rows [0,64) = gate features j0..j0+63, rows [64,128) = up features j0..j0+63
      const int r = et & 63, half = et >> 6;
      const int j = m_tile * 64 + r;
      if (j < g.ff)
        for (int c = half; c < ncol; c += 2) {
          const float gv = S[c * kSP + r], uv = S[c * kSP + 64 + r];
          const float sgv = gv / (1.f + __expf(-gv));
          g.act[(size_t)(n0 + c) * g.ff + j] = __float2bfloat16_rn(sgv * uv);
        }
      break;
    }
    case EPI_QKV: {
      const QkvFuse& q = g.qkv;
      const int hd = q.hd, half = hd >> 1;
      // per-column (token row) metadata, one thread per column
      __shared__ int s_pos[256], s_page[256];
      for (int c = et; c < ncol; c += 128) {
        const int row = q.row0 + n0 + c;
        const int pos = q.row_pos[row];
        s_pos[c] = pos;
        s_page[c] = q.page_table[(size_t)q.row_task[row] * q.pt_stride + (pos >> 4)];
      }
      epi_bar();
      const int pr = et & 63;                       // 128 features per tile = 64 (i, i + hd/2) pairs
      const int hl = pr / half, i = pr % half;      // head within tile, pair index
      const int f = m0 + hl * hd + i;               // feature of the first element
      if (f >= g.M) break;
      const int head = f / hd;
#pragma unroll 2
      for (int c = et >> 6; c < ncol; c += 2) {
        const int row = q.row0 + n0 + c;
        const int pos = s_pos[c];
        float x1 = S[c * kSP + hl * hd + i], x2 = S[c * kSP + hl * hd + i + half];
        if (head < q.nq + q.nkv) {
          const float cs = q.cos[(size_t)pos * half + i], sn = q.sin[(size_t)pos * half + i];
          const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
          x1 = y1;
          x2 = y2;
        }
        const bf16 b1 = __float2bfloat16_rn(x1), b2 = __float2bfloat16_rn(x2);
        if (head < q.nq) {
          bf16* qo = q.q_out + ((size_t)(n0 + c) * q.nq + head) * hd;
          qo[i] = b1;
          qo[i + half] = b2;
          if (q.q_cap) {
            float* qc = q.q_cap + ((size_t)row * q.nq + head) * hd;
            qc[i] = __bfloat162float(b1);
            qc[i + half] = __bfloat162float(b2);
          }
        } else {
          const int kind = head < q.nq + q.nkv ? 0 : 1;
          const int kvh = kind == 0 ? head - q.nq : head - q.nq - q.nkv;
          const int page = s_page[c];
          const int off = pos & 15;
          unsigned char* blk = (unsigned char*)q.pool +
                               (((size_t)page * q.nkv + kvh) * 2 + kind) * (size_t)(16 * hd * 2) + off * hd * 2;
          *(bf16*)(blk + (kv_swz_chunk(hd, off, i >> 3) << 4) + ((i & 7) << 1)) = b1;
          *(bf16*)(blk + (kv_swz_chunk(hd, off, (i + half) >> 3) << 4) + (((i + half) & 7) << 1)) = b2;
        }
      }
      break;
    }
    case EPI_ARGMAX: {
      const int m = m0 + et;
      if (g.out && m < g.M)
        for (int c = 0; c < ncol; ++c) g.out[(size_t)(n0 + c) * g.M + m] = S[c * kSP + et];
      for (int c = et; c < ncol; c += 128) {  // greedy: max over the tile's rows, lowest index on ties
        float bv = -INFINITY;
        int bi = INT_MAX;
        for (int r = 0; r < 128 && m0 + r < g.M; ++r) {
          const float v = S[c * kSP + r];
          if (v > bv) {
            bv = v;
            bi = m0 + r;
          }
        }
        g.part_val[(size_t)m_tile * g.N + n0 + c] = bv;
        g.part_idx[(size_t)m_tile * g.N + n0 + c] = bi;
      }
      break;
    }
    default:
      break;
  }
}

template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc(const __grid_constant__ TmaMap tmA, const __grid_constant__ TmaMap tmB, GemmArgs g) {
  using C = GemmCfg<BN>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int* is_last = reinterpret_cast<int*>(tmem_slot + 1);
  float* S = reinterpret_cast<float*>(smem);  // epilogue tile, reuses the ring after the mainloop

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // split fastest in launch order: a tile's split CTAs run together, so the last-CTA
  // reductions are spread over the kernel instead of piling up in the final wave
  const int split = blockIdx.x, m_tile = blockIdx.y, n_tile = blockIdx.z;
  const int kb0 = (int)(((long long)g.kb_total * split) / g.splits);
  const int kb1 = (int)(((long long)g.kb_total * (split + 1)) / g.splits);
  const int nkb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
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

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], C::STAGE);
        const int kc = (kb0 + i) * kBK;
        tma_load_2d(sA + s * C::A_BYTES, &tmA, kc, m_tile * 128, &full[s]);
        tma_load_2d(sB + s * C::B_BYTES, &tmB, kc, n_tile * BN, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc(128, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b0 = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          umma_f16(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                   (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5 (TMEM lane quarter = warp % 4)
    const int q = warp & 3;
    const int et = q * 32 + lane;  // row of the tile owned by this thread
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
    const int tile = n_tile * gridDim.y + m_tile;
    if (g.splits == 1) {
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) S[(c0 + j) * kSP + et] = v[j];
      }
    } else {
      // split-K: publish this partial (L2), the last CTA of the tile reduces in split order
      float* ws = g.ws + ((size_t)tile * g.splits + split) * (BN * 128);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) ws[(c0 + j) * 128 + et] = v[j];
      }
      __threadfence();
      epi_bar();
      if (et == 0) {
        const int prev = atomicAdd(&g.counters[tile], 1);
        *is_last = (prev == g.splits - 1);
        if (prev == g.splits - 1) g.counters[tile] = 0;  // ready for the next launch
      }
      epi_bar();
      if (!*is_last) goto epi_done;
      __threadfence();
      // reduce the splits in fixed order; 8 independent 16-byte L2 loads in flight per thread
      constexpr int NV = BN * 128 / 4;  // float4 per partial tile
      const float4* base = reinterpret_cast<const float4*>(g.ws + (size_t)tile * g.splits * (BN * 128));
#pragma unroll 1
      for (int j0 = 0; j0 < NV / 128; j0 += 8) {
        float4 acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
        for (int s = 0; s < g.splits; ++s) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcg(base + (size_t)s * NV + et + 128 * (j0 + u));
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            acc[u].x += v[u].x;
            acc[u].y += v[u].y;
            acc[u].z += v[u].z;
            acc[u].w += v[u].w;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e4 = 4 * (et + 128 * (j0 + u));
          float* d = S + (e4 >> 7) * kSP + (e4 & 127);
          d[0] = acc[u].x;
          d[1] = acc[u].y;
          d[2] = acc[u].z;
          d[3] = acc[u].w;
        }
      }
    }
    epi_bar();
    epi_apply<BN>(g, S, m_tile, n_tile, et);
  }
epi_done:
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

static int bn_for(int N) { return N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256; }

// Split-K so that the CTA count fills the 148 SMs (2 CTAs/SM) in as few waves as possible.
int gemm_choose_splits(int M, int N, int K, int max_splits) {
  const int bn = bn_for(N);
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int kb = K / kBK;
  const int slots = 2 * 148;
  int best = 1;
  double best_cost = 1e30;
  const int lim = std::max(1, std::min(max_splits, kb / 4));
  for (int s = 1; s <= lim; ++s) {
    const int ctas = tiles * s;
    const int waves = (ctas + slots - 1) / slots;
    // time ~ waves * (kb / s + fixed per-CTA overhead in k-blocks) ; partial traffic ~ s
    const double cost = waves * ((double)kb / s + 3.0) + 0.02 * s * tiles;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

int64_t gemm_ws_floats(int M, int N, int K, int splits) {
  const int bn = bn_for(N);
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  return splits > 1 ? (int64_t)tiles * splits * bn * 128 : 0;
}

template <int BN>
static void launch_bn(const TmaMap& a, const TmaMap& b, const GemmArgs& g, cudaStream_t s) {
  using C = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  dim3 grid(g.splits, (g.M + 127) / 128, (g.N + BN - 1) / BN);
  k_gemm_tc<BN><<<grid, kGemmThreads, C::SMEM, s>>>(a, b, g);
}

void launch_gemm_epi(const TmaMap& wmap, const GemmTmaSet& x, GemmArgs g, cudaStream_t s) {
  g.kb_total = g.K / kBK;
  if (g.splits < 1) g.splits = 1;
  if (g.N <= 32) launch_bn<32>(wmap, x.m32, g, s);
  else if (g.N <= 64) launch_bn<64>(wmap, x.m64, g, s);
  else if (g.N <= 128) launch_bn<128>(wmap, x.m128, g, s);
  else launch_bn<256>(wmap, x.m256, g, s);
}

}  // namespace rt
