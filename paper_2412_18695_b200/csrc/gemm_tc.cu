// gemm_tc.cu — dense projections on 5th-gen tensor cores.
//
//   out[s][n][m] = sum_{k in split s} W[m, k] * X[n, k]        (bf16 x bf16 -> fp32)
//
// Decode projections are skinny (N = running batch): the weight matrix goes in
// the UMMA M slot (128 rows per CTA tile) and the batch in N (32..256), so
// weights stream through HBM once per step (HBM-bound for N <~ 210).
// Structure (one output tile per CTA, 192 threads):
//   warp 0 lane 0 : TMA producer — cp.async.bulk.tensor.2d (SW128 K-major tiles of
//                   W [128 x 64] and X [BN x 64]) into a STAGES-deep smem ring,
//                   completion on "full" mbarriers (expect_tx);
//   warp 1        : TMEM allocator; lane 0 issues tcgen05.mma.cta_group::1.kind::f16
//                   (M=128, N=BN, K=16) x 4 per stage, tcgen05.commit frees the stage
//                   and finally signals the epilogue;
//   warps 2..5    : epilogue — tcgen05.ld.32x32b.x16 (TMEM lane quarter = warp % 4),
//                   fp32 partial store (coalesced along m) or fused lm_head argmax.
// Split-K over grid.z fills the 148 SMs when M/128 * N/BN is small (QKV: 48 tiles).
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
  static constexpr int STAGES = (BN <= 64) ? 4 : (BN == 128 ? 3 : 4);
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256 + 4 * BN * 8;
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

struct GemmArgs {
  int M, N, K, splits, kb_total;
  float* out;         // MODE 0: [splits][N][M]; MODE 1: logits [N][M] or null
  float* part_val;    // MODE 1: [n_mtiles][N]
  int32_t* part_idx;  // MODE 1
};

template <int BN, int MODE>
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
  float* red_v = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE + 256);  // [4][BN]
  int* red_i = reinterpret_cast<int*>(red_v + 4 * BN);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
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
    mbar_wait(done, 0);
    tc_fence_after();
    const int m = m_tile * 128 + q * 32 + lane;
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
    if (MODE == 0) {
      float* out = g.out + (size_t)split * g.N * g.M;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = n_tile * BN + c0 + j;
          if (n < g.N && m < g.M) out[(size_t)n * g.M + m] = v[j];
        }
      }
    } else {
      // fused greedy argmax over the 128 vocab rows of this tile (lowest index on ties)
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = n_tile * BN + c0 + j;
          float bv = (m < g.M) ? v[j] : -INFINITY;
          int bi = m;
          if (g.out && n < g.N && m < g.M) g.out[(size_t)n * g.M + m] = v[j];
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
            red_v[q * BN + c0 + j] = bv;
            red_i[q * BN + c0 + j] = bi;
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int c = threadIdx.x - 64; c < BN; c += 128) {
        const int n = n_tile * BN + c;
        if (n >= g.N) continue;
        float bv = red_v[c];
        int bi = red_i[c];
        for (int w = 1; w < 4; ++w) {
          const float ov = red_v[w * BN + c];
          const int oi = red_i[w * BN + c];
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        g.part_val[(size_t)m_tile * g.N + n] = bv;
        g.part_idx[(size_t)m_tile * g.N + n] = bi;
      }
    }
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

int gemm_choose_splits(int M, int N, int K, int max_splits) {
  const int bn = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int kb = K / kBK;
  int splits = 1;
  const int target = 2 * 148;
  if (tiles < target) splits = (target + tiles - 1) / tiles;
  if (splits > kb / 4) splits = kb / 4;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  return splits;
}

template <int BN, int MODE>
static void launch_bn(const TmaMap& a, const TmaMap& b, const GemmArgs& g, cudaStream_t s) {
  using C = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_tc<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  dim3 grid((g.M + 127) / 128, (g.N + BN - 1) / BN, g.splits);
  k_gemm_tc<BN, MODE><<<grid, kGemmThreads, C::SMEM, s>>>(a, b, g);
}

template <int MODE>
static void dispatch(const TmaMap& wmap, const GemmTmaSet& x, const GemmArgs& g, cudaStream_t s) {
  if (g.N <= 32) launch_bn<32, MODE>(wmap, x.m32, g, s);
  else if (g.N <= 64) launch_bn<64, MODE>(wmap, x.m64, g, s);
  else if (g.N <= 128) launch_bn<128, MODE>(wmap, x.m128, g, s);
  else launch_bn<256, MODE>(wmap, x.m256, g, s);
}

int launch_gemm(const TmaMap& wmap, const GemmTmaSet& xmaps, int M, int N, int K, float* out, int max_splits,
                cudaStream_t s) {
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.kb_total = K / kBK;
  g.splits = gemm_choose_splits(M, N, K, max_splits);
  g.out = out;
  dispatch<0>(wmap, xmaps, g, s);
  return g.splits;
}

void launch_gemm_fixed(const TmaMap& wmap, const GemmTmaSet& xmaps, int M, int N, int K, float* out, int splits,
                       cudaStream_t s) {
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.kb_total = K / kBK;
  g.splits = splits;
  g.out = out;
  dispatch<0>(wmap, xmaps, g, s);
}

void launch_gemm_argmax(const TmaMap& wmap, const GemmTmaSet& xmaps, int M, int N, int K, float* part_val,
                        int32_t* part_idx, float* logits, cudaStream_t s) {
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.kb_total = K / kBK;
  g.splits = 1;
  g.out = logits;
  g.part_val = part_val;
  g.part_idx = part_idx;
  dispatch<1>(wmap, xmaps, g, s);
}

}  // namespace rt
