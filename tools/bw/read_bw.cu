// Read-bandwidth ceiling probe for the decode attention's access pattern: every CTA (4 warps)
// streams 8 KiB blocks with cp.async.bulk into a per-warp ring completed on mbarriers and
// does no math, the blocks addressed through a page list like the KV pool.  Built by
// tools/read_bw.py (nvcc -shared), called through ctypes.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int BLOCK>
__global__ void __launch_bounds__(128) k_read(const unsigned char* base, const int* pages, int n_pages,
                                              unsigned* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smem + warp * STAGES * BLOCK;
  __shared__ __align__(8) uint64_t bar[4][STAGES];
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[warp][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // this warp's pages: a contiguous share of the list
  const long long W = (long long)gridDim.x * 4, w = (long long)blockIdx.x * 4 + warp;
  const int p0 = (int)(n_pages * w / W), p1 = (int)(n_pages * (w + 1) / W);
  const int n = p1 - p0;
  unsigned acc = 0;
  for (int i = 0; i < n + STAGES; ++i) {
    if (i >= STAGES) {  // consume page i - STAGES
      const int s = (i - STAGES) % STAGES;
      const uint32_t ph = ((i - STAGES) / STAGES) & 1;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&bar[warp][s])), "r"(ph) : "memory");
      acc += ring[s * BLOCK + lane * 4];
      __syncwarp();
    }
    if (i < n && lane == 0) {
      const int s = i % STAGES;
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[warp][s])), "r"(BLOCK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(ring + s * BLOCK)), "l"(base + (size_t)pages[p0 + i] * BLOCK), "r"(BLOCK), "r"(su32(&bar[warp][s]))
                   : "memory");
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

extern "C" int read_bw(const void* base, const int* pages, int n_pages, int ctas, int stages, void* sink, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  constexpr int B = 8192;
  switch (stages) {
#define C(S)                                                                                              \
  case S:                                                                                                 \
    cudaFuncSetAttribute(k_read<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * S * B);           \
    k_read<S, B><<<ctas, 128, 4 * S * B, s>>>((const unsigned char*)base, pages, n_pages, (unsigned*)sink); \
    break;
    C(2) C(3) C(4) C(5) C(6)
#undef C
    default: return -1;
  }
  return (int)cudaGetLastError();
}
